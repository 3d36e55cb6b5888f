"""Host volume type and ``.vol`` IO — the boundary type of every hot function.

Mirrors the reference's ``sfw3d.volumes`` contract (volumes.py:1-113): an
immutable float64 C-order (nx, ny, nz) array, z contiguous, validated finite,
read-only; the ``.vol`` format is ``b"SFW3DV01"``, three little-endian uint32
dims, then little-endian float64 payload. The B200 build adds one thing: a
per-(device, storage dtype) cache of the device copy, so a Volume handed to
several GPU calls (y in the solver loop) is uploaded once. The cache is safe
because the host array is read-only.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

MAGIC = b"SFW3DV01"
_HDR = struct.Struct("<8s3I")


class VolumeFormatError(ValueError):
    """Malformed ``.vol`` file: bad magic, size mismatch or non-finite payload."""


def _dims3(dims) -> tuple[int, int, int]:
    out = tuple(int(n) for n in dims)
    if len(out) != 3 or min(out) < 1:
        raise ValueError(f"dims must be three positive integers, got {out}")
    return out


class Volume:
    """Immutable dense float64 field on an (nx, ny, nz) voxel grid."""

    __slots__ = ("_data", "_dev")

    def __init__(self, data):
        arr = np.array(data, dtype=np.float64, order="C", copy=True) \
            if not (isinstance(data, np.ndarray) and data.dtype == np.float64
                    and data.flags.c_contiguous and not data.flags.writeable) \
            else data
        if arr.ndim != 3:
            raise ValueError(f"volume data must be 3D, got shape {arr.shape}")
        _dims3(arr.shape)
        if not np.isfinite(arr).all():
            raise ValueError("volume data contains non-finite values")
        if arr.flags.writeable:
            arr.setflags(write=False)
        object.__setattr__(self, "_data", arr)
        object.__setattr__(self, "_dev", {})

    def __setattr__(self, name, value):
        raise AttributeError("Volume is immutable")

    @property
    def data(self) -> np.ndarray:
        return self._data

    @property
    def dims(self) -> tuple[int, int, int]:
        return self._data.shape

    def __repr__(self) -> str:
        return f"Volume(dims={self.dims})"

    # -- device copies (B200 build) -----------------------------------------
    def device_tensor(self, dtype, device):
        """Device copy in the given torch dtype, uploaded once and cached."""
        import torch
        key = (str(device), dtype)
        t = self._dev.get(key)
        if t is None:
            import warnings
            with warnings.catch_warnings():  # read-only source: only read (pinned copy below)
                warnings.simplefilter("ignore", UserWarning)
                host = torch.from_numpy(self._data)
            if dtype != torch.float64:
                host = host.to(dtype)
            t = host.pin_memory().to(device, non_blocking=True)
            self._dev[key] = t
        return t

    @classmethod
    def from_device(cls, tensor) -> "Volume":
        """Host Volume from a device tensor (one D2H copy, float64)."""
        return cls(tensor.detach().to("cpu", dtype=__import__("torch").float64).numpy())


class GridGeometry:
    """Voxel grid geometry; spacing is one voxel per axis (volumes.py:62-74)."""

    __slots__ = ("_dims",)

    def __init__(self, dims):
        object.__setattr__(self, "_dims", _dims3(dims))

    def __setattr__(self, name, value):
        raise AttributeError("GridGeometry is immutable")

    @property
    def dims(self) -> tuple[int, int, int]:
        return self._dims

    @property
    def voxel_count(self) -> int:
        return self._dims[0] * self._dims[1] * self._dims[2]

    def __eq__(self, other):
        return isinstance(other, GridGeometry) and other._dims == self._dims

    def __hash__(self):
        return hash(self._dims)

    def __repr__(self) -> str:
        return f"GridGeometry(dims={self._dims})"


def zero_volume(dims) -> Volume:
    return Volume(np.zeros(_dims3(dims)))


def volume_norms(v: Volume) -> tuple[float, float]:
    """``(max |v_i|, sqrt(sum v_i^2))``."""
    flat = v.data.ravel()
    return (float(np.max(np.abs(flat))) if flat.size else 0.0, float(np.linalg.norm(flat)))


def write_volume(v: Volume, path) -> None:
    with open(Path(path), "wb") as fh:
        fh.write(_HDR.pack(MAGIC, *v.dims))
        fh.write(np.ascontiguousarray(v.data, dtype="<f8").tobytes())


def read_volume(path) -> Volume:
    path = Path(path)
    raw = path.read_bytes()
    if len(raw) < _HDR.size:
        raise VolumeFormatError(f"{path}: truncated header")
    magic, nx, ny, nz = _HDR.unpack_from(raw)
    if magic != MAGIC:
        raise VolumeFormatError(f"{path}: bad magic {magic!r}")
    dims = _dims3((nx, ny, nz))
    want = _HDR.size + 8 * nx * ny * nz
    if len(raw) != want:
        raise VolumeFormatError(
            f"{path}: payload size mismatch (header says {want} bytes, file has {len(raw)})")
    data = np.frombuffer(raw, dtype="<f8", offset=_HDR.size).reshape(dims)
    if not np.isfinite(data).all():
        raise VolumeFormatError(f"{path}: payload contains non-finite values")
    return Volume(data.astype(np.float64, copy=True))


# -- .vol IO straight to HBM (B200 build: SURVEY §8(f)4) ----------------------
def read_volume_device(path, device=None, precision: str | None = None):
    """A ``.vol`` file as a device tensor in the storage precision, without a
    host float64 Volume: the payload streams through pinned staging into HBM
    (sfw3d_volume_read); the format checks are the reference's
    (volumes.py:96-113) and raise VolumeFormatError."""
    import torch
    from . import _native as N
    p = str(Path(path)).encode()
    dims = np.zeros(3, np.int32)
    code = N.dtype_code(precision)
    try:
        N.check(N.lib().sfw3d_volume_info(p, N.i32_ptr(dims)))
        dev = N.device_index(device)
        out = torch.empty(tuple(int(d) for d in dims), dtype=N.torch_dtype(code),
                          device=f"cuda:{dev}")
        N.check(N.lib().sfw3d_volume_read(N.context(dev).handle, p, code, N.ptr(out)))
    except ValueError as e:
        raise VolumeFormatError(str(e)) from None
    return out


def write_volume_device(tensor, path) -> None:
    """Write a device volume (fp32 or fp64) as a ``.vol`` file (float64
    payload; bit-exact round trip for fp64)."""
    from . import _native as N
    from .forward import code_of
    t = tensor.contiguous()
    dev = t.device.index
    N.check(N.lib().sfw3d_volume_write(N.context(dev).handle, str(Path(path)).encode(), code_of(t),
                                       N.dims_arg(t.shape), N.ptr(t)))
