"""Forward imaging model on the B200: atoms, PSF blur, criterion, gradient.

Drop-in for ``sfw3d.forward`` (forward.py:1-263): same public names,
signatures, return types and exceptions. Bodies call the sm_100a C-ABI
(``_native``): K3 render, K4 separable PSF passes, K5 residual + ||.||^2,
K6 per-atom fp64 gradient reductions. ``workers`` is accepted for signature
compatibility and ignored (the GPU grid replaces ``map_ordered``,
_parallel.py:12-22). ``y_hat`` is accepted and ignored (there is no FFT).

Device-resident variants (suffix ``_dev``) take/return torch CUDA tensors
and are what the solvers and ``bench.py`` use inside their loops.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .measures import AtomParams, WeightedMeasure, measure_rows, total_mass
from .volumes import GridGeometry, Volume

#: unit-profile value below which an atom is exactly zero (forward.py:31-32)
TAIL_CUTOFF = 1e-12
_TAIL_EXPONENT = 2.0 * np.log(1.0 / TAIL_CUTOFF)

#: per-atom gradient column order (forward.py:36-37)
GRADIENT_COLUMNS = ("w", "m_x", "m_y", "m_z", "sigma", "d")


# ---------------------------------------------------------------------- PSF
class Psf:
    """Centred PSF kernel (origin voxel n//2 per axis), unit sum by default.

    forward.py:40-76. The device representation (three 1-D tap vectors when
    the kernel is separable, else its non-zero box) is built lazily per
    device by the C library. ``kernel_hat`` (the reference's cached FFT) is
    kept for API compatibility and computed on first access only.
    """

    def __init__(self, kernel: Volume, normalize: bool = True):
        data = kernel.data
        if normalize:
            s = float(data.sum())
            peak = float(np.abs(data).max()) if data.size else 0.0
            if abs(s) < 1e-12 * max(peak, 1.0):
                raise ValueError("kernel sum is ~0, cannot normalize to unit sum")
            kernel = Volume(data / s)
        self.kernel = kernel
        self._native = {}
        self._hat = None

    @property
    def dims(self) -> tuple[int, int, int]:
        return self.kernel.dims

    @property
    def kernel_hat(self) -> np.ndarray:
        """Reference compatibility only: a HOST FFT (the B200 path never uses it)."""
        if self._hat is None:
            import scipy.fft as sfft
            _warn_host_fft("Psf.kernel_hat", self.dims)
            self._hat = sfft.rfftn(sfft.ifftshift(self.kernel.data))
        return self._hat

    @classmethod
    def delta(cls, dims) -> "Psf":
        data = np.zeros(tuple(dims))
        data[tuple(n // 2 for n in data.shape)] = 1.0
        return cls(Volume(data), normalize=False)

    def is_centrosymmetric(self, tol: float = 1e-10) -> bool:
        """kernel(origin + o) == kernel(origin - o) for every offset o (the
        kernel is immutable: the answer is kept per tolerance — three passes over
        a 256^3 host array are 0.15 s of every table request otherwise)."""
        memo = self.__dict__.setdefault("_centro", {})
        if tol not in memo:
            k = self.kernel.data
            sh = np.roll(k, [-(n // 2) for n in k.shape], axis=(0, 1, 2))  # origin -> index 0
            mir = np.roll(sh[::-1, ::-1, ::-1], 1, axis=(0, 1, 2))
            scale = float(np.abs(sh).max()) or 1.0
            memo[tol] = bool(np.max(np.abs(sh - mir)) <= tol * scale)
        return memo[tol]

    def native(self, device: int):
        h = self._native.get(device)
        if h is None:
            ctx = N.context(device)
            hp = C.c_void_p()
            kd = np.ascontiguousarray(self.kernel.data)
            N.check(N.lib().sfw3d_psf_create(ctx.handle, N.dims_arg(self.dims), N.f64_ptr(kd),
                                             C.byref(hp)))
            h = _PsfHandle(hp)
            self._native[device] = h
        return h.handle

    def separable(self, device=None) -> bool:
        sep = C.c_int()
        N.check(N.lib().sfw3d_psf_info(self.native(N.device_index(device)), C.byref(sep), None, None))
        return bool(sep.value)


def _warn_host_fft(what: str, dims) -> None:
    if int(np.prod(dims)) >= (1 << 21):
        import warnings
        warnings.warn(f"{what}: computing a host FFT of a {dims} volume for reference "
                      "compatibility (the B200 path does not use it)", RuntimeWarning,
                      stacklevel=3)


_FOREIGN_PSF = None


def as_psf(psf) -> Psf:
    """This package's Psf for `psf`: itself, or (cached per object) a wrapper
    of a reference ``sfw3d.forward.Psf`` / any object with ``.kernel.data``
    (already normalised: the reference normalises in its constructor)."""
    global _FOREIGN_PSF
    if isinstance(psf, Psf):
        return psf
    if not hasattr(psf, "kernel") or not hasattr(psf.kernel, "data"):
        raise TypeError(f"expected a Psf, got {type(psf).__name__}")
    if _FOREIGN_PSF is None:
        import weakref
        _FOREIGN_PSF = weakref.WeakKeyDictionary()
    try:
        got = _FOREIGN_PSF.get(psf)
    except TypeError:  # (not weak-referenceable: wrap every time)
        return Psf(Volume(np.asarray(psf.kernel.data, dtype=np.float64)), normalize=False)
    if got is None:
        got = Psf(Volume(np.asarray(psf.kernel.data, dtype=np.float64)), normalize=False)
        _FOREIGN_PSF[psf] = got
    return got


class _PsfHandle:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if N._lib is not None and self.handle:
                N._lib.sfw3d_psf_destroy(self.handle)
        except Exception:
            pass


# ------------------------------------------------------------ device helpers
def _device():
    return N.device_index(None)


def to_dev(v, code: int | None = None, device=None):
    """Device tensor of a Volume / ndarray / tensor in the storage dtype."""
    import torch
    code = N.dtype_code() if code is None else code
    dt = N.torch_dtype(code)
    dev = torch.device("cuda", N.device_index(device))
    if isinstance(v, torch.Tensor):
        return v.to(dev, dt).contiguous()
    if isinstance(v, Volume):
        return v.device_tensor(dt, dev)
    if hasattr(v, "data") and isinstance(getattr(v, "data"), np.ndarray):  # reference Volume
        v = v.data
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev, dt)


def code_of(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return N.F64
    if t.dtype == torch.float32:
        return N.F32
    raise ValueError(f"unsupported device dtype {t.dtype}")


def psf_apply_dev(psf: Psf, x, adjoint: bool, out=None):
    """K4: H * x (adjoint=False) or H^T * x on the device."""
    import torch
    if tuple(x.shape) != tuple(psf.dims):
        raise ValueError(f"dims mismatch: volume {tuple(x.shape)} vs kernel {psf.dims}")
    dev = x.device.index
    ctx = N.context(dev)
    out = torch.empty_like(x) if out is None else out
    N.check(N.lib().sfw3d_psf_apply(ctx.handle, as_psf(psf).native(dev), code_of(x), N.ptr(x), N.ptr(out),
                                    1 if adjoint else 0))
    return out


def render_dev(rows: np.ndarray, dims, code: int | None = None, device=None, out=None):
    """K3: sum_i w_i G_i on the device (atoms summed in row order per voxel)."""
    import torch
    code = N.dtype_code() if code is None else code
    dev = N.device_index(device)
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
    if out is None:
        out = torch.empty(tuple(dims), dtype=N.torch_dtype(code), device=f"cuda:{dev}")
    ctx = N.context(dev)
    N.check(N.lib().sfw3d_render(ctx.handle, code, N.dims_arg(dims), N.f64_ptr(rows), rows.shape[0],
                                 N.ptr(out)))
    return out


def atom_sums_dev(field, rows: np.ndarray) -> np.ndarray:
    """K6/K7: raw (k, 6) inner products <P_c(atom), field> of unit atoms."""
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
    k = rows.shape[0]
    out = np.zeros((k, 6))
    if k == 0:
        return out
    ctx = N.context(field.device.index)
    N.check(N.lib().sfw3d_atom_sums(ctx.handle, code_of(field), N.dims_arg(field.shape),
                                    N.ptr(field), N.f64_ptr(rows), k, N.f64_ptr(out)))
    return out


def cost_grad_dev(psf: Psf, y, rows: np.ndarray, lam: float, want_grad: bool = True, back=None):
    """K3-K6 fused: (C, (k,6) gradient rows or None) against a device y."""
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
    k = rows.shape[0]
    dev = y.device.index
    ctx = N.context(dev)
    cost = C.c_double()
    grad = np.zeros((k, 6)) if want_grad else None
    N.check(N.lib().sfw3d_cost_grad(
        ctx.handle, as_psf(psf).native(dev), code_of(y), N.ptr(y), N.f64_ptr(rows), k, float(lam),
        C.byref(cost), N.f64_ptr(grad) if want_grad else None,
        N.ptr(back) if back is not None else None))
    return cost.value, grad


# ------------------------------------------------------------ public API
def convolve(v: Volume, psf: Psf) -> Volume:
    """Circular H * v (forward.py:79-87)."""
    if v.dims != psf.dims:
        raise ValueError(f"dims mismatch: volume {v.dims} vs kernel {psf.dims}")
    return Volume.from_device(psf_apply_dev(psf, to_dev(v), False))


def correlate_adjoint(v: Volume, psf: Psf) -> Volume:
    """Circular H^T * v (forward.py:90-94)."""
    if v.dims != psf.dims:
        raise ValueError(f"dims mismatch: volume {v.dims} vs kernel {psf.dims}")
    return Volume.from_device(psf_apply_dev(psf, to_dev(v), True))


def support_radius(sigma: float, d: float) -> int:
    """Radius beyond which the unit atom is below TAIL_CUTOFF (forward.py:97-99)."""
    return int(np.ceil(sigma * _TAIL_EXPONENT ** (1.0 / d)))


def render_atom(theta: AtomParams, w: float, geom: GridGeometry) -> Volume:
    """One weighted atom on the grid (forward.py:155-162)."""
    if not np.isfinite(w) or w < 0.0:
        raise ValueError(f"weight must be finite and >= 0, got {w}")
    if not (theta.sigma > 0.0 and theta.d > 0.0):
        raise ValueError(f"sigma and d must be positive, got {theta}")
    row = np.array([[float(w), *theta.m, theta.sigma, theta.d]])
    return Volume.from_device(render_dev(row, geom.dims))


def forward(measure: WeightedMeasure, psf: Psf, workers: int | None = None) -> Volume:
    """H * (sum of atoms) (forward.py:177-179)."""
    acc = render_dev(measure_rows(measure), psf.dims)
    return Volume.from_device(psf_apply_dev(psf, acc, False))


def criterion(y: Volume, measure: WeightedMeasure, psf: Psf, lam: float,
              workers: int | None = None) -> float:
    """0.5 ||y - H*sum w G||^2 + lam * sum w (forward.py:182-190)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    if y.dims != psf.dims:
        raise ValueError(f"dims mismatch: observation {y.dims} vs kernel {psf.dims}")
    c, _ = cost_grad_dev(psf, to_dev(y), measure_rows(measure), lam, want_grad=False)
    return c


@dataclass(frozen=True)
class CriterionGradient:
    """Per-atom derivative rows in GRADIENT_COLUMNS order, shape (k, 6)."""

    per_atom: np.ndarray

    def __post_init__(self):
        arr = np.asarray(self.per_atom, dtype=float)
        if arr.ndim != 2 or arr.shape[1] != len(GRADIENT_COLUMNS):
            raise ValueError(f"expected shape (k, 6), got {arr.shape}")
        object.__setattr__(self, "per_atom", arr)

    def flatten(self) -> np.ndarray:
        return self.per_atom.ravel()


def criterion_and_gradient(y: Volume, measure: WeightedMeasure, psf: Psf, lam: float,
                           workers: int | None = None,
                           y_hat: np.ndarray | None = None) -> tuple[float, CriterionGradient]:
    """Criterion and analytic gradient in one device pass (forward.py:232-257)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    if y.dims != psf.dims:
        raise ValueError(f"dims mismatch: observation {y.dims} vs kernel {psf.dims}")
    c, g = cost_grad_dev(psf, to_dev(y), measure_rows(measure), lam, want_grad=True)
    return c, CriterionGradient(g)


def criterion_gradient(y: Volume, measure: WeightedMeasure, psf: Psf, lam: float,
                       workers: int | None = None) -> CriterionGradient:
    return criterion_and_gradient(y, measure, psf, lam, workers)[1]


__all__ = [
    "TAIL_CUTOFF", "GRADIENT_COLUMNS", "Psf", "convolve", "correlate_adjoint", "support_radius",
    "render_atom", "forward", "criterion", "CriterionGradient", "criterion_and_gradient",
    "criterion_gradient", "total_mass",
]
