"""ctypes binding of the sm_100a C-ABI library ``_lib/libsfw3d_cuda.so``.

The library is the only compute path: there is no CPU fallback. Importing
this module never touches the GPU (so CPU-only tests can check that the
library loads and exports every symbol of ``include/sfw3d_cuda.h``); the
first call that needs a device raises ``RuntimeError`` when CUDA is absent.
Status codes map to the reference's exceptions:
EINVAL -> ValueError, ENONFINITE -> FloatingPointError.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import threading
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libsfw3d_cuda.so"

SFW3D_OK, SFW3D_EINVAL, SFW3D_ENONFINITE, SFW3D_ECUDA, SFW3D_ENOMEM = range(5)
F32, F64 = 0, 1

# every symbol include/sfw3d_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "sfw3d_abi_version", "sfw3d_last_error", "sfw3d_ctx_create", "sfw3d_ctx_destroy",
    "sfw3d_ctx_sync", "sfw3d_ctx_launches", "sfw3d_atom_geometry", "sfw3d_psf_create",
    "sfw3d_psf_info", "sfw3d_psf_destroy", "sfw3d_psf_apply", "sfw3d_render",
    "sfw3d_atom_sums", "sfw3d_cost_grad", "sfw3d_cost_grad_slab", "sfw3d_table_create", "sfw3d_table_info",
    "sfw3d_table_destroy", "sfw3d_eta_argmax", "sfw3d_dots", "sfw3d_nnlasso_cd", "sfw3d_nnlasso_qp",
    "sfw3d_residual", "sfw3d_ctx_profile", "sfw3d_ctx_profile_read", "sfw3d_probe_fp32",
    "sfw3d_table_candidate", "sfw3d_basis_fit", "sfw3d_basis_set_fit",
    "sfw3d_last_refine_count", "sfw3d_table_set_option", "sfw3d_eta_argmax_slab",
    "sfw3d_cost_grad_slab_dev", "sfw3d_render_slab", "sfw3d_atom_sums_slab",
    "sfw3d_volume_info", "sfw3d_volume_read", "sfw3d_volume_write",
    "sfw3d_lbfgsb_minimize", "sfw3d_refine_eta_max", "sfw3d_local_descent", "sfw3d_solve",
    "sfw3d_residual_ranged", "sfw3d_table_basis_passes",
)


class Argmax(C.Structure):
    _fields_ = [("pos", C.c_int32 * 3), ("cand", C.c_int32), ("value", C.c_double)]


_vp = C.c_void_p
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_dp = C.POINTER(C.c_double)

# x-slab data plane callbacks (include/sfw3d_cuda.h: sfw3d_halo_fn, sfw3d_allreduce_fn)
HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int,
                      C.c_int)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int)

class SolveOptions(C.Structure):
    """sfw3d_solve_options (include/sfw3d_cuda.h)."""
    _fields_ = [("lam", C.c_double), ("max_outer_iterations", C.c_int32), ("boosted", C.c_int32),
                ("eta_threshold", C.c_double), ("eta_slack", C.c_double), ("lasso_tol", C.c_double),
                ("lasso_max_iter", C.c_int32), ("descent_max_iter", C.c_int32),
                ("descent_gtol", C.c_double), ("descent_ftol", C.c_double),
                ("prune_rel_tol", C.c_double), ("duplicate_tol", C.c_double),
                ("lower", C.c_double * 5), ("upper", C.c_double * 5), ("window", C.c_int32 * 6),
                ("n_sigma", C.c_int32), ("n_shape", C.c_int32),
                ("sigma_grid", C.POINTER(C.c_double)), ("shape_grid", C.POINTER(C.c_double))]


class SolveRecord(C.Structure):
    """sfw3d_solve_record (include/sfw3d_cuda.h)."""
    _fields_ = [("index", C.c_int32), ("eta_max", C.c_double), ("criterion_before", C.c_double),
                ("criterion_after_lasso", C.c_double), ("criterion_after_descent", C.c_double),
                ("atom_count", C.c_int32), ("t_certificate", C.c_double), ("t_lasso", C.c_double),
                ("t_descent", C.c_double)]


# objective callback of the in-library L-BFGS-B (include/sfw3d_cuda.h: sfw3d_objective_fn)
OBJECTIVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                           C.POINTER(C.c_double))

_SIGNATURES = {
    "sfw3d_table_basis_passes": (C.c_int, [_vp, C.c_int, C.c_int, _i32p, _ip]),
    "sfw3d_residual_ranged": (C.c_int, [_vp, C.c_int, _ip, _vp, C.POINTER(_vp), _dp, _i32p, C.c_int,
                                        _vp, _dp]),
    "sfw3d_solve": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp, C.POINTER(SolveOptions), _vp, C.c_int, _dp,
                              _ip, _dp, _ip, C.POINTER(SolveRecord), _ip]),
    "sfw3d_lbfgsb_minimize": (C.c_int, [C.c_int, _dp, _dp, _dp, _i32p, C.c_int, C.c_double,
                                        C.c_double, C.c_int, C.c_int, C.c_int, OBJECTIVE_FN, _vp,
                                        _dp, _i32p]),
    "sfw3d_refine_eta_max": (C.c_int, [_vp, C.c_int, _ip, _vp, C.c_double, _dp, _dp, _dp, C.c_int,
                                       C.c_double, _dp, _dp, _i32p]),
    "sfw3d_local_descent": (C.c_int, [_vp, _vp, C.c_int, _vp, _dp, C.c_int, C.c_double, _dp, _dp,
                                      C.c_double, C.c_double, C.c_int, _dp, _i32p]),
    "sfw3d_abi_version": (C.c_int, []),
    "sfw3d_last_error": (C.c_char_p, []),
    "sfw3d_last_refine_count": (C.c_int, []),
    "sfw3d_ctx_create": (C.c_int, [C.c_int, _vp, C.POINTER(_vp)]),
    "sfw3d_ctx_destroy": (C.c_int, [_vp]),
    "sfw3d_ctx_sync": (C.c_int, [_vp]),
    "sfw3d_ctx_launches": (C.c_int64, [_vp]),
    "sfw3d_atom_geometry": (C.c_int, [_ip, _dp, C.c_int, _i32p, _i32p, _i32p, _i32p]),
    "sfw3d_psf_create": (C.c_int, [_vp, _ip, _dp, C.POINTER(_vp)]),
    "sfw3d_psf_info": (C.c_int, [_vp, _ip, _i32p, _i32p]),
    "sfw3d_psf_destroy": (C.c_int, [_vp]),
    "sfw3d_psf_apply": (C.c_int, [_vp, _vp, C.c_int, _vp, _vp, C.c_int]),
    "sfw3d_render": (C.c_int, [_vp, C.c_int, _ip, _dp, C.c_int, _vp]),
    "sfw3d_atom_sums": (C.c_int, [_vp, C.c_int, _ip, _vp, _dp, C.c_int, _dp]),
    "sfw3d_cost_grad": (C.c_int, [_vp, _vp, C.c_int, _vp, _dp, C.c_int, C.c_double, _dp, _dp, _vp]),
    "sfw3d_cost_grad_slab": (C.c_int, [_vp, _vp, C.c_int, _vp, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, _dp, _dp]),
    "sfw3d_cost_grad_slab_dev": (C.c_int, [_vp, _vp, C.c_int, _vp, _dp, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, _vp]),
    "sfw3d_render_slab": (C.c_int, [_vp, C.c_int, _ip, _dp, C.c_int, C.c_int, C.c_int, C.c_int, _vp]),
    "sfw3d_atom_sums_slab": (C.c_int, [_vp, C.c_int, _ip, _vp, _dp, C.c_int, C.c_int, C.c_int, C.c_int,
                                       _dp]),
    "sfw3d_volume_info": (C.c_int, [C.c_char_p, _i32p]),
    "sfw3d_volume_read": (C.c_int, [_vp, C.c_char_p, C.c_int, _vp]),
    "sfw3d_volume_write": (C.c_int, [_vp, C.c_char_p, C.c_int, _ip, _vp]),
    "sfw3d_table_create": (C.c_int, [_vp, _vp, C.c_int, _dp, C.c_int, _dp, C.c_double, C.c_int,
                                     C.c_double, C.POINTER(_vp)]),
    "sfw3d_table_info": (C.c_int, [_vp, C.c_int, _ip, _ip, _ip, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64), _dp, _dp]),
    "sfw3d_table_candidate": (C.c_int, [_vp, C.c_int, C.c_int, _ip, _ip, _dp, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), _dp]),
    "sfw3d_table_destroy": (C.c_int, [_vp]),
    "sfw3d_table_set_option": (C.c_int, [_vp, C.c_char_p, C.c_double]),
    "sfw3d_eta_argmax": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_double, _i32p, C.POINTER(Argmax),
                                   C.POINTER(Argmax), _vp]),
    "sfw3d_eta_argmax_slab": (C.c_int, [_vp, _vp, C.c_int, _vp, C.c_int, C.c_int, C.c_double, _i32p,
                                        HALO_FN, ALLREDUCE_FN, _vp, C.POINTER(Argmax),
                                        C.POINTER(Argmax)]),
    "sfw3d_dots": (C.c_int, [_vp, C.c_int, C.c_int64, C.POINTER(_vp), C.c_int, _vp, _dp]),
    "sfw3d_nnlasso_cd": (C.c_int, [_vp, C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_int, _dp,
                                   _i32p, _dp]),
    "sfw3d_nnlasso_qp": (C.c_int, [_vp, C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_int, _dp,
                                   _i32p, _dp]),
    "sfw3d_residual": (C.c_int, [_vp, C.c_int, C.c_int64, _vp, C.POINTER(_vp), _dp, C.c_int, _vp,
                                 _dp]),
    "sfw3d_basis_fit": (C.c_int, [_i32p, _i32p, C.c_double, C.c_double, C.c_int, _dp, _dp, _dp,
                                  _ip, _dp]),
    "sfw3d_basis_set_fit": (C.c_int, [_ip, C.c_int, _dp, C.c_int, _dp, C.c_int, C.c_double,
                                      C.c_int, C.c_double, C.c_int, _ip, _dp, _dp, _dp, _dp,
                                      _i32p]),
    "sfw3d_ctx_profile": (C.c_int, [_vp, C.c_int]),
    "sfw3d_ctx_profile_read": (C.c_int, [_vp, C.c_char_p, _dp, C.POINTER(C.c_int64)]),
    "sfw3d_probe_fp32": (C.c_int, [_vp, _dp]),
}

_lib = None

# "native": refine_eta_max / local_descent run the in-library L-BFGS-B (one C
# call per optimisation); "scipy": the reference's scipy.optimize loop over the
# same device evaluations (kept as the cross-check of the parity tests)
OPTIMIZER = "native"

# "native": sfw / bsfw run the whole outer loop inside the library (sfw3d_solve);
# "python": the host loop of solvers._solve over the same device calls (also
# taken when a step record is requested or OPTIMIZER is "scipy")
SOLVER = "native"
_lib_lock = threading.Lock()


def lib():
    """Load the CUDA library (raises loudly when it was not built)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not _LIB_PATH.exists():
                    raise RuntimeError(
                        f"sfw3d CUDA library not built: {_LIB_PATH} is missing "
                        "(run `make` or __graft_entry__.build()); there is no CPU fallback")
                handle = C.CDLL(str(_LIB_PATH))
                for name, (res, args) in _SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def lib_path() -> Path:
    return _LIB_PATH


def check(status: int) -> None:
    if status == SFW3D_OK:
        return
    msg = lib().sfw3d_last_error().decode(errors="replace")
    if status == SFW3D_EINVAL:
        raise ValueError(msg)
    if status == SFW3D_ENONFINITE:
        raise FloatingPointError(msg)
    if status == SFW3D_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def dims_arg(dims) -> "C.Array":
    return (C.c_int * 3)(*[int(n) for n in dims])


def f64_ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def i32_ptr(a: np.ndarray):
    return a.ctypes.data_as(_i32p)


def atom_geometry(dims, params: np.ndarray):
    """Host-only: support radius / box per atom exactly as forward.py:97-116."""
    p = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 6)
    k = p.shape[0]
    radius = np.zeros(k, np.int32)
    start = np.zeros((k, 3), np.int32)
    length = np.zeros((k, 3), np.int32)
    full = np.zeros((k, 3), np.int32)
    check(lib().sfw3d_atom_geometry(dims_arg(dims), f64_ptr(p), k, i32_ptr(radius),
                                    i32_ptr(start), i32_ptr(length), i32_ptr(full)))
    return radius, start, length, full


def basis_fit(lo, hi, sigma: float, d: float):
    """Host-only: (betas, weights, w0, max abs error) of the certificate basis fit."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    hi = np.ascontiguousarray(hi, dtype=np.int32)
    betas = np.zeros(64)
    weights = np.zeros(64)
    w0, err = C.c_double(), C.c_double()
    nt = C.c_int()
    check(lib().sfw3d_basis_fit(i32_ptr(lo), i32_ptr(hi), float(sigma), float(d), 64,
                                f64_ptr(betas), f64_ptr(weights), C.byref(w0), C.byref(nt),
                                C.byref(err)))
    k = min(nt.value, 64)
    return betas[:k], weights[:k], w0.value, err.value


def basis_set_fit(dims, sigmas, shapes, dtype: int, tol: float, max_terms: int = 256,
                  prune: int = -1, loose_tol: float = -1.0):
    """Host-only: the shared separable basis a table fits for the candidate
    grid (sigma-major): dict(betas [T], weights [C, T], w0 [C], fit_err [C],
    member [C] bool). prune / loose_tol as sfw3d_table_set_option (-1 = default)."""
    sg = np.ascontiguousarray(sigmas, dtype=np.float64)
    sh = np.ascontiguousarray(shapes, dtype=np.float64)
    nc = sg.size * sh.size
    betas = np.zeros(max_terms)
    weights = np.zeros((nc, max_terms))
    w0, err = np.zeros(nc), np.zeros(nc)
    member = np.zeros(nc, np.int32)
    nt = C.c_int()
    check(lib().sfw3d_basis_set_fit(dims_arg(dims), sg.size, f64_ptr(sg), sh.size, f64_ptr(sh),
                                    int(dtype), float(tol), int(prune), float(loose_tol),
                                    max_terms, C.byref(nt),
                                    f64_ptr(betas), f64_ptr(weights), f64_ptr(w0), f64_ptr(err),
                                    i32_ptr(member)))
    if nt.value > max_terms:
        raise ValueError(f"shared basis has {nt.value} terms > max_terms={max_terms}")
    k = nt.value
    return {"betas": betas[:k], "weights": weights[:, :k], "w0": w0, "fit_err": err,
            "member": member.astype(bool), "signed": member == 2}


# ------------------------------------------------------------------ devices
_state = threading.local()


def _torch():
    import torch
    return torch


def device_index(device=None) -> int:
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the sfw3d B200 path has no CPU fallback")
    if device is None:
        return torch.cuda.current_device()
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"not a CUDA device: {device!r}")
    return d.index if d.index is not None else torch.cuda.current_device()


class Context:
    """One C context per (device, stream); owns the library workspace."""

    def __init__(self, device: int, stream):
        self.device = device
        self.stream = stream
        h = _vp()
        check(lib().sfw3d_ctx_create(device, _vp(stream.cuda_stream), C.byref(h)))
        self.handle = h

    def sync(self):
        check(lib().sfw3d_ctx_sync(self.handle))

    @property
    def launches(self) -> int:
        return int(lib().sfw3d_ctx_launches(self.handle))

    def profile(self, enable: bool = True) -> None:
        """Enable (and reset) per-kernel-family CUDA-event timing."""
        check(lib().sfw3d_ctx_profile(self.handle, 1 if enable else 0))

    def profile_read(self, family: str) -> tuple[float, int]:
        """(total device ms, launches) of one kernel family since the reset."""
        ms = C.c_double()
        n = C.c_int64()
        check(lib().sfw3d_ctx_profile_read(self.handle, family.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def probe_fp32(self) -> float:
        """Measured FP32 FFMA peak of the device in TFLOP/s."""
        t = C.c_double()
        check(lib().sfw3d_probe_fp32(self.handle, C.byref(t)))
        return t.value

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.sfw3d_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict = {}


def context(device=None) -> Context:
    torch = _torch()
    dev = device_index(device)
    stream = torch.cuda.current_stream(dev)
    key = (dev, stream.cuda_stream)
    ctx = _contexts.get(key)
    if ctx is None:
        ctx = Context(dev, stream)
        _contexts[key] = ctx
    return ctx


def last_refine_count() -> int:
    """Voxels this thread's last certificate evaluation re-evaluated exactly."""
    return int(lib().sfw3d_last_refine_count())


def total_launches() -> int:
    return sum(c.launches for c in _contexts.values())


# ----------------------------------------------------------------- precision
_PRECISION = {"f64": F64, "f32": F32}
_precision_default = ["f64"]


def set_precision(name: str) -> None:
    """Storage precision of device volumes: "f64" (reference parity, default)
    or "f32" (fp32 storage, fp64 reductions; BASELINE configs 3-5)."""
    if name not in _PRECISION:
        raise ValueError("precision must be 'f64' or 'f32'")
    _precision_default[0] = name


def get_precision() -> str:
    return _precision_default[0]


@contextlib.contextmanager
def precision(name: str):
    old = get_precision()
    set_precision(name)
    try:
        yield
    finally:
        set_precision(old)


def dtype_code(name: str | None = None) -> int:
    return _PRECISION[name or get_precision()]


def torch_dtype(code: int):
    torch = _torch()
    return torch.float64 if code == F64 else torch.float32


def ptr(t) -> _vp:
    return _vp(t.data_ptr())

