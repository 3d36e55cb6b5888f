"""Dual certificate on the B200: grid scan fused with argmax, then refinement.

Drop-in for ``sfw3d.certificate`` (certificate.py:1-236). The grid stage
(eta_field) is the K1 direct-correlation kernel over every voxel x
(sigma, d) candidate with the fused windowed argmax; only the argmax
records (and, on request, the fields) leave the device. The continuous
stage (refine_eta_max) keeps scipy's L-BFGS-B on the host, as the reference
does, and evaluates eta and its 5-gradient with the K7 device reduction
against a device-resident back-projection H^T r.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
from scipy.optimize import minimize

from . import _native as N
from .forward import Psf, as_psf, atom_sums_dev, psf_apply_dev, to_dev
from .measures import AtomParams, DomainBounds, bounds_box, clamp_to_domain
from .volumes import Volume

MODES = {"auto": 0, "direct": 1}


def make_parameter_grids(bounds: DomainBounds, n_sigma: int = 8,
                         n_shape: int = 6) -> tuple[np.ndarray, np.ndarray]:
    """Geometric sigma samples, linear shape samples (certificate.py:37-49)."""
    if n_sigma < 1 or n_shape < 1:
        raise ValueError("grid sizes must be >= 1")
    return (np.geomspace(bounds.sigma_min, bounds.sigma_max, n_sigma),
            np.linspace(bounds.shape_min, bounds.shape_max, n_shape))


class _TableHandle:
    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        try:
            if N._lib is not None and self.handle:
                N._lib.sfw3d_table_destroy(self.handle)
        except Exception:
            pass


class AtomTemplateTable:
    """Per (sigma, d) candidate, the unit atom at the origin, held on the device.

    certificate.py:52-62 stores rfftn(H * G_ij); this build keeps the spatial
    G_ij and the PSF (the correlation is factorised, see eta.cu), and
    materialises ``template_hats`` on the host only if someone reads it.
    """

    def __init__(self, sigma_grid, shape_grid, dims, psf: Psf, tap_tol: float, mode: str,
                 basis_tol: float, options: dict | None = None):
        self.sigma_grid = sigma_grid
        self.shape_grid = shape_grid
        self.dims = tuple(dims)
        self.psf = psf
        self.tap_tol = float(tap_tol)
        self.mode = mode
        self.basis_tol = float(basis_tol)
        # evaluator options (sfw3d_table_set_option): prune, loose_tol, refine_cap
        self.options = {k: float(v) for k, v in (options or {}).items() if v is not None}
        self._native = {}
        self._hats = None

    def native(self, device: int):
        h = self._native.get(device)
        if h is None:
            ctx = N.context(device)
            hp = C.c_void_p()
            sg = np.ascontiguousarray(self.sigma_grid, dtype=np.float64)
            dg = np.ascontiguousarray(self.shape_grid, dtype=np.float64)
            N.check(N.lib().sfw3d_table_create(ctx.handle, self.psf.native(device), sg.size,
                                               N.f64_ptr(sg), dg.size, N.f64_ptr(dg),
                                               self.tap_tol, MODES[self.mode], self.basis_tol,
                                               C.byref(hp)))
            h = _TableHandle(hp)
            for key, val in self.options.items():
                N.check(N.lib().sfw3d_table_set_option(hp, key.encode(), val))
            self._native[device] = h
        return h.handle

    def info(self, device=None, precision: str | None = None) -> dict:
        """Evaluator split and executed taps per voxel for a storage precision."""
        code = N.dtype_code(precision)
        h = self.native(N.device_index(device))
        nc, nd, nb = C.c_int(), C.c_int(), C.c_int()
        dt, bt = C.c_int64(), C.c_int64()
        df, bf = C.c_double(), C.c_double()
        N.check(N.lib().sfw3d_table_info(h, code, C.byref(nc), C.byref(nd), C.byref(nb),
                                         C.byref(dt), C.byref(bt), C.byref(df), C.byref(bf)))
        cands = []
        for i in range(nc.value):
            ub, nt, fe, fl = C.c_int(), C.c_int(), C.c_double(), C.c_double()
            cdt, cbt = C.c_int64(), C.c_int64()
            N.check(N.lib().sfw3d_table_candidate(h, code, i, C.byref(ub), C.byref(nt),
                                                  C.byref(fe), C.byref(cdt), C.byref(cbt),
                                                  C.byref(fl)))
            s, d = divmod(i, len(self.shape_grid))
            cands.append({"sigma": float(self.sigma_grid[s]), "d": float(self.shape_grid[d]),
                          "path": ("direct", "basis", "basis+refine")[ub.value],
                          "terms": nt.value,
                          "fit_err": fe.value, "direct_taps": cdt.value, "basis_taps": cbt.value,
                          "flops_per_voxel": fl.value})
        npass = C.c_int()
        N.check(N.lib().sfw3d_table_basis_passes(h, code, 0, None, C.byref(npass)))
        ptaps = np.zeros(max(npass.value, 1), dtype=np.int32)
        N.check(N.lib().sfw3d_table_basis_passes(h, code, npass.value, N.i32_ptr(ptaps),
                                                 C.byref(npass)))
        return {"n_cand": nc.value, "n_direct": nd.value, "n_basis": nb.value,
                "basis_pass_taps": [int(v) for v in ptaps[:npass.value]],
                "direct_taps_per_voxel": dt.value, "basis_taps_per_voxel": bt.value,
                "direct_flops_per_voxel": df.value, "basis_flops_per_voxel": bf.value,
                "candidates": cands}

    @property
    def template_hats(self) -> np.ndarray:
        """Reference representation (n_sigma, n_shape, rfft dims), computed lazily."""
        if self._hats is None:
            import scipy.fft as sfft
            from .forward import _warn_host_fft
            _warn_host_fft("AtomTemplateTable.template_hats", self.dims)
            from .forward import render_dev  # device render, then host FFT (compatibility only)
            out = []
            for s in self.sigma_grid:
                for d in self.shape_grid:
                    atom = render_dev(np.array([[1.0, 0.0, 0.0, 0.0, s, d]]), self.dims, N.F64)
                    out.append(sfft.rfftn(atom.cpu().numpy()) * self.psf.kernel_hat)
            self._hats = np.stack(out).reshape(len(self.sigma_grid), len(self.shape_grid),
                                               *out[0].shape)
        return self._hats

    def entry(self, i_sigma: int, i_shape: int) -> np.ndarray:
        return self.template_hats[i_sigma, i_shape]


def build_template_table(psf: Psf, sigma_grid, shape_grid, bounds: DomainBounds | None = None,
                         workers: int | None = None, *, tap_tol: float = 0.0,
                         mode: str = "auto", basis_tol: float = 1e-9, prune: bool | None = None,
                         global_voxels: int | None = None, loose_tol: float | None = None,
                         refine_cap: int | None = None) -> AtomTemplateTable:
    """Candidate table for the (sigma, d) grid (certificate.py:65-97).

    Keyword-only extras: ``tap_tol`` skips template taps below it (0 keeps
    the reference's full 1e-12 support box); ``mode`` "auto" lets the
    library pick the fastest exact-to-``basis_tol`` evaluation per
    candidate, "direct" forces direct correlation. ``prune`` / ``global_voxels``
    (the voxel count of the default pruning rule) / ``loose_tol`` / ``refine_cap`` tune the shared separable basis (sfw3d_table_set_option;
    None keeps the library default: pruning by volume size, fp32 term
    selection at 1e-5, 65536 exactly re-evaluated voxels per call).
    """
    psf = as_psf(psf)
    sigma_grid = np.sort(np.asarray(sigma_grid, dtype=float))
    shape_grid = np.sort(np.asarray(shape_grid, dtype=float))
    if sigma_grid.size == 0 or shape_grid.size == 0:
        raise ValueError("parameter grids must be non-empty")
    if bounds is not None:
        if not (bounds.sigma_min <= sigma_grid[0] and sigma_grid[-1] <= bounds.sigma_max):
            raise ValueError("sigma grid extends outside the domain bounds")
        if not (bounds.shape_min <= shape_grid[0] and shape_grid[-1] <= bounds.shape_max):
            raise ValueError("shape grid extends outside the domain bounds")
    if not psf.is_centrosymmetric():
        raise ValueError("template table requires a centro-symmetric kernel")
    if mode not in MODES:
        raise ValueError(f"mode must be one of {sorted(MODES)}")
    opts = {"prune": None if prune is None else int(bool(prune)),
            "global_voxels": global_voxels, "loose_tol": loose_tol,
            "refine_cap": refine_cap}
    # Tables are immutable values: the same (kernel, grids, options) gives the
    # same table, so it is built once per Psf object and handed out again (a
    # solver called after lambda = c * max eta, or a regularisation path,
    # asks for the table it already has; config 3: 0.3 s of host work).
    cache = psf.__dict__.setdefault("_tables", {})
    key = (sigma_grid.tobytes(), shape_grid.tobytes(), float(tap_tol), mode, float(basis_tol),
           tuple(sorted((k, v) for k, v in opts.items() if v is not None)))
    table = cache.get(key)
    if table is None:
        table = AtomTemplateTable(sigma_grid, shape_grid, psf.dims, psf, tap_tol, mode, basis_tol,
                                  opts)
        if len(cache) >= 8:
            cache.pop(next(iter(cache)))
        cache[key] = table
    table.native(N.device_index(None))
    return table


def _position_window(bounds: DomainBounds | None, dims):
    """Integer box [ceil(lo), floor(hi)] clipped to the grid (certificate.py:100-111)."""
    if bounds is None:
        return tuple((0, n - 1) for n in dims)
    out = []
    for lo, hi, n in zip(bounds.pos_lower, bounds.pos_upper, dims):
        a, b = max(0, int(np.ceil(lo))), min(n - 1, int(np.floor(hi)))
        if a > b:
            raise ValueError("domain position bounds contain no integer grid point")
        out.append((a, b))
    return tuple(out)


@dataclass(frozen=True, eq=False)
class CertificateField:
    """Discrete argmax of eta over positions x (sigma, d), plus optional fields."""

    sigma_grid: np.ndarray
    shape_grid: np.ndarray
    argmax_position: tuple[int, int, int]
    argmax_sigma_index: int
    argmax_shape_index: int
    eta_max: float
    fields: tuple[Volume, ...] | None = None

    @property
    def argmax_params(self) -> AtomParams:
        return AtomParams(m=tuple(float(i) for i in self.argmax_position),
                          sigma=float(self.sigma_grid[self.argmax_sigma_index]),
                          d=float(self.shape_grid[self.argmax_shape_index]))


def eta_argmax_dev(residual, lam: float, table: AtomTemplateTable, window, keep_fields=False):
    """K1 on a device residual: (best Argmax, per-candidate list, fields tensor|None)."""
    import torch
    dev = residual.device.index
    ctx = N.context(dev)
    nc = len(table.sigma_grid) * len(table.shape_grid)
    win = np.array([v for ab in window for v in ab], dtype=np.int32)
    best = N.Argmax()
    per = (N.Argmax * nc)()
    fields = None
    if keep_fields:
        fields = torch.empty((nc, *table.dims), dtype=residual.dtype, device=residual.device)
    from .forward import code_of
    N.check(N.lib().sfw3d_eta_argmax(ctx.handle, table.native(dev), code_of(residual),
                                     N.ptr(residual), float(lam), N.i32_ptr(win), C.byref(best),
                                     per, N.ptr(fields) if fields is not None else None))
    return best, [per[i] for i in range(nc)], fields


def eta_field(residual: Volume, lam: float, table: AtomTemplateTable,
              bounds: DomainBounds | None = None, keep_fields: bool = True,
              workers: int | None = None) -> CertificateField:
    """eta at every integer position for each table entry (certificate.py:140-184)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    if residual.dims != table.dims:
        raise ValueError(f"dims mismatch: residual {residual.dims} vs table {table.dims}")
    return eta_field_dev(to_dev(residual), lam, table, bounds, keep_fields)


def eta_field_dev(residual, lam: float, table: AtomTemplateTable,
                  bounds: DomainBounds | None = None, keep_fields: bool = False) -> CertificateField:
    window = _position_window(bounds, table.dims)
    best, _, fields = eta_argmax_dev(residual, lam, table, window, keep_fields)
    i, j = divmod(int(best.cand), len(table.shape_grid))
    kept = None
    if keep_fields:
        host = fields.to("cpu", dtype=__import__("torch").float64).numpy()
        kept = tuple(Volume(host[c]) for c in range(host.shape[0]))
    return CertificateField(sigma_grid=table.sigma_grid, shape_grid=table.shape_grid,
                            argmax_position=tuple(int(p) for p in best.pos),
                            argmax_sigma_index=i, argmax_shape_index=j,
                            eta_max=float(best.value), fields=kept)


def refine_eta_max(residual: Volume, lam: float, psf: Psf, start: AtomParams,
                   bounds: DomainBounds, max_iter: int = 200,
                   gtol: float = 1e-8) -> tuple[AtomParams, float]:
    """Box-constrained L-BFGS-B ascent of eta from a grid seed (certificate.py:187-224)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    return refine_eta_max_dev(to_dev(residual), lam, psf, start, bounds, max_iter, gtol)


def refine_eta_max_dev(residual, lam: float, psf: Psf, start: AtomParams, bounds: DomainBounds,
                       max_iter: int = 200, gtol: float = 1e-8, back=None, info: dict | None = None):
    """The ascent as ONE C call (sfw3d_refine_eta_max): the in-library L-BFGS-B
    (scipy's algorithm and driver conventions, csrc/lbfgsb.cuh) evaluates eta
    and its 5-gradient with the device atom-sum kernel per step; no Python
    callback. `N.OPTIMIZER = "scipy"` selects the reference's own scipy loop
    over the same device evaluations (the cross-check of the tests)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    start = clamp_to_domain(start, bounds)
    if back is None:
        back = psf_apply_dev(psf, residual, True)
    from .forward import code_of
    ctx = N.context(back.device.index)
    if N.OPTIMIZER == "scipy":
        return _refine_scipy(ctx, back, lam, start, bounds, max_iter, gtol)
    box = np.array(bounds_box(bounds), dtype=np.float64)
    lo, hi = np.ascontiguousarray(box[:, 0]), np.ascontiguousarray(box[:, 1])
    x0 = np.ascontiguousarray(start.to_array(), dtype=np.float64)
    theta = np.empty(5)
    eta = C.c_double()
    stat = (C.c_int32 * 3)()
    N.check(N.lib().sfw3d_refine_eta_max(ctx.handle, code_of(back), N.dims_arg(back.shape),
                                         N.ptr(back), float(lam), N.f64_ptr(x0), N.f64_ptr(lo),
                                         N.f64_ptr(hi), int(max_iter), float(gtol),
                                         N.f64_ptr(theta), C.byref(eta), stat))
    if info is not None:
        info["lbfgsb"] = {"status": int(stat[0]), "iterations": int(stat[1]),
                          "evaluations": int(stat[2])}
    return clamp_to_domain(AtomParams.from_array(theta), bounds), float(eta.value)


def refine_eta_max_multistart(residual, lam: float, psf: Psf, starts, bounds: DomainBounds,
                              max_iter: int = 200, gtol: float = 1e-8, back=None):
    """Batched multi-start ascent: every start runs its own
    in-library L-BFGS-B on its own CUDA stream / library context from a host
    thread (the C calls release the GIL), all against ONE back-projection
    H^T r; the best refined (theta, eta) wins, ties to the earlier start. Not
    the reference's semantics — it refines only the grid argmax
    (certificate.py:227-236) — so the solvers do not use it by default; it is
    the tool for callers who want the ascent to escape a poor grid seed."""
    import threading
    import torch
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    starts = list(starts)
    if not starts:
        raise ValueError("at least one start is required")
    if back is None:
        back = psf_apply_dev(psf, residual, True)
    dev = back.device
    ready = torch.cuda.Event()
    ready.record(torch.cuda.current_stream(dev))
    out, err = [None] * len(starts), []

    def run(i):
        try:
            stream = torch.cuda.Stream(dev)
            with torch.cuda.stream(stream):
                stream.wait_event(ready)
                out[i] = refine_eta_max_dev(residual, lam, psf, starts[i], bounds, max_iter, gtol,
                                            back=back)
        except BaseException as exc:
            err.append(exc)

    threads = [threading.Thread(target=run, args=(i,)) for i in range(len(starts))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if err:
        raise err[0]
    best = 0
    for i in range(1, len(out)):
        if out[i][1] > out[best][1]:
            best = i
    return out[best]


def _refine_scipy(ctx, back, lam, start, bounds, max_iter, gtol):
    """certificate.py:201-224 with scipy's L-BFGS-B driving the device evaluations."""
    from .forward import code_of
    fn, handle, code = N.lib().sfw3d_atom_sums, ctx.handle, code_of(back)
    dims_a, bptr = N.dims_arg(back.shape), N.ptr(back)
    row = np.empty((1, 6))
    row[0, 0] = 1.0
    out = np.empty((1, 6))
    row_p, out_p = N.f64_ptr(row), N.f64_ptr(out)

    def neg_eta(vec):
        row[0, 1:] = vec
        N.check(fn(handle, code, dims_a, bptr, row_p, 1, out_p))
        s = out[0]
        val = float(s[0]) / lam
        grad = s[1:] / lam
        if not (np.isfinite(val) and np.isfinite(grad).all()):
            raise FloatingPointError(f"non-finite certificate value near {vec}")
        return -val, -grad

    box = bounds_box(bounds)
    start_val = -neg_eta(start.to_array())[0]
    res = minimize(neg_eta, start.to_array(), jac=True, method="L-BFGS-B", bounds=box,
                   options={"maxiter": max_iter, "gtol": gtol})
    if not np.isfinite(res.fun):
        raise FloatingPointError("certificate ascent diverged to a non-finite value")
    if -res.fun < start_val:
        return start, start_val
    return clamp_to_domain(AtomParams.from_array(res.x), bounds), float(-res.fun)


def certificate_max(residual: Volume, lam: float, table: AtomTemplateTable, psf: Psf,
                    bounds: DomainBounds, workers: int | None = None) -> tuple[AtomParams, float]:
    """Grid scan then continuous refinement (certificate.py:227-236)."""
    if lam <= 0.0:
        raise ValueError(f"lam must be > 0, got {lam}")
    if residual.dims != table.dims:
        raise ValueError(f"dims mismatch: residual {residual.dims} vs table {table.dims}")
    return certificate_max_dev(to_dev(residual), lam, table, psf, bounds)


def certificate_max_multistart_dev(residual, lam, table, psf, bounds, n_starts: int = 4):
    """Grid scan, then the batched multi-start ascent from the n_starts best
    per-candidate grid maxima (the reference's single start is the first)."""
    window = _position_window(bounds, table.dims)
    best, per, _ = eta_argmax_dev(residual, lam, table, window)
    nd = len(table.shape_grid)
    order = sorted(range(len(per)), key=lambda c: (-per[c].value, c))
    order = [int(best.cand)] + [c for c in order if c != int(best.cand)]
    starts = [AtomParams(m=tuple(float(v) for v in per[c].pos),
                         sigma=float(table.sigma_grid[c // nd]), d=float(table.shape_grid[c % nd]))
              for c in order[:max(1, n_starts)]]
    return refine_eta_max_multistart(residual, lam, psf, starts, bounds)


def certificate_max_dev(residual, lam, table, psf, bounds, info: dict | None = None):
    """Grid argmax then refinement on a device residual; `info` (optional)
    receives the grid seed ("start", "eta_grid") for step-level replays."""
    field = eta_field_dev(residual, lam, table, bounds, keep_fields=False)
    if info is not None:
        info["start"] = field.argmax_params
        info["eta_grid"] = field.eta_max
        info["cand"] = (field.argmax_sigma_index, field.argmax_shape_index)
    return refine_eta_max_dev(residual, lam, psf, field.argmax_params, bounds)
