"""Multi-GPU sharding of the hot path: one process per GPU.

Plumbing is torch.distributed (NCCL on the B200 box; gloo in the CPU tests).
What shards and which exchanges exist:

* certificate — the output grid is split into x-slabs (axis 0, the slowest
  axis). With a replicated residual every rank evaluates eta on its slab
  only (a window restriction, no halo needed) and the single collective is an
  all-gather of one 24-byte argmax record per rank, reduced with the
  reference's order (larger eta, then smaller sigma-major candidate, then
  smaller C-order position: certificate.py:161-172). With a slab-distributed
  residual the ranks first exchange periodic halos of the template radius.
* cost + gradient — atoms are split across ranks for the per-atom box
  reductions (K6, the dominant kernel at config 5) and the rows are
  all-gathered; the criterion value is computed once per rank (replicated
  volumes). Slab-local rendering is listed as next work in DESIGN.md.
* sums (Gram rows, ||r||^2) — fp64 all-reduce.

The functions take a `compute` callable where the per-rank work happens so
the same exchange logic runs with the CUDA kernels on the GPU and with the
CPU oracle in the gloo tests.
"""

from __future__ import annotations

import numpy as np


def _dist():
    import torch.distributed as dist
    return dist


def world():
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def slab_bounds(n: int, size: int, rank: int) -> tuple[int, int]:
    """Inclusive [x0, x1] of rank's x-slab; sizes differ by at most one plane."""
    if not 0 <= rank < size or n < size:
        raise ValueError("need 0 <= rank < size <= n")
    base, extra = divmod(n, size)
    x0 = rank * base + min(rank, extra)
    return x0, x0 + base + (1 if rank < extra else 0) - 1


def better(a, b) -> bool:
    """Total order of argmax records (value, cand, lin): eta desc, cand asc, lin asc."""
    if a[0] != b[0]:
        return a[0] > b[0]
    if a[1] != b[1]:
        return a[1] < b[1]
    return a[2] < b[2]


def combine_best(records):
    best = None
    for r in records:
        if r[0] != r[0]:  # NaN never wins
            continue
        if best is None or better(r, best):
            best = r
    return best


def allgather_best(record, group=None, device=None):
    """All-gather (value, cand, lin) records and return the global winner."""
    import torch
    dist = _dist()
    size = dist.get_world_size(group)
    t = torch.tensor([float(record[0]), float(record[1]), float(record[2])], dtype=torch.float64,
                     device=device)
    out = [torch.empty_like(t) for _ in range(size)]
    dist.all_gather(out, t, group=group)
    recs = [(float(o[0]), int(o[1]), int(o[2])) for o in (x.cpu() for x in out)]
    return combine_best(recs)


def allreduce_f64(values, group=None, device=None) -> np.ndarray:
    """Sum of float64 arrays over ranks (rank order does not matter for the
    tests' tolerance; NCCL's ring order is fixed for a fixed world size)."""
    import torch
    dist = _dist()
    t = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=device).clone()
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def halo_exchange(slab, halo: int, group=None):
    """Fill the periodic halos of an x-slab in place.

    `slab` has shape (n_local + 2*halo, ...): planes [halo, halo + n_local)
    are owned. Planes [0, halo) receive the left neighbour's last `halo`
    owned planes and [halo + n_local, end) the right neighbour's first ones
    (ring: rank 0's left neighbour is the last rank). Requires n_local >= halo.
    """
    import torch
    dist = _dist()
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    if halo == 0:
        return slab
    n_local = slab.shape[0] - 2 * halo
    if n_local < halo:
        raise ValueError("slab thinner than its halo")
    if size == 1:
        slab[:halo] = slab[n_local:n_local + halo]
        slab[halo + n_local:] = slab[halo:2 * halo]
        return slab
    left, right = (rank - 1) % size, (rank + 1) % size
    send_r = slab[n_local:n_local + halo].contiguous()   # my last owned -> right's low halo
    send_l = slab[halo:2 * halo].contiguous()             # my first owned -> left's high halo
    recv_l = torch.empty_like(send_r)
    recv_r = torch.empty_like(send_l)
    ops = [dist.P2POp(dist.isend, send_r, right, group), dist.P2POp(dist.irecv, recv_l, left, group),
           dist.P2POp(dist.isend, send_l, left, group), dist.P2POp(dist.irecv, recv_r, right, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    slab[:halo] = recv_l
    slab[halo + n_local:] = recv_r
    return slab


def sharded_argmax(compute, n: int, window, group=None, device=None):
    """Certificate over x-slabs: `compute(window_slab) -> (value, cand, lin)`
    for this rank's part of `window` (x range intersected with its slab);
    returns the global winner. Ranks whose slab misses the window contribute
    (-inf, big, big)."""
    dist = _dist()
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    x0, x1 = slab_bounds(n, size, rank)
    (wx0, wx1), wy, wz = window
    lo, hi = max(x0, wx0), min(x1, wx1)
    if lo <= hi:
        rec = compute(((lo, hi), wy, wz))
    else:
        rec = (float("-inf"), 2 ** 31, 2 ** 62)
    return allgather_best(rec, group, device)


def sharded_rows(compute_rows, k: int, group=None, device=None) -> np.ndarray:
    """Per-atom rows split over ranks: `compute_rows(i0, i1) -> (i1 - i0, 6)`;
    the full (k, 6) matrix is assembled with an fp64 all-reduce (each rank
    fills only its own atoms)."""
    dist = _dist()
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    base, extra = divmod(k, size)
    i0 = rank * base + min(rank, extra)
    i1 = i0 + base + (1 if rank < extra else 0)
    full = np.zeros((k, 6))
    if i1 > i0:
        full[i0:i1] = compute_rows(i0, i1)
    return allreduce_f64(full, group, device).reshape(k, 6)


# ------------------------------------------------------------- GPU helpers
def eta_field_sharded(residual, lam, table, bounds=None, group=None):
    """GPU certificate on this rank's x-slab of the window (replicated residual);
    returns the global (eta_max, candidate, (i, j, k))."""
    from .certificate import _position_window, eta_argmax_dev
    dims = table.dims

    def compute(win):
        best, _, _ = eta_argmax_dev(residual, lam, table, win)
        lin = (best.pos[0] * dims[1] + best.pos[1]) * dims[2] + best.pos[2]
        return (best.value, int(best.cand), int(lin))

    v, c, lin = sharded_argmax(compute, dims[0], _position_window(bounds, dims), group,
                               residual.device)
    pos = (lin // (dims[1] * dims[2]), (lin // dims[2]) % dims[1], lin % dims[2])
    return v, c, pos


def cost_grad_sharded(psf, y, rows, lam, group=None):
    """GPU criterion + gradient with the per-atom reductions split over ranks."""
    from .forward import atom_sums_dev, cost_grad_dev
    import torch
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
    back = torch.empty_like(y)
    # C and the back-projection H^T (model - y) once per rank (replicated)
    c, _ = cost_grad_dev(psf, y, rows, lam, want_grad=False, back=back)

    def compute_rows(i0, i1):
        s = atom_sums_dev(back, rows[i0:i1])
        out = np.empty_like(s)
        out[:, 0] = s[:, 0] + lam
        out[:, 1:] = rows[i0:i1, :1] * s[:, 1:]
        return out

    return c, sharded_rows(compute_rows, rows.shape[0], group, y.device)


# ------------------------------------- slab-local cost + gradient (GPU)
def psf_x_halo(kernel: np.ndarray) -> int:
    """x half-extent of the PSF's non-zero box (planes a slab needs each side)."""
    c = kernel.shape[0] // 2
    nzx = np.flatnonzero(np.abs(kernel).sum(axis=(1, 2)))
    return int(max(c - nzx.min(), nzx.max() - c))


def finish_cost_grad(half_sumsq: float, sums: np.ndarray, rows: np.ndarray, lam: float):
    """Rank-summed partials -> (C, (k, 6) gradient rows), forward.py:218-220
    and the criterion's lam * total mass (forward.py:182-190)."""
    # total_mass: sequential sum in row order (cumsum adds left to right)
    mass = float(np.cumsum(rows[:, 0])[-1]) if rows.shape[0] else 0.0
    g = np.empty_like(sums)
    g[:, 0] = sums[:, 0] + lam
    g[:, 1:] = rows[:, :1] * sums[:, 1:]
    return half_sumsq + lam * mass, g


class SlabCostGrad:
    """criterion_and_gradient (forward.py:232-257) sharded as x-slabs
    (SURVEY §8(e)): rank r owns planes [x0, x1] of the periodic (n, ny, nz)
    volume and keeps y on the window x0 - halo .. x1 + halo (halo = the PSF's
    x half-extent). Each rank renders only the clipped x-spans of the atoms
    meeting its window, convolves on the window, forms the residual on its own
    planes, back-projects it and takes the per-atom raw sums
    (sfw3d_cost_grad_slab). The one collective is the all-reduce of the
    6k + 1 fp64 partials (48 KB at k = 1000); the sum over ranks equals the
    single-volume C and gradient up to summation order."""

    def __init__(self, psf, dims, x0: int, x1: int):
        from .forward import Psf
        from .volumes import Volume
        self.dims = tuple(int(v) for v in dims)
        self.x0, self.x1 = int(x0), int(x1)
        self.halo = psf_x_halo(psf.kernel.data)
        n = self.dims[0]
        self.local_dims = (self.x1 - self.x0 + 1 + 2 * self.halo, self.dims[1], self.dims[2])
        if self.local_dims[0] > n:
            raise ValueError("slab + 2 halo planes exceed the volume: use the single-volume path")
        self.psf = Psf(Volume(local_psf_kernel(psf.kernel.data, self.local_dims)), normalize=False)
        import torch
        self.index = torch.arange(self.x0 - self.halo, self.x1 + self.halo + 1) % n

    def window(self, y):
        """This rank's window of a global observation (device or host tensor)."""
        return y.index_select(0, self.index.to(y.device)).contiguous()

    def partials(self, y_win, rows: np.ndarray):
        """(1/2 sum_slab r^2, (k, 6) raw sums) of this rank."""
        import ctypes as C
        from . import _native as N
        from .forward import code_of
        if tuple(y_win.shape) != tuple(self.local_dims):
            raise ValueError(f"y window shape {tuple(y_win.shape)} != {tuple(self.local_dims)}")
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        k = rows.shape[0]
        dev = y_win.device.index
        ctx = N.context(dev)
        half = C.c_double()
        sums = np.zeros((k, 6))
        N.check(N.lib().sfw3d_cost_grad_slab(
            ctx.handle, self.psf.native(dev), code_of(y_win), N.ptr(y_win), N.f64_ptr(rows), k,
            self.dims[0], self.x0, self.x1, self.halo, C.byref(half), N.f64_ptr(sums)))
        return half.value, sums

    def cost_grad(self, y_win, rows: np.ndarray, lam: float, group=None):
        """(C, (k, 6) rows) of the whole volume: partials all-reduced over the
        process group (this rank alone when no group is initialised)."""
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        half, sums = self.partials(y_win, rows)
        if world()[1] > 1:
            flat = allreduce_f64(np.concatenate([[half], sums.ravel()]), group, y_win.device)
            half, sums = float(flat[0]), flat[1:].reshape(-1, 6)
        return finish_cost_grad(half, sums, rows, lam)


# ------------------------------------------- slab-local certificate (GPU)
def slab_halo(psf, sigma_grid, shape_grid) -> int:
    """x-planes of halo an x-slab sub-volume needs so that eta on the slab is
    the global eta: the PSF's x-extent (b = H^T r) plus the largest candidate
    support radius (forward.py:97-99). The chained basis factors reach a few
    planes further with values below the 1e-12 truncation; the signed members'
    bounds cover those taps whatever data they meet (basis.cu)."""
    from .forward import support_radius
    k = psf.kernel.data
    c = k.shape[0] // 2
    nzx = np.flatnonzero(np.abs(k).sum(axis=(1, 2)))
    hx = int(max(c - nzx.min(), nzx.max() - c))
    r = max(support_radius(s, d) for s in sigma_grid for d in shape_grid)
    return hx + r


def local_psf_kernel(kernel: np.ndarray, local_dims) -> np.ndarray:
    """The kernel's non-zero box re-centred (origin n//2 per axis) in a volume
    of `local_dims`."""
    out = np.zeros(tuple(local_dims))
    src, dst = [], []
    for a in range(3):
        other = tuple(b for b in range(3) if b != a)
        ix = np.flatnonzero(np.abs(kernel).sum(axis=other))
        n, ln = kernel.shape[a], local_dims[a]
        lo, hi = ix.min() - n // 2, ix.max() - n // 2
        if ln // 2 + lo < 0 or ln // 2 + hi >= ln:
            raise ValueError("PSF support wider than the local sub-volume")
        src.append(slice(ix.min(), ix.max() + 1))
        dst.append(slice(ln // 2 + lo, ln // 2 + hi + 1))
    out[tuple(dst)] = kernel[tuple(src)]
    return out


class SlabCertificate:
    """Certificate of one rank's x-slab [x0, x1] computed on its own
    sub-volume: planes x0 - halo .. x1 + halo of the (periodic) residual.

    Every eta value on the slab equals the global one (the sub-volume holds
    all the residual the slab's b = H^T r and templates touch), so each rank
    runs the single-GPU certificate on (x1 - x0 + 1 + 2 halo) planes with the
    window restricted to its slab, and the only collective is the all-gather
    of 24-byte argmax records (combine_best: the reference's order). The
    redundant work is the 2 halo planes per slab plane count. The basis is
    pruned by the GLOBAL volume's rule (table option global_voxels) so every
    rank fits the same shared terms as one GPU would."""

    def __init__(self, psf, sigma_grid, shape_grid, dims, x0: int, x1: int, halo: int | None = None,
                 **table_kw):
        import torch
        from .certificate import build_template_table
        from .forward import Psf, support_radius
        from .volumes import Volume
        self.dims = tuple(int(v) for v in dims)
        self.x0, self.x1 = int(x0), int(x1)
        self.halo = int(slab_halo(psf, sigma_grid, shape_grid) if halo is None else halo)
        n = self.dims[0]
        rmax = max(support_radius(s, d) for s in sigma_grid for d in shape_grid)
        self.local_dims = (self.x1 - self.x0 + 1 + 2 * self.halo, self.dims[1], self.dims[2])
        if 2 * rmax + 1 >= n or 2 * rmax + 1 >= self.local_dims[0]:
            raise ValueError("candidate boxes span the x axis: slabs cannot shard this table")
        table_kw.setdefault("global_voxels", int(np.prod(self.dims)))
        self.psf = Psf(Volume(local_psf_kernel(psf.kernel.data, self.local_dims)), normalize=False)
        self.table = build_template_table(self.psf, sigma_grid, shape_grid, **table_kw)
        self.index = torch.arange(self.x0 - self.halo, self.x1 + self.halo + 1) % n

    def subvolume(self, residual):
        """This rank's sub-volume of a global residual (device or host tensor)."""
        return residual.index_select(0, self.index.to(residual.device)).contiguous()

    def argmax(self, sub, lam: float, window=None):
        """(eta, cand, global C-order index) of the slab's part of `window`
        (global coordinates; None = every voxel), or (-inf, big, big)."""
        from .certificate import eta_argmax_dev
        (wx0, wx1), wy, wz = window or ((0, self.dims[0] - 1), (0, self.dims[1] - 1),
                                        (0, self.dims[2] - 1))
        lo, hi = max(self.x0, wx0), min(self.x1, wx1)
        if lo > hi:
            return (float("-inf"), 2 ** 31, 2 ** 62)
        off = self.x0 - self.halo
        best, _, _ = eta_argmax_dev(sub, lam, self.table, ((lo - off, hi - off), wy, wz))
        x = (best.pos[0] + off) % self.dims[0]
        lin = (x * self.dims[1] + best.pos[1]) * self.dims[2] + best.pos[2]
        return (float(best.value), int(best.cand), int(lin))
