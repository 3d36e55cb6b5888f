"""Multi-GPU sharding of the hot path: one process per GPU,
x-slabs of the periodic volume (axis 0, the slowest), no replicated volumes.

* certificate (SlabCertificate -> sfw3d_eta_argmax_slab) — each rank holds
  the residual on its own planes only. b = H^T r and every shared basis term
  are computed on the owned planes: their z / y passes are plane-local, and
  before each x pass the library asks the transport to exchange the pass's
  halo planes with the two neighbours (sfw3d_halo_fn) — no plane is computed
  twice. Refined members read b with a template-radius halo (one more
  exchange); the refinement thresholds use the all-reduced |b| statistics and
  member maxima (sfw3d_allreduce_fn), so every rank collects the single-GPU
  candidate set on its slab. Per-candidate records are all-gathered and
  combined in the reference's order (eta desc, candidate asc, C-order asc).
* cost + gradient (SlabCostGrad -> sfw3d_cost_grad_slab) — y on the slab
  window (owned planes + the PSF's x half-extent, static during a solve),
  atom x-spans clipped to the window, residual masked to the slab; the 6k + 1
  fp64 partials are all-reduced ON THE DEVICE (one D2H per evaluation).
* sums (Gram rows, ||r||^2) — fp64 all-reduce.

Transports (`Comm`): TorchComm (torch.distributed: NCCL P2P / all-reduce on
the B200 box, gloo in the CPU tests), ThreadComm (ranks as threads of one
process sharing one GPU: the single-GPU tests of the data plane) and
SoloComm (one rank of a W-rank layout alone: per-rank timing only; its
halos are stand-in data).
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

    def partials_dev(self, y_win, rows: np.ndarray):
        """This rank's [1/2 sum_slab r^2, raw sums] as a DEVICE fp64 tensor,
        enqueued on the current stream without a host synchronisation."""
        import torch
        from . import _native as N
        from .forward import code_of
        if tuple(y_win.shape) != tuple(self.local_dims):
            raise ValueError(f"y window shape {tuple(y_win.shape)} != {tuple(self.local_dims)}")
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        k = rows.shape[0]
        dev = y_win.device.index
        out = torch.empty(1 + 6 * k, dtype=torch.float64, device=y_win.device)
        N.check(N.lib().sfw3d_cost_grad_slab_dev(
            N.context(dev).handle, self.psf.native(dev), code_of(y_win), N.ptr(y_win),
            N.f64_ptr(rows), k, self.dims[0], self.x0, self.x1, self.halo, N.ptr(out)))
        return out

    def cost_grad(self, y_win, rows: np.ndarray, lam: float, comm=None):
        """(C, (k, 6) rows) of the whole volume. The partials stay on the
        device through the all-reduce (TorchComm over NCCL: in-stream); one
        D2H per evaluation. comm=None: this rank alone."""
        import torch
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        part = self.partials_dev(y_win, rows)
        if comm is not None and comm.size > 1:
            if isinstance(comm, TorchComm) and _dist().get_backend(comm.group) == "nccl":
                _dist().all_reduce(part, group=comm.group)  # in place, on the current stream
                flat = part.cpu().numpy()
            else:
                flat = comm.allreduce(part.cpu().numpy(), "sum")
        else:
            flat = part.cpu().numpy()
        if not np.isfinite(flat).all():
            raise FloatingPointError("non-finite criterion gradient; atom parameters left the "
                                     "smooth regime")
        return finish_cost_grad(float(flat[0]), flat[1:].reshape(-1, 6), rows, lam)


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


# ----------------------------------------------------------- transports
def _runs(planes):
    """Consecutive runs of a list of ints: [(first, count)]."""
    out = []
    for p in planes:
        if out and p == out[-1][0] + out[-1][1]:
            out[-1] = (out[-1][0], out[-1][1] + 1)
        else:
            out.append((p, 1))
    return out


def halo_plan(bounds, n: int, rank: int, lo: int, hi: int):
    """Where rank's window halos come from: [(owner, window_row, owner_row, count)]
    for the lo planes below its slab and the hi planes above it (periodic),
    as contiguous runs per owner; owner_row is local to the owner's slab.
    Every rank computes every plan (the send lists are the peers' plans)."""
    x0, x1 = bounds[rank]
    own = x1 - x0 + 1
    rows = [(i, (x0 - lo + i) % n) for i in range(lo)]
    rows += [(lo + own + i, (x1 + 1 + i) % n) for i in range(hi)]
    starts = [b[0] for b in bounds]
    plan = []
    for row, g in rows:
        q = max(i for i, st in enumerate(starts) if st <= g)  # slab_bounds is ordered
        orow = g - bounds[q][0]
        if plan and plan[-1][0] == q and plan[-1][1] + plan[-1][3] == row \
                and plan[-1][2] + plan[-1][3] == orow:
            plan[-1] = (q, plan[-1][1], plan[-1][2], plan[-1][3] + 1)
        else:
            plan.append((q, row, orow, 1))
    return plan


class _Layout:
    """The x-slab layout every transport needs for multi-hop halos, and the
    halo bytes it has received (for the multi-GPU projections)."""

    halo_bytes = 0

    def _count(self, win, lo: int, hi: int) -> None:
        self.halo_bytes += (lo + hi) * win[0].numel() * win.element_size()

    def layout(self, n: int):
        self.n = int(n)
        self.bounds = [slab_bounds(self.n, self.size, r) for r in range(self.size)]
        self._plans = {}
        return self

    def _exchange_plan(self, lo: int, hi: int):
        """(sends [(peer, own_row, count)] in each receiver's plan order, recvs
        [(owner, window_row, count)], local copies [(window_row, own_row, count)])
        of one exchange; computed once per (lo, hi) — a certificate repeats
        the same dozen halo shapes every step."""
        key = (lo, hi)
        plan = self._plans.get(key)
        if plan is None:
            sends, recvs, local = [], [], []
            for q in range(self.size):
                if q == self.rank:
                    continue
                for owner, _, orow, cnt in halo_plan(self.bounds, self.n, q, lo, hi):
                    if owner == self.rank:
                        sends.append((q, orow, cnt))
            for owner, row, orow, cnt in halo_plan(self.bounds, self.n, self.rank, lo, hi):
                if owner == self.rank:
                    local.append((row, orow, cnt))
                else:
                    recvs.append((owner, row, cnt))
            plan = self._plans[key] = (sends, recvs, local)
        return plan


def _fill_halo_self(win, own: int, lo: int, hi: int) -> None:
    """Periodic halos from the rank's own planes (a ring of one)."""
    # plane x0 - lo + i  ==  owned plane (own - lo + i) mod own; copied in
    # contiguous runs (one copy per run, not per plane)
    def runs(dst0, count, src_of):
        i = 0
        while i < count:
            s0 = src_of(i)
            m = min(count - i, own - s0)  # run until the source wraps
            win[dst0 + i:dst0 + i + m] = win[lo + s0:lo + s0 + m]
            i += m
    runs(0, lo, lambda i: (own - lo + i) % own)
    runs(lo + own, hi, lambda i: i % own)


class TorchComm(_Layout):
    """torch.distributed transport: NCCL point-to-point / all-reduce on the
    GPUs (enqueued on the caller's current stream), gloo on CPU tensors."""

    def __init__(self, group=None):
        dist = _dist()
        self.group = group
        self.rank, self.size = dist.get_rank(group), dist.get_world_size(group)
        self.n = None

    def halo(self, win, own: int, lo: int, hi: int) -> None:
        """win: (lo + own + hi, ...) planes; fill [0, lo) with the lo global
        planes below this rank's slab and the top hi with those above it
        (each rank sends the peers' plans: single or multi-hop)."""
        dist = _dist()
        self._count(win, lo, hi)
        if self.size == 1:
            _fill_halo_self(win, own, lo, hi)
            return
        if self.n is None:
            raise RuntimeError("TorchComm.layout(n) must be called before halo exchanges")
        sends, recvs, local = self._exchange_plan(lo, hi)
        ops = [dist.P2POp(dist.isend, win[lo + orow:lo + orow + cnt], q, self.group)
               for q, orow, cnt in sends]
        ops += [dist.P2POp(dist.irecv, win[row:row + cnt], owner, self.group)
                for owner, row, cnt in recvs]
        for row, orow, cnt in local:
            win[row:row + cnt] = win[lo + orow:lo + orow + cnt]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        import torch
        dist = _dist()
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=dev).clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                        group=self.group)
        return t.cpu().numpy()

    def allgather(self, values) -> list:
        import torch
        dist = _dist()
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64), device=dev)
        out = [torch.empty_like(t) for _ in range(self.size)]
        dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]


class ThreadGroup:
    """Ranks as threads of one process sharing one GPU (each thread on its own
    CUDA stream): the single-GPU stand-in for NVLink in the tests. Exchanges
    synchronise the ranks' streams and copy device to device."""

    def __init__(self, size: int):
        import threading
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size

    def comm(self, rank: int) -> "ThreadComm":
        return ThreadComm(self, rank)


class ThreadComm(_Layout):
    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.size = group, rank, group.size
        self.n = None

    def _exchange(self, item):
        g = self.g
        g.slots[self.rank] = item
        g.barrier.wait()
        out = list(g.slots)
        g.barrier.wait()
        return out

    def halo(self, win, own: int, lo: int, hi: int) -> None:
        import torch
        self._count(win, lo, hi)
        torch.cuda.current_stream().synchronize()  # my owned planes are final
        g = self.g
        g.slots[self.rank] = ("halo", win, lo)
        g.barrier.wait()
        slots = list(g.slots)
        if any(sl[0] != "halo" for sl in slots):
            raise RuntimeError("ranks out of step: halo exchange met another collective")
        if self.size == 1:
            _fill_halo_self(win, own, lo, hi)
        else:
            if self.n is None:
                raise RuntimeError("ThreadComm.layout(n) must be called before halo exchanges")
            for owner, row, orow, cnt in halo_plan(self.bounds, self.n, self.rank, lo, hi):
                _, ow, olo = slots[owner]
                win[row:row + cnt].copy_(ow[olo + orow:olo + orow + cnt])
        torch.cuda.current_stream().synchronize()  # (owners may reuse their windows)
        g.barrier.wait()

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        arrs = self._exchange(np.array(values, dtype=np.float64))
        out = arrs[0].copy()
        for a in arrs[1:]:  # rank order: deterministic
            out = np.maximum(out, a) if op == "max" else out + a
        return out

    def allgather(self, values) -> list:
        return self._exchange(np.array(values, dtype=np.float64))


class SoloComm(_Layout):
    """Rank `rank` of a `size`-rank layout run ALONE on this GPU (no other
    process): halos are filled from the rank's own planes (stand-in data of the
    right size), reductions are the identity. Per-rank timing aid only."""

    def __init__(self, rank: int, size: int):
        self.rank, self.size = rank, size
        self.n = None

    def halo(self, win, own: int, lo: int, hi: int) -> None:
        self._count(win, lo, hi)
        _fill_halo_self(win, own, lo, hi)

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        return np.array(values, dtype=np.float64)

    def allgather(self, values) -> list:
        return [np.array(values, dtype=np.float64)]


_DT = {0: ("<f4", 4), 1: ("<f8", 8)}


class _DevBuf:
    """A raw device pointer as a torch-importable buffer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, code: int):
        self.__cuda_array_interface__ = {"shape": tuple(int(v) for v in shape),
                                         "typestr": _DT[code][0], "data": (int(ptr), False),
                                         "version": 3, "strides": None, "stream": None}


def slab_callbacks(comm, device: int):
    """ctypes halo / all-reduce callbacks of the library's x-slab data plane
    bound to a transport (keep the returned objects alive during the call)."""
    import traceback
    import torch
    from . import _native as N

    def halo(user, ptr, code, own, plane, lo, hi):
        try:
            win = torch.as_tensor(_DevBuf(ptr, (lo + own + hi, plane), code),
                                  device=f"cuda:{device}")
            comm.halo(win, own, lo, hi)
            return 0
        except Exception:  # (surfaced as the call's error status)
            traceback.print_exc()
            return 1

    def allreduce(user, vals, n, op):
        try:
            arr = np.ctypeslib.as_array(vals, shape=(n,))
            arr[:] = comm.allreduce(arr.copy(), "max" if op == 1 else "sum")
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    return N.HALO_FN(halo), N.ALLREDUCE_FN(allreduce)


# ------------------------------------------- slab certificate (GPU)
class SlabCertificate:
    """eta_field's grid stage (certificate.py:140-184) on this rank's x-slab
    [x0, x1] of the GLOBAL table's volume (sfw3d_eta_argmax_slab): the
    residual lives on the owned planes only; the x passes exchange their
    halos through `comm`; per-candidate records are all-gathered. The
    combined winner equals the single-GPU certificate's bit for bit (same
    kernels, same per-voxel arithmetic, same refinement thresholds)."""

    def __init__(self, table, x0: int, x1: int, comm):
        self.table = table
        self.dims = tuple(table.dims)
        self.x0, self.x1 = int(x0), int(x1)
        self.n_own = self.x1 - self.x0 + 1
        self.comm = comm
        comm.layout(self.dims[0])

    def owned(self, volume):
        """This rank's planes of a global volume (device or host tensor)."""
        return volume[self.x0:self.x1 + 1].contiguous()

    def argmax(self, r_owned, lam: float, window=None):
        """Global (eta, candidate, (i, j, k)) and the per-candidate global
        records [(eta, (i, j, k))] of `window` (global coordinates; None =
        every voxel). Collective: every rank calls it."""
        import ctypes as C
        from . import _native as N
        from .forward import code_of
        dims = self.dims
        if tuple(r_owned.shape) != (self.n_own, dims[1], dims[2]):
            raise ValueError(f"owned residual shape {tuple(r_owned.shape)} != "
                             f"{(self.n_own, dims[1], dims[2])}")
        (wx0, wx1), wy, wz = window or ((0, dims[0] - 1), (0, dims[1] - 1), (0, dims[2] - 1))
        lo, hi = max(self.x0, wx0), min(self.x1, wx1)
        mine = lo <= hi
        # (a rank whose slab misses the window still runs the collective
        # pipeline on its whole slab and contributes nothing)
        lwin = (lo - self.x0, hi - self.x0) if mine else (0, self.n_own - 1)
        w32 = np.array([*lwin, *wy, *wz], dtype=np.int32)
        dev = r_owned.device.index
        ctx = N.context(dev)
        halo, ared = slab_callbacks(self.comm, dev)
        nc = len(self.table.sigma_grid) * len(self.table.shape_grid)
        best = N.Argmax()
        per = (N.Argmax * nc)()
        N.check(N.lib().sfw3d_eta_argmax_slab(
            ctx.handle, self.table.native(dev), code_of(r_owned), N.ptr(r_owned), self.n_own,
            self.x0, float(lam), N.i32_ptr(w32), halo, ared, None, C.byref(best), per))
        plane = dims[1] * dims[2]
        rec = np.full(2 * nc, -np.inf)
        for c in range(nc):
            p = per[c]
            if mine and np.isfinite(p.value):
                rec[2 * c] = p.value
                rec[2 * c + 1] = ((self.x0 + p.pos[0]) * dims[1] + p.pos[1]) * dims[2] + p.pos[2]
        allr = self.comm.allgather(rec)
        out = []
        for c in range(nc):
            bv, bl = -np.inf, np.inf
            for r in allr:  # value desc, then the first C-order position
                v, lin = r[2 * c], r[2 * c + 1]
                if v > bv or (v == bv and lin < bl):
                    bv, bl = v, lin
            lin = int(bl) if np.isfinite(bl) else -1
            out.append((float(bv), (lin // plane, (lin // dims[2]) % dims[1], lin % dims[2])))
        gc = 0
        for c in range(nc):  # strict '>' over sigma-major candidates
            if out[c][0] > out[gc][0]:
                gc = c
        return out[gc][0], gc, out[gc][1], out
