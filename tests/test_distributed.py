"""World-size-2 (and 3) gloo tests of the multi-GPU exchange logic on CPU.

The per-rank compute is the CPU oracle here (tests only); on the B200 the
same transports carry the CUDA path's halos and partials
(distributed.TorchComm over NCCL: SlabCertificate, SlabCostGrad)."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, size, port, fn, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        q.put((rank, fn(rank, size)))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def spawn(fn, size=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_run, args=(r, size, port, fn, q)) for r in range(size)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def test_slab_bounds_cover_grid():
    from paper_2009_05473_b200.distributed import slab_bounds
    for n in (16, 17, 512):
        for size in (1, 2, 3, 8):
            seen = []
            for r in range(size):
                a, b = slab_bounds(n, size, r)
                seen.extend(range(a, b + 1))
            assert seen == list(range(n))


def test_combine_best_order():
    from paper_2009_05473_b200.distributed import combine_best
    recs = [(2.0, 3, 10), (2.0, 1, 50), (2.0, 1, 40), (1.0, 0, 0), (float("nan"), 0, 0)]
    assert combine_best(recs) == (2.0, 1, 40)


# ---------------------------------------------------------- rank bodies
def body_halo(rank, size):
    from paper_2009_05473_b200.distributed import halo_exchange, slab_bounds
    n, h = 12, 2
    full = torch.arange(n * 3, dtype=torch.float64).reshape(n, 3)
    x0, x1 = slab_bounds(n, size, rank)
    slab = torch.zeros((x1 - x0 + 1 + 2 * h, 3), dtype=torch.float64)
    slab[h:h + x1 - x0 + 1] = full[x0:x1 + 1]
    halo_exchange(slab, h)
    idx = [(x0 - h + i) % n for i in range(slab.shape[0])]
    return bool(torch.equal(slab, full[idx]))


def body_cert(rank, size):
    """Replicated residual, x-slab windows, all-gathered argmax == single process."""
    import sfw3d_oracle as O
    from paper_2009_05473_b200.distributed import sharded_argmax
    rng = np.random.default_rng(7)
    dims = (14, 12, 10)
    kernel = O.box_gaussian_psf(dims, (1.2, 1.2, 1.5), (2, 2, 3))
    r = rng.standard_normal(dims)
    hats = O.template_hats(O.psf_hat(kernel), dims, [1.0, 1.8], [1.6, 2.2])
    window = ((2, 11), (1, 10), (0, 9))

    def compute(win):
        pos, flat, val, _, _ = O.eta_field(r, 0.5, hats, 2, win)
        return (val, flat, (pos[0] * dims[1] + pos[1]) * dims[2] + pos[2])

    got = sharded_argmax(compute, dims[0], window)
    pos, flat, val, _, _ = O.eta_field(r, 0.5, hats, 2, window)
    want = (val, flat, (pos[0] * dims[1] + pos[1]) * dims[2] + pos[2])
    return got == want


def body_cert_halo(rank, size):
    """Slab-distributed b with periodic halos: a direct correlation on the owned
    planes only needs the template radius of halo."""
    import sfw3d_oracle as O
    from paper_2009_05473_b200.distributed import halo_exchange, slab_bounds
    rng = np.random.default_rng(3)
    dims = (12, 8, 8)
    b = rng.standard_normal(dims)
    R = 2
    off = np.arange(-R, R + 1)
    G = np.exp(-0.3 * (off[:, None, None] ** 2 + off[None, :, None] ** 2 + off[None, None, :] ** 2))
    x0, x1 = slab_bounds(dims[0], size, rank)
    slab = torch.zeros((x1 - x0 + 1 + 2 * R, *dims[1:]), dtype=torch.float64)
    slab[R:R + x1 - x0 + 1] = torch.from_numpy(b[x0:x1 + 1])
    halo_exchange(slab, R)
    s = slab.numpy()
    eta = np.zeros((x1 - x0 + 1, *dims[1:]))
    for a in off:
        for bb in off:
            for c in off:
                eta += G[a + R, bb + R, c + R] * np.roll(s, (-bb, -c), axis=(1, 2))[R + a:R + a + x1 - x0 + 1]
    ref = np.zeros(dims)
    for a in off:
        for bb in off:
            for c in off:
                ref += G[a + R, bb + R, c + R] * np.roll(b, (-a, -bb, -c), axis=(0, 1, 2))
    return float(np.max(np.abs(eta - ref[x0:x1 + 1])))


def body_rows(rank, size):
    import sfw3d_oracle as O
    from paper_2009_05473_b200.distributed import allreduce_f64, sharded_rows
    rng = np.random.default_rng(1)
    dims = (12, 12, 12)
    back = rng.standard_normal(dims)
    rows = np.column_stack([rng.uniform(0.5, 2, 7), rng.uniform(0, 12, (7, 3)),
                            rng.uniform(1, 2.5, 7), rng.uniform(1.5, 2.5, 7)])
    got = sharded_rows(lambda i0, i1: O.atom_rows(back, rows[i0:i1], 0.2), 7)
    s = allreduce_f64(np.array([rank + 1.0, 2.0]))
    return float(np.max(np.abs(got - O.atom_rows(back, rows, 0.2)))), s.tolist()


def body_torchcomm(rank, size):
    """TorchComm (the transport of the library's x-slab data plane): halos of
    lo / hi planes from the ring neighbours (wider than a slab: from several
    ranks), sum / max all-reduce, all-gather."""
    from paper_2009_05473_b200.distributed import TorchComm, slab_bounds
    n = 13
    comm = TorchComm().layout(n)
    full = torch.arange(n * 4, dtype=torch.float32).reshape(n, 4)
    x0, x1 = slab_bounds(n, size, rank)
    own = x1 - x0 + 1
    ok = True
    for lo, hi in ((2, 3), (0, 2), (3, 0), (1, 1), (8, 6), (13, 1)):  # (multi-hop halos)
        win = torch.full((lo + own + hi, 4), -1.0)
        win[lo:lo + own] = full[x0:x1 + 1]
        comm.halo(win, own, lo, hi)
        idx = [(x0 - lo + i) % n for i in range(win.shape[0])]
        ok &= bool(torch.equal(win, full[idx]))
    s = comm.allreduce(np.array([rank + 1.0, -rank]), "sum").tolist()
    m = comm.allreduce(np.array([rank + 1.0, -rank]), "max").tolist()
    g = [a.tolist() for a in comm.allgather(np.array([rank, 2.0 * rank]))]
    return ok, s, m, g


@pytest.mark.parametrize("size", [2, 3])
def test_torchcomm_transport(size):
    for ok, s, m, g in spawn(body_torchcomm, size).values():
        assert ok
        assert s == [sum(range(1, size + 1)), -sum(range(size))]
        assert m == [float(size), 0.0]
        assert g == [[r, 2.0 * r] for r in range(size)]


@pytest.mark.parametrize("size", [2, 3])
def test_halo_exchange(size):
    assert all(spawn(body_halo, size).values())


def test_sharded_certificate_matches_single_process():
    assert all(spawn(body_cert, 2).values())


def test_slab_halo_certificate():
    for err in spawn(body_cert_halo, 2).values():
        assert err < 1e-12


def test_sharded_rows_and_allreduce():
    for err, s in spawn(body_rows, 2).values():
        assert err == 0.0
        assert s == [3.0, 4.0]


def body_slab_cost_grad(rank, size):
    """The decomposition sfw3d_cost_grad_slab computes per rank, restated with
    the oracle: residual masked to the rank's x-slab, back-projected, raw
    per-atom sums; partials all-reduced and finished once."""
    import sfw3d_oracle as O
    from paper_2009_05473_b200.distributed import (allreduce_f64, finish_cost_grad, slab_bounds,
                                                   world)
    rng = np.random.default_rng(5)
    dims = (15, 10, 12)
    kernel = O.box_gaussian_psf(dims, (1.2, 1.0, 1.5), (2, 2, 3))
    khat = O.psf_hat(kernel)
    rows = np.column_stack([rng.uniform(0.5, 2, 6), rng.uniform(0, 15, 6), rng.uniform(0, 10, 6),
                            rng.uniform(0, 12, 6), rng.uniform(0.8, 1.5, 6), rng.uniform(1.8, 2.5, 6)])
    y = rng.standard_normal(dims)
    r = O.conv(O.render(rows, dims), khat) - y
    x0, x1 = slab_bounds(dims[0], size, rank)
    mask = np.zeros(dims)
    mask[x0:x1 + 1] = 1.0
    back = O.corr(r * mask, khat)
    part = O.atom_rows(back, rows, 0.0)      # [s0, w s1..w s5]
    raw = part.copy()
    raw[:, 1:] /= rows[:, :1]
    half = 0.5 * float(np.sum((r * mask) ** 2))
    flat = allreduce_f64(np.concatenate([[half], raw.ravel()]))
    c, g = finish_cost_grad(float(flat[0]), flat[1:].reshape(-1, 6), rows, 0.2)
    c0, g0, _ = O.criterion_and_gradient(y, rows, khat, 0.2)
    assert world() == (rank, size)
    return abs(c - c0) / abs(c0), float(np.max(np.abs(g - g0)) / np.max(np.abs(g0)))


@pytest.mark.parametrize("size", [2, 3])
def test_slab_cost_grad_decomposition(size):
    for ec, eg in spawn(body_slab_cost_grad, size).values():
        assert ec < 1e-13 and eg < 1e-12
