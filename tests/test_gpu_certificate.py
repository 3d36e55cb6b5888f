"""GPU tests of the certificate evaluators (direct correlation vs separable
Gaussian basis) against the oracle's FFT eta_field.

Bars: fp32 storage — eta within 1e-5 of eta_max (north-star bar) and the
argmax identical unless the top two differ by < 1e-6 relative; fp64 — the
direct path and the exact d = 2 separable path within 1e-10 of eta_max.
"""
import numpy as np
import pytest

import sfw3d_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2009_05473_b200 as pkg
    pkg.set_precision("f64")
    return pkg


def cfg4_like(n, seed=0):
    rng = np.random.default_rng(seed)
    dims = (n, n, n)
    kernel = O.box_gaussian_psf(dims, (3.0, 3.0, 3.0), (15, 15, 15))
    rows = np.column_stack([rng.uniform(5, 10, 12), rng.uniform(0, n, (12, 3)),
                            rng.uniform(1, 3, 12), rng.uniform(1.5, 3, 12)])
    r = rng.standard_normal(dims) + O.conv(O.render(rows, dims), O.psf_hat(kernel))
    return dims, kernel, r.astype(np.float32).astype(np.float64)


def test_table_fits(P):
    dims = (96, 96, 96)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (3, 3, 3), (15, 15, 15))), normalize=False)
    table = P.build_template_table(psf, [1.0, 1.5, 2.0, 3.0], [1.5, 2.0, 2.5, 3.0])
    with P.precision("f32"):
        info = table.info()
    members = [c for c in info["candidates"] if c["path"] == "basis"]
    for c in info["candidates"]:
        if c["d"] == 2.0:  # exactly one shared term (its own beta), weight 1
            assert c["path"] == "basis" and c["fit_err"] == 0.0
        elif c["d"] < 2.0:
            assert c["path"] == "basis" and c["fit_err"] <= 1e-9
        else:  # signed members: maxima refined exactly
            assert c["path"] == "basis+refine" and 0.0 < c["fit_err"] < 1.0
    # the shared terms' passes cost far less than the members' direct taps
    assert members[0]["basis_taps"] * 10 < sum(c["direct_taps"] for c in members)
    assert all(c["terms"] == members[0]["terms"] < 64 for c in members)
    with P.precision("f64"):
        info64 = table.info()
    for c in info64["candidates"]:
        if c["d"] == 2.0:  # exact: no refinement needed
            assert c["path"] == "basis" and c["fit_err"] == 0.0
        elif c["d"] > 2.0:  # signed members
            assert c["path"] == "basis+refine" and 0.0 < c["fit_err"] < 1e-3
        else:  # fp64: approximate basis, maxima refined exactly
            assert c["path"] == "basis+refine" and c["fit_err"] <= 1e-9


def test_eta_config2_f64_vs_oracle(P):
    """BASELINE config 2 geometry: 128^3 f64, anisotropic 17x17x33 PSF, 6 x 5
    candidates incl. d = 1.2 (full-axis boxes, R up to 85) — fp64 storage with
    the fp64 basis / direct split, against the FFT oracle."""
    rng = np.random.default_rng(12)
    dims = (128, 128, 128)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 4.0), (8, 8, 16))
    rows = np.column_stack([rng.uniform(0.5, 2, 20), rng.uniform(9, 118, (20, 3)),
                            rng.uniform(1, 3, 20), rng.uniform(1.2, 2.8, 20)])
    y = O.conv(O.render(rows, dims), O.psf_hat(kernel)) + 0.05 * rng.standard_normal(dims)
    sg, dg = np.geomspace(1, 3, 6), np.linspace(1.2, 2.8, 5)
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    win = ((9, 118), (9, 118), (9, 118))
    pos, flat, val, per, _ = O.eta_field(y, 0.7, hats, 5, win)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    table = P.build_template_table(psf, sg, dg)
    bounds = P.DomainBounds((9.0,) * 3, (118.0,) * 3, 1.0, 3.0, 1.2, 2.8)
    f = P.eta_field(P.Volume(y), 0.7, table, bounds=bounds, keep_fields=False)
    assert abs(f.eta_max - val) <= 1e-9 * abs(val)
    assert f.argmax_position == pos and f.argmax_sigma_index * 5 + f.argmax_shape_index == flat


@pytest.mark.parametrize("n", [64, 80])
def test_eta_f32_basis_vs_oracle(P, n):
    dims, kernel, r = cfg4_like(n)
    sg, dg = np.array([1.0, 1.5, 2.0, 3.0]), np.array([1.5, 2.0, 2.5, 3.0])
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    pos, flat, val, per, fields = O.eta_field(r, 1.0, hats, 4, None, keep_fields=True)
    ref = np.stack(fields)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    with P.precision("f32"):
        for mode in ("auto", "direct"):
            table = P.build_template_table(psf, sg, dg, mode=mode, tap_tol=1e-12)
            f = P.eta_field(P.Volume(r), 1.0, table, keep_fields=True)
            got = np.stack([v.data for v in f.fields])
            err = np.max(np.abs(got - ref)) / abs(val)
            assert err <= 1e-5, (mode, err)
            assert abs(f.eta_max - val) <= 1e-5 * abs(val)
            top = np.sort(np.array([v for _, v in per]))[::-1]
            if top[0] - top[1] > 1e-6 * abs(top[0]):
                assert f.argmax_sigma_index * 4 + f.argmax_shape_index == flat
            assert f.argmax_position == pos or abs(ref.ravel()[np.ravel_multi_index(
                f.argmax_position, dims) + flat * r.size] - val) <= 1e-6 * abs(val)


def test_eta_f64_separable_exact(P):
    dims, kernel, r = cfg4_like(48, seed=3)
    sg, dg = np.array([1.2, 2.4]), np.array([2.0])
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    _, _, val, _, fields = O.eta_field(r, 0.5, hats, 1, None, keep_fields=True)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    table = P.build_template_table(psf, sg, dg)
    assert table.info()["n_basis"] == 2
    f = P.eta_field(P.Volume(r), 0.5, table, keep_fields=True)
    got = np.stack([v.data for v in f.fields])
    assert np.max(np.abs(got - np.stack(fields))) <= 1e-10 * abs(val)


def test_eta_linearity(P):
    """eta(a r1 + b r2) = a eta(r1) + b eta(r2)."""
    dims, kernel, r1 = cfg4_like(40, seed=5)
    r2 = np.random.default_rng(9).standard_normal(dims)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    table = P.build_template_table(psf, [1.5, 2.5], [1.6, 2.0, 2.7])
    f1 = np.stack([v.data for v in P.eta_field(P.Volume(r1), 1.0, table).fields])
    f2 = np.stack([v.data for v in P.eta_field(P.Volume(r2), 1.0, table).fields])
    f3 = np.stack([v.data for v in P.eta_field(P.Volume(2.0 * r1 - 0.5 * r2), 1.0, table).fields])
    assert np.max(np.abs(f3 - (2.0 * f1 - 0.5 * f2))) <= 1e-10 * np.max(np.abs(f3))


def test_eta_f64_refined_maxima(P):
    """fp64 storage, d < 2 candidates on the shared basis with exact
    refinement: every candidate's windowed maximum and its position equal the
    oracle's (direct-equivalent) ones to 1e-10, and the approximate fields
    stay within the refinement bound E_c = (e_c + 2e-12) ||b||_1 / lam."""
    import torch
    dims, kernel, r = cfg4_like(56, seed=7)
    sg, dg = np.array([1.0, 1.7, 2.6]), np.array([1.3, 1.6, 1.9, 2.0])
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    win = ((4, 51), (6, 49), (3, 52))
    _, _, val, per, fields = O.eta_field(r, 0.8, hats, len(dg), win, keep_fields=True)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    table = P.build_template_table(psf, sg, dg)
    info = table.info()
    assert sum(c["path"] == "basis+refine" for c in info["candidates"]) == 9
    rd = torch.tensor(r, device="cuda")
    best, recs, fl = P.certificate.eta_argmax_dev(rd, 0.8, table, win, keep_fields=True)
    assert abs(best.value - val) <= 1e-10 * abs(val)
    for c, rec in enumerate(recs):
        pos, v = per[c]
        assert abs(rec.value - v) <= 1e-10 * abs(val), (c, rec.value, v)
        assert tuple(rec.pos) == tuple(pos), (c, tuple(rec.pos), pos)
    b = O.corr(r, O.psf_hat(kernel))  # H^T r
    l1 = np.abs(b).sum()
    got = fl.cpu().numpy()
    for c, cinfo in enumerate(info["candidates"]):
        if cinfo["path"] == "basis+refine":
            E = (cinfo["fit_err"] + 2e-12) * l1 / 0.8
            assert np.max(np.abs(got[c] - fields[c])) <= E


@pytest.mark.parametrize("prec,tol,cap", [("f32", 1e-5, None), ("f64", 1e-10, None),
                                          ("f32", 1e-5, "6")])
def test_signed_members_refined_maxima(P, prec, tol, cap):
    """d > 2 candidates on the shared basis with signed weights: an argmax-only
    evaluation refines every voxel within 2 E_c of each member's approximate
    maximum exactly, so each candidate's maximum and position equal the FFT
    oracle's (and the direct path's) to the storage bar; the refined set is
    small. With a refinement cap below the collected count (cap = 6), the
    members with the most near-maximal voxels fall back to the direct
    kernels and the rest are still refined."""
    import torch
    from paper_2009_05473_b200 import _native as N
    dims, kernel, r = cfg4_like(72, seed=11)
    sg, dg = np.array([1.0, 1.5, 2.0, 3.0]), np.array([1.5, 2.0, 2.5, 3.0])
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    win = ((3, 68), (0, 71), (5, 66))
    _, _, val, per, _ = O.eta_field(r, 0.9, hats, len(dg), win)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    with P.precision(prec):
        table = P.build_template_table(psf, sg, dg, tap_tol=1e-12,
                                       refine_cap=int(cap) if cap else None)
        paths = [c["path"] for c in table.info()["candidates"]]
        assert all(p == "basis+refine" for p, (s, d) in zip(paths, [(a, b) for a in sg for b in dg])
                   if d > 2.0)
        rd = torch.tensor(r, device="cuda", dtype=torch.float32 if prec == "f32" else torch.float64)
        best, recs, _ = P.certificate.eta_argmax_dev(rd, 0.9, table, win)
        count = N.last_refine_count()
        assert 0 < count <= (int(cap) if cap else 65536)
        dtab = P.build_template_table(psf, sg, dg, tap_tol=1e-12, mode="direct")
        _, drecs, _ = P.certificate.eta_argmax_dev(rd, 0.9, dtab, win)
    assert abs(best.value - val) <= tol * abs(val)
    for c, (rec, drec) in enumerate(zip(recs, drecs)):
        pos, v = per[c]
        assert abs(rec.value - v) <= tol * abs(val), (c, rec.value, v)
        assert abs(rec.value - drec.value) <= tol * abs(val), (c, rec.value, drec.value)
        assert tuple(rec.pos) == tuple(pos), (c, tuple(rec.pos), pos)


def _run_ranks(nranks, body):
    """Run body(rank, comm) on `nranks` threads of this process (one GPU, one
    CUDA stream per rank): the in-process stand-in for one process per GPU."""
    import threading
    import torch
    from paper_2009_05473_b200 import distributed as D
    group = D.ThreadGroup(nranks)
    out, errs = [None] * nranks, []

    def run(rank):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[rank] = body(rank, group.comm(rank))
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            group.barrier.abort()
    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_slab_certificate_halo_exchange_matches_global(P, nranks, prec):
    """Multi-GPU certificate data plane (distributed.SlabCertificate ->
    sfw3d_eta_argmax_slab): each rank holds only its own x-planes of the
    residual; b = H^T r and every basis term are computed on those planes with
    the x passes' halos exchanged between neighbours (here: ranks as threads
    on this GPU, device-to-device copies; at 8 ranks the 12-plane slabs are
    thinner than the halos, which then come from two ranks away). The
    combined per-candidate records
    equal the single-volume certificate's EXACTLY (same kernels, same
    per-voxel arithmetic, same refinement thresholds), and match the oracle."""
    import torch
    from paper_2009_05473_b200 import distributed as D
    dims = (96, 48, 64)
    rng = np.random.default_rng(5)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 1.5), (3, 3, 3))
    rows = np.column_stack([rng.uniform(5, 10, 6), rng.uniform(0, 48, (6, 3)),
                            rng.uniform(1, 2, 6), rng.uniform(1.8, 2.5, 6)])
    r = rng.standard_normal(dims) + O.conv(O.render(rows, dims), O.psf_hat(kernel))
    r = r.astype(np.float32).astype(np.float64)
    sg, dg = np.array([1.0, 1.5, 2.0]), np.array([1.8, 2.0, 2.5])
    psf = P.Psf(P.Volume(kernel), normalize=False)
    tdt = torch.float32 if prec == "f32" else torch.float64
    win = ((3, 90), (0, 47), (2, 60))
    with P.precision(prec):
        table = P.build_template_table(psf, sg, dg)
        rd = torch.tensor(r, device="cuda", dtype=tdt)
        best, recs, _ = P.certificate.eta_argmax_dev(rd, 0.7, table, win)

        def body(rank, comm):
            x0, x1 = D.slab_bounds(dims[0], nranks, rank)
            slab = D.SlabCertificate(table, x0, x1, comm)
            return slab.argmax(slab.owned(rd), 0.7, win)

        outs = _run_ranks(nranks, body)
    for v, c, pos, per in outs:  # every rank returns the same global result
        assert (v, c, pos) == (float(best.value), int(best.cand), tuple(best.pos))
        for rec, (pv, pp) in zip(recs, per):
            assert pv == float(rec.value) and pp == tuple(rec.pos)
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    opos, _, val, _, _ = O.eta_field(r, 0.7, hats, len(dg), win)
    assert tuple(best.pos) == tuple(opos)
    assert abs(best.value - val) <= (1e-5 if prec == "f32" else 1e-10) * abs(val)


def test_many_members_ring_slices_vs_oracle(P):
    """48 candidates (config 3's 8 sigma x 6 d grid) in fp32: the dense members
    go through mix_ring2_kernel in 16-member slices (copies with the first),
    the refinement's collect pass in matching 16-member V = 4 slices; every
    candidate's windowed maximum and position equal the FFT oracle's."""
    import torch
    rng = np.random.default_rng(12)
    dims = (48, 40, 64)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 1.5), (4, 4, 4))
    rows = np.column_stack([rng.uniform(3, 6, 5), rng.uniform(8, 36, (5, 3)),
                            rng.uniform(1, 3, 5), rng.uniform(1.5, 2.5, 5)])
    r = rng.standard_normal(dims) + O.conv(O.render(rows, dims), O.psf_hat(kernel))
    r = r.astype(np.float32).astype(np.float64)
    sg, dg = np.geomspace(1, 3, 8), np.linspace(1.5, 2.5, 6)
    win = ((2, 45), (0, 39), (3, 60))
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    _, _, val, per, _ = O.eta_field(r, 0.8, hats, len(dg), win)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    with P.precision("f32"):
        table = P.build_template_table(psf, sg, dg)
        assert table.info()["n_basis"] > 16
        rd = torch.tensor(r, device="cuda", dtype=torch.float32)
        best, recs, _ = P.certificate.eta_argmax_dev(rd, 0.8, table, win)
    assert abs(best.value - val) <= 1e-5 * abs(val)
    for c, rec in enumerate(recs):
        pos, v = per[c]
        assert abs(rec.value - v) <= 1e-5 * abs(val), (c, rec.value, v)
        assert tuple(rec.pos) == tuple(pos), (c, tuple(rec.pos), pos)


@pytest.mark.parametrize("nranks,prec,tc,tg", [(2, "f64", 1e-12, 1e-11), (3, "f64", 1e-12, 1e-11),
                                               (4, "f32", 1e-5, 1e-4)])
def test_slab_cost_grad_matches_global(P, nranks, prec, tc, tg):
    """Multi-GPU cost + gradient (distributed.SlabCostGrad through
    sfw3d_cost_grad_slab): the ranks run one after another on this GPU on
    their own windows; their partials summed equal the oracle's C and
    gradient. Atoms straddle the periodic x seam and (nranks = 2) meet a
    window through two periodic images."""
    import torch
    from paper_2009_05473_b200 import distributed as D
    rng = np.random.default_rng(31 + nranks)
    dims = (48, 20, 24)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.2, 2.0), (4, 3, 5))
    k = 40
    rows = np.column_stack([rng.uniform(0.5, 2, k), rng.uniform(0, 48, k), rng.uniform(0, 20, k),
                            rng.uniform(0, 24, k), rng.uniform(0.8, 1.5, k), rng.uniform(2.0, 2.8, k)])
    rows[:4, 1] = [0.2, 47.7, 23.9, 24.1]   # seam and slab-boundary centres
    y = rng.standard_normal(dims)
    c0, g0, _ = O.criterion_and_gradient(y, rows, O.psf_hat(kernel), 0.15)
    with P.precision(prec):
        psf = P.Psf(P.Volume(kernel), normalize=False)
        from paper_2009_05473_b200.forward import to_dev
        yd = to_dev(y)
        half, sums = 0.0, np.zeros((k, 6))
        for r in range(nranks):
            x0, x1 = D.slab_bounds(dims[0], nranks, r)
            sl = D.SlabCostGrad(psf, dims, x0, x1)
            h, s = sl.partials(sl.window(yd), rows)
            half += h
            sums += s
        torch.cuda.synchronize()
    c, g = D.finish_cost_grad(half, sums, rows, 0.15)
    assert abs(c - c0) <= tc * abs(c0)
    scale = np.maximum(np.max(np.abs(g0), axis=0), 1e-300)
    assert float(np.max(np.max(np.abs(g - g0), axis=0) / scale)) < tg


@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_cost_grad_threads_device_allreduce(P, nranks):
    """SlabCostGrad.cost_grad as a collective: ranks as threads on this GPU,
    partials left on the device (sfw3d_cost_grad_slab_dev) and all-reduced;
    every rank gets the oracle's C and gradient (fp64 bars)."""
    import torch
    from paper_2009_05473_b200 import distributed as D
    from paper_2009_05473_b200.forward import to_dev
    rng = np.random.default_rng(77)
    dims = (48, 20, 24)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.2, 2.0), (4, 3, 5))
    k = 30
    rows = np.column_stack([rng.uniform(0.5, 2, k), rng.uniform(0, 48, k), rng.uniform(0, 20, k),
                            rng.uniform(0, 24, k), rng.uniform(0.8, 1.5, k), rng.uniform(2.0, 2.8, k)])
    rows[:3, 1] = [0.3, 47.6, 16.0]
    y = rng.standard_normal(dims)
    c0, g0, _ = O.criterion_and_gradient(y, rows, O.psf_hat(kernel), 0.15)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    yd = to_dev(y)

    def body(rank, comm):
        x0, x1 = D.slab_bounds(dims[0], nranks, rank)
        sl = D.SlabCostGrad(psf, dims, x0, x1)
        return sl.cost_grad(sl.window(yd), rows, 0.15, comm)

    for c, g in _run_ranks(nranks, body):
        assert abs(c - c0) <= 1e-12 * abs(c0)
        assert np.max(np.abs(g - g0)) <= 1e-11 * np.max(np.abs(g0))
