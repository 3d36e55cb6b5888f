"""Step-level (teacher-forced) replay of a BASELINE config-2 BSFW solve
against the oracle.

The reference does not finish config 2 on CPU, so there is no
end-to-end golden; instead the GPU solve records the state every step started
from (solvers._solve(record=...)) and the oracle re-runs that step from the
SAME state:
  * certificate (certificate.py:140-184, 227-236): the grid argmax of
    y - sum w_i phi_i over the 6 x 5 candidates in the domain window (same
    voxel and candidate, eta within 1e-9 relative), then the L-BFGS-B refine
    from that seed (theta* within 1e-6, eta* within 1e-9 relative);
  * weight step (solvers.py:111-180): coordinate descent on the oracle Gram
    from the recorded atoms and warm start (weights within 1e-8 of max w);
  * final BSFW slide (solvers.py:197-240, 314-336): L-BFGS-B from the
    recorded start, both sides capped at 3 iterations (the oracle's f64
    criterion + gradient at 128^3 costs seconds per evaluation).
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


@pytest.fixture(scope="module")
def cfg2_solve(P):
    from paper_2009_05473_b200 import configs, solvers
    inst = configs.config2()
    khat = O.psf_hat(inst.kernel)
    clean = O.conv(O.render(inst.truth, inst.dims), khat)
    rng = np.random.default_rng(100)
    y = clean + O.power_snr_sigma(clean, inst.snr_db) * rng.standard_normal(inst.dims)
    b = inst.bounds
    sg, dg = solvers.make_parameter_grids(b, 6, 5)
    win = O.position_window(inst.dims, b.pos_lower, b.pos_upper)
    per = O.eta_maxima(y, 1.0, khat, sg, dg, win, threads=8)
    lam = inst.lam_factor * max(v for _, v in per)
    psf = P.Psf(P.Volume(inst.kernel), normalize=False)
    opts = P.SolverOptions(lam=lam, n_sigma=6, n_shape=5, max_outer_iterations=50)
    record = []
    res = solvers._solve(P.Volume(y), psf, opts, b, solvers.BSFW, record=record)
    return dict(inst=inst, khat=khat, y=y, lam=lam, sg=sg, dg=dg, win=win, psf=psf, res=res,
                record=record, box5=P.measures.bounds_box(b))


def _residual(y, khat, thetas, weights):
    phis = [O.phi(t.to_array(), khat, y.shape) for t in thetas]
    return O.residual(y, weights, phis)


def test_cfg2_solve_shape(cfg2_solve):
    res = cfg2_solve["res"]
    assert res.termination == "certificate"
    assert 15 <= len(res.measure) <= 40


def _cert_steps(c):
    return [r for r in c["record"] if r["step"] == "certificate"]


def _lasso_steps(c):
    return [r for r in c["record"] if r["step"] == "lasso"]


@pytest.mark.parametrize("part", range(4))
def test_cfg2_certificate_step_replay(cfg2_solve, part):
    """Every certificate step of the solve (split over 4 test items)."""
    c = cfg2_solve
    for st in _cert_steps(c)[part::4]:
        _replay_certificate(c, st)


def _replay_certificate(c, st):
    r = _residual(c["y"], c["khat"], st["thetas"], st["weights"])
    per = O.eta_maxima(r, c["lam"], c["khat"], c["sg"], c["dg"], c["win"], threads=8)
    flat = max(range(len(per)), key=lambda i: (per[i][1], -i))
    pos, val = per[flat]
    i, j = divmod(flat, len(c["dg"]))
    assert st["cand"] == (i, j) and tuple(st["start"].m) == tuple(float(p) for p in pos), st["k"]
    assert abs(st["eta_grid"] - val) <= 1e-9 * abs(val)
    back = O.corr(r, c["khat"])
    start = np.array([*pos, c["sg"][i], c["dg"][j]], dtype=float)
    theta, eta = O.refine_eta_max(back, c["lam"], start, c["box5"])
    assert abs(st["eta"] - eta) <= 1e-9 * abs(eta), (st["eta"], eta)
    np.testing.assert_allclose(st["theta"].to_array(), theta, atol=1e-6, rtol=0)


def test_cfg2_lasso_step_replay(cfg2_solve):
    """Every weight step of the solve."""
    c = cfg2_solve
    for st in _lasso_steps(c):
        _replay_lasso(c, st)


def _replay_lasso(c, st):
    phis = np.stack([O.phi(t.to_array(), c["khat"], c["y"].shape) for t in st["thetas"]])
    gram, b = O.gram_system(phis, c["y"])
    w, _, _ = O.cd_solve(gram, b, c["lam"], st["w_init"], tol=1e-6, max_iter=2000)
    assert np.max(np.abs(st["weights"] - w)) <= 1e-8 * max(1.0, np.max(np.abs(w)))


def test_cfg2_final_slide_replay(P, cfg2_solve):
    from paper_2009_05473_b200 import solvers
    from paper_2009_05473_b200.forward import to_dev
    c = cfg2_solve
    steps = [r for r in c["record"] if r["step"] == "descent"]
    assert steps, "BSFW ran no final slide"
    start = steps[-1]["start"]
    b = c["inst"].bounds
    got, cg, _ = solvers.local_descent_dev(to_dev(P.Volume(c["y"])), start, c["psf"], c["lam"], b,
                                           max_iter=3)
    rows0 = start.to_rows()
    want, cw = O.local_descent(c["y"], rows0, c["khat"], c["lam"], c["box5"], max_iter=3)
    assert abs(cg - cw) <= 1e-9 * abs(cw), (cg, cw)
    g = got.to_rows()
    assert g.shape == want.shape
    np.testing.assert_allclose(g[:, 1:4], want[:, 1:4], atol=1e-6, rtol=0)
    np.testing.assert_allclose(g[:, [0, 4, 5]], want[:, [0, 4, 5]], rtol=1e-6, atol=1e-9)
