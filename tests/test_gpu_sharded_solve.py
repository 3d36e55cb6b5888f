"""The x-slab sharded SFW / BSFW solve (sharded.sharded_solve: SURVEY §8(e),
BASELINE config 3's "full solve sharded ... at 1/2/4/8 GPUs") with ranks as
threads on this GPU (distributed.ThreadComm): every rank returns the same
result, equal to the single-GPU solve of the same observation at the
north-star bar (same atom count, positions within 1e-3 voxel, weights and
sigma / d within 1e-4 relative). The ranks hold only their own planes of y,
of every blurred atom and of the residual; Gram rows, ||r||^2, the refine's
atom sums and the descents' partials are all-reduced."""
import numpy as np
import pytest

import sfw3d_oracle as O
from test_gpu_certificate import _run_ranks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2009_05473_b200 as pkg
    pkg.set_precision("f64")
    return pkg


def _problem(P):
    rng = np.random.default_rng(17)
    dims = (96, 48, 48)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 1.5), (4, 4, 4))
    truth = np.column_stack([rng.uniform(1, 2, 6), rng.uniform(14, 82, 6), rng.uniform(10, 38, 6),
                             rng.uniform(10, 38, 6), rng.uniform(1.0, 1.6, 6),
                             rng.uniform(1.8, 2.2, 6)])
    truth[0, 1] = 31.6  # near a 2- and 3-rank slab boundary
    clean = O.conv(O.render(truth, dims), O.psf_hat(kernel))
    y = clean + O.power_snr_sigma(clean, 25.0) * rng.standard_normal(dims)
    bounds = P.DomainBounds((10.0, 6.0, 6.0), (86.0, 42.0, 42.0), 1.0, 1.6, 1.8, 2.2)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    sg, dg = P.make_parameter_grids(bounds, 3, 3)
    table = P.build_template_table(psf, sg, dg, bounds=bounds)
    lam = 0.1 * P.eta_field(P.Volume(y), 1.0, table, bounds=bounds, keep_fields=False).eta_max
    return y, psf, bounds, P.SolverOptions(lam=lam, n_sigma=3, n_shape=3, max_outer_iterations=30)


@pytest.mark.parametrize("algo,nranks", [("bsfw", 2), ("bsfw", 3), ("sfw", 2)])
def test_sharded_solve_matches_single_gpu(P, algo, nranks):
    from paper_2009_05473_b200.sharded import sharded_solve
    y, psf, bounds, opts = _problem(P)
    ref = getattr(P, algo)(P.Volume(y), psf, opts, bounds)
    outs = _run_ranks(nranks, lambda r, comm: sharded_solve(P.Volume(y), psf, opts, bounds, algo,
                                                            comm))
    want = ref.measure.to_rows()
    for res in outs:
        assert res.termination == ref.termination
        assert len(res.trace.records) == len(ref.trace.records)
        got = res.measure.to_rows()
        assert got.shape == want.shape
        for row in want:
            j = int(np.argmin(np.linalg.norm(got[:, 1:4] - row[1:4], axis=1)))
            assert np.linalg.norm(got[j, 1:4] - row[1:4]) < 1e-3
            np.testing.assert_allclose(got[j, [0, 4, 5]], row[[0, 4, 5]], rtol=1e-4)
        assert abs(res.criterion - ref.criterion) <= 1e-8 * abs(ref.criterion)
    assert all(np.array_equal(o.measure.to_rows(), outs[0].measure.to_rows()) for o in outs)
