"""GPU tests of the separable 1-D pass kernels (K4) across tile geometries:
the staged register-window tiles (pass_z2 contiguous, pass_tile2 strided:
partial row / column tiles, periodic wrap inside a staged row, wide and
narrow filters, odd offsets) and the fallbacks (short axes, rows wider than
the axis, z extents not a multiple of 4), checked against the oracle's FFT
circular convolution / correlation.

Bars: fp64 1e-12 of max|ref|; fp32 storage 2e-6 of max|ref| (fp32 FMA
chains of <= 89 taps)."""
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


GEOMS = [
    ((128, 128, 128), (2.0, 2.0, 2.0), (7, 7, 7)),      # staged tiles everywhere, full tiles
    ((97, 65, 192), (3.0, 1.0, 4.0), (15, 3, 15)),      # partial row / column tiles, To > n
    ((96, 192, 256), (9.0, 9.0, 9.0), (30, 44, 44)),    # 61- and 89-tap filters
    ((130, 64, 132), (0.5, 2.0, 0.7), (1, 9, 2)),       # z row wider than the axis
    ((48, 40, 36), (1.5, 1.5, 2.0), (3, 3, 4)),         # short axes
    ((40, 40, 64), (1.0, 4.0, 5.0), (3, 15, 17)),       # z taps wrap the axis
    ((24, 72, 200), (1.0, 3.0, 2.0), (2, 17, 6)),       # partial y and z tiles
    ((20, 18, 30), (1.0, 1.0, 1.0), (3, 3, 3)),         # nz % 4 != 0, stride % 64 != 0
    ((256, 16, 64), (6.0, 1.0, 1.0), (25, 3, 3)),       # wide fp32/fp64 strided tiles
]


@pytest.mark.parametrize("dims,sig,half", GEOMS)
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_psf_passes_vs_fft(P, dims, sig, half, prec):
    rng = np.random.default_rng(sum(dims))
    kernel = O.box_gaussian_psf(dims, sig, half)
    x = rng.standard_normal(dims)
    if prec == "f32":
        x = x.astype(np.float32).astype(np.float64)
    khat = O.psf_hat(kernel)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    tol = 2e-6 if prec == "f32" else 1e-12
    with P.precision(prec):
        fwd = P.convolve(P.Volume(x), psf).data
        adj = P.correlate_adjoint(P.Volume(x), psf).data
    for got, ref in ((fwd, O.conv(x, khat)), (adj, O.corr(x, khat))):
        err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        assert err <= tol, (dims, prec, err)
