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


def _rotated_psf(dims, half):
    """A non-separable kernel: anisotropic Gaussian with rotated axes on a box."""
    ax = [np.arange(-h, h + 1) for h in half]
    x, y, z = np.meshgrid(*ax, indexing="ij")
    u, v = 0.8 * x + 0.6 * y, -0.6 * x + 0.8 * y
    box = np.exp(-0.5 * ((u / 2.5) ** 2 + (v / 1.2) ** 2 + ((z + 0.3 * x) / 1.8) ** 2))
    k = np.zeros(dims)
    k[tuple(slice(n // 2 - h, n // 2 + h + 1) for n, h in zip(dims, half))] = box
    return k / k.sum()


@pytest.mark.parametrize("dims,half", [((96, 80, 64), (7, 7, 7)), ((33, 40, 30), (4, 3, 5))])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_nonseparable_psf_fft_path(P, dims, half, prec):
    """Non-separable kernels with more than 125 box taps go through cuFFT (the
    reference's own rfftn * H_hat, forward.py:79-94); odd dims included."""
    rng = np.random.default_rng(sum(dims))
    kernel = _rotated_psf(dims, half)
    x = rng.standard_normal(dims)
    if prec == "f32":
        x = x.astype(np.float32).astype(np.float64)
    khat = O.psf_hat(kernel)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    assert not psf.separable()
    tol = 2e-6 if prec == "f32" else 1e-12
    with P.precision(prec):
        fwd = P.convolve(P.Volume(x), psf).data
        adj = P.correlate_adjoint(P.Volume(x), psf).data
        rows = np.column_stack([rng.uniform(0.5, 2, 8), rng.uniform(0, 1, (8, 3)) * dims,
                                rng.uniform(1, 2, 8), rng.uniform(1.6, 2.4, 8)])
        meas = P.WeightedMeasure(tuple((P.AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]), r[0])
                                       for r in rows))
        c, g = P.criterion_and_gradient(P.Volume(x), meas, psf, 0.1)
    for got, ref in ((fwd, O.conv(x, khat)), (adj, O.corr(x, khat))):
        assert np.max(np.abs(got - ref)) <= tol * np.max(np.abs(ref))
    c0, g0, _ = O.criterion_and_gradient(x, rows, khat, 0.1)
    assert abs(c - c0) <= (1e-5 if prec == "f32" else 1e-12) * abs(c0)
    scale = np.max(np.abs(g0), axis=0)
    assert np.max(np.max(np.abs(g.per_atom - g0), axis=0) / scale) <= (1e-4 if prec == "f32" else 1e-11)


def test_certificate_with_nonseparable_psf(P):
    """eta_field with a non-separable (FFT-path) PSF against the oracle."""
    dims = (48, 40, 44)
    rng = np.random.default_rng(9)
    kernel = _rotated_psf(dims, (5, 5, 5))
    r = rng.standard_normal(dims)
    sg, dg = np.array([1.0, 1.6]), np.array([1.7, 2.0, 2.4])
    psf = P.Psf(P.Volume(kernel), normalize=False)
    table = P.build_template_table(psf, sg, dg)
    f = P.eta_field(P.Volume(r), 0.6, table, keep_fields=False)
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    pos, flat, val, _, _ = O.eta_field(r, 0.6, hats, len(dg))
    assert f.argmax_position == pos and abs(f.eta_max - val) <= 1e-10 * abs(val)
