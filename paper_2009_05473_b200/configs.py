"""Seeded synthetic instances of the BASELINE.json configs.

No public dataset is involved: every config is a recipe (atoms drawn from a
seeded numpy Generator in the order positions, sigma, d, w) rendered with
this package's own forward operator, except the config-4 residual, which is
generated on the host (``cfg4_residual_host``) so that the GPU arm and the
CPU reference arm of ``bench.py`` consume the identical array. Shapes, sizes and value distributions follow
BASELINE.json `configs`; unspecified items use the SURVEY Appendix A
choices, restated in each docstring.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .measures import DomainBounds


def box_psf_kernel(dims, sigmas, half) -> np.ndarray:
    """Box-truncated sampled Gaussian over -h..h per axis, centred at n//2, unit sum."""
    k = np.zeros(tuple(dims))
    ax = [np.exp(-0.5 * (np.arange(-h, h + 1) / s) ** 2) for s, h in zip(sigmas, half)]
    box = ax[0][:, None, None] * ax[1][None, :, None] * ax[2][None, None, :]
    k[tuple(slice(n // 2 - h, n // 2 + h + 1) for n, h in zip(dims, half))] = box
    return k / k.sum()


def _positions(rng, n_atoms, lo, hi, min_sep=None, max_tries=200000):
    pts = []
    tries = 0
    while len(pts) < n_atoms:
        tries += 1
        if tries > max_tries:
            raise RuntimeError("could not place atoms with the requested separation")
        p = rng.uniform(lo, hi, size=3)
        if min_sep is None or all(np.linalg.norm(p - q) >= min_sep for q in pts):
            pts.append(p)
    return np.array(pts)


@dataclass
class Instance:
    name: str
    dims: tuple
    kernel: np.ndarray
    truth: np.ndarray            # (N, 6) rows w, m, sigma, d
    bounds: DomainBounds | None
    sigma_grid: np.ndarray | None
    shape_grid: np.ndarray | None
    snr_db: float | None
    lam_factor: float | None
    precision: str


def config1(seed=0) -> Instance:
    """64^3 f64, N=5, m~U[8,56]^3, sigma~U[1.5,3], d~U[1.5,2.5], w~U[1,2]; PSF sigma_h=2 15^3;
    SNR 20 dB (power); lam = 0.1 max Phi*y; grid sigma{1.5,2,2.5,3} x d{1.5,2,2.5}."""
    rng = np.random.default_rng(seed)
    dims = (64, 64, 64)
    m = _positions(rng, 5, 8.0, 56.0)
    rows = np.column_stack([rng.uniform(1, 2, 5), m, rng.uniform(1.5, 3, 5), rng.uniform(1.5, 2.5, 5)])
    rows = rows[:, [0, 1, 2, 3, 4, 5]]
    return Instance("cfg1", dims, box_psf_kernel(dims, (2, 2, 2), (7, 7, 7)), rows,
                    DomainBounds((8.0,) * 3, (56.0,) * 3, 1.5, 3.0, 1.5, 2.5),
                    np.array([1.5, 2.0, 2.5, 3.0]), np.array([1.5, 2.0, 2.5]), 20.0, 0.1, "f64")


def config2(seed=0) -> Instance:
    """128^3 f64, N=20 (min sep 6, margin 9), sigma~U[1,3], d~U[1.2,2.8], w~U[0.5,2];
    PSF (1.5,1.5,4) on 17x17x33; SNR 15 dB; lam = 0.05 max Phi*y; 6 x 5 grid."""
    rng = np.random.default_rng(seed)
    dims = (128, 128, 128)
    m = _positions(rng, 20, 9.0, 118.0, min_sep=6.0)
    rows = np.column_stack([rng.uniform(0.5, 2, 20), m, rng.uniform(1, 3, 20), rng.uniform(1.2, 2.8, 20)])
    b = DomainBounds((9.0,) * 3, (118.0,) * 3, 1.0, 3.0, 1.2, 2.8)
    return Instance("cfg2", dims, box_psf_kernel(dims, (1.5, 1.5, 4.0), (8, 8, 16)), rows, b,
                    np.geomspace(1, 3, 6), np.linspace(1.2, 2.8, 5), 15.0, 0.05, "f64")


def config3(seed=0) -> Instance:
    """256^3 fp32 storage, N=100 (min sep 5), sigma~U[1,3], d~U[1.5,2.5], w log-U[0.3,3];
    PSF sigma_h=2.5 21^3; SNR 10 dB; assumed lam = 0.05 max Phi*y and an 8 x 6 grid."""
    rng = np.random.default_rng(seed)
    dims = (256, 256, 256)
    m = _positions(rng, 100, 9.0, 246.0, min_sep=5.0)
    w = np.exp(rng.uniform(np.log(0.3), np.log(3.0), 100))
    rows = np.column_stack([w, m, rng.uniform(1, 3, 100), rng.uniform(1.5, 2.5, 100)])
    b = DomainBounds((9.0,) * 3, (246.0,) * 3, 1.0, 3.0, 1.5, 2.5)
    return Instance("cfg3", dims, box_psf_kernel(dims, (2.5,) * 3, (10,) * 3), rows, b,
                    np.geomspace(1, 3, 8), np.linspace(1.5, 2.5, 6), 10.0, 0.05, "f32")


def config4(seed=0, n=512) -> Instance:
    """512^3 fp32 residual = N(0,1) + 200 blurred generalized Gaussians (assumed m~U[0,n)^3,
    sigma~U[1,3], d~U[1.5,3], w~U[5,10]); PSF sigma_h=3 31^3; 16 candidates
    sigma{1,1.5,2,3} x d{1.5,2,2.5,3}; window = every voxel."""
    rng = np.random.default_rng(seed)
    dims = (n, n, n)
    m = rng.uniform(0, n, size=(200, 3))
    rows = np.column_stack([rng.uniform(5, 10, 200), m, rng.uniform(1, 3, 200), rng.uniform(1.5, 3, 200)])
    return Instance("cfg4", dims, box_psf_kernel(dims, (3,) * 3, (15,) * 3), rows, None,
                    np.array([1.0, 1.5, 2.0, 3.0]), np.array([1.5, 2.0, 2.5, 3.0]), None, None, "f32")


def config5(seed=0, n=256, n_atoms=1000) -> Instance:
    """256^3 fp32 observation y = forward(truth) (no noise), N=1000 atoms m~U[0,n-1]^3
    (boxes wrap), sigma~U[1,3], d~U[1.5,2.5], w~U[0.5,2]; PSF sigma_h=2 15^3."""
    rng = np.random.default_rng(seed)
    dims = (n, n, n)
    m = rng.uniform(0, n - 1, size=(n_atoms, 3))
    rows = np.column_stack([rng.uniform(0.5, 2, n_atoms), m, rng.uniform(1, 3, n_atoms),
                            rng.uniform(1.5, 2.5, n_atoms)])
    return Instance("cfg5", dims, box_psf_kernel(dims, (2,) * 3, (7,) * 3), rows, None, None, None,
                    None, None, "f32")


def perturbations(truth: np.ndarray, count: int, std: float = 0.1, seed: int = 1):
    """cfg5: `count` perturbed parameter sets theta + std*N(0,1) on all 6 columns, w >= 0."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        p = truth + std * rng.standard_normal(truth.shape)
        p[:, 0] = np.maximum(p[:, 0], 0.0)
        p[:, 4] = np.maximum(p[:, 4], 0.5)
        p[:, 5] = np.maximum(p[:, 5], 1.05)
        out.append(p)
    return out


def _render_host(rows: np.ndarray, dims) -> np.ndarray:
    """Host rendering of generalized Gaussians for synthetic DATA generation
    (not a compute path): w exp(-|s - m|^d / (2 sigma^d)) on the periodic
    box round(m) +- ceil(sigma (2 ln 1e12)^(1/d)) per axis (boxes < n)."""
    out = np.zeros(tuple(dims))
    for w, mx, my, mz, sg, d in np.asarray(rows, dtype=float).reshape(-1, 6):
        r = int(np.ceil(sg * (2.0 * np.log(1e12)) ** (1.0 / d)))
        idx, off = [], []
        for m, n in zip((mx, my, mz), dims):
            span = np.arange(int(np.round(m)) - r, int(np.round(m)) + r + 1)
            idx.append(np.remainder(span, n))
            off.append(span - m)
        u2 = off[0][:, None, None] ** 2 + off[1][None, :, None] ** 2 + off[2][None, None, :] ** 2
        out[np.ix_(*idx)] += w * np.exp(-0.5 * u2 ** (0.5 * d) / sg ** d)
    return out


def cfg4_residual_host(inst: Instance, seed: int = 4) -> np.ndarray:
    """Config-4 residual as a host float32 array: N(0,1) i.i.d. noise (numpy
    Generator(seed)) + the 200 generalized Gaussians blurred by the PSF
    (circular, through scipy.fft). Both bench arms use this exact array."""
    import os
    import scipy.fft as sfft
    dims = inst.dims
    workers = os.cpu_count() or 1
    atoms = _render_host(inst.truth, dims)
    khat = sfft.rfftn(sfft.ifftshift(inst.kernel), workers=workers)
    blurred = sfft.irfftn(sfft.rfftn(atoms, workers=workers) * khat, s=dims, workers=workers)
    del atoms, khat
    r = np.random.default_rng(seed).standard_normal(dims, dtype=np.float32)
    r += blurred.astype(np.float32)
    return r


def observation_host(inst: Instance, seed: int = 0) -> np.ndarray:
    """y = H * truth + white noise at the config's power SNR, as a host float64
    array (numpy Generator(seed) noise, circular blur through scipy.fft):
    identical on every rank of a sharded run (which builds it independently)."""
    import os
    import scipy.fft as sfft
    dims = inst.dims
    workers = os.cpu_count() or 1
    khat = sfft.rfftn(sfft.ifftshift(inst.kernel), workers=workers)
    clean = sfft.irfftn(sfft.rfftn(_render_host(inst.truth, dims), workers=workers) * khat, s=dims,
                        workers=workers)
    sigma = float(np.sqrt(np.mean(clean ** 2) / 10 ** (inst.snr_db / 10)))
    y = clean + sigma * np.random.default_rng(seed).standard_normal(dims)
    if inst.precision == "f32":
        y = y.astype(np.float32).astype(np.float64)
    return y
