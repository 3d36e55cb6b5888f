"""Cost of one certificate ascent (refine_eta_max) at config 3: evaluations
per ascent, wall time per evaluation (one sfw3d_atom_sums call, k = 1) and
the device time of its kernels."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import refine_eta_max_dev  # noqa: E402
from paper_2009_05473_b200.forward import atom_sums_dev, psf_apply_dev, render_dev  # noqa: E402

inst = configs.config3(0)
P.set_precision(inst.precision)
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
code = N.dtype_code()
clean = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, code), False)
r = 0.01 * torch.randn(inst.dims, device="cuda", dtype=clean.dtype) + clean
back = psf_apply_dev(psf, r, True)
ctx = N.context()
for sigma, d in ((1.0, 2.5), (2.0, 2.0), (3.0, 1.5)):
    row = np.array([[1.0, *inst.truth[0, 1:4], sigma, d]])
    for _ in range(5):
        atom_sums_dev(back, row)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        atom_sums_dev(back, row)
    wall = (time.perf_counter() - t0) / 200
    ctx.profile(True)
    for _ in range(20):
        atom_sums_dev(back, row)
    fam = {f: ctx.profile_read(f) for f in ("atom_sums", "render", "psf_pass")}
    ctx.profile(False)
    print(f"sigma={sigma} d={d}: {1e6 * wall:.1f} us/eval wall; device {fam}")
    start = P.AtomParams(m=tuple(np.round(inst.truth[0, 1:4])), sigma=sigma, d=d)
    info = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th, eta = refine_eta_max_dev(r, 1.0, psf, start, inst.bounds, back=back, info=info)
    dt = time.perf_counter() - t0
    print(f"   refine: {1e3 * dt:.2f} ms, {info['lbfgsb']}, {1e6 * dt / info['lbfgsb']['evaluations']:.1f} us/eval")
