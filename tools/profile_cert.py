"""One certificate evaluation (BASELINE config 4 recipe) for ncu captures.

    python tools/profile_cert.py --n 512 [--mode auto|direct] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import eta_argmax_dev  # noqa: E402
from paper_2009_05473_b200.forward import cost_grad_dev, psf_apply_dev, render_dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--mode", default="auto")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--costgrad", action="store_true")
a = ap.parse_args()
P.set_precision("f32")
if a.costgrad:
    inst = configs.config5()
    psf = P.Psf(P.Volume(inst.kernel), normalize=False)
    y = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
    perts = configs.perturbations(inst.truth, 4)
    for i in range(a.reps):
        c, _ = cost_grad_dev(psf, y, perts[i % 4], 0.1)
    print("C", c)
else:
    inst = configs.config4(n=a.n)
    psf = P.Psf(P.Volume(inst.kernel), normalize=False)
    table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, tap_tol=1e-12, mode=a.mode)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    r = torch.randn(inst.dims, generator=g, device="cuda", dtype=torch.float32)
    r += psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
    win = tuple((0, n - 1) for n in inst.dims)
    for _ in range(a.reps):
        best, _, _ = eta_argmax_dev(r, 1.0, table, win)
    print("best", best.value, tuple(best.pos), best.cand)
torch.cuda.synchronize()
