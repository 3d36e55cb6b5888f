"""Config-4 (or --n 256) certificate: step time and the per-candidate maxima,
to compare pass variants (e.g. SFW3D_ZY=0/1) for speed and bitwise equality."""
import argparse
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import eta_argmax_dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
a = ap.parse_args()
P.set_precision("f32")
inst = configs.config4(n=a.n)
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, tap_tol=1e-12)
r = torch.from_numpy(configs.cfg4_residual_host(inst)).cuda()
win = tuple((0, d - 1) for d in inst.dims)
for _ in range(3):
    best, per, _ = eta_argmax_dev(r, 1.0, table, win)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    best, per, _ = eta_argmax_dev(r, 1.0, table, win)
e1.record()
torch.cuda.synchronize()
ctx = N.context()
ctx.profile(True)
eta_argmax_dev(r, 1.0, table, win)
fam = {f: ctx.profile_read(f) for f in ("eta_basis", "eta_basis_wide", "eta_basis_zy", "eta_mix", "eta_refine", "psf_pass")}
ctx.profile(False)
vals = np.array([p.value for p in per])
pos = [tuple(p.pos) for p in per]
print("ms/step %.3f" % (e0.elapsed_time(e1) / 10), {k: (round(v[0], 3), v[1]) for k, v in fam.items() if v[1]})
print("digest", hashlib.sha1(vals.tobytes() + np.array(pos).tobytes()).hexdigest()[:16], "best", best.value, tuple(best.pos), best.cand)
