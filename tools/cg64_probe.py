"""Config-2 shaped fp64 cost + gradient (128^3, k atoms): wall per evaluation and
per-family device time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.forward import cost_grad_dev, psf_apply_dev, render_dev  # noqa: E402

inst = configs.config2(0)
P.set_precision("f64")
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
y = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F64), False)
rows = inst.truth.copy()
rows[:, 1:4] += 0.1
ctx = N.context(0)
for _ in range(3):
    cost_grad_dev(psf, y, rows, 0.1)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    cost_grad_dev(psf, y, rows, 0.1)
wall = (time.perf_counter() - t0) / 50
ctx.profile(True)
for _ in range(10):
    cost_grad_dev(psf, y, rows, 0.1)
fam = {f: ctx.profile_read(f) for f in ("render", "psf_pass", "sumsq", "atom_sums")}
ctx.profile(False)
print("k", len(rows), "wall ms/eval %.3f" % (1e3 * wall), {k: (round(v[0] / 10, 4), v[1] // 10) for k, v in fam.items()})
