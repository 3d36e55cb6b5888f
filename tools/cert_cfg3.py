"""Per-family device time of one config-3 certificate (256^3 fp32, 8 x 6
candidates) on a synthetic residual."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import eta_argmax_dev  # noqa: E402
from paper_2009_05473_b200.forward import psf_apply_dev, render_dev  # noqa: E402

inst = configs.config3(0)
P.set_precision("f32")
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
r = 0.01 * torch.randn(inst.dims, device="cuda") + psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, bounds=inst.bounds)
win = ((0, inst.dims[0] - 1), (0, inst.dims[1] - 1), (0, inst.dims[2] - 1))
for _ in range(3):
    eta_argmax_dev(r, 1.0, table, win)
torch.cuda.synchronize()
ctx = N.context()
ctx.profile(True)
eta_argmax_dev(r, 1.0, table, win)
fam = {f: ctx.profile_read(f) for f in ("eta_direct", "eta_basis", "eta_mix", "eta_refine", "psf_pass", "pad", "argmax")}
ctx.profile(False)
info = table.info()
print({k: (round(v[0], 3), v[1]) for k, v in fam.items() if v[1]}, "refined", N.last_refine_count(),
      "members", info["n_basis"], "direct", info["n_direct"])
