"""Per-family device time of one config-2 (128^3 f64) or config-3 (256^3
fp32) certificate on a synthetic residual: python tools/cert_cfg3.py [2|3]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import eta_argmax_dev  # noqa: E402
from paper_2009_05473_b200.forward import psf_apply_dev, render_dev  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = {2: configs.config2, 3: configs.config3}[cfg](0)
P.set_precision(inst.precision)
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
code = N.dtype_code()
clean = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, code), False)
r = 0.01 * torch.randn(inst.dims, device="cuda", dtype=clean.dtype) + clean
table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, bounds=inst.bounds)
win = ((0, inst.dims[0] - 1), (0, inst.dims[1] - 1), (0, inst.dims[2] - 1))
for _ in range(3):
    eta_argmax_dev(r, 1.0, table, win)
torch.cuda.synchronize()
ctx = N.context()
ctx.profile(True)
eta_argmax_dev(r, 1.0, table, win)
fam = {f: ctx.profile_read(f) for f in ("eta_direct", "eta_basis", "eta_basis_wide", "eta_mix", "eta_refine", "psf_pass", "pad", "argmax")}
ctx.profile(False)
info = table.info()
print({k: (round(v[0], 3), v[1]) for k, v in fam.items() if v[1]}, "refined", N.last_refine_count(),
      "members", info["n_basis"], "direct", info["n_direct"])
