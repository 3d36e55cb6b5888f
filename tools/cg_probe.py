"""Config-5 cost + gradient breakdown: wall time per synchronous call, device
time per kernel family (library CUDA events), and the algorithmic rooflines
of render / atom sums (FP32 and MUFU work per atom-voxel)."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.forward import cost_grad_dev, psf_apply_dev, render_dev  # noqa: E402

P.set_precision("f32")
inst = configs.config5()
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
y = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
perts = configs.perturbations(inst.truth, 20)
ctx = N.context(0)
for i in range(5):
    cost_grad_dev(psf, y, perts[i], 0.1)
torch.cuda.synchronize()
reps = 50
t0 = time.perf_counter()
for i in range(reps):
    cost_grad_dev(psf, y, perts[i % 20], 0.1)
wall = (time.perf_counter() - t0) / reps
ctx.profile(True)
for i in range(10):
    cost_grad_dev(psf, y, perts[i], 0.1)
fam = {f: ctx.profile_read(f) for f in ("render", "psf_pass", "sumsq", "atom_sums")}
ctx.profile(False)
_, _, ln, _ = N.atom_geometry(inst.dims, perts[0])
sbox = float(np.prod(ln, axis=1).sum())
print(json.dumps({"wall_ms": 1e3 * wall, "evals_per_s": 1 / wall,
                  "device_ms": {k: v[0] / 10 for k, v in fam.items()},
                  "launches": {k: v[1] / 10 for k, v in fam.items()},
                  "sum_box_voxels": sbox}, indent=1))
