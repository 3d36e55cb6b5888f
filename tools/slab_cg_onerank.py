"""Per-rank time of the x-slab cost + gradient (distributed.SlabCostGrad) on
BASELINE config 5 (256^3 fp32, N = 1000): each rank of a W-rank layout is run
alone on this GPU (only one GPU is available to this build), device-timed with
CUDA events around synchronous sfw3d_cost_grad_slab calls; also checks that
the W ranks' partials summed reproduce the single-volume C and gradient.
Prints one JSON line per W."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs, distributed as D  # noqa: E402
from paper_2009_05473_b200.forward import cost_grad_dev, psf_apply_dev, render_dev  # noqa: E402

P.set_precision("f32")
inst = configs.config5()
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
y = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
perts = configs.perturbations(inst.truth, 100)
steps = 20
c_ref, g_ref = cost_grad_dev(psf, y, perts[0], 0.1)
for w in (1, 2, 4, 8):
    per_rank, half, sums = [], 0.0, np.zeros_like(g_ref)
    for r in range(w):
        x0, x1 = D.slab_bounds(inst.dims[0], w, r)
        if w == 1:
            t0 = time.perf_counter()
            for i in range(steps):
                cost_grad_dev(psf, y, perts[i % 100], 0.1)
            per_rank.append((time.perf_counter() - t0) / steps * 1e3)
            half, sums = None, None
            continue
        sl = D.SlabCostGrad(psf, inst.dims, x0, x1)
        yw = sl.window(y)
        h, s = sl.partials(yw, perts[0])
        half += h
        sums += s
        for i in range(3):
            sl.partials(yw, perts[i])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(steps):
            sl.partials(yw, perts[i % 100])
        per_rank.append((time.perf_counter() - t0) / steps * 1e3)
    out = {"W": w, "per_rank_ms": per_rank, "max_rank_ms": max(per_rank),
           "timing": "wall clock per synchronous C-ABI call, ranks run one at a time"}
    if half is not None:
        c, g = D.finish_cost_grad(half, sums, perts[0], 0.1)
        out["rel_err_C"] = abs(c - c_ref) / abs(c_ref)
        sc = np.maximum(np.max(np.abs(g_ref), axis=0), 1e-300)
        out["rel_err_grad_colwise"] = float(np.max(np.max(np.abs(g - g_ref), axis=0) / sc))
    print(json.dumps(out), flush=True)
