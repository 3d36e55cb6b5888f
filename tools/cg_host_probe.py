"""Host-side cost of one cost+grad call (config 5): cProfile over 50 calls."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.forward import cost_grad_dev, psf_apply_dev, render_dev  # noqa: E402

P.set_precision("f32")
inst = configs.config5()
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
y = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
perts = configs.perturbations(inst.truth, 10)
for i in range(3):
    cost_grad_dev(psf, y, perts[i], 0.1)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(50):
    cost_grad_dev(psf, y, perts[i % 10], 0.1)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
