"""Wall time vs device time of one certificate grid stage (config 3 / 4):
python tools/eta_wall.py [3|4]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs  # noqa: E402
from paper_2009_05473_b200.certificate import eta_argmax_dev  # noqa: E402
from paper_2009_05473_b200.forward import psf_apply_dev, render_dev  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = {3: configs.config3, 4: configs.config4}[cfg](0)
P.set_precision("f32")
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
clean = psf_apply_dev(psf, render_dev(inst.truth, inst.dims, N.F32), False)
r = 0.01 * torch.randn(inst.dims, device="cuda") + clean
table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, bounds=inst.bounds,
                               tap_tol=float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
win = P.certificate._position_window(inst.bounds, inst.dims)
for _ in range(3):
    eta_argmax_dev(r, 1.0, table, win)
torch.cuda.synchronize()
ctx = N.context()
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    eta_argmax_dev(r, 1.0, table, win)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
ctx.profile(True)
for _ in range(reps):
    eta_argmax_dev(r, 1.0, table, win)
fam = {f: ctx.profile_read(f) for f in ("eta_direct", "eta_basis", "eta_basis_wide", "eta_mix", "eta_refine",
                                       "psf_pass", "pad", "argmax")}
ctx.profile(False)
dev = sum(v[0] for v in fam.values()) / reps
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    eta_argmax_dev(r, 1.0, table, win)
e1.record()
torch.cuda.synchronize()
print(f"cfg{cfg}: wall {1e3 * wall:.3f} ms, stream-event {e0.elapsed_time(e1) / reps:.3f} ms, "
      f"kernel families {dev:.3f} ms, refined {N.last_refine_count()}",
      {k: round(v[0] / reps, 3) for k, v in fam.items() if v[1]})
