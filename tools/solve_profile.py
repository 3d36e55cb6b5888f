"""Where a config-2 / config-3 solve spends its time: wall time and call
counts of the certificate's grid stage, refine (+ its atom-sum callbacks),
the residual, the weight step and the descent. python tools/solve_profile.py [3]"""
import collections
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from paper_2009_05473_b200 import certificate as Cm, forward as F, solvers as S  # noqa: E402
import run_solve  # noqa: E402

T = collections.defaultdict(float)
Nc = collections.Counter()


def wrap(mod, name, key):
    f = getattr(mod, name)

    def g(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f(*a, **k)
        torch.cuda.synchronize()
        T[key] += time.perf_counter() - t0
        Nc[key] += 1
        return out
    setattr(mod, name, g)


wrap(Cm, "eta_field_dev", "eta_grid")
wrap(Cm, "eta_argmax_dev", "eta_argmax_dev")
wrap(Cm, "_position_window", "position_window")
_ef = Cm.eta_field_dev
REF = []


FAM = collections.defaultdict(float)


def ef(*a, **k):
    from paper_2009_05473_b200 import _native as N
    ctx = N.context()
    ctx.profile(True)
    out = _ef(*a, **k)
    for f in ("eta_direct", "eta_basis", "eta_basis_wide", "eta_mix", "eta_refine", "psf_pass", "pad", "argmax"):
        FAM[f] += ctx.profile_read(f)[0]
    ctx.profile(False)
    REF.append(N.last_refine_count())
    return out


Cm.eta_field_dev = ef
wrap(Cm, "refine_eta_max_dev", "refine")
wrap(Cm, "atom_sums_dev", "refine_atom_sums")
wrap(S, "residual_dev", "residual")
wrap(S, "_lasso_on", "lasso_solve")
wrap(S, "phi_dev", "phi")
wrap(S, "dots_dev", "dots")
wrap(S, "cost_grad_dev", "descent_cost_grad")
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r = run_solve.run(cfg, "bsfw")
print({k: r[k] for k in ("solve_s", "outer_iterations", "atoms", "split_s")})
for k in sorted(T, key=lambda k: -T[k]):
    print(f"  {k:20s} {T[k]:8.3f} s  {Nc[k]:6d} calls  {1e3 * T[k] / max(Nc[k], 1):8.3f} ms/call")
import numpy as np  # noqa: E402
print("refined voxels per certificate: median", int(np.median(REF)), "max", max(REF),
      "sum", sum(REF), "last 10", REF[-10:])
print("eta device ms per call:", {k: round(v / max(len(REF), 1), 3) for k, v in FAM.items() if v})
