"""Per-call LASSO statistics of a config-3 solve: atoms k, CD sweeps, device
time per call (wraps solvers.cd_dev)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_2009_05473_b200 import solvers  # noqa: E402

calls = []
_orig = solvers.cd_dev


def cd_dev(gram, b, lam, w_init, tol, max_iter, device=None, **kw):
    t0 = time.perf_counter()
    out = _orig(gram, b, lam, w_init, tol, max_iter, device, **kw)
    if out is not None:
        calls.append((b.size, out[1], out[2], time.perf_counter() - t0))
    return out


solvers.cd_dev = cd_dev
sys.argv = ["run_solve.py", "--config", sys.argv[1] if len(sys.argv) > 1 else "3"]
exec(open(Path(__file__).resolve().parent / "run_solve.py").read())
ks = np.array([c[0] for c in calls])
sw = np.array([c[1] for c in calls])
ts = np.array([c[3] for c in calls])
print("calls", len(calls), "total s %.3f" % ts.sum(), "sweeps mean %.0f max %d" % (sw.mean(), sw.max()),
      "us/sweep/coord %.3f" % (1e6 * (ts / np.maximum(sw * ks, 1)).mean()),
      "reasons", {r: sum(1 for c in calls if c[2] == r) for r in ("kkt", "stall", "cap")})
for c in calls[::20]:
    print(c)
