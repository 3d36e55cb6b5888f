"""First-call vs steady-state wall time of the config-1 BSFW solve (table and
basis memoisation, allocator warm-up): python tools/first_solve_probe.py"""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np, torch
import paper_2009_05473_b200 as P
import sfw3d_oracle as O
from paper_2009_05473_b200 import solvers
g = np.load(ROOT / 'tests' / 'golden' / 'config1.npz')
P.set_precision("f64")
dims = (64, 64, 64)
psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (2, 2, 2), (7, 7, 7))), normalize=False)
bounds = P.DomainBounds(pos_lower=(8.0,) * 3, pos_upper=(56.0,) * 3, sigma_min=1.5, sigma_max=3.0, shape_min=1.5, shape_max=2.5)
sg, dg = np.array([1.5, 2.0, 2.5, 3.0]), np.array([1.5, 2.0, 2.5])
solvers.make_parameter_grids = lambda b, ns, nd: (sg, dg)
import paper_2009_05473_b200.solvers as S
orig = S._solve_native
def timed(*a, **k):
    t0 = time.perf_counter(); r = orig(*a, **k); print("   _solve_native %.3f" % (time.perf_counter() - t0)); return r
S._solve_native = timed
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = P.bsfw(P.Volume(g["y"]), psf, P.SolverOptions(lam=float(g["lam"]), max_outer_iterations=20), bounds)
    print("solve %d: %.3f s, trace total %.3f, table %.3f, steps %.3f" % (i, time.perf_counter() - t0, res.trace.t_total, res.trace.t_table, sum(res.trace.step_time(s) for s in ("certificate", "lasso", "descent"))))
