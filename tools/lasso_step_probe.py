"""Per-call cost of the weight step's volume kernels at config 3 with k phis:
dots of one phi against k (full volume vs x support), residual (full vs ranged)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N, configs, solvers  # noqa: E402
from paper_2009_05473_b200.forward import code_of  # noqa: E402

inst = configs.config3(0)
P.set_precision(inst.precision)
psf = P.Psf(P.Volume(inst.kernel), normalize=False)
code = N.dtype_code()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
thetas = [P.AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]) for r in inst.truth[:k]]
phis = [solvers.phi_dev(t, psf, code) for t in thetas]
y = torch.randn(inst.dims, device="cuda", dtype=phis[0].dtype)
w = np.abs(np.random.default_rng(0).standard_normal(k))
nx = inst.dims[0]
xr = np.zeros((k, 2), dtype=np.int32)
for i, p in enumerate(phis):
    on = torch.any(p.reshape(nx, -1) != 0, dim=1).cpu().numpy()
    idx = np.flatnonzero(on)
    if on.all():
        xr[i] = (0, nx - 1)
    elif on[0] and on[-1]:
        gap = np.flatnonzero(~on)
        xr[i] = (gap[-1] + 1, gap[0] - 1)
    else:
        xr[i] = (idx[0], idx[-1])
print("mean support planes", np.mean((xr[:, 1] - xr[:, 0]) % nx + 1))
ctx = N.context(0)


def timeit(f, n=10):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n


print("dots full      %.3f ms" % timeit(lambda: solvers.dots_dev(phis, phis[-1])))
print("residual full  %.3f ms" % timeit(lambda: solvers.residual_dev(y, w, phis)))
out = torch.empty_like(y)
ss = C.c_double()
arr = (C.c_void_p * k)(*[t.data_ptr() for t in phis])
print("residual ranged %.3f ms" % timeit(lambda: N.check(N.lib().sfw3d_residual_ranged(
    ctx.handle, code_of(y), N.dims_arg(y.shape), N.ptr(y), arr, N.f64_ptr(w),
    xr.ctypes.data_as(C.POINTER(C.c_int32)), k, N.ptr(out), C.byref(ss)))))
print("phi (render + 3 passes) %.3f ms" % timeit(lambda: solvers.phi_dev(thetas[0], psf, code)))
g = np.eye(k) + 0.01
print("lasso qp %.3f ms" % timeit(lambda: solvers.cd_dev(g, np.ones(k), 0.1, np.zeros(k), 1e-6, 2000, 0, "qp")))
