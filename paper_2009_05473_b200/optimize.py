"""The in-library L-BFGS-B behind a Python objective (sfw3d_lbfgsb_minimize).

The single-GPU solver runs its two optimisations entirely inside the library
(sfw3d_refine_eta_max, sfw3d_local_descent). The x-slab solver's objectives
contain a collective (the all-reduce of the per-rank partial sums), which the
Python side owns, so they go through this callback form of the same
optimiser: every rank runs the same iterates on the same reduced values.

Replaces scipy.optimize.minimize(method="L-BFGS-B") at certificate.py:217-218
and solvers.py:231-232 (same options: maxcor 10, ftol, gtol, maxiter,
maxfun 15000, maxls 20)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

STATUS = ("CONVERGENCE: NORM OF PROJECTED GRADIENT <= PGTOL",
          "CONVERGENCE: RELATIVE REDUCTION OF F <= FACTR*EPSMCH",
          "STOP: TOTAL NO. OF ITERATIONS REACHED LIMIT",
          "STOP: TOTAL NO. OF F AND G EVALUATIONS EXCEEDS LIMIT",
          "ABNORMAL: LINE SEARCH GAVE UP")


@dataclass
class Result:
    x: np.ndarray
    fun: float
    status: int
    nit: int
    nfev: int

    @property
    def success(self) -> bool:
        return self.status in (0, 1)

    @property
    def message(self) -> str:
        return STATUS[self.status] if 0 <= self.status < len(STATUS) else f"status {self.status}"


def minimize(fun, x0, bounds, maxiter: int = 15000, gtol: float = 1e-5,
             ftol: float = 2.220446049250313e-09, maxcor: int = 10, maxfun: int = 15000,
             maxls: int = 20) -> Result:
    """L-BFGS-B of fun(x) -> (f, grad) over the box `bounds` [(lo|None, hi|None)]."""
    x = np.array(x0, dtype=np.float64).ravel().copy()
    n = x.size
    lo, hi, nbd = np.zeros(n), np.zeros(n), np.zeros(n, dtype=np.int32)
    for i, (a, b) in enumerate(bounds):
        if a is not None and b is not None:
            nbd[i], lo[i], hi[i] = 2, a, b
        elif a is not None:
            nbd[i], lo[i] = 1, a
        elif b is not None:
            nbd[i], hi[i] = 3, b
    raised = []

    def objective(_user, xp, fp, gp):
        try:
            f, g = fun(np.ctypeslib.as_array(xp, (n,)).copy())
            fp[0] = float(f)
            np.ctypeslib.as_array(gp, (n,))[:] = np.asarray(g, dtype=np.float64).ravel()
            return 0
        except BaseException as exc:  # carried across the C frame, re-raised below
            raised.append(exc)
            return N.SFW3D_EINVAL

    cb = N.OBJECTIVE_FN(objective)
    f = C.c_double()
    info = (C.c_int32 * 3)()
    rc = N.lib().sfw3d_lbfgsb_minimize(n, N.f64_ptr(x), N.f64_ptr(lo), N.f64_ptr(hi),
                                       nbd.ctypes.data_as(C.POINTER(C.c_int32)), int(maxcor),
                                       float(ftol), float(gtol), int(maxiter), int(maxfun),
                                       int(maxls), cb, None, C.byref(f), info)
    if raised:
        raise raised[0]
    N.check(rc)
    return Result(x=x, fun=float(f.value), status=int(info[0]), nit=int(info[1]), nfev=int(info[2]))
