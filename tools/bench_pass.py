"""Time the 1-D pass kernels at 512^3 fp32 for narrow and wide separable
kernels: adjoint PSF application (z, y, x passes), per-family device time."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_05473_b200 as P  # noqa: E402
from paper_2009_05473_b200 import _native as N  # noqa: E402
from paper_2009_05473_b200.configs import box_psf_kernel  # noqa: E402
from paper_2009_05473_b200.forward import psf_apply_dev  # noqa: E402

n = int(os.environ.get("N", "512"))
dims = (n, n, n)
x = torch.randn(dims, device="cuda", dtype=torch.float32)
ctx = N.context()
for half in (4, 7, 11, 15, 44):
    psf = P.Psf(P.Volume(box_psf_kernel(dims, (3.0,) * 3, (half,) * 3)), normalize=False)
    out = torch.empty_like(x)
    for _ in range(2):
        psf_apply_dev(psf, x, True, out)
    torch.cuda.synchronize()
    ctx.profile(True)
    for _ in range(5):
        psf_apply_dev(psf, x, True, out)
    ms, cnt = ctx.profile_read("psf_pass")
    ctx.profile(False)
    per = ms / cnt
    gbs = 2 * x.numel() * 4 / (per / 1e3) / 1e9
    print(f"taps={2 * half + 1}: "
          f"{per:.3f} ms/pass (avg of z,y,x) -> {gbs:.0f} GB/s (read+write)")
