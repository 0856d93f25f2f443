"""Time the projector pair (forward / adjoint) and one PDHG step at config 3."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402


def timed(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


n = 512
R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
for dt in (torch.float32, torch.float64):
    u = torch.rand(n, n, dtype=dt, device="cuda")
    y = torch.rand(60, 725, dtype=dt, device="cuda")
    tf = timed(lambda: R.forward(u))
    ta = timed(lambda: R.adjoint(y))
    print(f"{dt}: forward {tf:.1f} us  adjoint {ta:.1f} us  "
          f"({62996804 / tf / 1e3:.1f} / {62996804 / ta / 1e3:.1f} Gtap/s)")
