"""BASELINE config 3 (512^2 CT, 60 x 725, PDHGSkip-2, fp32 state): time a
warm 2000-iteration run, then run a short one whose kernels ncu can capture
(``--launch-skip`` past the setup):  python tools/profile_ct.py [prec] [iters]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
n = 512
R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
s = R.forward(phantoms.config3_phantom(0, n))
b = phantoms.config3_noisy(s, 0)
prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit", precision=prec)
sp = prob.saddle_problem
st = 1.0 / np.sqrt(sp.norm_K_sq)
y0 = np.zeros(60 * 725 + 2 * n * n)
psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st, psb.SkipConfig(0.1, 0), 64)  # warm
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st, psb.SkipConfig(0.1, 0), iters)
e1.record()
torch.cuda.synchronize()
print(f"{prec}: {iters / (e0.elapsed_time(e1) / 1e3):.1f} it/s over {iters} iterations", flush=True)
