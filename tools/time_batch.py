"""Resident config-4 run timing, repeated: python tools/time_batch.py [n_problems] [K] [reps]
(PSB_DEBUG_TIMES=1 prints the per-launch queue statistics)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import batched, phantoms  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
idx = np.arange(n)
b = torch.from_numpy(phantoms.config4_batch(idx, 256)).cuda()
coins = batched.coin_table(0.1, idx, 5 + K)
ts = []
for r in range(reps):
    s = psb.BatchedTvDenoise(b, 0.1, 50, precision="fp32")
    s.run_proxskip(coins[:5], 1.0, 0.1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.run_proxskip(coins[5:], 1.0, 0.1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} K={K}: ms {[round(t, 2) for t in ts]} -> {K / (min(ts) * 1e-3):.1f} batch it/s (best), "
      f"{K / (float(np.median(ts)) * 1e-3):.1f} (median)")
