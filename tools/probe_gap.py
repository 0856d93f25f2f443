"""Where does the device-resident bench region spend its time? (diagnostic)"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import batched  # noqa: E402

idx = np.arange(4096)
b_host = bench.make_inputs(idx)
coins = batched.coin_table(0.1, idx, 300)
s = psb.BatchedTvDenoise(b_host, 0.1, 50, precision="fp32")
for rep in range(3):
    s.reset()
    s.run_proxskip(coins[:5], 1.0, 0.1)
    torch.cuda.synchronize()
    f = np.zeros(295)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    s.run_proxskip(coins[5:], 1.0, 0.1, fgp_time=f)
    e1.record()
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    tot = e0.elapsed_time(e1) / 1e3
    print(f"rep {rep}: region {tot:.3f}s  kernels {f.sum():.3f}s  gaps {tot - f.sum():.3f}s  "
          f"host {h1 - h0:.3f}s  -> {295 / tot:.1f} it/s", flush=True)
