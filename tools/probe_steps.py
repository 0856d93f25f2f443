"""Device-resident config-4 throughput vs number of timed steps (diagnostic)."""
import os
import sys

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
for W, K, ft in ((3, 30, False), (3, 100, False), (3, 100, True), (3, 295, False), (50, 100, False)):
    s.reset()
    s.run_proxskip(coins[:W], 1.0, 0.1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f = np.zeros(K) if ft else None
    e0.record()
    s.run_proxskip(coins[W:W + K], 1.0, 0.1, fgp_time=f)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    per = [] if f is None else f
    print(f"W={W} K={K} fgp_time={ft}: {K / t:.1f} it/s  active={int(coins[W:W+K].sum())}", flush=True)
