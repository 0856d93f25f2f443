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
for variant in ("events", "plain", "graph", "events", "plain", "graph"):
    s.reset()
    s.run_proxskip(coins[:5], 1.0, 0.1)
    torch.cuda.synchronize()
    f = np.zeros(295) if variant == "events" else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    s.run_proxskip(coins[5:], 1.0, 0.1, fgp_time=f, use_graph=variant == "graph")
    h_launch = time.perf_counter() - h0
    e1.record()
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    tot = e0.elapsed_time(e1) / 1e3
    kern = f.sum() if f is not None else float("nan")
    print(f"{variant:6s}: region {tot:.3f}s  kernels {kern:.3f}s  host-return {h_launch:.3f}s  "
          f"-> {295 / tot:.1f} it/s", flush=True)
