"""Phase timing of the config-4 public entry point run_proxskip_batched."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import _arrays as AR  # noqa: E402
from paper_2411_00688_b200 import batched  # noqa: E402

idx = np.arange(4096)
b_host = bench.make_inputs(idx)
b_pin = torch.from_numpy(b_host).pin_memory()
for rep in range(int(os.environ.get("REPS", "4"))):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    coins = batched.coin_table(0.1, idx, 300)
    t.append(time.perf_counter())
    s = psb.BatchedTvDenoise(b_pin, 0.1, 50, precision="fp32")
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    s.run_proxskip(coins, 1.0, 0.1)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    s.check_finite()
    x = AR.like(s.x, b_pin)
    t.append(time.perf_counter())
    d = np.diff(t)
    print(f"rep {rep}: coins {d[0]:.3f}s  build+H2D {d[1]:.3f}s  run {d[2]:.3f}s  "
          f"check+D2H {d[3]:.3f}s  total {t[-1] - t[0]:.3f}s  -> {300 / (t[-1] - t[0]):.1f} it/s",
          flush=True)
    del s, x
    torch.cuda.empty_cache()
