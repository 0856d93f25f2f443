"""Per-step device time distribution of the config-4 cluster path (diagnostic)."""
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
for rep in range(int(os.environ.get("REPS", "3"))):
    s.reset()
    s.run_proxskip(coins[:3], 1.0, 0.1)
    f = np.zeros(295)
    s.run_proxskip(coins[3:298], 1.0, 0.1, fgp_time=f)
    torch.cuda.synchronize()
    act = coins[3:298].sum(axis=1)
    per = f / np.maximum(act, 1) * 1e6  # us per problem-prox
    q = np.percentile(per, [5, 50, 95, 100])
    slow = np.nonzero(per > 1.3 * np.median(per))[0]
    print(f"rep {rep}: total {f.sum():.3f}s  us/problem p5 {q[0]:.1f} p50 {q[1]:.1f} p95 {q[2]:.1f} "
          f"max {q[3]:.1f}  slow steps {len(slow)}: {slow[:20].tolist()}", flush=True)
