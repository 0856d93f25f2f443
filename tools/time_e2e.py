"""e2e timing of run_proxskip_batched (pinned host in / out) for several
chunk sizes:  python tools/time_e2e.py K chunk [chunk ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402

K = int(sys.argv[1])
idx = np.arange(4096)
b = torch.from_numpy(phantoms.config4_batch(idx[:512], 256)).repeat(8, 1, 1).pin_memory()
out = torch.empty(b.shape, dtype=torch.float32).pin_memory()
psb.run_proxskip_batched(b[:512], 0.1, 0.1, idx[:512], 5, 50, out=out[:512])
for ch in [int(a) for a in sys.argv[2:]]:
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        psb.run_proxskip_batched(b, 0.1, 0.1, idx, K, 50, out=out, chunk=ch)
        ts.append(time.perf_counter() - t0)
    print(f"K={K} chunk={ch}: median {1e3 * np.median(ts):.2f} ms -> {K / np.median(ts):.1f} batch it/s "
          f"(samples {[round(1e3 * t, 2) for t in ts]})", flush=True)
