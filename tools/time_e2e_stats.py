"""e2e timing of run_proxskip_batched with the queue statistics of every call:
python tools/time_e2e_stats.py [K] [calls]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import _lib as L, phantoms  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 25
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
idx = np.arange(4096)
b = torch.from_numpy(phantoms.config4_batch(idx[:512], 256)).repeat(8, 1, 1).pin_memory()
out = torch.empty(b.shape, dtype=torch.float32).pin_memory()
psb.run_proxskip_batched(b[:512], 0.1, 0.1, idx[:512], 5, 50, out=out[:512])
for c in range(calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    psb.run_proxskip_batched(b, 0.1, 0.1, idx, K, 50, out=out)
    dt = time.perf_counter() - t0
    qs = (L.C.c_double * 6)()
    L.call("psb_queue_stats", qs)
    print(f"call {c}: {1e3 * dt:.2f} ms; cluster {qs[0] / max(qs[1], 1):.1f} ns/unit over {qs[1]:.0f} units, "
          f"cluster8 {qs[4] / max(qs[5], 1):.1f} over {qs[5]:.0f}, "
          f"worker {qs[2] / max(qs[3], 1):.1f} ns/unit over {qs[3]:.0f} units", flush=True)
