"""Cluster-kernel timing probe: ns per cost unit (one FGP inner iteration of
one 256^2 problem) from the run's queue statistics, for a given inner budget.
  PSB_NO_SMWORK=1 python tools/time_cluster.py [inner ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import _lib as L, batched, phantoms  # noqa: E402

idx = np.arange(1184) * 7 % 4096
b = torch.from_numpy(phantoms.config4_batch(idx, 256)).cuda()
for inner in [int(a) for a in sys.argv[1:]] or [50]:
    s = psb.BatchedTvDenoise(b, 0.1, inner, precision="fp32")
    coins = batched.coin_table(0.1, idx, 25)
    s.run_proxskip(coins[:5], 1.0, 0.1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.run_proxskip(coins[5:], 1.0, 0.1)
    e1.record()
    torch.cuda.synchronize()
    qs = (L.C.c_double * 6)()
    L.call("psb_queue_stats", qs)
    calls = int(coins[5:].sum())
    print(f"inner {inner}: {e0.elapsed_time(e1):.2f} ms, {calls} prox calls, cluster "
          f"{qs[0] / max(qs[1], 1):.1f} ns/unit, cluster8 {qs[4] / max(qs[5], 1):.1f}, worker {qs[2] / max(qs[3], 1):.1f} ns/unit, "
          f"{1e6 * e0.elapsed_time(e1) / (calls * inner):.1f} ns per problem-iteration overall",
          flush=True)
