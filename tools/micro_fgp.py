"""Micro-timings of the single-problem FGP paths (persistent vs per-launch) and config 1."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402


def t_prox(n, inner, persist, reps=20):
    os.environ["PSB_NO_PERSIST"] = "0" if persist else "1"
    x = torch.randn((n, n), device="cuda")
    st = psb.TvProxState.cold((n, n), inner)
    psb.tv_prox(x, 0.5, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        psb.tv_prox(x, 0.5, st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / inner  # us per inner iteration


for n in (256, 512, 1024):
    for persist in (False, True):
        print(f"tv_prox {n}^2 persist={persist}: {t_prox(n, 50, persist):.2f} us / inner iteration")
_, b = phantoms.config1_data(0)
for rep in range(3):
    prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=100, precision="mixed")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0, psb.SkipConfig(0.1, 0), 500)
    torch.cuda.synchronize()
    print(f"config 1 run: {(time.perf_counter() - t0) * 1e3:.2f} ms")
