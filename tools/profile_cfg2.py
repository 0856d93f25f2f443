"""Config 2 (512^2 deblur ProxSkip, 1000 x FGP-50, p = 0.2): where the time of
one run call goes (host wall vs device events), for tuning."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
UG = {"auto": None, "1": True, "0": False}[sys.argv[2] if len(sys.argv) > 2 else "auto"]
truth = phantoms.random_shapes((512, 512), 10, np.random.default_rng(0), rects=False)
k = psb.gaussian_kernel(9, 2.0)
b = phantoms.add_noise(psb.blur_forward(truth, k), 0.01, 0)
A = psb.blur_map(k, b.shape)
prob = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
L = prob.prox_problem.smooth.lipschitz
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
    pr.A.norm_sq_estimate = L
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, log = psb.run_proxskip(pr.prox_problem, np.zeros_like(b), None, 1.0 / L,
                              psb.SkipConfig(0.2, 0), K, use_graph=UG)
    e1.record()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"graph={UG} rep {rep}: build {1e3*(t1-t0):.2f} ms, run call {1e3*(t2-t1):.2f} ms (wall to sync "
          f"{1e3*(t3-t1):.2f}), device events {e0.elapsed_time(e1):.2f} ms, "
          f"elapsed_s[-1] {log.records[-1].elapsed_s*1e3 if log and log.records else -1:.2f} ms",
          flush=True)
