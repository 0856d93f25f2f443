import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2411_00688_b200 as psb
from paper_2411_00688_b200 import phantoms
truth = phantoms.random_shapes((512, 512), 10, np.random.default_rng(0), rects=False)
k = psb.gaussian_kernel(9, 2.0)
b = phantoms.add_noise(psb.blur_forward(truth, k), 0.01, 0)
A = psb.blur_map(k, b.shape)
for rep in range(3):
    pr = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
    L = 0.9939912746344076
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, log = psb.run_fista(pr.prox_problem, np.zeros_like(b), 1.0 / L, 100)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"fista 100 it: {1e3*(t1-t0):.1f} ms", flush=True)
