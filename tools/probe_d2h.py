import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_00688_b200 import _arrays as AR  # noqa: E402
x = torch.rand(4096, 256, 256, device="cuda")
ref_cpu = torch.empty(1)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); a = AR.like(x, ref_cpu); t1 = time.perf_counter()
    h = AR.to_host(x[:512]); t2 = time.perf_counter()
    d = AR.to_dev(a, torch.float32); torch.cuda.synchronize(); t3 = time.perf_counter()
    e = AR.to_dev(h, torch.float32); torch.cuda.synchronize(); t4 = time.perf_counter()
    assert torch.equal(d, x) and torch.equal(e, x[:512]) and np.array_equal(h, x[:512].double().cpu().numpy())
    print(f"like(cpu f32 1GB) {t1-t0:.3f}s  to_host(f64 256MB) {t2-t1:.3f}s  "
          f"to_dev(tensor 1GB) {t3-t2:.3f}s  to_dev(numpy f64 256MB) {t4-t3:.3f}s")
