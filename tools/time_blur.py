"""Time the fused blur gradient g = A^T(A u - b) at config 2 (512^2, 9x9)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import operators as O  # noqa: E402

k = psb.gaussian_kernel(9, 2.0)
for dt in (torch.float64, torch.float32):
    u = torch.rand(512, 512, dtype=dt, device="cuda")
    b = torch.rand(512, 512, dtype=dt, device="cuda")
    gb = torch.empty_like(u)
    fn = lambda: O.blur_grad_dev(u, b, k, out=gb)
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            for _ in range(100):
                fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"TS={os.environ.get('PSB_BLUR_TS', 32)} {dt}: {e0.elapsed_time(e1) * 10:.2f} us per call")

# calibration: an elementwise kernel over the same 512^2 fp64 arrays, and a
# plain torch copy, in the same graph setup
from paper_2411_00688_b200 import _lib as L  # noqa: E402
for name, fn in [("lincomb", lambda: L.call("psb_lincomb", L.F64, 1.0, L.ptr(u64), 2.0, L.ptr(b64),
                                             L.ptr(o64), u64.numel(), L.stream())),
                 ("torch copy", lambda: o64.copy_(u64))]:
    u64 = torch.rand(512, 512, dtype=torch.float64, device="cuda")
    b64 = torch.rand_like(u64)
    o64 = torch.empty_like(u64)
    fn()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g):
            for _ in range(100):
                fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 10:.2f} us per call")
