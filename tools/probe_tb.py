"""Time tv_prox (fp32, 512^2, FGP-50) with the temporally blocked kernel and
with the one-launch-per-iteration streaming kernel (PSB_NO_TB=1)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_00688_b200 as psb  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
inner = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x = torch.randn((n, n), device="cuda", dtype=torch.float32)
for tb in ("0", "1"):
    os.environ["PSB_NO_TB"] = "1" if tb == "0" else "0"
    st = psb.TvProxState.cold((n, n), inner)
    for _ in range(3):
        psb.tv_prox(x, 0.3, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        psb.tv_prox(x, 0.3, st)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50
    print(f"n={n} inner={inner} tb={tb}: {t*1e3:.1f} us per prox, {t*1e3/inner:.2f} us per inner iteration", flush=True)
