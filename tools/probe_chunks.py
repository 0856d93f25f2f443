"""e2e of run_proxskip_batched (pinned float32 host in, host out) for several chunk sizes."""
import os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2411_00688_b200 as psb  # noqa: E402
idx = np.arange(4096)
b_pin = torch.from_numpy(bench.make_inputs(idx)).pin_memory()
psb.run_proxskip_batched(b_pin[:512], 0.1, 0.1, idx[:512], 20, 50)  # warm-up
for chunk in [int(c) for c in sys.argv[1:]]:
    ts = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, cnt = psb.run_proxskip_batched(b_pin, 0.1, 0.1, idx, 300, 50, chunk=chunk)
        ts.append(time.perf_counter() - t0)
    print(f"chunk {chunk}: " + " ".join(f"{300/t:.1f}" for t in ts) + " it/s", flush=True)
