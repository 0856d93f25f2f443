import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2411_00688_b200 as psb
from paper_2411_00688_b200 import batched, phantoms
n = int(sys.argv[1]); K = 60
idx = np.arange(n)
b = np.stack([phantoms.config4_problem(int(i))[1] for i in idx]).astype(np.float32)
coins = batched.coin_table(0.1, idx, K)
s = psb.BatchedTvDenoise(b, 0.1, 50, precision="fp32")
s.run_proxskip(coins[:5], 1.0, 0.1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); s.run_proxskip(coins[5:], 1.0, 0.1); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1)
nprox = int(coins[5:].sum())
print(f"n={n} ratio={os.environ.get('PSB_SM_RATIO')} time {t:.2f} ms, prox calls {nprox}, per-iteration-per-machine {t*1e3/(nprox*50):.3f} us")
