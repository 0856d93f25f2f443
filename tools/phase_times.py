import ctypes as C, os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["PSB_NO_SMWORK"] = "1"
import paper_2411_00688_b200 as psb
from paper_2411_00688_b200 import _lib as L, batched, phantoms
idx = np.arange(1184) * 7 % 4096
b = torch.from_numpy(phantoms.config4_batch(idx, 256)).cuda()
for inner in (10, 50, 200):
    s = psb.BatchedTvDenoise(b, 0.1, inner, precision="fp32")
    coins = batched.coin_table(0.1, idx, 25)
    lib = L.LIB
    z = (C.c_double * 16)()
    dbg = lib.psb_debug_phases if os.environ.get('PSB_CLUSTER8') == '0' else lib.psb_debug_phases8
    dbg(z); base = np.array(z[:])
    s.run_proxskip(coins, 1.0, 0.1); torch.cuda.synchronize()
    dbg(z); v = (np.array(z[:]) - base)
    # cluster 0 did some number of calls; print ns per call-phase ratios
    print(inner, "prologue", v[0:3], "inner", v[4:7], "epilogue", v[8:11])
