"""Micro-benchmark of the 256x256 FGP paths (cluster-resident vs streaming).

Runs N problems with every coin firing (p = 1) so each outer iteration is one
prox call per problem, for inner budgets 1 and 50; the slope gives the cost
of one inner iteration.  Used for ncu captures (-k regex:fgp_cluster).

  python tools/profile_fgp.py [--n 64] [--iters 3] [--mode cluster|stream]
"""

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402


def run(n, iters, inner, mode, reps=3):
    return min(_run(n, iters, inner, mode) for _ in range(reps))


def _run(n, iters, inner, mode):
    os.environ["PSB_NO_CLUSTER"] = "1" if mode == "stream" else "0"
    b = np.stack([phantoms.config4_problem(i, 256)[1] for i in range(min(n, 8))]).astype(np.float32)
    b = np.concatenate([b] * ((n + 7) // 8))[:n]
    s = psb.BatchedTvDenoise(b, 0.1, inner)
    coins = np.ones((iters, n), dtype=np.uint8)
    s.run_proxskip(coins[:1], 1.0, 1.0)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.run_proxskip(coins, 1.0, 1.0)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--mode", default="cluster")
    ap.add_argument("--inner", type=int, default=0)
    a = ap.parse_args()
    if a.inner:
        t = run(a.n, a.iters, a.inner, a.mode)
        print(f"{a.mode} n={a.n} inner={a.inner}: {t * 1e3:.3f} ms")
        return
    for mode in ("cluster", "stream"):
        t1 = run(a.n, a.iters, 1, mode)
        t50 = run(a.n, a.iters, 50, mode)
        per_inner = (t50 - t1) / (49 * a.iters)
        px_it = a.n * 65536 / per_inner
        print(f"{mode}: n={a.n} t(inner=1)={t1 * 1e3:.3f} ms t(inner=50)={t50 * 1e3:.3f} ms "
              f"per inner iteration (all {a.n} problems) {per_inner * 1e6:.2f} us "
              f"-> {px_it / 1e9:.1f} Gpx-it/s")


if __name__ == "__main__":
    main()
