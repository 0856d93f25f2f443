"""Config-5 strong scaling projected from one GPU.

At N ranks, rank r owns planes slab_bounds(1024, r, N) of the 1024^3 volume
and runs the overlapped schedule of run_proxskip_slabs: per FGP inner
iteration an interior launch (no halo) and an edge launch (the two boundary
planes, after the neighbours' new dual planes arrived).  The transfer itself
is 3 planes x 4 MB per neighbour per inner iteration, issued while the
interior launch (~1 ms at N = 8) runs.  Here every distinct rank shape (one or
two neighbours) is timed alone on one B200 with the exchange replaced by a
no-op (halo rings left as they are), i.e. the per-rank device time with the
transfer fully hidden; prints T_1 / (N * T_N) for the slowest rank.  Only one
GPU is available in this run, so the NVLink transfer is not measured."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import volume3d as v3  # noqa: E402


class NullExchange:
    def setup(self, slabs):
        pass

    def begin_prox(self, slabs):
        pass

    def wait_ring(self, slabs, m):
        pass

    def send(self, slabs, m):
        pass

    def finish(self, slabs):
        pass

    def agree_bad(self, k):
        return k


def main(side=1024, K=200, inner=20):
    coins = psb.SkipConfig(0.1, 0).coins(K)
    g = torch.Generator(device="cuda").manual_seed(0)
    out = {}
    for n in (1, 2, 4, 8):
        ranks = sorted({0, min(1, n - 1)})
        worst, per = 0.0, {}
        for r in ranks:
            z0, z1 = v3.slab_bounds(side, r, n)
            b = torch.rand((z1 - z0, side, side), generator=g, device="cuda")
            slab = v3.Slab3D(b, z0, side, 0.08, inner, precision="fp32")
            del b
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            v3.run_proxskip_slabs([slab], coins, gamma=1.0, p=0.1, exchange=NullExchange())
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            per[r] = round(t, 5)
            worst = max(worst, t)
            del slab
            torch.cuda.empty_cache()
        out[n] = worst
        print(json.dumps({"config": 5, "n": n, "slowest_rank_s": worst, "outer_it_s": K / worst,
                          "projected_efficiency": out[1] / (n * worst), "per_rank_s": per,
                          "prox_calls": int(coins.sum()), "inner": inner}), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
