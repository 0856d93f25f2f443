"""BASELINE config 5 on N GPUs: z-slab decomposed 3-D ProxSkip TV denoising,
one slab per rank, launched with torchrun (one process per GPU):

  python -m torch.distributed.run --nnodes=1 --nproc-per-node N \\
      --master-addr 127.0.0.1 --master-port P tools/run_config5_dist.py \\
      [--side 1024] [--iters 200] [--inner 20] [--exchange peer|nccl] [--check]

--exchange peer: the edge kernels store their new dual planes into the
neighbours' receive rings over NVLink (CUDA IPC), ordered by device flags
(volume3d.PeerExchange.dist); the process group (gloo) only swaps handles
and agrees on divergence.  --exchange nccl: send buffers + NCCL P2P on a side
stream (volume3d.DistExchange).  --check: rank 0 also runs the whole volume
on its device and the gathered slabs must equal it bit for bit (small sides).
--share-device runs every rank on cuda:0 (protocol check on a 1-GPU box;
peer exchange only).  Prints one JSON line (rank 0): device time = max over
ranks (CUDA events)."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms, volume3d as v3  # noqa: E402


def volume(side, seed=0):
    """Seeded noisy ellipsoid volume, identical on every rank (host numpy for
    small sides, the device generator of tools/bench_configs.cfg5 otherwise)."""
    if side <= 128:
        vol = phantoms.random_ellipsoids((side, side, side), 50, np.random.default_rng(seed))
        return torch.from_numpy(phantoms.add_noise(vol, 0.1, seed).astype(np.float32)).cuda()
    return phantoms.config5_volume(side, seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--side", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--inner", type=int, default=20)
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--exchange", choices=["peer", "nccl"], default="peer")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--share-device", action="store_true")
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", 0))
    dev = 0 if a.share_device else local
    torch.cuda.set_device(dev)
    backend = "nccl" if a.exchange == "nccl" else "gloo"
    dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    if a.share_device and a.exchange == "nccl":
        raise SystemExit("--share-device needs --exchange peer (NCCL rejects duplicate GPUs)")
    b = volume(a.side)
    z0, z1 = v3.slab_bounds(a.side, rank, world)
    slab = v3.Slab3D(b[z0:z1].clone(), z0, a.side, 0.08, a.inner, precision="fp32")
    bfull = b if (a.check and rank == 0) else None
    del b
    ex = v3.PeerExchange.dist(slab, None) if a.exchange == "peer" else v3.DistExchange()
    coins = psb.SkipConfig(a.p, 0).coins(a.iters)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    v3.run_proxskip_slabs([slab], coins, gamma=1.0, p=a.p, exchange=ex)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64)
    if backend == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t = float(t.item())
    ok = None
    if a.check:
        parts = [None] * world
        dist.all_gather_object(parts, (z0, slab.x.cpu().numpy()))
        if rank == 0:
            x1, _ = v3.proxskip_denoise3d(bfull, 0.08, a.p, 0, a.iters, a.inner, n_slabs=1,
                                          precision="fp32")
            xd = np.concatenate([x for _, x in sorted(parts, key=lambda r: r[0])])
            ok = bool(np.array_equal(xd, x1.cpu().numpy() if torch.is_tensor(x1) else x1))
    if hasattr(ex, "close"):
        ex.close()
    if rank == 0:
        n_prox = int(coins.sum())
        print(json.dumps({"config": 5, "n_ranks": world, "side": a.side, "exchange": a.exchange,
                          "share_device": a.share_device, "outer_it_s": a.iters / t,
                          "seconds": t, "prox_calls": n_prox, "inner": a.inner,
                          "bitwise_equal_whole_volume": ok}), flush=True)
    dist.destroy_process_group()
    if ok is False:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
