"""Throughput of all five BASELINE configs on one GPU (secondary report).

bench.py prints the single contract line (config 4).  This script times the
other configs through the same public API so DESIGN.md can quote them:
outer iterations/s of the native run drivers (metrics off, setup excluded,
as harness.py:413-420 times), FGP inner iterations/s, and the FGP kernels'
algorithmic HBM rate (28 B/px-iter 2-D, 40 B/voxel-iter 3-D) against the
measured peak.  Usage: python tools/bench_configs.py [--configs 1,2,3,5]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms, volume3d as v3  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps=3):
    fn()  # warm-up (graph instantiation, allocator)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts), ts


def cfg1():
    _, b = phantoms.config1_data(0)
    K, inner = 500, 100
    coins = psb.SkipConfig(0.1, 0).coins(K)

    def run():
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=inner,
                                  precision="mixed")
        run.x, _ = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                    psb.SkipConfig(0.1, 0), K)
    t, ts = timed(run)
    n_inner = int(coins.sum()) * inner
    return {"config": 1, "outer_it_s": K / t, "inner_it_s": n_inner / t,
            "mpx_iter_s": n_inner * 65536 / t / 1e6, "seconds": t, "prox_calls": int(coins.sum()),
            "note": "includes problem build + graph capture/instantiate inside the timed call"}


def cfg2():
    truth = phantoms.random_shapes((512, 512), 10, np.random.default_rng(0), rects=False)
    k = psb.gaussian_kernel(9, 2.0)
    b = phantoms.add_noise(psb.blur_forward(truth, k), 0.01, 0)
    A = psb.blur_map(k, b.shape)
    prob = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
    L = prob.prox_problem.smooth.lipschitz
    K = 1000
    coins = psb.SkipConfig(0.2, 0).coins(K)

    def run():
        pr = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
        pr.A.norm_sq_estimate = L
        run.x, _ = psb.run_proxskip(pr.prox_problem, np.zeros_like(b), None, 1.0 / L,
                                    psb.SkipConfig(0.2, 0), K)
    t, _ = timed(run, reps=2)
    n_inner = int(coins.sum()) * 50
    # FISTA comparator (prox every iteration, native driver algo 1); one
    # untimed call first (lazy kernel loading)
    pr = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
    psb.run_fista(pr.prox_problem, np.zeros_like(b), 1.0 / L, 5)
    pr = psb.build_tv_recon(A, b, 0.02, inner_budget=50, precision="mixed")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    psb.run_fista(pr.prox_problem, np.zeros_like(b), 1.0 / L, 100)
    torch.cuda.synchronize()
    tf = (time.perf_counter() - t0) / 100
    return {"config": 2, "L": L, "outer_it_s": K / t, "inner_it_s": n_inner / t,
            "mpx_iter_s": n_inner * 512 * 512 / t / 1e6, "seconds": t,
            "prox_calls": int(coins.sum()), "fista_it_s": 1.0 / tf}


def cfg3():
    n = 512
    u = phantoms.shepp_like(n, 10, np.random.default_rng(0))
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
    s = R.forward(u)
    b = phantoms.add_noise(s, 0.01 * s.max(), 0)
    out = {"config": 3}
    for prec in ("mixed", "fp32"):
        prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit", precision=prec)
        sp = prob.saddle_problem
        st = 1.0 / np.sqrt(sp.norm_K_sq)
        y0 = np.zeros(60 * 725 + 2 * n * n)
        K = 2000

        def run():
            run.x, _ = psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st,
                                         psb.SkipConfig(0.1, 0), K)
        t, _ = timed(run, reps=2)

        def run_p():
            run_p.x, _ = psb.run_pdhg(sp, np.zeros((n, n)), y0, st, st, K)
        tp, _ = timed(run_p, reps=1)
        out[prec] = {"Knsq": sp.norm_K_sq, "pdhgskip2_it_s": K / t, "pdhg_it_s": K / tp,
                     "taps_per_s_fwd_adj": 2 * 62996804 * K / t}
    return out


def cfg3i(inner=50, K=2000, p=0.1):
    """PDHGSkip-2 on the implicit CT saddle problem (K = A,
    TV in the warm-started FGP prox with u >= 0) at config-3 geometry, through
    the native driver psb_ct_implicit_run; PDHG (p = 1) alongside."""
    n = 512
    u = phantoms.shepp_like(n, 10, np.random.default_rng(0))
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
    s = R.forward(u)
    b = phantoms.add_noise(s, 0.01 * s.max(), 0)
    out = {"config": "3i", "inner": inner, "p": p, "iters": K}
    coins = psb.SkipConfig(p, 0).coins(K)
    for prec in ("mixed", "fp32"):
        prob = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=inner,
                                            precision=prec)
        nsq = prob.saddle_problem.norm_K_sq

        def run():
            pr = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=inner,
                                              precision=prec)
            pr.saddle_problem.norm_K_sq = nsq
            st = 1.0 / np.sqrt(nsq)
            run.x, _ = psb.run_pdhgskip2(pr.saddle_problem, np.zeros((n, n)), np.zeros((60, 725)),
                                         None, st, st, psb.SkipConfig(p, 0), K)
        t, _ = timed(run, reps=2)

        def run_p():
            pr = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=inner,
                                              precision=prec)
            pr.saddle_problem.norm_K_sq = nsq
            st = 1.0 / np.sqrt(nsq)
            run_p.x, _ = psb.run_pdhg(pr.saddle_problem, np.zeros((n, n)), np.zeros((60, 725)),
                                      st, st, K // 10)
        tp, _ = timed(run_p, reps=1)
        out[prec] = {"Anorm_sq": nsq, "pdhgskip2_it_s": K / t, "pdhg_it_s": (K // 10) / tp,
                     "prox_calls": int(coins.sum())}
    return out


def cfg8f():
    """SURVEY 8(f) rows 2-4 through the native drivers: dual-ROF light-prox
    ProxSkip / PGD / FISTA (denoise-dual), reference-solution generators,
    PDHGSkip-1 on the explicit CT splitting, and the device IterationLog."""
    out = {"config": "8f"}
    n = 256
    u = phantoms.random_shapes((n, n), 10, np.random.default_rng(0))
    b = phantoms.add_noise(u, 0.05, 0)
    dual = psb.build_dual_rof(b, 0.5)
    g = 1.0 / dual.smooth.lipschitz
    K = 20000
    for name, run in (("proxskip_p0.3", lambda: psb.run_proxskip(dual.prox_problem(), dual.zero_dual(),
                                                                 None, g, psb.SkipConfig(0.3, 0), K)),
                      ("pgd", lambda: psb.run_pgd(dual.prox_problem(), dual.zero_dual(), g, K)),
                      ("fista", lambda: psb.run_fista(dual.prox_problem(), dual.zero_dual(), g, K))):
        t, _ = timed(run, reps=2)
        out[f"dual_rof_{name}_it_s"] = K / t
    t, _ = timed(lambda: psb.run_aprojgd(dual.smooth, dual.projector, dual.zero_dual(), g, 100000),
                 reps=1)
    out["aprojgd_dual_100k_seconds"] = t
    # CT explicit (config 3 geometry, fp64 state): preconditioned PDHG, PDHGSkip-1
    R = psb.radon_map(psb.RadonGeometry(image_side=512, n_angles=60, n_bins=725))
    s = R.forward(phantoms.shepp_like(512, 10, np.random.default_rng(0)))
    bb = phantoms.add_noise(s, 0.01 * s.max(), 0)
    for prec in ("mixed", "fp32"):
        prob = psb.build_tv_recon(R, bb, 0.05, nonneg=True, splitting="explicit", precision=prec)
        sp = prob.saddle_problem
        t, _ = timed(lambda: psb.run_pdhg_preconditioned(sp, 1000), reps=1)
        out[f"pdhg_precond_{prec}_it_s"] = 1000 / t
        st = 1.0 / np.sqrt(sp.norm_K_sq)
        y0 = np.zeros(60 * 725 + 2 * 512 * 512)
        t, _ = timed(lambda: psb.run_pdhgskip1(sp, np.zeros((512, 512)), y0, st, st, 9.0,
                                               psb.SkipConfig(0.1, 0), 2000), reps=1)
        out[f"pdhgskip1_{prec}_it_s"] = 2000 / t
    # device IterationLog: config 1 with rel_error + objective every iteration
    _, b1 = phantoms.config1_data(0)
    ref = b1
    for mode in ("passive", "device_log"):
        def run():
            prob = psb.build_tv_recon(psb.identity_map(b1.shape), b1, 0.1, inner_budget=100,
                                      precision="mixed")
            log = None if mode == "passive" else psb.IterationLog(
                reference=ref, objective_fn=psb.device_objective(prob))
            psb.run_proxskip(prob.prox_problem, np.zeros_like(b1), None, 1.0,
                             psb.SkipConfig(0.1, 0), 500, log)
        t, _ = timed(run, reps=2)
        out[f"config1_{mode}_it_s"] = 500 / t
    return out


def config5_volume(side=1024):
    """Config-5 input on the device (seeded): phantoms.config5_volume."""
    return phantoms.config5_volume(side, 0)


def cfg5(side=1024, K=200, inner=20):
    b = config5_volume(side)
    D = H = W = side
    coins = psb.SkipConfig(0.1, 0).coins(K)
    slab = v3.Slab3D(b, 0, D, 0.08, inner, precision="fp32")
    del b
    ev = []
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    v3.run_proxskip_slabs([slab], coins, gamma=1.0, p=0.1, fgp_events=ev)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    tf = sum(a.elapsed_time(bb) for a, bb in ev) / 1e3
    n_inner = int(coins.sum()) * inner
    nvox = D * H * W
    bytes_fgp = int(coins.sum()) * nvox * (28 + (inner - 1) * 40)
    return {"config": 5, "side": side, "outer_it_s": K / t, "inner_it_s": n_inner / t,
            "mvox_iter_s": n_inner * nvox / t / 1e6, "seconds": t, "prox_calls": int(coins.sum()),
            "fgp_seconds": tf, "fgp_gbs": bytes_fgp / tf / 1e9, "fgp_frac": bytes_fgp / tf / 1e9 / peak()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--side5", type=int, default=1024)
    args = ap.parse_args()
    fns = {"1": cfg1, "2": cfg2, "3": cfg3, "3i": cfg3i, "8f": cfg8f, "5": lambda: cfg5(args.side5)}
    for c in args.configs.split(","):
        r = fns[c]()
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
