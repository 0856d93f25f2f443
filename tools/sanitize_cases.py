"""Small cases for compute-sanitizer (memcheck / racecheck /
synccheck on the stencil and halo kernels).  Each case runs one hot kernel
family at a small size and checks its result against the plain streaming
path, so a run under the sanitizer is also a functional check:

  compute-sanitizer --tool memcheck  python tools/sanitize_cases.py --case cluster
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py --case tb
  ...

Cases: cluster (fgp_cluster_run_kernel, 16-CTA clusters, DSMEM st.async +
mbarriers), smworker (fgp_sm_run_kernel through the device work queue),
queue (both kernels sharing the queue, PDL placement), streamed (host input
chunks + stream memory operations), tb (temporally blocked fgp2d_tb_kernel,
512^2), stream2d (fgp2d_iter_kernel), fgp3d (fgp3d_march_kernel, TMA tiles),
slabs (3-slab peer-memory halo exchange, one stream per slab), ct (Radon
projector pair + PDHG kernels), blur (fused blur gradient + ProxSkip pre).
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    case = ap.parse_args().case
    import torch
    import paper_2411_00688_b200 as psb
    from paper_2411_00688_b200 import phantoms, volume3d as v3

    if case in ("cluster", "smworker", "queue", "streamed"):
        if case == "cluster":
            os.environ["PSB_NO_SMWORK"] = "1"
        if case == "smworker":
            os.environ["PSB_SM_ONLY"] = "1"
        n = 12 if case == "cluster" else 40
        idx = np.arange(n) * 97 % 4096
        b = phantoms.config4_batch(idx, 256)
        K, inner, p = 6, 4, 0.4
        if case == "streamed":
            x, c = psb.run_proxskip_batched(torch.from_numpy(b).pin_memory(), 0.1, p, idx, K,
                                            inner, chunk=8)
            x = x.numpy()
        else:
            x, c = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
            x = x.cpu().numpy()
        os.environ.pop("PSB_NO_SMWORK", None)
        os.environ.pop("PSB_SM_ONLY", None)
        os.environ["PSB_NO_CLUSTER"] = "1"
        xs, cs = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
        assert np.array_equal(c, cs)
        err = max(rel(x[j], xs[j].cpu().numpy()) for j in range(n))
        assert err < 2e-6, err
    elif case == "tb":
        _, b, _ = phantoms.config2_data(0, 512)
        st = psb.TvProxState.cold(b.shape, 23)
        u = psb.tv_prox(torch.from_numpy(b).float().cuda(), 0.1, st)  # temporally blocked
        os.environ["PSB_NO_TB"] = "1"
        st2 = psb.TvProxState.cold(b.shape, 23)
        u2 = psb.tv_prox(torch.from_numpy(b).float().cuda(), 0.1, st2)
        err = rel(u.cpu(), u2.cpu())
        assert err < 1e-5, err
    elif case == "stream2d":
        x = np.random.default_rng(1).random((3, 77, 130)).astype(np.float32)
        for j in range(3):
            st = psb.TvProxState.cold(x[j].shape, 9)
            psb.tv_prox(torch.from_numpy(x[j]).cuda(), 0.2, st)
    elif case in ("fgp3d", "slabs"):
        vol = phantoms.random_ellipsoids((40, 48, 64), 8, np.random.default_rng(3))
        b = phantoms.add_noise(vol, 0.1, 3).astype(np.float32)
        x1, _ = v3.proxskip_denoise3d(b, 0.08, 0.3, 0, 12, 5)
        if case == "slabs":
            x3, _ = v3.proxskip_denoise3d(b, 0.08, 0.3, 0, 12, 5, n_slabs=3, exchange="peer")
            assert np.array_equal(np.asarray(x1), np.asarray(x3))
    elif case == "ct":
        n = 48
        R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=12, n_bins=67))
        s = R.forward(phantoms.shepp_like(n, 5, np.random.default_rng(2)))
        for prec in ("fp32", "mixed"):
            prob = psb.build_tv_recon(R, s, 0.05, nonneg=True, splitting="explicit",
                                      precision=prec)
            sp = prob.saddle_problem
            st = 1.0 / np.sqrt(sp.norm_K_sq)
            psb.run_pdhgskip2(sp, np.zeros((n, n)), np.zeros(12 * 67 + 2 * n * n), None, st, st,
                              psb.SkipConfig(0.3, 0), 15)
    elif case == "blur":
        _, b, _ = phantoms.config2_data(0, 96)
        A = psb.blur_map(psb.gaussian_kernel(9, 2.0), b.shape)
        prob = psb.build_tv_recon(A, b, 0.02, inner_budget=7)
        L = prob.prox_problem.smooth.lipschitz
        psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0 / L,
                         psb.SkipConfig(0.3, 0), 12)
    else:
        raise SystemExit(f"unknown case {case}")
    torch.cuda.synchronize()
    print(f"case {case}: ok")


if __name__ == "__main__":
    main()
