"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``imgskip`` from /root/reference/pkg/src (read-only), evaluates the
hot-path functions on small seeded inputs and writes ``tests/golden/ref_*.npz``.
The fixtures are committed; nothing on the GPU box reads /root/reference.
Tests pin ``oracle/`` against these files (tests/test_oracle_golden.py) and the
CUDA path against the oracle.
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import imgskip as m
    from imgskip.operators import radon_system_matrix
    from imgskip.problems import objective_tv
    from imgskip.solvers import IterationLog

    out = {}

    # -- operators ----------------------------------------------------------
    rng = np.random.default_rng(100)
    u = rng.standard_normal((7, 9))
    q = rng.standard_normal((2, 7, 9))
    out["op_u"], out["op_q"] = u, q
    out["op_grad"] = m.grad_forward(u)
    out["op_div"] = m.divergence(q)
    out["op_ball"] = m.project_ball(3.0 * q, 0.7)
    out["op_tv"] = np.array(m.tv_value(u))
    qi = rng.integers(-50, 50, size=(2, 5, 8)).astype(np.float64)
    out["op_qint"], out["op_divint"] = qi, m.divergence(qi)

    taps = m.gaussian_kernel(9, 2.0).weights
    out["blur_taps"] = taps
    ub = rng.standard_normal((16, 20))
    out["blur_u"] = ub
    out["blur_fwd"] = m.blur_forward(ub, m.gaussian_kernel(9, 2.0))
    out["blur_adj"] = m.blur_adjoint(ub, m.gaussian_kernel(9, 2.0))
    k5 = m.gaussian_kernel(5, 1.2)
    out["blur5_fwd"] = m.blur_forward(ub, k5)
    out["blur_L_32"] = np.array(m.blur_map(m.gaussian_kernel(9, 2.0), (32, 32)).norm_sq())
    out["grad_L_16"] = np.array(m.power_method(m.grad_map((16, 16))))

    for tag, (n, na, nb) in {"r1": (16, 7, 23), "r2": (33, 12, 47), "r3": (64, 60, 91)}.items():
        geom = m.RadonGeometry(image_side=n, n_angles=na, n_bins=nb)
        mat = radon_system_matrix(geom)
        op = m.radon_map(geom)
        rr = np.random.default_rng(7 + n)
        xu = rr.standard_normal((n, n))
        ys = rr.standard_normal((na, nb))
        out[f"{tag}_shape"] = np.array([n, na, nb])
        out[f"{tag}_x"], out[f"{tag}_y"] = xu, ys
        out[f"{tag}_fwd"] = op.forward(xu)
        out[f"{tag}_adj"] = op.adjoint(ys)
        out[f"{tag}_nnz"] = np.array(mat.nnz)
        out[f"{tag}_rowsum"] = np.asarray(mat.sum(axis=1)).ravel()
        out[f"{tag}_colsum"] = np.asarray(mat.sum(axis=0)).ravel()

    # -- TV prox --------------------------------------------------------------
    rng = np.random.default_rng(5)
    x = rng.standard_normal((12, 9))
    out["tv_x"] = x
    st = m.TvProxState.cold((12, 9), 7)
    out["tv_u1"] = m.tv_prox(x, 0.3, st)
    out["tv_q1"] = st.q_warm.copy()
    out["tv_u2"] = m.tv_prox(x, 0.3, st)            # warm start, same weight
    out["tv_u3"] = m.tv_prox(x, 0.05, st)           # weight change -> reprojection
    out["tv_q3"] = st.q_warm.copy()
    out["tv_count"] = np.array(st.total_inner_iterations)
    st = m.TvProxState.cold((12, 9), 11, nonneg=True)
    out["tv_nn"] = m.tv_prox(x - 0.5, 0.2, st)
    st = m.TvProxState.cold((12, 9), 9, accelerated=False)
    out["tv_plain"] = m.tv_prox(x, 0.3, st)
    st = m.TvProxState.cold((12, 9), 200)
    m.tv_prox(x, 0.25, st)
    out["tv_gap"] = np.array(m.dual_gap_rof(x, st.q_warm, 0.25))

    # -- coins ----------------------------------------------------------------
    out["coins"] = np.stack([m.SkipConfig(0.1, s).stream().random(64) for s in range(4)])

    # -- ProxSkip / PGD denoising (config-1 path, small) ----------------------
    b = m.add_noise(m.gen_shapes_phantom(24, 20), 0.1, 3)
    out["dn_b"] = b

    def traj(run):
        xs, flags = [], []
        log = IterationLog(callback=lambda r, xx: (xs.append(xx.copy()), flags.append(r.prox_applied)))
        run(log)
        return np.stack(xs), np.array(flags)

    prob = m.build_tv_recon(m.identity_map(b.shape), b, 0.1, inner_budget=7)
    xs, fl = traj(lambda log: m.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                             m.SkipConfig(0.3, 5), 25, log))
    out["dn_ps_traj"], out["dn_ps_flags"] = xs, fl
    out["dn_ps_inner"] = np.array(prob.tv_state.total_inner_iterations)
    out["dn_ps_obj"] = np.array(objective_tv(xs[-1], prob))
    prob = m.build_tv_recon(m.identity_map(b.shape), b, 0.1, inner_budget=7)
    xs, _ = traj(lambda log: m.run_pgd(prob.prox_problem, np.zeros_like(b), 1.0, 6, log))
    out["dn_pgd_traj"] = xs

    # -- deblurring with FISTA / ProxSkip (config-2 path, small) -------------
    kern = m.gaussian_kernel(9, 2.0)
    A = m.blur_map(kern, (32, 32))
    truth = m.gen_shapes_phantom(32, 32)
    bb = m.add_noise(A.forward(truth), 0.01, 1)
    out["db_b"] = bb
    prob = m.build_tv_recon(A, bb, 0.02, inner_budget=5)
    L = prob.prox_problem.smooth.lipschitz
    out["db_L"] = np.array(L)
    xs, fl = traj(lambda log: m.run_proxskip(prob.prox_problem, np.zeros_like(bb), None, 1.0 / L,
                                             m.SkipConfig(0.2, 0), 20, log))
    out["db_ps_traj"], out["db_ps_flags"] = xs, fl
    out["db_ps_obj"] = np.array(objective_tv(xs[-1], prob))
    prob = m.build_tv_recon(A, bb, 0.02, inner_budget=5)
    prob.A.norm_sq_estimate = L
    xs, _ = traj(lambda log: m.run_fista(prob.prox_problem, np.zeros_like(bb), 1.0 / L, 8, log))
    out["db_fista_traj"] = xs

    # -- CT with PDHG / PDHGSkip-2, explicit splitting (config-3 path, small)
    n = 16
    geom = m.RadonGeometry(image_side=n, n_angles=7, n_bins=23)
    R = m.radon_map(geom)
    ph = m.gen_disc_phantom(n)
    sino = R.forward(ph)
    sino = m.add_noise(sino, 0.01 * sino.max(), 2)
    out["ct_b"] = sino
    prob = m.build_tv_recon(R, sino, 0.05, nonneg=True, splitting="explicit")
    sp_ = prob.saddle_problem
    out["ct_Knsq"] = np.array(sp_.norm_K_sq)
    step = 1.0 / np.sqrt(sp_.norm_K_sq)
    y0 = np.zeros(sp_.K.range_shape)
    xs, fl = traj(lambda log: m.run_pdhgskip2(sp_, np.zeros((n, n)), y0, None, step, step,
                                              m.SkipConfig(0.1, 0), 40, log))
    out["ct_skip_traj"], out["ct_skip_flags"] = xs, fl
    xs, _ = traj(lambda log: m.run_pdhg(sp_, np.zeros((n, n)), y0, step, step, 15, log))
    out["ct_pdhg_traj"] = xs
    # CT, implicit saddle form
    prob = m.build_tv_saddle_implicit(R, sino, 0.05, nonneg=True, inner_budget=6)
    spi = prob.saddle_problem
    out["cti_nsq"] = np.array(spi.norm_K_sq)
    st_ = 1.0 / np.sqrt(spi.norm_K_sq)
    xs, fl = traj(lambda log: m.run_pdhgskip2(spi, np.zeros((n, n)), np.zeros(R.range_shape), None,
                                              st_, st_, m.SkipConfig(0.3, 1), 12, log))
    out["cti_skip_traj"], out["cti_skip_flags"] = xs, fl

    path = os.path.join(HERE, "ref_hotpath.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays")


if __name__ == "__main__":
    main()
