"""Golden vectors for the SURVEY 8(f) rows (dual-ROF light-prox problems,
PDHGSkip-1, diagonal preconditioning), produced by the REFERENCE itself.

    python tests/golden/make_golden_next.py   ->  tests/golden/ref_next.npz
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    import imgskip as m
    from imgskip.solvers import IterationLog

    out = {}

    def traj(run):
        xs, flags = [], []
        run(IterationLog(callback=lambda r, x: (xs.append(np.array(x, copy=True)),
                                                flags.append(r.prox_applied))))
        return np.stack(xs), np.array(flags)

    # -- dual ROF (problems.py:22-84) ------------------------------------------
    b = m.add_noise(m.gen_shapes_phantom(16, 16), 0.05, 0)
    out["dr_b"] = b
    prob = m.build_dual_rof(b, 0.5)
    q0 = prob.zero_dual()
    g = 1.0 / prob.smooth.lipschitz
    xs, fl = traj(lambda log: m.run_proxskip(prob.prox_problem(), q0, None, g, m.SkipConfig(0.3, 1),
                                             30, log))
    out["dr_ps_traj"], out["dr_ps_flags"] = xs, fl
    out["dr_ps_primal"] = m.primal_from_dual(xs[-1], b)
    xs, _ = traj(lambda log: m.run_pgd(prob.prox_problem(), q0, g, 10, log))
    out["dr_pgd_traj"] = xs
    xs, _ = traj(lambda log: m.run_aprojgd(prob.smooth, prob.projector, q0, g, 10, log))
    out["dr_aprojgd_traj"] = xs
    rng = np.random.default_rng(3)
    qr = 0.3 * rng.standard_normal((2, 16, 16))
    out["dr_q"] = qr
    hub = m.build_dual_rof(b, 0.55, 0.1)
    out["dr_hub_grad"] = hub.smooth.grad(qr)
    out["dr_hub_obj"] = np.array(hub.smooth.objective(qr))
    out["dr_hub_L"] = np.array(hub.smooth.lipschitz)
    xs, _ = traj(lambda log: m.run_gd(prob.smooth, q0, g, 5, log))
    out["dr_gd_traj"] = xs

    # -- abs maps of grad_map (operators.py:81-94) -----------------------------
    D = m.grad_map((9, 13))
    u = rng.standard_normal((9, 13))
    qq = rng.standard_normal((2, 9, 13))
    out["abs_u"], out["abs_q"] = u, qq
    out["abs_grad"] = D.abs_forward(u)
    out["abs_div"] = D.abs_adjoint(qq)

    # -- CT explicit: PDHGSkip-1, diagonal steps, preconditioned PDHG ----------
    n = 16
    R = m.radon_map(m.RadonGeometry(image_side=n, n_angles=7, n_bins=23))
    sino = R.forward(m.gen_disc_phantom(n))
    sino = m.add_noise(sino, 0.01 * sino.max(), 2)
    out["ct_b"] = sino
    prob = m.build_tv_recon(R, sino, 0.05, nonneg=True, splitting="explicit")
    sp = prob.saddle_problem
    s = 1.0 / np.sqrt(sp.norm_K_sq)
    out["ct_nsq"] = np.array(sp.norm_K_sq)
    y0 = np.zeros(sp.K.range_shape)
    p = 0.3
    xs, fl = traj(lambda log: m.run_pdhgskip1(sp, np.zeros((n, n)), y0, s, s, 1.0 / p - 1.0,
                                              m.SkipConfig(p, 2), 20, log))
    out["ct_skip1_traj"], out["ct_skip1_flags"] = xs, fl
    from imgskip.solvers import diagonal_steps
    sig, tau = diagonal_steps(sp.K)
    out["ct_sigma"], out["ct_tau"] = sig, tau
    xs, _ = traj(lambda log: m.run_pdhg_preconditioned(sp, 20, log))
    out["ct_precond_traj"] = xs

    path = os.path.join(HERE, "ref_next.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays")


if __name__ == "__main__":
    main()
