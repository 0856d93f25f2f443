"""SURVEY 8(f) rows on the device against reference golden vectors
(tests/golden/make_golden_next.py): dual-ROF light-prox problems
(problems.py:22-84) with ProxSkip / PGD / AProjGD / GD, PDHGSkip-1
(skip.py:82-114), diagonal preconditioning (solvers.py:212-234) and the
absolute gradient maps (operators.py:81-94)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gn():
    with np.load(os.path.join(HERE, "golden", "ref_next.npz")) as z:
        return {k: z[k] for k in z.files}


def _traj():
    xs, flags = [], []
    return xs, flags, psb.IterationLog(callback=lambda r, x: (xs.append(np.array(x, copy=True)),
                                                             flags.append(r.prox_applied)))


def test_dual_rof_drivers(gn):
    b = gn["dr_b"]
    prob = psb.build_dual_rof(b, 0.5)
    q0 = prob.zero_dual()
    g = 1.0 / prob.smooth.lipschitz
    xs, fl, log = _traj()
    psb.run_proxskip(prob.prox_problem(), q0, None, g, psb.SkipConfig(0.3, 1), 30, log)
    np.testing.assert_array_equal(np.array(fl), gn["dr_ps_flags"])
    np.testing.assert_allclose(np.stack(xs), gn["dr_ps_traj"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(psb.primal_from_dual(xs[-1], b), gn["dr_ps_primal"], rtol=1e-12,
                               atol=1e-13)
    xs, _, log = _traj()
    psb.run_pgd(prob.prox_problem(), q0, g, 10, log)
    np.testing.assert_allclose(np.stack(xs), gn["dr_pgd_traj"], rtol=1e-12, atol=1e-13)
    xs, _, log = _traj()
    psb.run_aprojgd(prob.smooth, prob.projector, q0, g, 10, log)
    np.testing.assert_allclose(np.stack(xs), gn["dr_aprojgd_traj"], rtol=1e-12, atol=1e-13)
    xs, _, log = _traj()
    psb.run_gd(prob.smooth, q0, g, 5, log)
    np.testing.assert_allclose(np.stack(xs), gn["dr_gd_traj"], rtol=1e-12, atol=1e-13)


def test_dual_huber_gradient_objective(gn):
    hub = psb.build_dual_rof(gn["dr_b"], 0.55, 0.1)
    assert hub.smooth.lipschitz == pytest.approx(float(gn["dr_hub_L"]), rel=1e-15)
    g = hub.smooth.grad(gn["dr_q"])
    np.testing.assert_allclose(g.cpu().numpy(), gn["dr_hub_grad"], rtol=1e-13, atol=1e-14)
    assert hub.smooth.objective(gn["dr_q"]) == pytest.approx(float(gn["dr_hub_obj"]), rel=1e-13)
    with pytest.raises(ValueError):
        psb.build_dual_rof(gn["dr_b"], 0.0)


def test_abs_grad_maps(gn):
    D = psb.grad_map((9, 13))
    np.testing.assert_array_equal(D.abs_forward(gn["abs_u"]), gn["abs_grad"])
    np.testing.assert_array_equal(D.abs_adjoint(gn["abs_q"]), gn["abs_div"])


def _ct(gn):
    R = psb.radon_map(psb.RadonGeometry(image_side=16, n_angles=7, n_bins=23))
    prob = psb.build_tv_recon(R, gn["ct_b"], 0.05, nonneg=True, splitting="explicit",
                              precision="fp64")
    sp = prob.saddle_problem
    sp.norm_K_sq = float(gn["ct_nsq"])
    return sp


def test_pdhgskip1(gn):
    sp = _ct(gn)
    s = 1.0 / np.sqrt(float(gn["ct_nsq"]))
    p = 0.3
    xs, fl, log = _traj()
    psb.run_pdhgskip1(sp, np.zeros((16, 16)), np.zeros(7 * 23 + 512), s, s, 1.0 / p - 1.0,
                      psb.SkipConfig(p, 2), 20, log)
    np.testing.assert_array_equal(np.array(fl), gn["ct_skip1_flags"])
    np.testing.assert_allclose(np.stack(xs), gn["ct_skip1_traj"], rtol=1e-10, atol=1e-12)
    # staircase: x is constant on skipped iterations (test_skip.py:165-179)
    for k in range(1, 20):
        if not fl[k]:
            np.testing.assert_array_equal(xs[k], xs[k - 1])


def test_diagonal_preconditioning(gn):
    sp = _ct(gn)
    sig, tau = psb.diagonal_steps(sp.K)
    np.testing.assert_allclose(sig.cpu().numpy(), gn["ct_sigma"], rtol=1e-12)
    np.testing.assert_allclose(tau.cpu().numpy(), gn["ct_tau"], rtol=1e-12)
    xs, _, log = _traj()
    psb.run_pdhg_preconditioned(sp, 20, log)
    np.testing.assert_allclose(np.stack(xs), gn["ct_precond_traj"], rtol=1e-10, atol=1e-12)


def test_bernoulli_op():
    x = np.array([2.0, -4.0])
    np.testing.assert_allclose(psb.bernoulli_op(x, 0.25, True), x / 0.25)
    np.testing.assert_array_equal(psb.bernoulli_op(x, 0.25, False), 0.0)
    with pytest.raises(ValueError):
        psb.bernoulli_op(x, 0.0, True)
