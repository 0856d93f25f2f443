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


def test_aprojgd_dual_fused_fgp_path(gn):
    """run_aprojgd on the plain dual-ROF problem with a passive log is one FGP
    burst; it reproduces the reference trajectory's end point and the stepped
    (observed) run bit for bit over a longer run."""
    b = gn["dr_b"]
    prob = psb.build_dual_rof(b, 0.5)
    g = 1.0 / prob.smooth.lipschitz
    q, log = psb.run_aprojgd(prob.smooth, prob.projector, prob.zero_dual(), g, 10)
    np.testing.assert_allclose(q, gn["dr_aprojgd_traj"][-1], rtol=1e-12, atol=1e-13)
    assert [r.prox_count for r in log.records] == list(range(1, 11))
    q_fast, _ = psb.run_aprojgd(prob.smooth, prob.projector, prob.zero_dual(), g, 300)
    xs, _, lg = _traj()
    q_step, _ = psb.run_aprojgd(prob.smooth, prob.projector, prob.zero_dual(), g, 300, lg)
    np.testing.assert_allclose(q_fast, q_step, rtol=1e-13, atol=1e-14)


def test_pdhg_preconditioned_native(gn):
    sp = _ct(gn)
    x, log = psb.run_pdhg_preconditioned(sp, 20)
    np.testing.assert_allclose(x, gn["ct_precond_traj"][-1], rtol=1e-10, atol=1e-12)
    assert len(log.records) == 20


def test_compute_reference_solution(gn):
    R = psb.radon_map(psb.RadonGeometry(image_side=16, n_angles=7, n_bins=23))
    sino = R.forward(gn["abs_u"][:9, :9].repeat(2, 0).repeat(2, 1)[:16, :16] ** 2)
    sp_prob = psb.build_tv_recon(R, sino, 0.05, nonneg=True, splitting="explicit",
                                 precision="fp64")
    ref = psb.compute_reference_solution(sp_prob, 20000)
    assert ref.provenance["method"] == "pdhg-preconditioned-explicit"
    assert ref.provenance["self_consistency_error"] <= psb.SELF_CONSISTENCY_TOL
    # the split run is exactly one run
    x1, _ = psb.run_pdhg_preconditioned(sp_prob.saddle_problem, 20000)
    np.testing.assert_array_equal(ref.u_star, x1)
    with pytest.raises(psb.ReferenceRejectedError):
        psb.compute_reference_solution(sp_prob, 10)
    b = np.random.default_rng(1).random((16, 16))
    dual = psb.build_dual_rof(b, 0.2)
    ref_d = psb.compute_reference_solution(dual, 6000)
    assert ref_d.provenance["method"] == "aprojgd-dual"
    q, _ = psb.run_aprojgd(dual.smooth, dual.projector, dual.zero_dual(), 1.0 / 8.0, 6000)
    np.testing.assert_array_equal(ref_d.u_star, psb.primal_from_dual(q, b))


def test_dual_rof_fused_drivers_match_reference_and_stepping(gn):
    """Passive logs run the dual-ROF problems in the native driver
    (csrc/dualrof.cu): the end points equal the reference trajectories, and
    longer runs are bitwise the observed (stepped) runs -- same operations in
    the same order."""
    b = gn["dr_b"]
    prob = psb.build_dual_rof(b, 0.5)
    q0 = prob.zero_dual()
    g = 1.0 / prob.smooth.lipschitz
    q, log = psb.run_proxskip(prob.prox_problem(), q0, None, g, psb.SkipConfig(0.3, 1), 30)
    np.testing.assert_allclose(q, gn["dr_ps_traj"][-1], rtol=1e-12, atol=1e-13)
    np.testing.assert_array_equal([r.prox_applied for r in log.records], gn["dr_ps_flags"])
    q, _ = psb.run_pgd(prob.prox_problem(), q0, g, 10)
    np.testing.assert_allclose(q, gn["dr_pgd_traj"][-1], rtol=1e-12, atol=1e-13)
    q, _ = psb.run_fista(prob.prox_problem(), q0, g, 10)
    np.testing.assert_allclose(q, gn["dr_aprojgd_traj"][-1], rtol=1e-12, atol=1e-13)
    q, _ = psb.run_gd(prob.smooth, q0, g, 5)
    np.testing.assert_allclose(q, gn["dr_gd_traj"][-1], rtol=1e-12, atol=1e-13)

    rng = np.random.default_rng(8)
    b2 = rng.random((48, 64))
    for huber in (0.0, 0.1):
        pr = psb.build_dual_rof(b2, 0.3, huber)
        z = pr.zero_dual()
        g = 1.0 / pr.smooth.lipschitz
        runs = {
            "proxskip": lambda log: psb.run_proxskip(pr.prox_problem(), z, None, g,
                                                     psb.SkipConfig(0.2, 3), 300, log),
            "pgd": lambda log: psb.run_pgd(pr.prox_problem(), z, g, 200, log),
            "fista": lambda log: psb.run_fista(pr.prox_problem(), z, g, 200, log),
            "gd": lambda log: psb.run_gd(pr.smooth, z, g, 100, log),
            "aprojgd": lambda log: psb.run_aprojgd(pr.smooth, pr.projector, z, g, 200, log),
        }
        for name, run in runs.items():
            fast, _ = run(None)
            stepped, _ = run(psb.IterationLog(callback=lambda r, x: None))
            if name == "aprojgd" and huber == 0.0:
                # plain dual: the FGP-kernel path (different but exact-order kernel)
                np.testing.assert_allclose(fast, stepped, rtol=1e-12, atol=1e-14)
            else:
                np.testing.assert_array_equal(fast, stepped, err_msg=f"{name} huber={huber}")


def test_pdhgskip1_native_driver(gn):
    """PDHGSkip-1 on the explicit CT splitting in the native driver (passive
    log): the reference's end point, coin accounting, and the stepped run."""
    sp = _ct(gn)
    s = 1.0 / np.sqrt(float(gn["ct_nsq"]))
    p = 0.3
    x, log = psb.run_pdhgskip1(sp, np.zeros((16, 16)), np.zeros(7 * 23 + 512), s, s, 1.0 / p - 1.0,
                               psb.SkipConfig(p, 2), 20)
    np.testing.assert_allclose(x, gn["ct_skip1_traj"][-1], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal([r.prox_applied for r in log.records], gn["ct_skip1_flags"])
    assert log.records[-1].prox_count == int(np.sum(gn["ct_skip1_flags"]))
    xs, _, lg = _traj()
    xstep, _ = psb.run_pdhgskip1(sp, np.zeros((16, 16)), np.zeros(7 * 23 + 512), s, s,
                                 1.0 / p - 1.0, psb.SkipConfig(p, 2), 20, lg)
    np.testing.assert_allclose(x, xstep, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("diag", [True, False])
def test_pdhg_explicit_blur_graph_replay_equals_stepped(monkeypatch, diag):
    """PDHG on the explicit blur splitting K = [blur; D] (the deblurring
    reference-solution path, harness.py:246-251 -> solvers.py:227-234) has no
    fused kernel: a passive run replays one captured CUDA graph per
    iteration.  Same kernels, same iterates as the stepped loop, bit for bit;
    a non-finite iterate raises with the stepped loop's iteration."""
    from paper_2411_00688_b200 import phantoms
    _, b, _ = phantoms.config2_data(0, 48)
    A = psb.blur_map(psb.gaussian_kernel(9, 2.0), b.shape)
    prob = psb.build_tv_recon(A, b, 0.02, nonneg=True, splitting="explicit", precision="fp64")
    sp = prob.saddle_problem
    y0 = np.zeros(48 * 48 * 3)
    if diag:
        run = lambda: psb.run_pdhg_preconditioned(sp, 40)  # noqa: E731
    else:
        s = 1.0 / np.sqrt(sp.norm_K_sq)
        run = lambda: psb.run_pdhg(sp, np.zeros((48, 48)), y0, s, s, 40)  # noqa: E731
    xg, log = run()
    assert len(log.records) == 40
    monkeypatch.setenv("PSB_NO_GRAPH_PDHG", "1")
    xs, _ = run()
    np.testing.assert_array_equal(xg, xs)
    # divergence: a NaN in the data poisons the iterate at the first step
    bad = b.copy()
    bad[3, 4] = np.nan
    pb = psb.build_tv_recon(A, bad, 0.02, splitting="explicit", precision="fp64")
    ks = []
    for flag in ("1", "0"):
        monkeypatch.setenv("PSB_NO_GRAPH_PDHG", flag)
        with pytest.raises(psb.DivergenceError) as ei:
            s = 1.0 / np.sqrt(pb.saddle_problem.norm_K_sq)
            psb.run_pdhg(pb.saddle_problem, np.zeros((48, 48)), y0, s, s, 20)
        ks.append(ei.value.iteration)
    assert ks[0] == ks[1]
