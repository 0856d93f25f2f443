"""Pin the CPU oracle against golden vectors produced by the reference itself.

The vectors come from tests/golden/make_golden.py (imports /root/reference).
Elementwise/stencil results must be bit-identical; CSR-ordered sums and BLAS
reductions are compared at 1e-13 relative.
"""

import numpy as np
import pytest

from oracle import imgskip_cpu as oc
from oracle import tv3d_cpu as o3


def test_grad_div_ball_tv(golden):
    g = golden
    np.testing.assert_array_equal(oc.fd_grad(g["op_u"]), g["op_grad"])
    np.testing.assert_array_equal(oc.fd_div(g["op_q"]), g["op_div"])
    np.testing.assert_array_equal(oc.fd_div(g["op_qint"]), g["op_divint"])
    np.testing.assert_array_equal(oc.ball_project(3.0 * g["op_q"], 0.7), g["op_ball"])
    assert oc.tv_total(g["op_u"]) == float(g["op_tv"])


def test_blur(golden):
    g = golden
    taps = oc.gauss_taps(9, 2.0)
    np.testing.assert_array_equal(taps, g["blur_taps"])
    np.testing.assert_array_equal(oc.conv_periodic(g["blur_u"], taps), g["blur_fwd"])
    np.testing.assert_array_equal(oc.corr_periodic(g["blur_u"], taps), g["blur_adj"])
    np.testing.assert_array_equal(oc.conv_periodic(g["blur_u"], oc.gauss_taps(5, 1.2)),
                                  g["blur5_fwd"])
    assert oc.blur_op(taps, (32, 32)).norm_sq() == pytest.approx(float(g["blur_L_32"]), rel=1e-14)
    assert oc.power_iteration(oc.grad_op((16, 16))) == pytest.approx(float(g["grad_L_16"]),
                                                                     rel=1e-14)


@pytest.mark.parametrize("tag", ["r1", "r2", "r3"])
def test_radon(golden, tag):
    g = golden
    n, na, nb = (int(v) for v in g[f"{tag}_shape"])
    m = oc.radon_matrix(n, oc.default_angles(na), nb)
    assert m.nnz == int(g[f"{tag}_nnz"])
    op = oc.radon_op(n, na, nb)
    np.testing.assert_allclose(op.fwd(g[f"{tag}_x"]), g[f"{tag}_fwd"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(op.adj(g[f"{tag}_y"]), g[f"{tag}_adj"], rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(np.asarray(m.sum(axis=1)).ravel(), g[f"{tag}_rowsum"], rtol=1e-13)
    np.testing.assert_allclose(np.asarray(m.sum(axis=0)).ravel(), g[f"{tag}_colsum"], rtol=1e-13)


def test_tv_prox_sequence(golden):
    g = golden
    x = g["tv_x"]
    st = oc.FgpState.zeros(x.shape, 7)
    np.testing.assert_array_equal(oc.fgp_prox(x, 0.3, st), g["tv_u1"])
    np.testing.assert_array_equal(st.q, g["tv_q1"])
    np.testing.assert_array_equal(oc.fgp_prox(x, 0.3, st), g["tv_u2"])
    np.testing.assert_array_equal(oc.fgp_prox(x, 0.05, st), g["tv_u3"])
    np.testing.assert_array_equal(st.q, g["tv_q3"])
    assert st.inner_total == int(g["tv_count"])
    st = oc.FgpState.zeros(x.shape, 11, nonneg=True)
    np.testing.assert_array_equal(oc.fgp_prox(x - 0.5, 0.2, st), g["tv_nn"])
    st = oc.FgpState.zeros(x.shape, 9, accelerated=False)
    np.testing.assert_array_equal(oc.fgp_prox(x, 0.3, st), g["tv_plain"])
    st = oc.FgpState.zeros(x.shape, 200)
    oc.fgp_prox(x, 0.25, st)
    assert oc.rof_gap(x, st.q, 0.25) == pytest.approx(float(g["tv_gap"]), rel=1e-12, abs=1e-15)


def test_coins(golden):
    for s in range(4):
        draws = np.random.Generator(np.random.Philox(s)).random(64)
        np.testing.assert_array_equal(draws, golden["coins"][s])
        np.testing.assert_array_equal(oc.coin_draws(0.1, s, 64), golden["coins"][s] < 0.1)


def _collect():
    xs, flags = [], []
    return xs, flags, (lambda k, x, n, th: (xs.append(x.copy()), flags.append(th)))


def test_proxskip_denoise_trajectory(golden):
    g = golden
    b = g["dn_b"]
    pr = oc.make_recon(oc.identity_op(b.shape), b, 0.1, inner=7)
    xs, fl, obs = _collect()
    oc.proxskip(pr.grad, pr.prox, np.zeros_like(b), None, 1.0, 0.3, 5, 25, obs)
    np.testing.assert_array_equal(np.stack(xs), g["dn_ps_traj"])
    np.testing.assert_array_equal(np.array(fl), g["dn_ps_flags"])
    assert pr.tv.inner_total == int(g["dn_ps_inner"])
    assert oc.tv_objective(xs[-1], pr) == pytest.approx(float(g["dn_ps_obj"]), rel=1e-13)
    pr = oc.make_recon(oc.identity_op(b.shape), b, 0.1, inner=7)
    xs, _, obs = _collect()
    oc.pgd(pr.grad, pr.prox, np.zeros_like(b), 1.0, 6, obs)
    np.testing.assert_array_equal(np.stack(xs), g["dn_pgd_traj"])


def test_deblur_trajectories(golden):
    g = golden
    b = g["db_b"]
    A = oc.blur_op(oc.gauss_taps(9, 2.0), b.shape)
    pr = oc.make_recon(A, b, 0.02, inner=5)
    assert pr.L == pytest.approx(float(g["db_L"]), rel=1e-14)
    L = float(g["db_L"])
    xs, fl, obs = _collect()
    oc.proxskip(pr.grad, pr.prox, np.zeros_like(b), None, 1.0 / L, 0.2, 0, 20, obs)
    np.testing.assert_array_equal(np.array(fl), g["db_ps_flags"])
    np.testing.assert_allclose(np.stack(xs), g["db_ps_traj"], rtol=1e-12, atol=1e-13)
    pr = oc.make_recon(A, b, 0.02, inner=5)
    xs, _, obs = _collect()
    oc.fista(pr.grad, pr.prox, np.zeros_like(b), 1.0 / L, 8, obs)
    np.testing.assert_allclose(np.stack(xs), g["db_fista_traj"], rtol=1e-12, atol=1e-13)


def test_ct_pdhg_trajectories(golden):
    g = golden
    sino = g["ct_b"]
    R = oc.radon_op(16, 7, 23)
    pr = oc.make_recon(R, sino, 0.05, nonneg=True, splitting="explicit")
    assert pr.K_nsq == pytest.approx(float(g["ct_Knsq"]), rel=1e-12)
    nsq = float(g["ct_Knsq"])
    s = 1.0 / np.sqrt(nsq)
    y0 = np.zeros(pr.K.ran)
    xs, fl, obs = _collect()
    oc.pdhgskip2(pr.K, pr.prox_fstar, pr.prox_g, nsq, np.zeros((16, 16)), y0, None, s, s,
                 0.1, 0, 40, obs)
    np.testing.assert_array_equal(np.array(fl), g["ct_skip_flags"])
    np.testing.assert_allclose(np.stack(xs), g["ct_skip_traj"], rtol=1e-11, atol=1e-12)
    xs, _, obs = _collect()
    oc.pdhg(pr.K, pr.prox_fstar, pr.prox_g, nsq, np.zeros((16, 16)), y0, s, s, 15, obs)
    np.testing.assert_allclose(np.stack(xs), g["ct_pdhg_traj"], rtol=1e-11, atol=1e-12)
    pr = oc.make_saddle_implicit(R, sino, 0.05, nonneg=True, inner=6)
    nsq = float(g["cti_nsq"])
    s = 1.0 / np.sqrt(nsq)
    xs, fl, obs = _collect()
    oc.pdhgskip2(pr.K, pr.prox_fstar, pr.prox_g, nsq, np.zeros((16, 16)), np.zeros(R.ran), None,
                 s, s, 0.3, 1, 12, obs)
    np.testing.assert_array_equal(np.array(fl), g["cti_skip_flags"])
    np.testing.assert_allclose(np.stack(xs), g["cti_skip_traj"], rtol=1e-11, atol=1e-12)


def test_3d_plane_constant_matches_2d_reference(golden):
    # A volume of identical planes has zero z-differences, so every plane of
    # the 3-D prox must equal the reference 2-D prox at the same step (1/8).
    x2 = golden["tv_x"]
    vol = np.broadcast_to(x2, (4,) + x2.shape).copy()
    st = o3.Fgp3State.zeros(vol.shape, 7)
    u = o3.fgp_prox3(vol, 0.3, st, step=0.125)
    for z in range(4):
        np.testing.assert_array_equal(u[z], golden["tv_u1"])
    np.testing.assert_array_equal(st.q[0], 0.0)


def test_3d_div_is_negative_transpose():
    rng = np.random.default_rng(0)
    shape = (3, 4, 5)
    u = rng.integers(-20, 20, size=shape).astype(np.float64)
    q = rng.integers(-20, 20, size=(3,) + shape).astype(np.float64)
    assert np.sum(o3.fd_grad3(u) * q) == -np.sum(u * o3.fd_div3(q))


def test_3d_gap_vanishes():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((5, 6, 7))
    st = o3.Fgp3State.zeros(x.shape, 3000)
    u = o3.fgp_prox3(x, 0.2, st)
    obj = lambda v: 0.5 * np.sum((v - x) ** 2) + 0.2 * o3.tv_total3(v)
    base = obj(u)
    for seed in range(5):
        d = np.random.default_rng(seed).standard_normal(x.shape)
        d /= np.linalg.norm(d)
        assert obj(u + 1e-3 * d) >= base - 1e-9
