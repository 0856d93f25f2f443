"""GPU parity for the CT path (BASELINE config 3): matrix-free projector pair
and the fused PDHG / PDHGSkip-2 kernels against the reference golden vectors
and the CPU oracle (scipy CSR, as in operators.py:218-292)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms  # noqa: E402
from oracle import imgskip_cpu as oc  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


@pytest.mark.parametrize("tag", ["r1", "r2", "r3"])
def test_radon_pair_vs_reference_csr(golden, tag):
    g = golden
    n, na, nb = (int(v) for v in g[f"{tag}_shape"])
    op = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=na, n_bins=nb))
    np.testing.assert_allclose(op.forward(g[f"{tag}_x"]), g[f"{tag}_fwd"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(op.adjoint(g[f"{tag}_y"]), g[f"{tag}_adj"], rtol=1e-12, atol=1e-12)
    # row / column sums of the implied matrix
    np.testing.assert_allclose(op.forward(np.ones((n, n))).ravel(), g[f"{tag}_rowsum"], rtol=1e-12,
                               atol=1e-12)
    np.testing.assert_allclose(op.adjoint(np.ones((na, nb))).ravel(), g[f"{tag}_colsum"],
                               rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("n,na,nb,sp", [(10, 7, 15, 1.0), (31, 13, 40, 1.0), (64, 60, 91, 1.0),
                                        (20, 9, 41, 0.5), (16, 5, 16, 1.3)])
def test_radon_adjoint_identity_and_oracle(n, na, nb, sp):
    geom = psb.RadonGeometry(image_side=n, n_angles=na, n_bins=nb, bin_spacing=sp)
    op = psb.radon_map(geom)
    ref = oc.radon_op(n, na, nb, bin_spacing=sp)
    for seed in range(5):
        rng = np.random.default_rng(seed)
        x, y = rng.standard_normal((n, n)), rng.standard_normal((na, nb))
        ax, aty = op.forward(x), op.adjoint(y)
        np.testing.assert_allclose(ax, ref.fwd(x), rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(aty, ref.adj(y), rtol=1e-12, atol=1e-12)
        defect = abs(np.sum(ax * y) - np.sum(x * aty)) / (np.linalg.norm(ax) * np.linalg.norm(y))
        assert defect < 1e-12


def test_radon_full_geometry_fp32():
    geom = psb.RadonGeometry(image_side=512, n_angles=60, n_bins=725)
    op = psb.radon_map(geom)
    ref = oc.radon_op(512, 60, 725)
    u = phantoms.shepp_like(512, 10, np.random.default_rng(0))
    s32 = op.forward(torch.tensor(u, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    assert rel(s32, ref.fwd(u)) < 1e-6
    y = np.random.default_rng(1).standard_normal((60, 725))
    a32 = op.adjoint(torch.tensor(y, dtype=torch.float32, device="cuda")).double().cpu().numpy()
    assert rel(a32, ref.adj(y)) < 1e-6


def _traj():
    xs, flags = [], []
    return xs, flags, psb.IterationLog(callback=lambda r, x: (xs.append(x.copy()),
                                                             flags.append(r.prox_applied)))


def test_ct_explicit_trajectories_fp64(golden):
    g = golden
    sino = g["ct_b"]
    R = psb.radon_map(psb.RadonGeometry(image_side=16, n_angles=7, n_bins=23))
    prob = psb.build_tv_recon(R, sino, 0.05, nonneg=True, splitting="explicit", precision="fp64")
    sp = prob.saddle_problem
    assert sp.norm_K_sq == pytest.approx(float(g["ct_Knsq"]), rel=1e-10)
    nsq = float(g["ct_Knsq"])
    sp.norm_K_sq = nsq
    s = 1.0 / np.sqrt(nsq)
    y0 = np.zeros(7 * 23 + 2 * 256)
    xs, fl, log = _traj()
    psb.run_pdhgskip2(sp, np.zeros((16, 16)), y0, None, s, s, psb.SkipConfig(0.1, 0), 40, log)
    np.testing.assert_array_equal(np.array(fl), g["ct_skip_flags"])
    np.testing.assert_allclose(np.stack(xs), g["ct_skip_traj"], rtol=1e-10, atol=1e-12)
    # native driver (passive log) reaches the same iterate
    x, _ = psb.run_pdhgskip2(sp, np.zeros((16, 16)), y0, None, s, s, psb.SkipConfig(0.1, 0), 40)
    np.testing.assert_allclose(x, g["ct_skip_traj"][-1], rtol=1e-10, atol=1e-12)
    xs, _, log = _traj()
    psb.run_pdhg(sp, np.zeros((16, 16)), y0, s, s, 15, log)
    np.testing.assert_allclose(np.stack(xs), g["ct_pdhg_traj"], rtol=1e-10, atol=1e-12)


def test_pdhgskip2_p1_is_pdhg():
    n = 24
    geom = psb.RadonGeometry(image_side=n, n_angles=9, n_bins=35)
    R = psb.radon_map(geom)
    b = R.forward(phantoms.shepp_like(n, 4, np.random.default_rng(2)))
    prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit", precision="fp64")
    sp = prob.saddle_problem
    s = 1.0 / np.sqrt(sp.norm_K_sq)
    y0 = np.zeros(9 * 35 + 2 * n * n)
    xa, _ = psb.run_pdhg(sp, np.zeros((n, n)), y0, s, s, 30)
    xb, _ = psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, s, s, psb.SkipConfig(1.0, 0), 30)
    np.testing.assert_array_equal(xa, xb)


def test_pdhg_step_rule_enforced():
    R = psb.radon_map(psb.RadonGeometry(image_side=8, n_angles=3, n_bins=12))
    prob = psb.build_tv_recon(R, np.zeros((3, 12)), 0.05, splitting="explicit")
    with pytest.raises(ValueError):
        psb.run_pdhg(prob.saddle_problem, np.zeros((8, 8)), np.zeros(36 + 128), 2.0, 2.0, 3)


@pytest.mark.slow
def test_config3_full_geometry_parity_150_iters():
    """Config 3 at full geometry (512^2, 60 angles, 725 bins, alpha=0.05,
    nonneg, PDHGSkip-2 p=0.1): 150 of the 2000 iterations so the CSR oracle
    finishes in well under a minute; objective via the unguarded formula (D8)."""
    n = 512
    u_true = phantoms.shepp_like(n, 10, np.random.default_rng(0))
    ref_op = oc.radon_op(n, 60, 725)
    s = ref_op.fwd(u_true)
    b = phantoms.add_noise(s, 0.01 * s.max(), 0)
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
    prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit", precision="mixed")
    sp = prob.saddle_problem
    assert sp.norm_K_sq == pytest.approx(29740.8629, rel=2e-3)
    st = 1.0 / np.sqrt(sp.norm_K_sq)
    y0 = np.zeros(60 * 725 + 2 * n * n)
    x, log = psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st, psb.SkipConfig(0.1, 0), 150)
    pr = oc.make_recon(ref_op, b, 0.05, nonneg=True, splitting="explicit", K_nsq=sp.norm_K_sq)
    xr, _, _, n_prox, _ = oc.pdhgskip2(pr.K, pr.prox_fstar, pr.prox_g, pr.K_nsq, np.zeros((n, n)),
                                      y0, None, st, st, 0.1, 0, 150)
    assert log.records[-1].prox_count == n_prox
    assert rel(x, xr) < 1e-4
    o_dev = psb.objective_tv(x, prob, guarded=False)
    o_ref = oc.tv_objective(xr, pr, guarded=False)
    assert abs(o_dev - o_ref) / abs(o_ref) < 1e-5


def test_ct_implicit_saddle_pdhgskip2_fp64(golden):
    """PDHGSkip-2 on the implicit saddle form (K = A, TV in
    the warm-started FGP prox with nonneg) -- build_tv_saddle_implicit,
    problems.py:162-184 -- against the reference trajectory."""
    g = golden
    sino = g["ct_b"]
    R = psb.radon_map(psb.RadonGeometry(image_side=16, n_angles=7, n_bins=23))
    prob = psb.build_tv_saddle_implicit(R, sino, 0.05, nonneg=True, inner_budget=6,
                                        precision="fp64")
    sp = prob.saddle_problem
    assert sp.norm_K_sq == pytest.approx(float(g["cti_nsq"]), rel=1e-10)
    s = 1.0 / np.sqrt(float(g["cti_nsq"]))
    sp.norm_K_sq = float(g["cti_nsq"])
    xs, fl, log = _traj()
    psb.run_pdhgskip2(sp, np.zeros((16, 16)), np.zeros((7, 23)), None, s, s,
                      psb.SkipConfig(0.3, 1), 12, log)
    np.testing.assert_array_equal(np.array(fl), g["cti_skip_flags"])
    np.testing.assert_allclose(np.stack(xs), g["cti_skip_traj"], rtol=1e-10, atol=1e-12)


@pytest.mark.slow
def test_config3_fp32_tent_gather_full_run_vs_fp64():
    """The fp32 CT path (tent-weight gather, csrc/radon.cu pixel_gather_tent)
    over the full config-3 run (512^2, 60 x 725, PDHGSkip-2 p=0.1, 2000
    iterations) against the exact fp64 path, which is pinned to the reference
    by the golden trajectories above: rel-L2(u) <= 1e-4, objective <= 1e-5."""
    n = 512
    u_true = phantoms.shepp_like(n, 10, np.random.default_rng(0))
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=725))
    s = R.forward(u_true)
    b = phantoms.add_noise(s, 0.01 * s.max(), 0)
    out = {}
    for prec in ("fp64", "fp32"):
        prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit", precision=prec)
        sp = prob.saddle_problem
        sp.norm_K_sq = 29740.8629  # same steps for both arms
        st = 1.0 / np.sqrt(sp.norm_K_sq)
        x, log = psb.run_pdhgskip2(sp, np.zeros((n, n)), np.zeros(60 * 725 + 2 * n * n), None, st,
                                   st, psb.SkipConfig(0.1, 0), 2000)
        out[prec] = (x, psb.objective_tv(x, prob, guarded=False))
    assert rel(out["fp32"][0], out["fp64"][0]) < 1e-4
    assert abs(out["fp32"][1] - out["fp64"][1]) / abs(out["fp64"][1]) < 1e-5


def test_ct_implicit_native_driver_matches_reference_fp64(golden):
    """The native implicit driver (psb_ct_implicit_run, passive log) reaches the
    reference's final iterate and the same TvProxState accounting."""
    g = golden
    R = psb.radon_map(psb.RadonGeometry(image_side=16, n_angles=7, n_bins=23))
    prob = psb.build_tv_saddle_implicit(R, g["ct_b"], 0.05, nonneg=True, inner_budget=6,
                                        precision="fp64")
    sp = prob.saddle_problem
    sp.norm_K_sq = float(g["cti_nsq"])
    s = 1.0 / np.sqrt(sp.norm_K_sq)
    x, log = psb.run_pdhgskip2(sp, np.zeros((16, 16)), np.zeros((7, 23)), None, s, s,
                               psb.SkipConfig(0.3, 1), 12)
    np.testing.assert_allclose(x, g["cti_skip_traj"][-1], rtol=1e-10, atol=1e-12)
    np.testing.assert_array_equal([r.prox_applied for r in log.records], g["cti_skip_flags"])
    n_prox = int(np.sum(g["cti_skip_flags"]))
    assert prob.tv_state.total_inner_iterations == 6 * n_prox
    assert prob.tv_state.last_weight == (s / 0.3) * 0.05


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-12), ("mixed", 1e-4), ("fp32", 1e-4)])
def test_ct_implicit_native_vs_oracle(prec, tol):
    """64^2 implicit CT (nonneg, PDHGSkip-2 p=0.2, 60 iterations, FGP-20)
    against the oracle; then PDHG (p=1) through run_pdhg on the same driver."""
    n, na, nb = 64, 30, 91
    u_true = phantoms.shepp_like(n, 6, np.random.default_rng(3))
    ref_op = oc.radon_op(n, na, nb)
    sino = ref_op.fwd(u_true)
    b = phantoms.add_noise(sino, 0.01 * sino.max(), 3)
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=na, n_bins=nb))
    for p, iters in ((0.2, 60), (1.0, 25)):
        prob = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=20,
                                            precision=prec)
        sp = prob.saddle_problem
        pr = oc.make_saddle_implicit(ref_op, b, 0.05, nonneg=True, inner=20)
        nsq = pr.K_nsq
        sp.norm_K_sq = nsq
        st = 1.0 / np.sqrt(nsq)
        if p < 1.0:
            x, log = psb.run_pdhgskip2(sp, np.zeros((n, n)), np.zeros((na, nb)), None, st, st,
                                       psb.SkipConfig(p, 4), iters)
            assert log.records[-1].prox_count == int(np.sum(oc.coin_draws(p, 4, iters)))
        else:
            x, _ = psb.run_pdhg(sp, np.zeros((n, n)), np.zeros((na, nb)), st, st, iters)
        xr = oc.pdhgskip2(pr.K, pr.prox_fstar, pr.prox_g, nsq, np.zeros((n, n)),
                          np.zeros((na, nb)), None, st, st, p, 4, iters)[0]
        assert rel(x, xr) < tol, (p, rel(x, xr))


@pytest.mark.parametrize("prec", ["fp32", "mixed", "fp64"])
@pytest.mark.parametrize("variant", ["pdhgskip2", "pdhg", "implicit"])
def test_transposed_forward_gather_is_bitwise(prec, variant):
    """The native run drivers give the forward projector a transposed copy of
    xbar (steep rays gather along memory rows); the stepped path (a callback
    log: one step per Python call) gathers from xbar itself.  Same taps in the
    same order: the iterates agree bit for bit."""
    n = 96
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=60, n_bins=137))
    b = R.forward(phantoms.shepp_like(n, 6, np.random.default_rng(3)))
    b = phantoms.add_noise(b, 0.01 * b.max(), 3)
    split = "implicit" if variant == "implicit" else "explicit"

    def run(stepped):
        if split == "explicit":
            prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit",
                                      precision=prec)
            y0 = np.zeros(60 * 137 + 2 * n * n)
        else:
            prob = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=5,
                                                precision=prec)
            y0 = np.zeros((60, 137))
        sp = prob.saddle_problem
        sp.norm_K_sq = 4000.0
        s = 1.0 / np.sqrt(sp.norm_K_sq)
        log = psb.IterationLog(callback=lambda rec, x: None) if stepped else None
        if variant == "pdhg":
            x, _ = psb.run_pdhg(sp, np.zeros((n, n)), y0, s, s, 25, log)
        else:
            x, _ = psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, s, s,
                                     psb.SkipConfig(0.3, 1), 25, log)
        return x

    if variant == "implicit":
        # the stepped implicit path composes operator-level kernels (A^T y,
        # prox steps) whose grouping differs from the fused driver's at the
        # last bit; the transposed gather itself is covered bitwise above
        tol = 1e-4 if prec == "fp32" else 1e-12
        np.testing.assert_allclose(run(False), run(True), rtol=tol, atol=tol)
    else:
        np.testing.assert_array_equal(run(False), run(True))
