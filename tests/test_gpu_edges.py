"""Edge cases on the device: ragged and minimal shapes (vector and scalar
kernel variants), non-aligned widths, empty runs, nonneg clamps in the
cluster path, non-finite inputs, and size-independent properties at large
sizes -- the reference's validation behaviour (test_operators.py:98-112,
test_tv.py:36-43, test_skip.py:42-46, test_solvers.py:60-68) included."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import phantoms, volume3d  # noqa: E402
from paper_2411_00688_b200.operators import div_dev  # noqa: E402
from oracle import imgskip_cpu as oc  # noqa: E402
from oracle import tv3d_cpu as o3  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


SHAPES = [(2, 2), (2, 3), (3, 2), (5, 7), (17, 33), (64, 130), (130, 64), (129, 257), (2, 300)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("nonneg", [False, True])
def test_tv_prox_ragged_shapes_fp64_bitwise(shape, nonneg):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    st = psb.TvProxState.cold(shape, 9, nonneg=nonneg, dtype=torch.float64)
    ref = oc.FgpState.zeros(shape, 9, nonneg=nonneg)
    for wgt in (0.3, 0.3, 0.7):  # warm start + re-projection on the weight change
        u = psb.tv_prox(x, wgt, st)
        ur = oc.fgp_prox(x, wgt, ref)
        np.testing.assert_array_equal(u, ur)
    np.testing.assert_array_equal(st.q_warm, ref.q)
    assert st.total_inner_iterations == ref.inner_total == 27


@pytest.mark.parametrize("shape", SHAPES)
def test_tv_prox_ragged_shapes_fp32(shape):
    rng = np.random.default_rng(7 + sum(shape))
    x = rng.standard_normal(shape)
    st = psb.TvProxState.cold(shape, 20)
    ref = oc.FgpState.zeros(shape, 20)
    u = psb.tv_prox(x, 0.25, st)
    ur = oc.fgp_prox(x, 0.25, ref)
    assert rel(u, ur) < 2e-6


def test_validation_matches_reference():
    with pytest.raises(ValueError):
        psb.grad_forward(np.zeros((1, 5)))
    with pytest.raises(ValueError):
        psb.divergence(np.zeros((2, 1, 5)))
    with pytest.raises(ValueError):
        psb.TvProxState.cold((5, 7), 0)
    with pytest.raises(ValueError):
        psb.tv_prox(np.zeros((4, 4)), 0.0, psb.TvProxState.cold((4, 4), 3))
    with pytest.raises(ValueError):
        psb.SkipConfig(0.0, 0)
    with pytest.raises(ValueError):
        psb.SkipConfig(1.2, 0)
    with pytest.raises(ValueError):
        psb.RadonGeometry(image_side=8, n_angles=4, n_bins=6)
    with pytest.raises(ValueError):
        psb.block_stack(psb.identity_map((4, 4)), psb.grad_map((5, 5)))
    A = psb.identity_map((6, 6))
    with pytest.raises(ValueError):
        psb.build_tv_recon(A, np.zeros((6, 6)), -1.0)
    with pytest.raises(ValueError):
        psb.build_tv_recon(A, np.zeros((6, 6)), 0.1, splitting="magic")
    with pytest.raises(ValueError):
        psb.build_tv_recon(A, np.zeros((6, 6)), 0.1, inner_budget=0)
    prob = psb.build_tv_recon(A, np.zeros((6, 6)), 0.1)
    with pytest.raises(ValueError):
        psb.run_proxskip(prob.prox_problem, np.zeros((6, 6)), None, 0.0, psb.SkipConfig(0.5, 0), 3)
    with pytest.raises(ValueError):
        psb.run_pgd(prob.prox_problem, np.zeros((6, 6)), -1.0, 3)


@pytest.mark.parametrize("prec", ["mixed", "fp64"])
def test_zero_iterations_return_a_copy(prec):
    b = np.random.default_rng(1).random((16, 16))
    prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=5, precision=prec)
    x0 = np.full_like(b, 0.5)
    x, log = psb.run_proxskip(prob.prox_problem, x0, None, 1.0, psb.SkipConfig(0.3, 0), 0)
    np.testing.assert_array_equal(x, x0)
    assert x is not x0 and log.records == []
    assert prob.tv_state.total_inner_iterations == 0


def test_run_with_no_coin_fired():
    """A run whose coins never fire executes only skip updates (skip.py:72-74)."""
    b = np.random.default_rng(2).random((256, 256))
    seed = next(s for s in range(1000) if not psb.SkipConfig(0.05, s).coins(4).any())
    for prec in ("mixed", "fp32"):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=5, precision=prec)
        x, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                  psb.SkipConfig(0.05, seed), 4)
        ref = oc.make_recon(oc.identity_op(b.shape), b, 0.1, inner=5)
        xr = oc.proxskip(ref.grad, ref.prox, np.zeros_like(b), None, 1.0, 0.05, seed, 4)[0]
        assert rel(x, xr) < 1e-6
        assert log.records[-1].prox_count == 0


def test_cluster_path_nonneg_matches_oracle():
    """256^2 fp32 problems take the cluster kernel; nonneg selects its clamped
    instantiation (tv.py:65,76)."""
    u = phantoms.random_shapes((256, 256), 8, np.random.default_rng(3))
    b = phantoms.add_noise(u, 0.2, 3) - 0.1
    prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, nonneg=True, inner_budget=20,
                              precision="fp32")
    x, _ = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                            psb.SkipConfig(0.2, 4), 30)
    pr = oc.make_recon(oc.identity_op(b.shape), b, 0.1, nonneg=True, inner=20)
    xr = oc.proxskip(pr.grad, pr.prox, np.zeros_like(b), None, 1.0, 0.2, 4, 30)[0]
    assert rel(x, xr) < 1e-5


@pytest.mark.parametrize("n,shape", [(1, (256, 256)), (3, (40, 72)), (2, (33, 17))])
def test_batched_odd_batches_and_shapes(n, shape):
    rng = np.random.default_rng(n)
    b = rng.random((n,) + shape)
    seeds = np.arange(n) + 11
    x, counts = psb.run_proxskip_batched(b, 0.1, 0.3, seeds, 12, 8, precision="fp32")
    for i in range(n):
        xr, _, npx, _ = oc.proxskip_denoise(b[i], 0.1, 0.3, int(seeds[i]), 12, 8)
        assert counts[i] == npx
        assert rel(x[i], xr) < 2e-5


def test_nonfinite_input_raises_divergence():
    b = np.random.default_rng(4).random((256, 256))
    b[3, 5] = np.nan
    for prec in ("fp32", "mixed"):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=5,
                                  precision=prec)
        with pytest.raises(psb.DivergenceError) as ei:
            psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                             psb.SkipConfig(0.5, 0), 5)
        assert ei.value.iteration == 0 and ei.value.algorithm == "proxskip"


@pytest.mark.parametrize("shape", [(3, 5, 7), (4, 9, 130), (6, 2, 2), (2, 33, 20)])
def test_tv_prox3d_ragged_fp64_bitwise(shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    st = volume3d.TvProxState3D(shape, 6, dtype=torch.float64)
    ref = o3.Fgp3State.zeros(shape, 6)
    for wgt in (0.2, 0.5):
        u = volume3d.tv_prox3d(x, wgt, st)
        ur = o3.fgp_prox3(x, wgt, ref)
        np.testing.assert_array_equal(u, ur)


def test_radon_minimal_geometries():
    for n, na, nb in ((2, 1, 2), (3, 2, 3), (8, 1, 8)):
        op = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=na, n_bins=nb))
        ref = oc.radon_op(n, na, nb)
        x = np.random.default_rng(n).random((n, n))
        y = np.random.default_rng(na).random((na, nb))
        np.testing.assert_allclose(op.forward(x), ref.fwd(x), rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(op.adjoint(y), ref.adj(y), rtol=1e-12, atol=1e-13)


def test_large_tv_prox_properties():
    """4096^2 fp32: size-independent properties -- the dual iterate is
    feasible (|q| <= w), u = x + div q, and the ROF duality gap shrinks with
    the inner budget (tv.py:92-105)."""
    n = 4096
    x = torch.rand((n, n), device="cuda", dtype=torch.float32)
    gaps = []
    for inner in (10, 40):
        st = psb.TvProxState.cold((n, n), inner)
        u = psb.tv_prox(x, 0.05, st)
        q = st.slots[0].double()
        # the fp32 ball projection (radius w (1 - 2^-20), common.cuh) keeps the
        # dual iterate inside the reference's feasibility ball exactly
        assert float(torch.sqrt(q[0] ** 2 + q[1] ** 2).max()) <= 0.05
        div = div_dev(q)
        assert float((u.double() - (x.double() + div)).abs().max()) < 1e-5
        # the fp32 state itself passes dual_gap_rof's check (tv.py:98-100)
        gaps.append(psb.dual_gap_rof(x.double(), st.slots[0], 0.05))
    assert gaps[1] < gaps[0]


@pytest.mark.parametrize("prec", ["mixed", "fp64"])
def test_fista_native_equals_stepped_denoise(prec):
    """FISTA on the identity fidelity: the native driver (passive log) and the
    stepped run (observing log) execute the same operations."""
    b = np.random.default_rng(9).random((40, 52))
    out = []
    for log in (None, psb.IterationLog(callback=lambda r, x: None)):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=7, precision=prec)
        x, _ = psb.run_fista(prob.prox_problem, np.zeros_like(b), 1.0, 25, log)
        out.append(x)
    if prec == "fp64":
        np.testing.assert_array_equal(out[0], out[1])
    else:
        assert rel(out[0], out[1]) < 1e-12


@pytest.mark.parametrize("prec,shape", [("fp64", (40, 52)), ("mixed", (256, 256))])
def test_pgd_native_equals_stepped(prec, shape):
    """run_pgd with a passive log runs the native driver as ProxSkip(p = 1),
    which is PGD operation for operation (skip.py:62-64)."""
    b = np.random.default_rng(10).random(shape)
    out = []
    for log in (None, psb.IterationLog(callback=lambda r, x: None)):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=7, precision=prec)
        x, lg = psb.run_pgd(prob.prox_problem, np.zeros_like(b), 1.0, 12, log)
        out.append(x)
        assert lg.records[-1].prox_count == 12
    if prec == "fp64":
        np.testing.assert_array_equal(out[0], out[1])
    else:
        assert rel(out[0], out[1]) < 2e-6  # cluster kernel (fp32 FGP) vs streaming path


def test_c_host_through_the_abi(tmp_path):
    """A plain C program (tests/c_host/tv_prox_demo.c) drives the library
    through include/psb200.h only -- context, buffers, copies, the fp64 TV
    prox twice (warm start) -- and matches the oracle bit for bit."""
    import os
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    libdir = os.path.join(root, "paper_2411_00688_b200")
    exe = tmp_path / "tv_prox_demo"
    subprocess.run([gcc, "-O2", "-std=c11", os.path.join(root, "tests", "c_host", "tv_prox_demo.c"),
                    "-I", os.path.join(root, "include"), "-L", libdir, "-lpsb200",
                    f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    H, W, inner, wgt = 37, 61, 12, 0.3
    x = np.random.default_rng(11).standard_normal((H, W))
    x.tofile(tmp_path / "in.bin")
    subprocess.run([str(exe), str(H), str(W), str(inner), str(wgt), str(tmp_path / "in.bin"),
                    str(tmp_path / "out.bin")], check=True)
    u = np.fromfile(tmp_path / "out.bin", dtype=np.float64).reshape(H, W)
    st = oc.FgpState.zeros((H, W), inner)
    oc.fgp_prox(x, wgt, st)
    np.testing.assert_array_equal(u, oc.fgp_prox(x, wgt, st))


def test_device_coin_table_is_numpys_philox_stream():
    """psb_coin_table (SeedSequence + Philox4x64-10 on the device) reproduces
    Generator(Philox(seed)).random() < p bit for bit (skip.py:27-28)."""
    seeds = [0, 1, 7, 4095, 2 ** 31 + 5, 2 ** 32, 2 ** 40 + 3, 2 ** 62 + 11] + list(range(100, 140))
    for p in (0.1, 0.5, 1.0):
        t = psb.coin_table(p, seeds, 301)
        assert t.shape == (301, len(seeds)) and t.dtype == np.uint8
        for j, s in enumerate(seeds):
            draws = np.random.Generator(np.random.Philox(s)).random(301)
            np.testing.assert_array_equal(t[:, j], (draws < p).astype(np.uint8))
    big = psb.coin_table(0.1, np.arange(4096), 300)
    assert abs(big.mean() - 0.1) < 0.005
    with pytest.raises(ValueError):
        psb.coin_table(0.0, [1], 3)
