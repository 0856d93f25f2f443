"""The cluster-resident 256x256 ProxSkip path (csrc/fgp_cluster.cu) against the
streaming kernels and the CPU oracle."""

import os

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


def _batch(idx):
    return np.stack([phantoms.config4_problem(int(i))[1] for i in idx])


def _run(b, idx, K, inner, p, stream_only, precision="fp32", graph=False):
    old = os.environ.get("PSB_NO_CLUSTER")
    os.environ["PSB_NO_CLUSTER"] = "1" if stream_only else "0"
    try:
        return psb.run_proxskip_batched(b, 0.1, p, idx, K, inner, precision=precision,
                                        use_graph=graph)
    finally:
        if old is None:
            os.environ.pop("PSB_NO_CLUSTER")
        else:
            os.environ["PSB_NO_CLUSTER"] = old


@pytest.mark.parametrize("graph", [False, True])
def test_cluster_matches_streaming_and_oracle(graph):
    idx = np.array([0, 5, 4095, 77, 1234])
    b = _batch(idx)
    K, inner, p = 40, 12, 0.25
    xc, cc = _run(b, idx, K, inner, p, stream_only=False, graph=graph)
    xs, cs = _run(b, idx, K, inner, p, stream_only=True)
    np.testing.assert_array_equal(cc, cs)
    for j, i in enumerate(idx):
        assert rel(xc[j], xs[j]) < 2e-6
        xr, _, n_prox, _ = oc.proxskip_denoise(b[j], 0.1, p, int(i), K, inner)
        assert cc[j] == n_prox
        assert rel(xc[j], xr) < 1e-5


def test_cluster8_in_a_captured_graph_matches_stream_launch():
    """More problems than 16-CTA clusters fit: the batch runs on the 8-CTA
    tensor-memory kernel; its launch inside a captured CUDA graph gives the
    stream launch's bits and the streaming kernels' values."""
    idx = np.arange(20) * 101 % 4096
    b = _batch(idx)
    K, inner, p = 30, 9, 0.3
    xg, cg = _run(b, idx, K, inner, p, stream_only=False, graph=True)
    xc, cc = _run(b, idx, K, inner, p, stream_only=False, graph=False)
    xs, cs = _run(b, idx, K, inner, p, stream_only=True)
    np.testing.assert_array_equal(cg, cc)
    np.testing.assert_array_equal(cg, cs)
    np.testing.assert_array_equal(np.asarray(xg), np.asarray(xc))
    for j in range(len(idx)):
        assert rel(xg[j], xs[j]) < 2e-6


def test_cluster_kernels_nonneg_instantiation(monkeypatch):
    """The nonneg = True instantiations (u clamped at 0 inside every FGP
    iteration and in the finalize, tv.py:77,89): 8-CTA kernel, 16-CTA kernel, SM
    workers and the streaming kernels agree, and match the oracle with a
    nonnegativity-constrained TV prox."""
    from paper_2411_00688_b200 import batched
    idx = np.arange(20) * 37 % 4096
    b = _batch(idx).astype(np.float32) - 0.35   # data with negative parts: the clamp is active
    K, inner, p = 24, 11, 0.3
    coins = batched.coin_table(p, idx, K)
    outs = {}
    for name, env in (("c8", {"PSB_CLUSTER8": "1", "PSB_NO_SMWORK": "1"}),
                      ("c16", {"PSB_CLUSTER8": "0", "PSB_NO_SMWORK": "1"}),
                      ("sm", {"PSB_SM_ONLY": "1"}),
                      ("stream", {"PSB_NO_CLUSTER": "1"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = psb.BatchedTvDenoise(torch.from_numpy(b).cuda(), 0.1, inner, precision="fp32", nonneg=True)
        s.run_proxskip(coins, 1.0, p)
        outs[name] = (s.x.clone(), s.prox_count.copy())
        for k in env:
            monkeypatch.delenv(k)
    for name in ("c16", "sm"):
        assert torch.equal(outs["c8"][0], outs[name][0]), name
        np.testing.assert_array_equal(outs["c8"][1], outs[name][1])
    xs = outs["stream"][0].cpu().numpy()
    xc = outs["c8"][0].cpu().numpy()
    for j in (0, 7, 19):
        assert rel(xc[j], xs[j]) < 2e-6
        pr = oc.make_recon(oc.identity_op(b[j].shape), b[j].astype(np.float64), 0.1,
                           splitting="implicit", inner=inner, nonneg=True)
        xr, _, n_prox, _ = oc.proxskip(pr.grad, pr.prox, np.zeros(b[j].shape), None, 1.0 / pr.L, p,
                                       int(idx[j]), K)
        assert outs["c8"][1][j] == n_prox
        assert rel(xc[j], xr) < 1e-5


def test_cluster_kernels_plain_fgp(monkeypatch):
    """accelerated = False (the plain projected-gradient inner loop, beta = 0
    in every iteration, tv.py:79-81): the run kernels agree bit for bit and
    match the streaming kernels."""
    from paper_2411_00688_b200 import batched
    idx = np.arange(18) * 41 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 20, 8, 0.35
    coins = batched.coin_table(p, idx, K)
    outs = {}
    for name, env in (("c8", {"PSB_CLUSTER8": "1", "PSB_NO_SMWORK": "1"}),
                      ("c16", {"PSB_CLUSTER8": "0", "PSB_NO_SMWORK": "1"}),
                      ("sm", {"PSB_SM_ONLY": "1"}),
                      ("stream", {"PSB_NO_CLUSTER": "1"})):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = psb.BatchedTvDenoise(torch.from_numpy(b).cuda(), 0.1, inner, precision="fp32",
                                 accelerated=False)
        s.run_proxskip(coins, 1.0, p)
        outs[name] = s.x.clone()
        for k in env:
            monkeypatch.delenv(k)
    assert torch.equal(outs["c8"], outs["c16"])
    assert torch.equal(outs["c8"], outs["sm"])
    xs, xc = outs["stream"].cpu().numpy(), outs["c8"].cpu().numpy()
    for j in range(len(idx)):
        assert rel(xc[j], xs[j]) < 2e-6


def test_cluster_warm_restart_reprojection_and_state():
    """Two runs on the same solver: the second uses a different p, so the prox
    weight changes and the warm start is re-projected (tv.py:68-69); x and h
    carry over; deferred skips span the run boundary via the flush."""
    idx = np.arange(3)
    b = _batch(idx)
    K1, K2, inner = 25, 30, 10
    solvers = {}
    for mode in ("cluster", "stream"):
        os.environ["PSB_NO_CLUSTER"] = "1" if mode == "stream" else "0"
        s = psb.BatchedTvDenoise(b, 0.1, inner, precision="fp32")
        s.run_proxskip(psb.coin_table(0.3, idx, K1), 1.0, 0.3)
        s.run_proxskip(psb.coin_table(0.15, idx + 100, K2), 1.0, 0.15)
        s.check_finite()
        solvers[mode] = s
    os.environ.pop("PSB_NO_CLUSTER")
    a, c = solvers["cluster"], solvers["stream"]
    for j in range(3):
        assert rel(a.x[j].cpu().numpy(), c.x[j].cpu().numpy()) < 2e-6
        assert rel(a.h[j].cpu().numpy(), c.h[j].cpu().numpy()) < 1e-4
        assert rel(a.slots[j, 0].cpu().numpy(), c.slots[j, 0].cpu().numpy()) < 1e-5
    np.testing.assert_array_equal(a.prox_count, c.prox_count)
    # oracle: the same two-run sequence with one FgpState per problem
    for j, i in enumerate(idx):
        pr = oc.make_recon(oc.identity_op(b[j].shape), b[j].astype(np.float64), 0.1, inner=inner)
        x, h, _, _ = oc.proxskip(pr.grad, pr.prox, np.zeros((256, 256)), None, 1.0, 0.3, int(i), K1)
        x, h, _, _ = oc.proxskip(pr.grad, pr.prox, x, h, 1.0, 0.15, int(i) + 100, K2)
        assert rel(a.x[j].cpu().numpy(), x) < 1e-5


def test_cluster_mixed_precision_single_problem_matches_oracle():
    truth, b = phantoms.config1_data(seed=2)
    prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=30, precision="mixed")
    x, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0, psb.SkipConfig(0.2, 2),
                              60)
    xr, _, n_prox, inner = oc.proxskip_denoise(b, 0.1, 0.2, 2, 60, 30)
    assert log.records[-1].prox_count == n_prox
    assert prob.tv_state.total_inner_iterations == inner
    assert rel(x, xr) < 1e-6


def test_cluster_divergence_reports_iteration():
    idx = np.arange(2)
    b = _batch(idx).astype(np.float32)
    b[1, 10, 10] = np.inf
    coins = psb.coin_table(0.3, idx, 20)
    s = psb.BatchedTvDenoise(b, 0.1, 5)
    s.run_proxskip(coins, 1.0, 0.3)
    with pytest.raises(psb.DivergenceError) as ei:
        s.check_finite()
    # problem 1's first iterate is already non-finite (iteration 0)
    assert ei.value.iteration == 0


def test_cluster_occupancy_query():
    import ctypes
    from paper_2411_00688_b200 import _lib as L
    n = ctypes.c_int(0)
    L.call("psb_cluster_max_active", ctypes.byref(n))
    assert n.value >= 1
    print("max active 16-CTA clusters:", n.value)


@pytest.mark.parametrize("mode", ["queue", "sm_only"])
def test_cluster_with_sm_workers_matches_streaming_and_oracle(mode, monkeypatch):
    """More problems than resident clusters: the SMs the clusters leave run
    fgp_sm_run_kernel, both kernels claiming from one device work queue
    ("queue"); PSB_SM_ONLY=1 hands the whole batch to the SM workers."""
    idx = np.arange(40) * 97 % 4096
    b = _batch(idx)
    K, inner, p = 30, 10, 0.2
    if mode == "sm_only":
        monkeypatch.setenv("PSB_SM_ONLY", "1")
    xc, cc = _run(b, idx, K, inner, p, stream_only=False)
    xs, cs = _run(b, idx, K, inner, p, stream_only=True)
    np.testing.assert_array_equal(cc, cs)
    for j in range(len(idx)):
        assert rel(xc[j], xs[j]) < 2e-6, j
    for j in (0, 17, 39):
        xr, _, n_prox, _ = oc.proxskip_denoise(b[j], 0.1, p, int(idx[j]), K, inner)
        assert cc[j] == n_prox
        assert rel(xc[j], xr) < 1e-5


def test_sm_workers_warm_restart_and_divergence(monkeypatch):
    """Two run segments on one solver with SM workers (x, h, warm starts carry
    over), and a non-finite problem reported with its first bad iteration."""
    idx = np.arange(20)
    b = _batch(idx).astype(np.float32)
    b[13, 5, 5] = np.nan
    monkeypatch.setenv("PSB_SM_ONLY", "1")
    s = psb.BatchedTvDenoise(b, 0.1, 8, precision="fp32")
    s.run_proxskip(psb.coin_table(0.3, idx, 12), 1.0, 0.3)
    s.run_proxskip(psb.coin_table(0.3, idx + 500, 9), 1.0, 0.3)
    monkeypatch.setenv("PSB_NO_CLUSTER", "1")
    r = psb.BatchedTvDenoise(b, 0.1, 8, precision="fp32")
    r.run_proxskip(psb.coin_table(0.3, idx, 12), 1.0, 0.3)
    r.run_proxskip(psb.coin_table(0.3, idx + 500, 9), 1.0, 0.3)
    for j in range(20):
        if j == 13:
            continue
        assert rel(s.x[j].cpu().numpy(), r.x[j].cpu().numpy()) < 2e-6
        assert rel(s.slots[j, 0].cpu().numpy(), r.slots[j, 0].cpu().numpy()) < 1e-5
    with pytest.raises(psb.DivergenceError) as ei:
        s.check_finite()
    assert ei.value.iteration == 0


def test_problem_range_calls_equal_one_shot():
    """BatchedTvDenoise.run_proxskip on problem ranges (lo, hi) in separate
    calls equals one call over the whole batch, bit for bit (problems are
    independent; cluster and SM-worker kernels share the arithmetic)."""
    idx = np.arange(50) * 31 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 20, 6, 0.25
    coins = psb.coin_table(p, idx, K)
    one = psb.BatchedTvDenoise(b, 0.1, inner)
    one.run_proxskip(coins, 1.0, p)
    parts = psb.BatchedTvDenoise(b, 0.1, inner)
    for lo in range(0, 50, 16):
        hi = min(50, lo + 16)
        parts.run_proxskip(np.ascontiguousarray(coins[:, lo:hi]), 1.0, p, lo=lo, hi=hi)
    np.testing.assert_array_equal(parts.prox_count, one.prox_count)
    assert torch.equal(parts.x, one.x)
    assert torch.equal(parts.h, one.h)
    assert torch.equal(parts.slots[:, 0], one.slots[:, 0])


@pytest.mark.parametrize("host", ["numpy", "pinned", "pageable"])
def test_host_inputs_equal_device_run(host):
    idx = np.arange(12) * 31 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 20, 6, 0.25
    x_ref, c_ref = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    src = b.astype(np.float64) if host == "numpy" else torch.from_numpy(b)
    if host == "pinned":
        src = src.pin_memory()
    x, c = psb.run_proxskip_batched(src, 0.1, p, idx, K, inner)
    np.testing.assert_array_equal(c, c_ref)
    x = x if isinstance(x, np.ndarray) else x.numpy()
    np.testing.assert_array_equal(x.astype(np.float32), x_ref.cpu().numpy())


def test_sm_worker_and_cluster_kernels_bitwise_equal(monkeypatch):
    """The same problems run entirely on the SM workers (PSB_SM_ONLY=1), on
    the clusters only (PSB_NO_SMWORK=1) and through the shared work queue give
    identical bits: which kernel claims a problem never changes a result."""
    idx = np.arange(24) * 53 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 25, 7, 0.3
    xq, cq = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    monkeypatch.setenv("PSB_SM_ONLY", "1")
    xs, cs = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    monkeypatch.delenv("PSB_SM_ONLY")
    monkeypatch.setenv("PSB_NO_SMWORK", "1")
    xc, cc = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    np.testing.assert_array_equal(cs, cc)
    np.testing.assert_array_equal(cq, cc)
    assert torch.equal(xs, xc)
    assert torch.equal(xq, xc)


def test_cluster8_kernel_bitwise_equals_cluster16(monkeypatch):
    """The 8-CTA cluster kernel (csrc/fgp_cluster8.cu: 16 px per thread, z and
    q_{k-1} in tensor memory; the default for fp32 outer state) gives the
    16-CTA kernel's (PSB_CLUSTER8=0) bits, and so does the mixed launch (2):
    warm restarts with re-projection, odd / even inner budgets, nonneg off,
    the streamed (cold, host input) path, and a diverging problem's iteration."""
    idx = np.arange(40) * 53 % 4096
    b = _batch(idx).astype(np.float32)
    for K, inner, p in ((25, 7, 0.3), (12, 50, 0.2), (9, 1, 0.5)):
        outs = []
        for c8 in ("0", "1", "2"):
            monkeypatch.setenv("PSB_CLUSTER8", c8)
            monkeypatch.setenv("PSB_NO_SMWORK", "1")
            s = psb.BatchedTvDenoise(torch.from_numpy(b).cuda(), 0.1, inner, precision="fp32")
            from paper_2411_00688_b200 import batched
            coins = batched.coin_table(p, idx, 2 * K)
            s.run_proxskip(coins[:K], 1.0, p)
            s.run_proxskip(coins[K:], 1.0, 0.5 * p + 0.1)  # weight changes: re-projection
            outs.append((s.x.clone(), s.h.clone(), s.slots[:, 0].clone(), s.prox_count.copy()))
            monkeypatch.delenv("PSB_NO_SMWORK")
            xh, ch = psb.run_proxskip_batched(b, 0.1, p, idx, K, inner)  # streamed host run
            outs[-1] += (torch.as_tensor(xh).clone(), np.asarray(ch).copy())
        for other in outs[1:]:
            for u, v in zip(outs[0], other):
                if isinstance(u, torch.Tensor):
                    assert torch.equal(u, v)
                else:
                    np.testing.assert_array_equal(u, v)
    bad = b[:3].copy()
    bad[1, 100, 100] = np.inf
    ks = []
    for c8 in ("0", "1"):
        monkeypatch.setenv("PSB_CLUSTER8", c8)
        with pytest.raises(psb.DivergenceError) as ei:
            psb.run_proxskip_batched(torch.from_numpy(bad).cuda(), 0.1, 0.3, idx[:3], 20, 5)
        ks.append(ei.value.iteration)
    assert ks[0] == ks[1]


@pytest.mark.parametrize("host", ["numpy", "numpy64", "pinned", "pageable"])
def test_streamed_host_run_equals_resident_run(host):
    """Host input streams in chunks (kernels wait on per-chunk ready flags,
    results leave per chunk behind a device counter); results bit-identical
    to the run on device-resident input."""
    idx = np.arange(60) * 29 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 24, 6, 0.25
    x_ref, c_ref = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    src = {"numpy": b, "numpy64": b.astype(np.float64)}.get(host)
    if src is None:
        src = torch.from_numpy(b)
    if host == "pinned":
        src = src.pin_memory()
    x, c = psb.run_proxskip_batched(src, 0.1, p, idx, K, inner, chunk=16)
    np.testing.assert_array_equal(c, c_ref)
    x = x if isinstance(x, np.ndarray) else x.numpy()
    np.testing.assert_array_equal(x.astype(np.float32), x_ref.cpu().numpy())


@pytest.mark.parametrize("pinned", [True, False])
def test_streamed_run_into_caller_buffer(pinned):
    """out=: the streamed run writes x into the caller's CPU buffer (DMA when
    page-locked) -- the same bits as the resident run; a wrong buffer is a
    ValueError."""
    idx = np.arange(40) * 31 % 4096
    b = _batch(idx).astype(np.float32)
    K, inner, p = 20, 5, 0.3
    x_ref, c_ref = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, p, idx, K, inner)
    src = torch.from_numpy(b).pin_memory()
    out = torch.full(b.shape, float("nan"), dtype=torch.float32)
    if pinned:
        out = out.pin_memory()
    x, c = psb.run_proxskip_batched(src, 0.1, p, idx, K, inner, chunk=16, out=out)
    assert x is out
    np.testing.assert_array_equal(c, c_ref)
    np.testing.assert_array_equal(out.numpy(), x_ref.cpu().numpy())
    with pytest.raises(ValueError):
        psb.run_proxskip_batched(src, 0.1, p, idx, K, inner, chunk=16,
                                 out=torch.empty((3, 256, 256), dtype=torch.float32))


_SERIAL_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2411_00688_b200 as psb
from paper_2411_00688_b200 import phantoms
idx = np.arange(48) * 37 % 4096
b = np.stack([phantoms.config4_problem(int(i))[1] for i in idx]).astype(np.float32)
x_ref, c_ref = psb.run_proxskip_batched(torch.from_numpy(b).cuda(), 0.1, 0.3, idx, 12, 5)
x, c = psb.run_proxskip_batched(torch.from_numpy(b).pin_memory(), 0.1, 0.3, idx, 12, 5, chunk=8)
assert np.array_equal(c, c_ref)
assert np.array_equal(x.numpy(), x_ref.cpu().numpy())
print("serial ok")
"""


def test_streamed_run_under_serialised_execution():
    """CUDA_LAUNCH_BLOCKING=1 serialises every launch: the streamed host-input
    path must not depend on the copy stream running beside the waiting run
    kernels (its H2D copies are enqueued before the run), so it completes
    quickly with the resident run's bits instead of timing out."""
    import subprocess
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1")
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c", _SERIAL_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "serial ok" in r.stdout
    assert time.time() - t0 < 120  # no 20 s device-wait timeouts
