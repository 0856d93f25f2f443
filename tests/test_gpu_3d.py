"""GPU parity for the 3-D path (BASELINE config 5): the 3-D FGP kernel against
the oracle restatement (oracle/tv3d_cpu.py, itself pinned to the reference's
2-D prox), and the z-slab decomposition against the whole volume."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402,F401
from paper_2411_00688_b200 import phantoms, volume3d as v3  # noqa: E402
from oracle import tv3d_cpu as o3  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def test_plane_constant_volume_equals_reference_2d(golden):
    x2 = golden["tv_x"]
    vol = np.broadcast_to(x2, (4,) + x2.shape).copy()
    st = v3.TvProxState3D(vol.shape, 7, dtype=torch.float64, step=0.125)
    u = v3.tv_prox3d(vol, 0.3, st)
    for z in range(4):
        np.testing.assert_array_equal(u[z], golden["tv_u1"])
    np.testing.assert_array_equal(st.q_warm[0], 0.0)


@pytest.mark.parametrize("shape", [(2, 2, 2), (3, 5, 7), (9, 13, 37), (17, 8, 70)])
@pytest.mark.parametrize("inner", [1, 3])
def test_tv_prox3d_fp64_bitwise(shape, inner):
    rng = np.random.default_rng(sum(shape) + inner)
    x = rng.standard_normal(shape)
    st = v3.TvProxState3D(shape, inner, dtype=torch.float64)
    so = o3.Fgp3State.zeros(shape, inner)
    for w in (0.2, 0.2, 0.05):
        np.testing.assert_array_equal(v3.tv_prox3d(x, w, st), o3.fgp_prox3(x, w, so))
        np.testing.assert_array_equal(st.q_warm, so.q)


def test_tv_prox3d_fp32_tolerance():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((40, 48, 64))
    st = v3.TvProxState3D(x.shape, 20)
    so = o3.Fgp3State.zeros(x.shape, 20)
    for _ in range(2):
        assert rel(v3.tv_prox3d(x, 0.3, st), o3.fgp_prox3(x, 0.3, so)) < 1e-5


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("n_slabs", [2, 3, 5])
@pytest.mark.parametrize("exchange", ["direct", "copy", "peer"])
def test_slab_decomposition_is_exact(precision, n_slabs, exchange):
    """Overlapped slab schedule (interior launch, then the edge planes once the
    halo ring slot arrived) == the whole volume, bit for bit, for the three
    data paths: edge kernels storing into the neighbours' rings, send buffers +
    copies (NCCL's), and one stream per slab ordered only by device flags
    (the peer-memory protocol of the multi-GPU run)."""
    vol = phantoms.random_ellipsoids((23, 20, 36), 6, np.random.default_rng(1))
    b = phantoms.add_noise(vol, 0.1, 1)
    x1, s1 = v3.proxskip_denoise3d(b, 0.08, 0.3, 4, 20, 5, n_slabs=1, precision=precision)
    xn, sn = v3.proxskip_denoise3d(b, 0.08, 0.3, 4, 20, 5, n_slabs=n_slabs, precision=precision,
                                   exchange=exchange)
    np.testing.assert_array_equal(x1, xn)
    assert s1[0].prox_count == sn[-1].prox_count
    for s in sn:  # the warm start left in slot 0 matches the whole volume's
        np.testing.assert_array_equal(s.q[0].cpu().numpy(),
                                      s1[0].q[0][:, s.z0:s.z0 + s.D].cpu().numpy())


@pytest.mark.parametrize("exchange", ["direct", "peer"])
def test_thin_slabs_exact(exchange):
    """Slabs of one and two planes (no interior; both edges on one plane)."""
    vol = phantoms.random_ellipsoids((9, 16, 40), 4, np.random.default_rng(2))
    b = phantoms.add_noise(vol, 0.1, 2)
    x1, _ = v3.proxskip_denoise3d(b, 0.08, 0.4, 6, 12, 4, n_slabs=1, precision="fp64")
    xn, sn = v3.proxskip_denoise3d(b, 0.08, 0.4, 6, 12, 4, n_slabs=7, precision="fp64",
                                   exchange=exchange)
    assert sorted({s.D for s in sn}) == [1, 2]
    np.testing.assert_array_equal(x1, xn)


def test_config5_reduced_size_vs_oracle():
    """Config 5 inputs at 48^3 (50 ellipsoids, noise 0.1, alpha 0.08, p 0.1,
    FGP-20, step 1/12, 200 outer) against the 3-D oracle; fp32 device path,
    2 emulated slabs."""
    n = 48
    vol = phantoms.random_ellipsoids((n, n, n), 50, np.random.default_rng(0)).astype(np.float64)
    b = phantoms.add_noise(vol, 0.1, 0)
    x, slabs = v3.proxskip_denoise3d(b, 0.08, 0.1, 0, 200, 20, n_slabs=2, precision="fp32")
    xr, _, n_prox, _ = o3.proxskip_denoise3(b, 0.08, 0.1, 0, 200, 20)
    assert slabs[0].prox_count == n_prox
    assert rel(x, xr) < 1e-4
    obj = lambda u: 0.5 * np.sum((u - b) ** 2) + 0.08 * o3.tv_total3(u)
    assert abs(obj(x) - obj(xr)) / obj(xr) < 1e-5


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_deferred_skips_are_bitwise_identical(precision):
    vol = phantoms.random_ellipsoids((12, 20, 36), 6, np.random.default_rng(3))
    b = phantoms.add_noise(vol, 0.1, 3)
    xa, _ = v3.proxskip_denoise3d(b, 0.08, 0.2, 9, 37, 4, n_slabs=2, precision=precision,
                                  defer_skips=True)
    xb, _ = v3.proxskip_denoise3d(b, 0.08, 0.2, 9, 37, 4, n_slabs=2, precision=precision,
                                  defer_skips=False)
    np.testing.assert_array_equal(xa, xb)


@pytest.mark.parametrize("shape,n_slabs", [((23, 20, 36), 3), ((9, 33, 260), 2), ((40, 17, 128), 1)])
def test_tma_staging_is_bitwise_the_cp_async_path(monkeypatch, shape, n_slabs):
    """The fp32 3-D kernel stages planes with tensor-map TMA tiles (zero-filled
    out of range) by default; PSB_NO_TMA3D=1 selects the per-lane cp.async
    staging.  Same values reach the arithmetic, so the runs agree bit for bit
    (slab halo planes, band edges and ragged tiles included)."""
    vol = phantoms.random_ellipsoids(shape, 5, np.random.default_rng(5))
    b = phantoms.add_noise(vol, 0.1, 5)
    xa, sa = v3.proxskip_denoise3d(b, 0.08, 0.3, 2, 15, 6, n_slabs=n_slabs, precision="fp32")
    monkeypatch.setenv("PSB_NO_TMA3D", "1")
    xb, sb = v3.proxskip_denoise3d(b, 0.08, 0.3, 2, 15, 6, n_slabs=n_slabs, precision="fp32")
    np.testing.assert_array_equal(xa, xb)
    for p, q in zip(sa, sb):
        np.testing.assert_array_equal(p.q.cpu().numpy(), q.q.cpu().numpy())


@pytest.mark.parametrize("n", [2, 3])
def test_peer_exchange_across_processes(n):
    """The multi-GPU wiring of the config-5 peer exchange (CUDA IPC handles
    swapped over a gloo group, edge kernels storing into the other process's
    rings, flags written / waited on by stream memory operations) with n
    processes sharing this box's one GPU: the gathered slabs equal the
    whole-volume run bit for bit.  A protocol check, not a timing (no kernel
    waits on another; the streams do)."""
    import os
    import socket
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tools", "run_config5_dist.py"), "--side", "40", "--iters", "30",
           "--inner", "5", "--p", "0.3", "--check", "--share-device"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"bitwise_equal_whole_volume": true' in r.stdout


def test_proxskip_denoise3d_into_caller_buffer():
    """out=: x lands in the caller's (page-locked) CPU buffer -- the same bits
    as the default return; a wrong buffer is a ValueError."""
    vol = phantoms.random_ellipsoids((24, 20, 36), 5, np.random.default_rng(8))
    b = torch.from_numpy(phantoms.add_noise(vol, 0.1, 8).astype(np.float32)).pin_memory()
    x_ref, _ = v3.proxskip_denoise3d(b, 0.08, 0.3, 0, 9, 4)
    out = torch.full(b.shape, float("nan"), dtype=torch.float32).pin_memory()
    x, _ = v3.proxskip_denoise3d(b, 0.08, 0.3, 0, 9, 4, out=out)
    assert x is out
    assert torch.equal(out, x_ref)
    with pytest.raises(ValueError):
        v3.proxskip_denoise3d(b, 0.08, 0.3, 0, 9, 4, out=torch.empty((3, 3, 3)))
