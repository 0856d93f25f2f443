"""Temporally blocked FGP (fgp2d_tb_kernel: TBI = 10 inner iterations per
launch on 64 x 64 register windows -- a 44 x 44 output tile plus a 10-pixel
halo) against the one-launch-per-iteration streaming kernel (PSB_NO_TB=1) --
same per-pixel formulas, different instruction selection, so agreement to
2e-6 absolute -- and against the CPU oracle."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import _lib as L  # noqa: E402
from oracle import imgskip_cpu as oc  # noqa: E402


def _prox_batch(x, q0, weight, inner, rep, nonneg, active, tb):
    """psb_tv_prox2d on a (N, H, W) batch; returns (u, slot 0)."""
    import os
    old = os.environ.get("PSB_NO_TB")
    os.environ["PSB_NO_TB"] = "0" if tb else "1"
    try:
        n, H, W = x.shape
        xd = torch.from_numpy(x).cuda()
        q = torch.zeros((n, 3, 2, H, W), dtype=torch.float32, device="cuda")
        q[:, 0] = torch.from_numpy(q0).cuda()
        u = torch.zeros_like(xd)
        act = torch.tensor(active, dtype=torch.int32, device="cuda")
        reps = torch.tensor([rep] * len(active), dtype=torch.uint8, device="cuda")
        L.call("psb_tv_prox2d", L.F32, L.ptr(xd), H * W, L.ptr(q), 6 * H * W, L.ptr(act),
               len(active), float(weight), None, 0, L.ptr(reps), H, W, inner, 1, int(nonneg),
               0.125, L.ptr(u), H * W, L.stream())
        torch.cuda.synchronize()
        return u.cpu().numpy(), q[:, 0].cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("PSB_NO_TB")
        else:
            os.environ["PSB_NO_TB"] = old


@pytest.mark.parametrize("shape", [(33, 47), (64, 64), (100, 300), (256, 256), (512, 512)])
@pytest.mark.parametrize("inner", [5, 17, 50])
def test_tb_equals_streaming(shape, inner):
    rng = np.random.default_rng(sum(shape) + inner)
    n = 3
    x = rng.standard_normal((n,) + shape).astype(np.float32)
    q0 = (0.05 * rng.standard_normal((n, 2) + shape)).astype(np.float32)
    q0[:, 0, -1, :] = 0.0  # a warm start the FGP produced (zero on the last row / column)
    q0[:, 1, :, -1] = 0.0
    for rep, nonneg, active in ((0, 0, [0, 1, 2]), (1, 0, [2, 0]), (0, 1, [1])):
        ut, qt = _prox_batch(x, q0, 0.3, inner, rep, nonneg, active, True)
        us, qs = _prox_batch(x, q0, 0.3, inner, rep, nonneg, active, False)
        for e in active:
            np.testing.assert_allclose(ut[e], us[e], rtol=0, atol=2e-6)
            np.testing.assert_allclose(qt[e], qs[e], rtol=0, atol=2e-6)
        untouched = [i for i in range(n) if i not in active]
        for i in untouched:
            assert np.all(ut[i] == 0)


def test_tb_prox_matches_oracle_sequence():
    """Warm-started sequence of tv_prox calls (fp32, TB path), including a
    weight change (re-projection), vs the float64 oracle."""
    rng = np.random.default_rng(7)
    b = rng.standard_normal((96, 80))
    st = psb.TvProxState.cold(b.shape, 20)
    ost = oc.FgpState.zeros(b.shape, 20)
    for wgt in (0.3, 0.3, 0.5):
        u = psb.tv_prox(b, wgt, st)
        ur = oc.fgp_prox(b, wgt, ost)
        assert float(np.linalg.norm(u - ur) / np.linalg.norm(ur)) < 1e-5
