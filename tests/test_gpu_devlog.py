"""Device-side IterationLog (paper_2411_00688_b200/devlog.py):
a log with a reference solution / device objective / tol runs inside the
native drivers with an iterate history and batched reductions, and must
produce the same records, stopping iteration and final state as the
synchronous per-iteration observation path (the reference's semantics,
solvers.py:61-104)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2411_00688_b200 as psb  # noqa: E402
from paper_2411_00688_b200 import devlog, phantoms  # noqa: E402


def _denoise_data(n=64, seed=0):
    rng = np.random.default_rng(seed)
    u = phantoms.random_shapes((n, n), 6, rng)
    return phantoms.add_noise(u, 0.1, seed)


def _logs(prob, ref, tol=None, sync=False):
    cb = (lambda r, x: None) if sync else None
    st = prob.tv_state if prob.tv_state is not None else None
    return psb.IterationLog(reference=ref, objective_fn=psb.device_objective(prob),
                            inner_counter=(lambda: st.total_inner_iterations) if st else None,
                            tol=tol, callback=cb)


def _compare(la, lb, rtol=1e-11):
    assert len(la.records) == len(lb.records)
    for ra, rb in zip(la.records, lb.records):
        assert (ra.iteration, ra.prox_count, ra.inner_iter_count, ra.prox_applied) == \
            (rb.iteration, rb.prox_count, rb.inner_iter_count, rb.prox_applied)
        for a, b in ((ra.l2_rel_error, rb.l2_rel_error), (ra.objective, rb.objective)):
            assert (a is None) == (b is None)
            if a is not None:
                assert a == pytest.approx(b, rel=rtol)


@pytest.mark.parametrize("prec", ["mixed", "fp64"])
def test_denoise_device_log_matches_sync_observation(prec):
    b = _denoise_data()
    ref, _ = psb.run_pgd(psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=50,
                                            precision=prec).prox_problem, b, 1.0, 40)
    out = {}
    for sync in (False, True):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=20, precision=prec)
        log = _logs(prob, ref, sync=sync)
        x, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                  psb.SkipConfig(0.2, 3), 90, log)
        out[sync] = (x, log, prob.tv_state.total_inner_iterations)
    _compare(out[False][1], out[True][1])
    np.testing.assert_array_equal(out[False][0], out[True][0])
    assert out[False][2] == out[True][2]


def test_tol_stop_mid_chunk_lands_on_the_same_iteration(monkeypatch):
    b = _denoise_data(seed=1)
    prob0 = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=20)
    ref, _ = psb.run_pgd(prob0.prox_problem, b, 1.0, 60)
    # tol between the errors of iterations 36 and 37 of a logged run
    probe = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=20)
    _, lg = psb.run_proxskip(probe.prox_problem, np.zeros_like(b), None, 1.0,
                             psb.SkipConfig(0.3, 5), 80, _logs(probe, ref))
    errs = [r.l2_rel_error for r in lg.records]
    stop = next(k for k in range(30, 80) if errs[k] < errs[k - 1])
    tol = 0.5 * (errs[stop] + errs[stop - 1])
    # a 16-iteration history forces several chunks and a replay inside one
    monkeypatch.setattr(devlog, "HIST_BYTES", 16 * b.size * 8)
    out = {}
    for sync in (False, True):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=20)
        x, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                  psb.SkipConfig(0.3, 5), 80, _logs(prob, ref, tol=tol, sync=sync))
        out[sync] = (x, log, prob.tv_state)
    _compare(out[False][1], out[True][1])
    assert out[False][1].records[-1].l2_rel_error < tol
    np.testing.assert_array_equal(out[False][0], out[True][0])
    assert out[False][2].total_inner_iterations == out[True][2].total_inner_iterations
    np.testing.assert_array_equal(out[False][2].q_warm, out[True][2].q_warm)


def test_deblur_device_log():
    n = 64
    truth = phantoms.random_shapes((n, n), 5, np.random.default_rng(2), rects=False)
    k = psb.gaussian_kernel(9, 2.0)
    b = phantoms.add_noise(psb.blur_forward(truth, k), 0.01, 2)
    A = psb.blur_map(k, b.shape)
    out = {}
    for sync in (False, True):
        prob = psb.build_tv_recon(A, b, 0.02, inner_budget=10, precision="mixed")
        L = prob.prox_problem.smooth.lipschitz
        x, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0 / L,
                                  psb.SkipConfig(0.2, 0), 40, _logs(prob, truth, sync=sync))
        out[sync] = (x, log)
    _compare(out[False][1], out[True][1], rtol=1e-9)
    np.testing.assert_allclose(out[False][0], out[True][0], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("splitting", ["explicit", "implicit"])
def test_ct_device_log(splitting):
    n, na, nb = 32, 15, 47
    R = psb.radon_map(psb.RadonGeometry(image_side=n, n_angles=na, n_bins=nb))
    u_true = phantoms.shepp_like(n, 5, np.random.default_rng(4))
    s = R.forward(u_true)
    b = phantoms.add_noise(s, 0.01 * s.max(), 4)
    out = {}
    for sync in (False, True):
        if splitting == "explicit":
            prob = psb.build_tv_recon(R, b, 0.05, nonneg=True, splitting="explicit",
                                      precision="fp64")
            y0 = np.zeros(na * nb + 2 * n * n)
        else:
            prob = psb.build_tv_saddle_implicit(R, b, 0.05, nonneg=True, inner_budget=10,
                                                precision="fp64")
            y0 = np.zeros((na, nb))
        sp = prob.saddle_problem
        st = 1.0 / np.sqrt(sp.norm_K_sq)
        x, log = psb.run_pdhgskip2(sp, np.zeros((n, n)), y0, None, st, st, psb.SkipConfig(0.3, 1),
                                   50, _logs(prob, u_true, sync=sync))
        out[sync] = (x, log)
    _compare(out[False][1], out[True][1], rtol=1e-9)
    np.testing.assert_allclose(out[False][0], out[True][0], rtol=1e-10, atol=1e-12)
    assert any(r.objective == np.inf for r in out[False][1].records) or \
        all(np.isfinite(r.objective) for r in out[False][1].records)


def test_device_log_csv_deterministic(tmp_path):
    """Criterion 10 of the reference acceptance suite (test_acceptance.py:345-367):
    two runs give byte-identical CSVs modulo elapsed_s."""
    b = _denoise_data(seed=7)
    ref = b
    rows = []
    for i in range(2):
        prob = psb.build_tv_recon(psb.identity_map(b.shape), b, 0.1, inner_budget=10)
        _, log = psb.run_proxskip(prob.prox_problem, np.zeros_like(b), None, 1.0,
                                  psb.SkipConfig(0.3, 0), 60, _logs(prob, ref))
        path = tmp_path / f"{i}.csv"
        psb.emit_csv(log.records, str(path))
        rows.append([",".join(f for j, f in enumerate(line.split(",")) if j != 1)
                     for line in path.read_text().splitlines()])
    assert rows[0] == rows[1]
    assert rows[0][0] == psb.CSV_HEADER.replace(",elapsed_s", "")
