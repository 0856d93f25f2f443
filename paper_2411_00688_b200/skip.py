"""ProxSkip and PDHGSkip-2 on the device (skip.py of the reference).

Coins: one ``Generator(Philox(seed)).random()`` draw per iteration, compared
with p (skip.py:27-28, 67, 136).  The whole coin sequence is drawn on the host
up front -- bit-identical to the reference's stream -- so the GPU never
generates randomness and the fused drivers know the skip pattern in advance.

Fast path: a problem assembled by ``problems.build_tv_recon`` with an
identity fidelity (BASELINE configs 1/4) and a passive IterationLog runs the
whole outer loop inside the native driver (psb_proxskip_denoise_run: fused
pre/FGP/post kernels, optionally one CUDA graph).  Every other case runs the
same kernels step by step from Python and observes each iteration exactly
like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from . import tensor as T
from .errors import DivergenceError
from .operators import apply_adjoint, apply_forward
from .devlog import device_loggable, run_logged
from .solvers import IterationLog, RunRecord, _check_finite, _check_step_rule, _dev, _ensure_log

INT32_MAX = 2 ** 31 - 1


@dataclass
class SkipConfig:
    """Skip probability + seed of the per-run Bernoulli stream (skip.py:16-28)."""

    p: float
    seed: int = 0

    def __post_init__(self):
        if not 0.0 < self.p <= 1.0:
            raise ValueError(f"SkipConfig: p must be in (0, 1], got {self.p}")

    def stream(self):
        return np.random.Generator(np.random.Philox(self.seed))

    def coins(self, iters):
        """theta_k = stream().random() < p for k < iters (host, uint8)."""
        return (self.stream().random(iters) < self.p).astype(np.uint8)


def optimal_probability(mu, L):  # noqa: N803  (the reference's parameter name)
    """sqrt(mu / L) (skip.py:31-35)."""
    if mu <= 0 or L <= 0 or mu > L:
        raise ValueError(f"optimal_probability: need 0 < mu <= L, got mu={mu}, L={L}")
    return float(np.sqrt(mu / L))


def _finish_passive(log, coins, elapsed, base_inner, inner_iters):
    """Fill the records of a passive log after a fused run."""
    counts = np.cumsum(coins.astype(np.int64))
    for k in range(len(coins)):
        inner = base_inner + inner_iters * int(counts[k]) if log.inner_counter is not None else 0
        log.records.append(RunRecord(k + 1, float(elapsed[k]), int(counts[k]), inner, None, None,
                                     bool(coins[k])))


def run_proxskip(problem, x0, h0, gamma, skip, iters, log=None, *, use_graph=None):
    """ProxSkip (skip.py:46-79).  Returns (x_final, IterationLog)."""
    if gamma <= 0:
        raise ValueError("run_proxskip: gamma must be positive")
    log = _ensure_log(log)
    dual = getattr(problem, "_dual_rof", None)
    if dual is not None and log.passive and iters >= 1:
        from .solvers import _dual_rof_fused
        return _dual_rof_fused(dual, "proxskip", x0, gamma, iters, log, skip=skip, h0=h0)
    fused = getattr(problem, "_fused", None)
    if (fused is not None and fused.get("kind") in ("denoise", "deblur")
            and (log.passive or device_loggable(log))):
        return _proxskip_tv_fused(problem, fused, x0, h0, gamma, skip, iters, log, use_graph)
    log.start(AR.is_host(x0))
    p = skip.p
    coins = skip.coins(iters)
    dt = getattr(problem, "outer_dtype", torch.float64)
    x = AR.to_dev(x0, dt).clone()
    h = AR.to_dev(h0, dt).clone() if h0 is not None else torch.zeros_like(x)
    hc = gamma - gamma / p
    pg = p / gamma
    prox_count = 0
    step = fused is not None and fused.get("kind") == "denoise"
    for k in range(iters):
        theta = bool(coins[k])
        if step:
            x, h = _denoise_step(problem, fused, x, h, gamma, p, hc, pg, theta, k)
        else:
            g = _dev(problem.smooth.grad(x), x)
            t = T.lincomb(1.0, x, -gamma, g)
            xhat = T.lincomb(1.0, t, gamma, h)
            if theta:
                xn = _dev(problem.prox_g(T.lincomb(1.0, t, hc, h), gamma / p), x)
            else:
                xn = xhat
            h = T.lincomb(1.0, h, pg, T.lincomb(1.0, xn, -1.0, xhat))
            x = xn
        prox_count += theta
        _check_finite(x, k, "proxskip")
        if log.observe(k + 1, x, prox_count, theta):
            break
    return AR.like(x, x0), log


# -- fused identity-fidelity path (configs 1 / 4) ------------------------------

_ONE = {}


def _coin_dev(theta):
    key = (torch.cuda.current_device(), bool(theta))
    if key not in _ONE:
        _ONE[key] = torch.tensor([1 if theta else 0], dtype=torch.uint8, device="cuda")
    return _ONE[key]


def _denoise_step(problem, fused, x, h, gamma, p, hc, pg, theta, k):
    """One outer iteration with the same kernels the native driver uses."""
    st = problem.tv_state
    b = fused["b_dev"]
    H, W = st.shape
    HW = H * W
    dto, dtf = L.dcode(x.dtype), L.dcode(st.dtype)
    z = fused.setdefault("z", torch.empty((H, W), dtype=st.dtype, device="cuda"))
    bad = fused.setdefault("bad", torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda"))
    L.call("psb_proxskip_pre", dto, dtf, L.ptr(x), L.ptr(b), 1, L.ptr(h), L.ptr(z), 1, HW,
           L.ptr(_coin_dev(theta)), gamma, hc, L.ptr(bad), k, L.stream())
    if theta:
        weight = (gamma / p) * problem.alpha  # prox_g(z, gamma/p) -> tv_prox(z, step*alpha)
        rep = int(st.last_weight is not None and st.last_weight != weight)
        from .tv import INNER_STEP
        betas = fused.setdefault("betas", _betas(st.inner_iters))
        for it in range(st.inner_iters):
            bprev = betas[it - 1] if (st.accelerated and it > 0) else 0.0
            L.call("psb_fgp2d_iter", dtf, L.ptr(z), HW, L.ptr(st.slots), 6 * HW, None, 1, weight,
                   None, rep, None, H, W, it, bprev, INNER_STEP, int(st.nonneg), L.stream())
        L.call("psb_proxskip_post", dto, dtf, L.ptr(x), L.ptr(b), 1, L.ptr(h), L.ptr(z),
               L.ptr(st.slots), 6 * HW, None, 1, H, W, st.inner_iters, int(st.nonneg), gamma, pg,
               L.ptr(bad), k, L.stream())
        st.last_weight = weight
        st.total_inner_iterations += st.inner_iters
    return x, h


def _betas(n):
    out, t = [], 1.0
    for _ in range(n):
        t1 = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
        out.append((t - 1.0) / t1)
        t = t1
    return out


def _tv_snapshot(st, *tensors):
    return ([t.clone() if t is not None else None for t in tensors], st.slots.clone() if st else None,
            st.last_weight if st else None, st.total_inner_iterations if st else 0)


def _tv_restore(snap, st, *tensors):
    saved, slots, lw, tot = snap
    for t, v in zip(tensors, saved):
        if t is not None:
            t.copy_(v)
    if st is not None:
        st.slots.copy_(slots)
        st.last_weight = lw
        st.total_inner_iterations = tot


def _drive(log, iters, coins, shape, dtype, chunk, state, tensors, base_inner, inner_per_prox):
    """Passive log: one native call for the whole run.  Device-loggable log:
    chunked native calls with an iterate history (devlog.run_logged)."""
    if log.passive:
        el = chunk(0, coins, None)
        _finish_passive(log, coins[:iters], el, base_inner, inner_per_prox)
        return
    run_logged(log, iters, coins, shape, dtype, chunk, lambda: _tv_snapshot(state, *tensors),
               lambda sn: _tv_restore(sn, state, *tensors), inner_per_prox, base_inner)


def _proxskip_tv_fused(problem, fused, x0, h0, gamma, skip, iters, log, use_graph,
                       fgp_time=None, algo="proxskip"):
    """Whole run inside the native driver (psb_proxskip_denoise_run /
    psb_proxskip_deblur_run): no host round trip per iteration.  algo="fista"
    runs FISTA (solvers.py:148-168) in the same driver (every coin set)."""
    log.start(AR.is_host(x0))
    st = problem.tv_state
    H, W = st.shape
    dt = problem.outer_dtype
    x = AR.to_dev(x0, dt).clone()
    h = AR.to_dev(h0, dt).clone() if h0 is not None else torch.zeros_like(x)
    z = torch.empty((H, W), dtype=st.dtype, device="cuda")
    coins = skip.coins(iters)
    bad = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
    if use_graph is None:
        use_graph = H * W <= 1024 * 1024
    aux = None
    if algo == "fista":  # x_prev (= x0) and xbar buffers
        aux = torch.empty((2,) + tuple(x.shape), dtype=dt, device="cuda")
        aux[0].copy_(x)
    base_inner = st.total_inner_iterations
    vp = L.C.c_void_p
    if fused["kind"] == "deblur":
        ker = fused["kernel"]
        sep = bool(fused["separable"] and ker.factor is not None)
        w2 = np.ascontiguousarray(ker.weights, dtype=np.float64)
        w1 = np.ascontiguousarray(ker.factor if sep else np.zeros(1), dtype=np.float64)
        g = torch.empty_like(x)
        scratch = None if sep else torch.empty_like(x)

    def chunk(k0, cc, hist):
        cc = np.ascontiguousarray(cc, dtype=np.uint8)
        K = len(cc)
        lw = np.array([np.nan if st.last_weight is None else st.last_weight], dtype=np.float64)
        pc = np.zeros(1, dtype=np.int64)
        el = np.zeros(max(K, 1), dtype=np.float64)
        bad.fill_(INT32_MAX)
        ft = fgp_time.ctypes.data_as(vp) if (fgp_time is not None and hist is None) else None
        tail = (cc.ctypes.data_as(vp), K, float(gamma), float(skip.p), float(problem.alpha),
                st.inner_iters, int(bool(st.accelerated)), int(bool(st.nonneg)),
                lw.ctypes.data_as(vp), pc.ctypes.data_as(vp), L.ptr(bad), int(bool(use_graph)),
                el.ctypes.data_as(vp), ft, L.ptr(hist), 1 if algo == "fista" else 0, L.ptr(aux),
                L.stream())
        if fused["kind"] == "denoise":
            L.call("psb_proxskip_denoise_run", L.dcode(dt), L.dcode(st.dtype), L.ptr(x),
                   L.ptr(fused["b_dev"]), L.ptr(h), L.ptr(z), L.ptr(st.slots), 1, H, W, *tail)
        else:
            L.call("psb_proxskip_deblur_run", L.dcode(dt), L.dcode(st.dtype), L.ptr(x),
                   L.ptr(fused["b_dev"]), L.ptr(h), L.ptr(z), L.ptr(st.slots), L.ptr(g),
                   L.ptr(scratch), H, W, w2.ctypes.data_as(vp), w1.ctypes.data_as(vp), ker.size,
                   int(sep), *tail)
        k_bad = int(bad.item())
        if k_bad != INT32_MAX:
            raise DivergenceError(k0 + k_bad, algo)
        st.last_weight = None if np.isnan(lw[0]) else float(lw[0])
        st.total_inner_iterations += st.inner_iters * int(pc[0])
        return el

    _drive(log, iters, coins, (H, W), dt, chunk, st, (x, h), base_inner, st.inner_iters)
    return AR.like(x, x0), log


def bernoulli_op(x, p, draw):
    """x/p on a success draw, zeros otherwise (skip.py:38-43)."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"bernoulli_op: p must be in (0, 1], got {p}")
    t = AR.to_dev(x, torch.float64)
    return AR.like(T.lincomb(1.0 / p, t) if draw else torch.zeros_like(t), x)


def run_pdhgskip1(problem, x0, y0, sigma, tau, omega, skip, iters, log=None):
    """PDHGSkip-1 (skip.py:82-114): on a success draw xhat = (prox(x - s K^T y) - x)/p,
    else 0 (prox and K^T skipped); x <- x + xhat/(1 + omega);
    y <- prox_{tau f*}(y + tau K(x + xhat))."""
    if sigma <= 0 or tau <= 0:
        raise ValueError("run_pdhgskip1: steps must be positive")
    if omega < 0:
        raise ValueError("run_pdhgskip1: omega must be nonnegative")
    log = _ensure_log(log)
    fused = getattr(problem, "_fused", None)
    if (fused is not None and fused["kind"] == "ct_explicit" and np.isscalar(sigma)
            and np.isscalar(tau) and (log.passive or device_loggable(log))):
        # native driver: psb_pdhg_run variant 2 (K^T and the prox on success draws only)
        return _pdhg_family_fused(problem, x0, y0, None, sigma, tau, skip, iters, log,
                                  "pdhgskip1", omega=omega)
    log.start(AR.is_host(x0))
    p = skip.p
    coins = skip.coins(iters)
    K = problem.K
    x = AR.to_dev(x0, torch.float64).clone()
    y = AR.to_dev(y0, torch.float64).clone()
    prox_count = 0
    for k in range(iters):
        theta = bool(coins[k])
        if theta:
            px = _dev(problem.prox_g(T.lincomb(1.0, x, -sigma, apply_adjoint(K, y)), sigma), x)
            xhat = T.lincomb(1.0 / p, T.lincomb(1.0, px, -1.0, x))
            prox_count += 1
        else:
            xhat = torch.zeros_like(x)
        x_new = T.lincomb(1.0, x, 1.0 / (1.0 + omega), xhat)
        y = _dev(problem.prox_fstar(T.lincomb(1.0, y, tau, apply_forward(K, T.lincomb(1.0, x_new, 1.0, xhat))), tau), y)
        x = x_new
        _check_finite(x, k, "pdhgskip1")
        if log.observe(k + 1, x, prox_count, theta):
            break
    return AR.like(x, x0), log


# -- PDHGSkip-2 (skip.py:117-150) ----------------------------------------------

def run_pdhgskip2(problem, x0, y0, h0, sigma, tau, skip, iters, log=None):
    """PDHG with a ProxSkip control variate on the primal prox (Alg. 6)."""
    _check_step_rule(sigma, tau, problem.norm_K_sq)
    fused = getattr(problem, "_fused", None)
    if fused is not None and np.isscalar(sigma) and np.isscalar(tau):
        if fused["kind"] == "ct_implicit":
            if log is None or log.passive or device_loggable(log):
                return _ct_implicit_fused(problem, x0, y0, h0, sigma, tau, skip, iters, log,
                                          "pdhgskip2")
        else:
            return _pdhg_family_fused(problem, x0, y0, h0, sigma, tau, skip, iters, log,
                                      "pdhgskip2")
    log = _ensure_log(log)
    log.start(AR.is_host(x0))
    p = skip.p
    coins = skip.coins(iters)
    K = problem.K
    x = AR.to_dev(x0, torch.float64).clone()
    y = AR.to_dev(y0, torch.float64).clone()
    h = AR.to_dev(h0, torch.float64).clone() if h0 is not None else torch.zeros_like(x)
    hc = sigma - sigma / p
    ps = p / sigma
    prox_count = 0
    for k in range(iters):
        kty = apply_adjoint(K, y)
        theta = bool(coins[k])
        t = T.lincomb(1.0, x, -sigma, kty)
        xhat = T.lincomb(1.0, t, sigma, h)
        if theta:
            xn = _dev(problem.prox_g(T.lincomb(1.0, t, hc, h), sigma / p), x)
            prox_count += 1
        else:
            xn = xhat
        xbar = T.lincomb(2.0, xn, -1.0, x)
        y = _dev(problem.prox_fstar(T.lincomb(1.0, y, tau, apply_forward(K, xbar)), tau), y)
        h = T.lincomb(1.0, h, ps, T.lincomb(1.0, xn, -1.0, xhat))
        x = xn
        _check_finite(x, k, "pdhgskip2")
        if log.observe(k + 1, x, prox_count, theta):
            break
    return AR.like(x, x0), log


def _ct_implicit_fused(problem, x0, y0, h0, sigma, tau, skip, iters, log, algo, use_graph=True):
    """Whole PDHGSkip-2 / PDHG run on the implicit CT saddle problem inside the
    native driver (psb_ct_implicit_run): Radon gather + outer update, FGP prox
    on coin iterations, forward projection + fidelity dual prox -- no host
    round trip per iteration.  Passive and device-loggable logs (devlog.py);
    other observing logs step through the generic driver with the same kernels."""
    f = problem._fused
    st = f["tv_state"]
    dt = f["dtype"]
    log = _ensure_log(log)
    log.start(AR.is_host(x0))
    g, _ = f["geom"].device()
    n = g.n
    x = AR.to_dev(x0, dt).clone()
    y = AR.to_dev(y0, dt).clone().reshape(-1)
    h = AR.to_dev(h0, dt).clone() if h0 is not None else torch.zeros_like(x)
    xbar = torch.empty_like(x)
    z = torch.empty((n, n), dtype=st.dtype, device="cuda")
    p = skip.p if skip is not None else 1.0
    coins = skip.coins(iters) if skip is not None else np.ones(iters, dtype=np.uint8)
    bad = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
    base_inner = st.total_inner_iterations
    vp = L.C.c_void_p

    def chunk(k0, cc, hist):
        cc = np.ascontiguousarray(cc, dtype=np.uint8)
        K = len(cc)
        lw = np.array([np.nan if st.last_weight is None else st.last_weight], dtype=np.float64)
        pc = np.zeros(1, dtype=np.int64)
        el = np.zeros(max(K, 1), dtype=np.float64)
        bad.fill_(INT32_MAX)
        L.call("psb_ct_implicit_run", L.dcode(dt), L.dcode(st.dtype), L.C.byref(g), L.ptr(x),
               L.ptr(y), L.ptr(h), L.ptr(xbar), L.ptr(z), L.ptr(st.slots), L.ptr(f["b_dev"]),
               cc.ctypes.data_as(vp), K, float(sigma), float(tau), float(p), float(f["alpha"]),
               st.inner_iters, int(bool(st.accelerated)), int(bool(st.nonneg)),
               lw.ctypes.data_as(vp), pc.ctypes.data_as(vp), L.ptr(bad), int(bool(use_graph)),
               el.ctypes.data_as(vp), L.ptr(hist), L.stream())
        k_bad = int(bad.item())
        if k_bad != INT32_MAX:
            raise DivergenceError(k0 + k_bad, algo)
        st.last_weight = None if np.isnan(lw[0]) else float(lw[0])
        st.total_inner_iterations += st.inner_iters * int(pc[0])
        return el

    _drive(log, iters, coins, (n, n), dt, chunk, st, (x, y, h), base_inner, st.inner_iters)
    log.y_final = y
    return AR.like(x, x0), log


def _pdhg_family_fused(problem, x0, y0, h0, sigma, tau, skip, iters, log, algo, use_graph=True,
                       omega=0.0):
    """PDHG (skip is None) / PDHGSkip-2 on K = [A; D] with the fused kernels of
    csrc/radon.cu.  Passive logs run the whole loop natively (psb_pdhg_run);
    observing logs step it from here with the same kernels."""
    f = problem._fused
    dt = f["dtype"]
    log = _ensure_log(log)
    log.start(AR.is_host(x0))
    g, _ = f["geom"].device()
    x = AR.to_dev(x0, dt).clone()
    y = AR.to_dev(y0, dt).clone().reshape(-1)
    is_skip = skip is not None
    variant = 0 if not is_skip else (2 if algo == "pdhgskip1" else 1)
    h = None
    if variant == 1:
        h = AR.to_dev(h0, dt).clone() if h0 is not None else torch.zeros_like(x)
    xbar = torch.empty_like(x)
    bad = torch.full((1,), INT32_MAX, dtype=torch.int32, device="cuda")
    p = skip.p if is_skip else 1.0
    coins = skip.coins(iters) if is_skip else np.ones(iters, dtype=np.uint8)
    # diagonal (preconditioned) steps of run_pdhg_preconditioned: device arrays
    sig_a = None if np.isscalar(sigma) else AR.to_dev(sigma, dt).reshape(-1)
    tau_a = None if np.isscalar(tau) else AR.to_dev(tau, dt).reshape(-1)
    sig_s = float(sigma) if sig_a is None else 0.0
    tau_s = float(tau) if tau_a is None else 0.0
    if log.passive or device_loggable(log):
        def chunk(k0, cc, hist):
            cc = np.ascontiguousarray(cc, dtype=np.uint8)
            K = len(cc)
            el = np.zeros(max(K, 1))
            bad.fill_(INT32_MAX)
            L.call("psb_pdhg_run", L.dcode(dt), L.C.byref(g), L.ptr(x), L.ptr(y), L.ptr(h),
                   L.ptr(xbar), L.ptr(f["b_dev"]), cc.ctypes.data_as(L.C.c_void_p), K,
                   sig_s, tau_s, L.ptr(sig_a), L.ptr(tau_a), float(p), float(f["alpha"]),
                   int(bool(f["nonneg"])), variant, float(omega), L.ptr(bad), int(bool(use_graph)),
                   el.ctypes.data_as(L.C.c_void_p),
                   L.ptr(hist), L.stream())
            k_bad = int(bad.item())
            if k_bad != INT32_MAX:
                raise DivergenceError(k0 + k_bad, algo)
            return el

        _drive(log, iters, coins, tuple(x.shape), dt, chunk, None, (x, y, h), 0, 0)
    else:
        hc = sigma - sigma / p if is_skip else 0.0
        ps = p / sigma if is_skip else 0.0
        n_prox = 0
        for k in range(iters):
            th = int(coins[k])
            L.call("psb_pdhg_step", L.dcode(dt), L.C.byref(g), L.ptr(x), L.ptr(y), L.ptr(h),
                   L.ptr(xbar), L.ptr(f["b_dev"]), L.ptr(bad), k, th, float(sigma), float(tau),
                   float(hc), float(ps), float(f["alpha"]), int(bool(f["nonneg"])), L.stream())
            n_prox += th
            if int(bad.item()) != INT32_MAX:
                raise DivergenceError(k, algo)
            if log.observe(k + 1, x, n_prox, bool(th)):
                break
    log.y_final = y
    return AR.like(x, x0), log
