"""Float64 numpy restatement of the reference ``imgskip`` hot path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): used by tests as the
parity checker and by ``bench.py`` as the timed CPU baseline.  It restates the
published algorithm of the reference package; each function cites the
reference ``file:line`` (relative to ``/root/reference/pkg/src/imgskip``).

Elementwise arithmetic follows the reference's operation order exactly (numpy
rounds every binary op separately), so the oracle is bit-identical to the
reference on every golden vector (``tests/test_oracle_golden.py``); the device
double-precision debug path is bit-identical to this oracle in turn.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.sparse as sp

# tv.py:16 -- 1/L for the 2-D dual problem, ||D||^2 <= 8.
STEP_2D = 0.125
# problems.py:18 -- analytic ||D||^2 bound used for the explicit splitting.
GRAD_BOUND = 8.0


# ---------------------------------------------------------------------------
# finite differences (operators.py:44-71)
# ---------------------------------------------------------------------------

def fd_grad(u):
    """Neumann forward differences, channel 0 = rows (operators.py:44-57)."""
    u = np.asarray(u, dtype=np.float64)
    if u.ndim != 2 or min(u.shape) < 2:
        raise ValueError(f"fd_grad: need a 2-D grid with sides >= 2, got {u.shape}")
    out = np.zeros((2,) + u.shape)
    np.subtract(u[1:, :], u[:-1, :], out=out[0, :-1, :])
    np.subtract(u[:, 1:], u[:, :-1], out=out[1, :, :-1])
    return out


def fd_div(q):
    """Divergence = -D^T; four masked accumulations in the reference order
    (operators.py:60-71): +qy (rows < H-1), -qy shifted, +qx (cols < W-1),
    -qx shifted."""
    q = np.asarray(q, dtype=np.float64)
    if q.ndim != 3 or q.shape[0] != 2 or min(q.shape[1:]) < 2:
        raise ValueError(f"fd_div: expected (2, H, W) with H, W >= 2, got {q.shape}")
    d = np.zeros(q.shape[1:])
    d[:-1, :] += q[0, :-1, :]
    d[1:, :] -= q[0, :-1, :]
    d[:, :-1] += q[1, :, :-1]
    d[:, 1:] -= q[1, :, :-1]
    return d


# ---------------------------------------------------------------------------
# pointwise proxes (proximal.py:10-41)
# ---------------------------------------------------------------------------

def ball_project(q, radius):
    """radius * q / max(radius, |q|) per pixel (proximal.py:10-21)."""
    if radius <= 0:
        raise ValueError(f"ball_project: radius must be positive, got {radius}")
    q = np.asarray(q, dtype=np.float64)
    norm = np.sqrt(q[0] ** 2 + q[1] ** 2)
    return q * (radius / np.maximum(radius, norm))


def clamp_nonneg(u):
    """max(u, 0) (proximal.py:39-41)."""
    return np.maximum(np.asarray(u, dtype=np.float64), 0.0)


# ---------------------------------------------------------------------------
# TV and its inexact prox (tv.py:19-105)
# ---------------------------------------------------------------------------

def tv_total(u):
    """Isotropic TV, sum of |grad u| (tv.py:19-22)."""
    g = fd_grad(u)
    return float(np.sqrt(g[0] ** 2 + g[1] ** 2).sum())


@dataclass
class FgpState:
    """Warm start + accounting of the inexact prox (tv.py:25-50)."""

    q: np.ndarray
    n_inner: int
    accelerated: bool = True
    nonneg: bool = False
    inner_total: int = 0
    prev_weight: Optional[float] = None

    @staticmethod
    def zeros(shape, n_inner, accelerated=True, nonneg=False):
        if n_inner < 1:
            raise ValueError("FgpState: n_inner must be >= 1")
        return FgpState(np.zeros((2,) + tuple(shape)), n_inner, accelerated, nonneg)


def fista_betas(n):
    """Momentum weights beta_k = (t_k - 1)/t_{k+1}, t_0 = 1 (tv.py:72-80).
    Index k is the coefficient applied after inner iteration k+1."""
    out = []
    t = 1.0
    for _ in range(n):
        t1 = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        out.append((t - 1.0) / t1)
        t = t1
    return out


def fgp_prox(x, weight, st: FgpState):
    """FGP / accelerated dual projected gradient for prox_{weight TV}
    (tv.py:53-89).  Mutates ``st`` exactly like the reference."""
    if weight <= 0:
        raise ValueError(f"fgp_prox: weight must be positive, got {weight}")
    x = np.asarray(x, dtype=np.float64)
    cl = clamp_nonneg if st.nonneg else (lambda v: v)
    q0 = st.q
    if st.prev_weight is not None and st.prev_weight != weight:   # tv.py:68-69
        q0 = ball_project(q0, weight)
    if st.accelerated:
        y = q0
        q_old = q0
        for beta in fista_betas(st.n_inner):
            q_new = ball_project(y + STEP_2D * fd_grad(cl(x + fd_div(y))), weight)
            y = q_new + beta * (q_new - q_old)
            q_old = q_new
        q_fin = q_new
    else:                                                           # tv.py:82-84
        q_fin = q0
        for _ in range(st.n_inner):
            q_fin = ball_project(q_fin + STEP_2D * fd_grad(cl(x + fd_div(q_fin))), weight)
    st.q = q_fin
    st.prev_weight = weight
    st.inner_total += st.n_inner
    return cl(x + fd_div(q_fin))


def rof_gap(x, q, weight):
    """ROF prox duality gap at u = x + div q (tv.py:92-105)."""
    q = np.asarray(q, dtype=np.float64)
    if np.any(np.sqrt(q[0] ** 2 + q[1] ** 2) > weight * (1.0 + 1e-10)):
        raise ValueError("rof_gap: q is infeasible")
    dq = fd_div(q)
    u = x + dq
    p = 0.5 * l2(u - x) ** 2 + weight * tv_total(u)
    d = -0.5 * l2(dq + x) ** 2 + 0.5 * l2(x) ** 2
    return p - d


# ---------------------------------------------------------------------------
# vector helpers (tensor.py:17-51)
# ---------------------------------------------------------------------------

def inner(a, b):
    return float(np.dot(np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()))


def l2(a):
    return float(np.linalg.norm(np.asarray(a, np.float64).ravel()))


def relerr(x, ref):
    den = l2(ref)
    if den == 0.0:
        raise ZeroDivisionError("relerr: zero reference")
    return l2(np.asarray(x, np.float64) - ref) / den


# ---------------------------------------------------------------------------
# linear maps (operators.py:18-39, 109-390)
# ---------------------------------------------------------------------------

@dataclass
class Op:
    """forward/adjoint pair + cached ||A||^2 (operators.py:18-39)."""

    dom: tuple
    ran: tuple
    fwd: Callable
    adj: Callable
    nsq: Optional[float] = None

    def norm_sq(self, iters=100, seed=0):
        if self.nsq is None:
            self.nsq = power_iteration(self, iters, seed)
        return self.nsq


def power_iteration(op: Op, iters=100, seed=0):
    """Rayleigh quotient of A^T A after ``iters`` normalised power steps from a
    default_rng(seed) normal start (operators.py:368-390)."""
    if iters < 1:
        raise ValueError("power_iteration: iters must be >= 1")
    v = np.random.default_rng(seed).standard_normal(op.dom)
    est = 0.0
    for _ in range(iters):
        av = op.fwd(v)
        if l2(av) == 0.0:
            return 0.0
        w = op.adj(av)
        est = inner(v, w) / inner(v, v)
        nw = l2(w)
        if nw == 0.0:
            return 0.0
        v = w / nw
    return float(est)


def identity_op(shape):
    """operators.py:297-307 (norm fixed at 1)."""
    f = lambda v: np.array(v, dtype=np.float64)
    return Op(tuple(shape), tuple(shape), f, f, 1.0)


def grad_op(shape, nsq=None):
    """operators.py:74-104 (signed part only)."""
    return Op(tuple(shape), (2,) + tuple(shape), fd_grad, lambda q: -fd_div(q), nsq)


def gauss_taps(size, sigma):
    """Normalised truncated 2-D Gaussian (operators.py:131-137)."""
    if size % 2 == 0 or size < 1:
        raise ValueError(f"gauss_taps: size must be odd, got {size}")
    r = np.arange(size) - size // 2
    g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / (2.0 * sigma ** 2))
    return g / g.sum()


def conv_periodic(u, taps):
    """Circular convolution, 81 shifted accumulations in the reference's
    (a outer, b inner) order (operators.py:149-158)."""
    u = np.asarray(u, dtype=np.float64)
    k = taps.shape[0]
    c = k // 2
    acc = np.zeros_like(u)
    for a in range(k):
        for b in range(k):
            if taps[a, b] != 0.0:
                acc += taps[a, b] * np.roll(u, (a - c, b - c), axis=(0, 1))
    return acc


def corr_periodic(r, taps):
    """Adjoint of conv_periodic (operators.py:161-172)."""
    r = np.asarray(r, dtype=np.float64)
    k = taps.shape[0]
    c = k // 2
    acc = np.zeros_like(r)
    for a in range(k):
        for b in range(k):
            if taps[a, b] != 0.0:
                acc += taps[a, b] * np.roll(r, (c - a, c - b), axis=(0, 1))
    return acc


def blur_op(taps, shape):
    return Op(tuple(shape), tuple(shape), lambda u: conv_periodic(u, taps),
              lambda r: corr_periodic(r, taps))


def default_angles(n_angles):
    """Uniform over [0, pi) (operators.py:209-211)."""
    return np.arange(n_angles) * (np.pi / n_angles)


def ray_lattice(n, n_bins, bin_spacing=1.0):
    """Sample lattice of the ray-driven projector (operators.py:224-229):
    (center, step positions, bin offsets)."""
    center = (n - 1) / 2.0
    half = n / np.sqrt(2.0)
    n_steps = int(np.ceil(2.0 * half)) + 1
    steps = np.linspace(-half, half, n_steps)
    offsets = (np.arange(n_bins) - (n_bins - 1) / 2.0) * bin_spacing
    return center, steps, offsets


def radon_matrix(n, angles, n_bins, bin_spacing=1.0):
    """Ray-driven bilinear system matrix, duplicates summed by COO->CSR
    (operators.py:218-263)."""
    center, steps, offsets = ray_lattice(n, n_bins, bin_spacing)
    rr, cc, vv = [], [], []
    for ia, th in enumerate(np.asarray(angles, np.float64)):
        c, s = np.cos(th), np.sin(th)
        px = offsets[:, None] * c + steps[None, :] * (-s) + center
        py = offsets[:, None] * s + steps[None, :] * c + center
        ix = np.floor(px).astype(np.int64)
        iy = np.floor(py).astype(np.int64)
        fx = px - ix
        fy = py - iy
        ray = ia * n_bins + np.broadcast_to(np.arange(n_bins)[:, None], px.shape)
        for oy, ox, w in ((0, 0, (1 - fy) * (1 - fx)), (0, 1, (1 - fy) * fx),
                          (1, 0, fy * (1 - fx)), (1, 1, fy * fx)):
            yy, xx = iy + oy, ix + ox
            ok = (yy >= 0) & (yy < n) & (xx >= 0) & (xx < n) & (w > 0)
            rr.append(ray[ok])
            cc.append(yy[ok] * n + xx[ok])
            vv.append(w[ok])
    m = sp.coo_matrix((np.concatenate(vv), (np.concatenate(rr), np.concatenate(cc))),
                      shape=(len(angles) * n_bins, n * n))
    return m.tocsr()


def radon_op(n, n_angles, n_bins, bin_spacing=1.0, angles=None):
    """operators.py:266-292."""
    ang = default_angles(n_angles) if angles is None else np.asarray(angles, np.float64)
    m = radon_matrix(n, ang, n_bins, bin_spacing)
    mt = m.T.tocsr()
    rs = (len(ang), n_bins)
    return Op((n, n), rs, lambda u: (m @ np.asarray(u, np.float64).ravel()).reshape(rs),
              lambda y: (mt @ np.asarray(y, np.float64).ravel()).reshape(n, n))


def stack_ops(a: Op, d: Op):
    """K = [a; d] with a flat range (operators.py:323-365)."""
    na = int(np.prod(a.ran))
    nd = int(np.prod(d.ran))

    def fwd(x):
        return np.concatenate([a.fwd(x).ravel(), d.fwd(x).ravel()])

    def adj(y):
        y = np.asarray(y, np.float64)
        return a.adj(y[:na].reshape(a.ran)) + d.adj(y[na:].reshape(d.ran))

    return Op(a.dom, (na + nd,), fwd, adj)


# ---------------------------------------------------------------------------
# problems (problems.py:101-192)
# ---------------------------------------------------------------------------

@dataclass
class Recon:
    """1/2||Au-b||^2 + alpha TV(u) in one of the two splittings."""

    A: Op
    b: np.ndarray
    alpha: float
    nonneg: bool
    splitting: str
    grad: Optional[Callable] = None          # implicit: A^T(Au - b)
    prox: Optional[Callable] = None          # implicit: prox_{step g}
    L: Optional[float] = None
    tv: Optional[FgpState] = None
    K: Optional[Op] = None                   # explicit / saddle
    prox_fstar: Optional[Callable] = None
    prox_g: Optional[Callable] = None
    K_nsq: Optional[float] = None


def make_recon(A: Op, b, alpha, nonneg=False, splitting="implicit", inner=100,
               accelerated=True, K_nsq=None):
    """build_tv_recon (problems.py:101-159).  ``K_nsq`` (test convenience)
    seeds the cached ||K||^2 of the explicit splitting instead of running the
    power method, exactly like setting LinearMap.norm_sq_estimate."""
    if alpha <= 0:
        raise ValueError("make_recon: alpha must be positive")
    b = np.asarray(b, np.float64)
    pr = Recon(A, b, alpha, nonneg, splitting)
    if splitting == "implicit":
        st = FgpState.zeros(A.dom, inner, accelerated, nonneg)
        pr.tv = st
        pr.grad = lambda u: A.adj(A.fwd(u) - b)
        pr.L = A.norm_sq()
        pr.prox = lambda u, step: fgp_prox(u, step * alpha, st)
    elif splitting == "explicit":
        D = grad_op(A.dom, GRAD_BOUND)
        K = stack_ops(A, D)
        nf = int(np.prod(A.ran))

        def pfs(y, step):                                          # problems.py:139-146
            yf = y[:nf].reshape(A.ran)
            sf = step[:nf].reshape(A.ran) if isinstance(step, np.ndarray) else step
            fid = (yf - sf * b) / (1.0 + sf)
            tvb = ball_project(y[nf:].reshape(D.ran), alpha)
            return np.concatenate([fid.ravel(), tvb.ravel()])

        pr.K = K
        pr.prox_fstar = pfs
        pr.prox_g = (lambda u, s: clamp_nonneg(u)) if nonneg else (
            lambda u, s: np.array(u, dtype=np.float64))
        if K_nsq is not None:
            K.nsq = K_nsq
        pr.K_nsq = K.norm_sq()
    else:
        raise ValueError(f"make_recon: unknown splitting {splitting!r}")
    return pr


def make_saddle_implicit(A: Op, b, alpha, nonneg=False, inner=100, accelerated=True):
    """build_tv_saddle_implicit (problems.py:162-184)."""
    b = np.asarray(b, np.float64)
    pr = Recon(A, b, alpha, nonneg, "implicit")
    st = FgpState.zeros(A.dom, inner, accelerated, nonneg)
    pr.tv = st
    pr.K = A
    pr.prox_fstar = lambda y, s: (y - s * b) / (1.0 + s)
    pr.prox_g = lambda u, s: fgp_prox(u, s * alpha, st)
    pr.K_nsq = A.norm_sq()
    return pr


def tv_objective(u, pr: Recon, guarded=True):
    """objective_tv (problems.py:187-192); ``guarded=False`` drops the +inf
    nonnegativity guard."""
    u = np.asarray(u, np.float64)
    if guarded and pr.nonneg and float(u.min()) < -1e-12:
        return np.inf
    return 0.5 * l2(pr.A.fwd(u) - pr.b) ** 2 + pr.alpha * tv_total(u)


# ---------------------------------------------------------------------------
# drivers (solvers.py:116-209, skip.py:16-150)
# ---------------------------------------------------------------------------

def coin_draws(p, seed, n):
    """The per-run Bernoulli stream: Philox(seed).random() < p, one draw per
    iteration (skip.py:27-28, 67, 136)."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"coin_draws: p must be in (0, 1], got {p}")
    return np.random.Generator(np.random.Philox(seed)).random(n) < p


class DivergedAt(RuntimeError):
    """Mirror of errors.DivergenceError (errors.py:4-11)."""

    def __init__(self, k, algo):
        self.iteration, self.algorithm = k, algo
        super().__init__(f"{algo} diverged: non-finite iterate at iteration {k}")


def _finite_or_raise(x, k, algo):                                  # solvers.py:111-113
    if not np.all(np.isfinite(x)):
        raise DivergedAt(k, algo)


def proxskip(grad, prox, x0, h0, gamma, p, seed, iters, observe=None):
    """ProxSkip (skip.py:46-79).  ``observe(k, x, n_prox, theta)`` is called
    after every iteration; returns (x, h, n_prox, thetas)."""
    if gamma <= 0:
        raise ValueError("proxskip: gamma must be positive")
    coins = coin_draws(p, seed, iters)
    x = np.array(x0, dtype=np.float64)
    h = np.zeros_like(x) if h0 is None else np.array(h0, dtype=np.float64)
    hc = gamma - gamma / p
    n_prox = 0
    for k in range(iters):
        g = grad(x)
        xhat = x - gamma * g + gamma * h
        if coins[k]:
            xn = prox((x - gamma * g) + hc * h, gamma / p)
            n_prox += 1
        else:
            xn = xhat
        h = h + (p / gamma) * (xn - xhat)
        x = xn
        _finite_or_raise(x, k, "proxskip")
        if observe is not None:
            observe(k, x, n_prox, bool(coins[k]))
    return x, h, n_prox, coins


def pgd(grad, prox, x0, gamma, iters, observe=None):
    """ISTA (solvers.py:131-145)."""
    x = np.array(x0, dtype=np.float64)
    for k in range(iters):
        x = prox(x - gamma * grad(x), gamma)
        _finite_or_raise(x, k, "pgd")
        if observe is not None:
            observe(k, x, k + 1, True)
    return x


def fista(grad, prox, x0, gamma, iters, observe=None):
    """FISTA, Beck-Teboulle t-sequence (solvers.py:148-168)."""
    x = np.array(x0, dtype=np.float64)
    xp = x
    t = 1.0
    for k in range(iters):
        t1 = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        xb = x + ((t - 1.0) / t1) * (x - xp)
        xp = x
        x = prox(xb - gamma * grad(xb), gamma)
        t = t1
        _finite_or_raise(x, k, "fista")
        if observe is not None:
            observe(k, x, k + 1, True)
    return x


def check_steps(sigma, tau, nsq):                                  # solvers.py:177-184
    if sigma <= 0 or tau <= 0:
        raise ValueError("pdhg: steps must be positive")
    if sigma * tau * nsq > 1.0 + 1e-10:
        raise ValueError(f"pdhg: step rule violated, {sigma * tau * nsq}")


def pdhg(K: Op, prox_fstar, prox_g, nsq, x0, y0, sigma, tau, iters, observe=None):
    """PDHG with theta = 1 (solvers.py:187-209)."""
    check_steps(sigma, tau, nsq)
    x = np.array(x0, dtype=np.float64)
    y = np.array(y0, dtype=np.float64)
    for k in range(iters):
        xn = prox_g(x - sigma * K.adj(y), sigma)
        xb = 2.0 * xn - x
        y = prox_fstar(y + tau * K.fwd(xb), tau)
        x = xn
        _finite_or_raise(x, k, "pdhg")
        if observe is not None:
            observe(k, x, k + 1, True)
    return x, y


def pdhgskip2(K: Op, prox_fstar, prox_g, nsq, x0, y0, h0, sigma, tau, p, seed, iters,
              observe=None):
    """PDHGSkip-2 (skip.py:117-150); returns (x, y, h, n_prox, coins)."""
    check_steps(sigma, tau, nsq)
    coins = coin_draws(p, seed, iters)
    x = np.array(x0, dtype=np.float64)
    y = np.array(y0, dtype=np.float64)
    h = np.zeros_like(x) if h0 is None else np.array(h0, dtype=np.float64)
    hc = sigma - sigma / p
    n_prox = 0
    for k in range(iters):
        kty = K.adj(y)
        xhat = x - sigma * kty + sigma * h
        if coins[k]:
            xn = prox_g((x - sigma * kty) + hc * h, sigma / p)
            n_prox += 1
        else:
            xn = xhat
        xb = 2.0 * xn - x
        y = prox_fstar(y + tau * K.fwd(xb), tau)
        h = h + (p / sigma) * (xn - xhat)
        x = xn
        _finite_or_raise(x, k, "pdhgskip2")
        if observe is not None:
            observe(k, x, n_prox, bool(coins[k]))
    return x, y, h, n_prox, coins


# ---------------------------------------------------------------------------
# batched denoising (BASELINE config 4): a per-problem loop over the above
# ---------------------------------------------------------------------------

def proxskip_denoise(b, alpha, p, seed, iters, inner, x0=None):
    """One config-1/config-4 problem: identity fidelity, implicit TV prox,
    gamma = 1/||I||^2 = 1 (problems.py:117-132, skip.py:46-79).
    Returns (x, h, n_prox, inner_total)."""
    pr = make_recon(identity_op(b.shape), b, alpha, splitting="implicit", inner=inner)
    x0 = np.zeros_like(b) if x0 is None else x0
    x, h, n_prox, _ = proxskip(pr.grad, pr.prox, x0, None, 1.0 / pr.L, p, seed, iters)
    return x, h, n_prox, pr.tv.inner_total


__all__ = [n for n in dir() if not n.startswith("_")]
