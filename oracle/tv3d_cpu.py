"""3-D restatement of the reference TV prox.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  The reference is
2-D only (operators.py:51-53 rejects other ranks); this module generalises
operators.py:44-71, proximal.py:10-21 and tv.py:53-89 to a (D, H, W) volume
with three dual channels (z, y, x), Neumann zeros on the last plane of each
axis and the 3-D dual step 1/12 (||grad_3D||^2 <= 12; the reference's 1/8 in
tv.py:16 is the 2-D bound).  It is pinned against the 2-D reference prox on
plane-constant volumes (q_z stays 0, so every plane must equal the 2-D prox
run with the same step) in ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .imgskip_cpu import fista_betas

STEP_3D = 1.0 / 12.0


def fd_grad3(u):
    u = np.asarray(u, dtype=np.float64)
    if u.ndim != 3 or min(u.shape) < 2:
        raise ValueError(f"fd_grad3: need a 3-D grid with sides >= 2, got {u.shape}")
    g = np.zeros((3,) + u.shape)
    np.subtract(u[1:], u[:-1], out=g[0, :-1])
    np.subtract(u[:, 1:], u[:, :-1], out=g[1, :, :-1])
    np.subtract(u[:, :, 1:], u[:, :, :-1], out=g[2, :, :, :-1])
    return g


def fd_div3(q):
    """-D^T in the 2-D reference's accumulation order, z first."""
    q = np.asarray(q, dtype=np.float64)
    d = np.zeros(q.shape[1:])
    d[:-1] += q[0, :-1]
    d[1:] -= q[0, :-1]
    d[:, :-1] += q[1, :, :-1]
    d[:, 1:] -= q[1, :, :-1]
    d[:, :, :-1] += q[2, :, :, :-1]
    d[:, :, 1:] -= q[2, :, :, :-1]
    return d


def ball_project3(q, radius):
    q = np.asarray(q, dtype=np.float64)
    norm = np.sqrt(q[0] ** 2 + q[1] ** 2 + q[2] ** 2)
    return q * (radius / np.maximum(radius, norm))


def tv_total3(u):
    g = fd_grad3(u)
    return float(np.sqrt(g[0] ** 2 + g[1] ** 2 + g[2] ** 2).sum())


@dataclass
class Fgp3State:
    q: np.ndarray
    n_inner: int
    nonneg: bool = False
    inner_total: int = 0
    prev_weight: Optional[float] = None

    @staticmethod
    def zeros(shape, n_inner, nonneg=False):
        if n_inner < 1:
            raise ValueError("Fgp3State: n_inner must be >= 1")
        return Fgp3State(np.zeros((3,) + tuple(shape)), n_inner, nonneg)


def fgp_prox3(x, weight, st: Fgp3State, step=STEP_3D):
    """Accelerated FGP in 3-D; same control flow as tv.py:53-89."""
    if weight <= 0:
        raise ValueError("fgp_prox3: weight must be positive")
    x = np.asarray(x, dtype=np.float64)
    cl = (lambda v: np.maximum(v, 0.0)) if st.nonneg else (lambda v: v)
    q0 = st.q
    if st.prev_weight is not None and st.prev_weight != weight:
        q0 = ball_project3(q0, weight)
    y = q0
    q_old = q0
    for beta in fista_betas(st.n_inner):
        q_new = ball_project3(y + step * fd_grad3(cl(x + fd_div3(y))), weight)
        y = q_new + beta * (q_new - q_old)
        q_old = q_new
    st.q = q_new
    st.prev_weight = weight
    st.inner_total += st.n_inner
    return cl(x + fd_div3(q_new))


def proxskip_denoise3(b, alpha, p, seed, iters, inner, step=STEP_3D):
    """Config-5 outer loop: identity fidelity, gamma = 1 (skip.py:46-79)."""
    from .imgskip_cpu import coin_draws
    coins = coin_draws(p, seed, iters)
    st = Fgp3State.zeros(b.shape, inner)
    x = np.zeros_like(b)
    h = np.zeros_like(b)
    gamma = 1.0
    hc = gamma - gamma / p
    n_prox = 0
    for k in range(iters):
        g = x - b
        xhat = x - gamma * g + gamma * h
        if coins[k]:
            xn = fgp_prox3((x - gamma * g) + hc * h, (gamma / p) * alpha, st, step)
            n_prox += 1
        else:
            xn = xhat
        h = h + (p / gamma) * (xn - xhat)
        x = xn
    return x, h, n_prox, st
