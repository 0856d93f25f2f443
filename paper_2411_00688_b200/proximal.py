"""Pointwise projections on the device (proximal.py:10-41 of the reference)."""

from __future__ import annotations

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L


def _dt(a):
    return a.dtype if isinstance(a, torch.Tensor) and a.dtype in (torch.float32, torch.float64) \
        else torch.float64


def project_ball(q, alpha):
    """alpha * q / max(alpha, |q|) per pixel of a (2, H, W) field (proximal.py:10-21)."""
    if alpha <= 0:
        raise ValueError(f"project_ball: alpha must be positive, got {alpha}")
    t = AR.to_dev(q, _dt(q))
    if t.dim() < 2 or t.shape[0] != 2:
        raise ValueError(f"project_ball: expected a (2, ...) field, got {tuple(t.shape)}")
    out = torch.empty_like(t)
    L.call("psb_project_ball2d", L.dcode(t.dtype), L.ptr(t), L.ptr(out), 1, t[0].numel(),
           float(alpha), L.stream())
    return AR.like(out, q)


def project_nonneg(u):
    """Elementwise max(u, 0) (proximal.py:39-41)."""
    t = AR.to_dev(u, _dt(u))
    out = torch.empty_like(t)
    L.call("psb_project_nonneg", L.dcode(t.dtype), L.ptr(t), L.ptr(out), t.numel(), L.stream())
    return AR.like(out, u)


def prox_l2_fidelity(x, b, tau):
    """Prox of z -> 0.5||z - b||^2 at x with step tau: (x + tau b)/(1 + tau);
    tau a scalar or an array of x's shape (diagonal steps) (proximal.py:44-55)."""
    xt = AR.to_dev(x, _dt(x))
    bt = AR.to_dev(b, xt.dtype)
    if tuple(xt.shape) != tuple(bt.shape):
        raise ValueError(f"prox_l2_fidelity: shape mismatch {tuple(xt.shape)} vs {tuple(bt.shape)}")
    out = torch.empty_like(xt)
    if np.isscalar(tau):
        if tau == 0.0:
            return AR.like(xt.clone(), x)
        L.call("psb_prox_l2_fidelity", L.dcode(xt.dtype), L.ptr(xt), float(tau), None, L.ptr(bt),
               L.ptr(out), xt.numel(), L.stream())
    else:
        ta = AR.to_dev(tau, xt.dtype)
        if tuple(ta.shape) != tuple(xt.shape):
            raise ValueError(f"prox_l2_fidelity: tau shape {tuple(ta.shape)} vs {tuple(xt.shape)}")
        L.call("psb_prox_l2_fidelity", L.dcode(xt.dtype), L.ptr(xt), 0.0, L.ptr(ta), L.ptr(bt),
               L.ptr(out), xt.numel(), L.stream())
    return AR.like(out, x)


def prox_zero(x):
    """Identity (proximal.py:68-70)."""
    return AR.like(AR.to_dev(x, _dt(x)).clone(), x)
