"""Pointwise projections on the device (proximal.py:10-41 of the reference)."""

from __future__ import annotations

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


def prox_zero(x):
    """Identity (proximal.py:68-70)."""
    return AR.like(AR.to_dev(x, _dt(x)).clone(), x)
