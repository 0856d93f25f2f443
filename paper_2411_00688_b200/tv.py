"""Isotropic TV and its warm-started inexact prox on the device (tv.py of the reference).

``tv_prox`` runs ``state.inner_iters`` FGP iterations of the fused sm_100a
stencil kernel (csrc/fgp2d.cu), one launch per inner iteration, with the
Beck-Teboulle momentum table computed in double on the host.  The dual warm
start lives on the device in three rotating slots; ``state.q_warm`` hands back
a float64 numpy copy so reference-style inspection keeps working.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from . import tensor as T
from .operators import div_dev

INNER_STEP = 1.0 / 8.0  # 1/L of the 2-D dual problem, ||D||^2 <= 8 (tv.py:16)

PRECISIONS = {
    # name: (outer-state dtype, FGP dtype)
    "fp32": (torch.float32, torch.float32),
    "mixed": (torch.float64, torch.float32),
    "fp64": (torch.float64, torch.float64),
}


def tv_value(u):
    """sum of |grad u| (tv.py:19-22), fp64 accumulation on the device."""
    t = AR.to_dev(u, u.dtype if isinstance(u, torch.Tensor) else torch.float64)
    if t.dim() != 2 or min(t.shape) < 2:
        raise ValueError(f"tv_value: need a 2-D grid with both sides >= 2, got {tuple(t.shape)}")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L.call("psb_tv2d", L.dcode(t.dtype), L.ptr(t), 1, t.shape[0], t.shape[1], L.ptr(out), L.stream())
    return float(out[0])


@dataclass
class TvProxState:
    """Warm start + accounting of repeated TV prox calls (tv.py:25-50).

    ``slots`` is a (3, 2, H, W) device buffer; slot 0 holds the warm start
    between calls.  ``dtype`` is the FGP arithmetic type (float32 by default;
    float64 reproduces the reference bit for bit).
    """

    slots: torch.Tensor
    inner_iters: int
    accelerated: bool = True
    nonneg: bool = False
    total_inner_iterations: int = 0
    last_weight: Optional[float] = field(default=None)

    @classmethod
    def cold(cls, shape, inner_iters, accelerated=True, nonneg=False, dtype=torch.float32):
        if inner_iters < 1:
            raise ValueError("TvProxState: inner_iters must be >= 1")
        shape = tuple(shape)
        return cls(slots=AR.zeros((3, 2) + shape, dtype), inner_iters=inner_iters,
                   accelerated=accelerated, nonneg=nonneg)

    @property
    def dtype(self):
        return self.slots.dtype

    @property
    def shape(self):
        return tuple(self.slots.shape[2:])

    @property
    def q_warm_device(self):
        return self.slots[0]

    @property
    def q_warm(self):
        return AR.to_host(self.slots[0])

    @q_warm.setter
    def q_warm(self, value):
        self.slots[0].copy_(AR.to_dev(value, self.dtype))


def tv_prox(x, weight, state: TvProxState):
    """Approximate prox_{weight*TV}(x) (+ optional u >= 0) by exactly
    ``state.inner_iters`` FGP iterations on the dual (tv.py:53-89)."""
    if weight <= 0:
        raise ValueError(f"tv_prox: weight must be positive, got {weight}")
    xd = AR.to_dev(x, state.dtype)
    H, W = state.shape
    if tuple(xd.shape) != (H, W):
        raise ValueError(f"tv_prox: input shape {tuple(xd.shape)} != state shape {(H, W)}")
    u = torch.empty_like(xd)
    rep = int(state.last_weight is not None and state.last_weight != weight)
    L.call("psb_tv_prox2d", L.dcode(state.dtype), L.ptr(xd), H * W, L.ptr(state.slots), 6 * H * W,
           None, 1, float(weight), None, rep, None, H, W, state.inner_iters,
           int(bool(state.accelerated)), int(bool(state.nonneg)), INNER_STEP, L.ptr(u), H * W,
           L.stream())
    state.last_weight = weight
    state.total_inner_iterations += state.inner_iters
    if AR.is_host(x):
        return AR.to_host(u)
    return u if u.dtype == x.dtype else u.to(x.dtype)


def dual_gap_rof(x, q, weight):
    """ROF prox duality gap at u = x + div q (tv.py:92-105)."""
    qd = AR.to_dev(q, q.dtype if isinstance(q, torch.Tensor) and q.dtype == torch.float32
                   else torch.float64)
    xd = AR.to_dev(x, torch.float64)
    if qd.dim() != 3 or qd.shape[0] != 2:
        raise ValueError(f"dual_gap_rof: expected a (2, H, W) field, got {tuple(qd.shape)}")
    qd = qd.contiguous()
    cnt = torch.empty(1, dtype=torch.float64, device="cuda")
    L.call("psb_count_outside_ball", L.dcode(qd.dtype), L.ptr(qd), qd[0].numel(),
           float(weight * (1.0 + 1e-10)), L.ptr(cnt), L.stream())
    if float(cnt.item()) > 0:
        raise ValueError("dual_gap_rof: q lies outside the feasibility ball")
    dq = div_dev(qd.double())
    u = T.lincomb(1.0, xd, 1.0, dq)
    primal = 0.5 * float(T.reduce_sumsq(u, xd)) + weight * tv_value(u)
    dual = -0.5 * float(T.reduce_sumsq(T.lincomb(1.0, dq, 1.0, xd))) + 0.5 * float(T.reduce_sumsq(xd))
    return primal - dual
