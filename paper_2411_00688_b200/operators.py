"""Linear operators with matched adjoints, evaluated on the device.

Mirrors operators.py of the reference (names, signatures, shapes).  Each map
carries a ``kind`` tag so the fused drivers can recognise the structure they
accelerate (identity fidelity -> x - b fused; blur -> separable periodic
kernel; radon -> matrix-free ray-driven projector pair).  ``forward`` /
``adjoint`` accept numpy (returned as numpy float64) or CUDA tensors
(returned on the device).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any, Callable, Optional

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from . import tensor as T


@dataclass
class LinearMap:
    """forward/adjoint pair + cached norm estimate (operators.py:18-39)."""

    domain_shape: tuple
    range_shape: tuple
    forward: Callable
    adjoint: Callable
    norm_sq_estimate: Optional[float] = None
    abs_forward: Optional[Callable] = None
    abs_adjoint: Optional[Callable] = None
    kind: str = "generic"
    params: Any = field(default=None, repr=False)

    def norm_sq(self, iters=100, seed=0):
        if self.norm_sq_estimate is None:
            self.norm_sq_estimate = power_method(self, iters=iters, seed=seed)
        return self.norm_sq_estimate


def _fdtype(a):
    if isinstance(a, torch.Tensor) and a.dtype == torch.float32:
        return torch.float32
    return torch.float64


def _wrap(dev_fn):
    """Lift a device->device function to the numpy-or-tensor public surface."""
    def f(a):
        t = AR.to_dev(a, _fdtype(a))
        return AR.like(dev_fn(t), a)
    f.device_fn = dev_fn
    return f


# -- finite differences (operators.py:44-104) ---------------------------------

def grad_dev(u):
    if u.dim() != 2 or min(u.shape) < 2:
        raise ValueError(f"grad_forward: need a 2-D grid with both sides >= 2, got {tuple(u.shape)}")
    H, W = u.shape
    g = torch.empty((2, H, W), dtype=u.dtype, device="cuda")
    L.call("psb_grad2d", L.dcode(u.dtype), L.ptr(u), L.ptr(g), 1, H, W, L.stream())
    return g


def div_dev(q):
    if q.dim() != 3 or q.shape[0] != 2 or min(q.shape[1:]) < 2:
        raise ValueError(f"divergence: expected (2, H, W) with H, W >= 2, got {tuple(q.shape)}")
    H, W = q.shape[1:]
    d = torch.empty((H, W), dtype=q.dtype, device="cuda")
    L.call("psb_div2d", L.dcode(q.dtype), L.ptr(q), L.ptr(d), 1, H, W, L.stream())
    return d


grad_forward = _wrap(grad_dev)
grad_forward.__doc__ = "Neumann forward differences, (2, H, W) (operators.py:44-57)."
divergence = _wrap(div_dev)
divergence.__doc__ = "Discrete divergence = -grad^T (operators.py:60-71)."


def grad_map(shape, norm_sq_estimate=None):
    """LinearMap of grad_forward on a fixed grid (operators.py:74-104)."""
    h, w = shape
    return LinearMap(
        domain_shape=(h, w), range_shape=(2, h, w), forward=grad_forward,
        adjoint=_wrap(lambda q: T.lincomb(-1.0, div_dev(q))),
        norm_sq_estimate=norm_sq_estimate, kind="grad")


# -- identity (operators.py:297-307) ------------------------------------------

def identity_map(shape):
    shape = tuple(shape)
    copy = _wrap(lambda t: t.clone())
    return LinearMap(shape, shape, copy, copy, norm_sq_estimate=1.0,
                     abs_forward=copy, abs_adjoint=copy, kind="identity")


# -- composition (operators.py:323-365) ---------------------------------------

def block_stack(a, d):
    """K x = (a x, d x) with a flat range; K^T y sums the block adjoints."""
    if tuple(a.domain_shape) != tuple(d.domain_shape):
        raise ValueError(f"block_stack: domain mismatch {a.domain_shape} vs {d.domain_shape}")
    na = int(np.prod(a.range_shape))
    nd = int(np.prod(d.range_shape))

    def fwd(x):
        fa, fd = _dev_apply(a.forward, x), _dev_apply(d.forward, x)
        return torch.cat([fa.reshape(-1), fd.reshape(-1)])

    def adj(y):
        if y.shape != (na + nd,):
            raise ValueError(f"block_stack adjoint: expected ({na + nd},), got {tuple(y.shape)}")
        ya = y[:na].reshape(a.range_shape)
        yd = y[na:].reshape(d.range_shape)
        return T.lincomb(1.0, _dev_apply(a.adjoint, ya), 1.0, _dev_apply(d.adjoint, yd))

    return LinearMap(tuple(a.domain_shape), (na + nd,), _wrap(fwd), _wrap(adj), kind="stack",
                     params=(a, d))


def _dev_apply(fn, t):
    dev = getattr(fn, "device_fn", None)
    if dev is not None:
        return dev(t)
    r = fn(t)
    return r if isinstance(r, torch.Tensor) else AR.to_dev(r, t.dtype)


def apply_forward(op, t):
    """Device-tensor forward of any LinearMap (used by the drivers)."""
    return _dev_apply(op.forward, t)


def apply_adjoint(op, t):
    return _dev_apply(op.adjoint, t)


# -- norm estimate (operators.py:368-390) -------------------------------------

def power_method(op, iters=100, seed=0):
    """Rayleigh quotient of A^T A after ``iters`` normalised power steps from
    the reference's start vector default_rng(seed).standard_normal."""
    if iters < 1:
        raise ValueError("power_method: iters must be >= 1")
    x = AR.to_dev(np.random.default_rng(seed).standard_normal(op.domain_shape), torch.float64)
    est = 0.0
    for _ in range(iters):
        y = apply_forward(op, x)
        if float(T.reduce_sumsq(y)) == 0.0:
            return 0.0
        z = apply_adjoint(op, y)
        est = float(T.reduce_dot(x, z)) / float(T.reduce_sumsq(x))
        nz = float(T.reduce_sumsq(z)) ** 0.5
        if nz == 0.0:
            return 0.0
        x = T.lincomb(1.0 / nz, z)
    return float(est)
