"""Vector-space primitives on the device (tensor.py:17-51 of the reference).

Reductions accumulate in fp64 on the GPU with a fixed two-pass order
(csrc/reduce.cu); results agree with numpy's BLAS/pairwise sums to ~1e-15
relative.  Inputs may be numpy arrays or CUDA tensors.
"""

from __future__ import annotations

import math

import numpy as np

import torch

from . import _arrays as AR
from . import _lib as L


def _dev(a):
    return AR.to_dev(a, a.dtype if isinstance(a, torch.Tensor) and a.dtype in (torch.float32, torch.float64)
                     else torch.float64)


def reduce_sumsq(a, b=None):
    """sum((a - b)^2) in fp64 on the device (b optional); returns a 0-d device tensor."""
    a = _dev(a)
    if b is not None:
        b = _dev(b)
        if a.dtype != b.dtype:
            a, b = a.double(), b.double()
        if b.numel() != a.numel():
            raise ValueError(f"shape mismatch {tuple(a.shape)} vs {tuple(b.shape)}")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L.call("psb_sumsq", L.dcode(a.dtype), L.ptr(a), L.ptr(b), 1, a.numel(), L.ptr(out), L.stream())
    return out[0]


def reduce_dot(a, b):
    a, b = _dev(a), _dev(b)
    if a.dtype != b.dtype:
        a, b = a.double(), b.double()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L.call("psb_dot", L.dcode(a.dtype), L.ptr(a), L.ptr(b), 1, a.numel(), L.ptr(out), L.stream())
    return out[0]


def count_nonfinite(a):
    a = _dev(a)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    L.call("psb_count_nonfinite", L.dcode(a.dtype), L.ptr(a), a.numel(), L.ptr(out), L.stream())
    return out[0]


def dot(a, b):
    """Euclidean inner product (tensor.py:17-25)."""
    if tuple(a.shape) != tuple(b.shape) and math.prod(a.shape) != math.prod(b.shape):
        raise ValueError(f"dot: length mismatch {math.prod(a.shape)} vs {math.prod(b.shape)}")
    return float(reduce_dot(a, b))


def norm2(a):
    """Euclidean norm (tensor.py:28-30)."""
    return math.sqrt(float(reduce_sumsq(a)))


def rel_error(x, ref):
    """norm2(x - ref) / norm2(ref) (tensor.py:42-51)."""
    if tuple(x.shape) != tuple(ref.shape):
        raise ValueError(f"rel_error: shape mismatch {tuple(x.shape)} vs {tuple(ref.shape)}")
    den = norm2(ref)
    if den == 0.0:
        raise ZeroDivisionError("rel_error: zero reference")
    return math.sqrt(float(reduce_sumsq(x, ref))) / den


def lincomb(a, x, b=0.0, y=None, out=None):
    """(a*x) + (b*y) elementwise on the device, each product rounded once."""
    x = _dev(x)
    if y is not None:
        y = AR.to_dev(y, x.dtype)
        if y.numel() != x.numel():
            raise ValueError(f"shape mismatch {tuple(x.shape)} vs {tuple(y.shape)}")
    if out is None:
        out = torch.empty_like(x)
    L.call("psb_lincomb", L.dcode(x.dtype), float(a), L.ptr(x), float(b), L.ptr(y), L.ptr(out),
           x.numel(), L.stream())
    return out


def axpby(alpha, x, beta, y):
    """Elementwise alpha*x + beta*y (tensor.py:33-39)."""
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError(f"axpby: shape mismatch {tuple(x.shape)} vs {tuple(y.shape)}")
    return AR.like(lincomb(alpha, x, beta, y), x)


def axpy_arr(x, sign, s, y):
    """x + sign * (s .* y) with an array coefficient s (diagonal PDHG steps)."""
    x = _dev(x)
    s = AR.to_dev(s, x.dtype)
    y = AR.to_dev(y, x.dtype)
    out = torch.empty_like(x)
    L.call("psb_axpy_arr", L.dcode(x.dtype), L.ptr(x), int(sign), L.ptr(s), L.ptr(y), L.ptr(out),
           x.numel(), L.stream())
    return out


def scaled(x, sign, s, y):
    """x + sign * s * y for a scalar or array step s, rounded like the reference."""
    if isinstance(s, (int, float, np.floating)):
        return lincomb(1.0, x, sign * float(s), y)
    return axpy_arr(x, sign, s, y)


def fidprox(v, t, b):
    """(v - t b) / (1 + t), t scalar or array (problems.py:143-144)."""
    v = _dev(v)
    b = AR.to_dev(b, v.dtype).reshape(v.shape)
    out = torch.empty_like(v)
    if isinstance(t, (int, float, np.floating)):
        L.call("psb_fidprox", L.dcode(v.dtype), L.ptr(v), float(t), None, L.ptr(b), L.ptr(out),
               v.numel(), L.stream())
    else:
        ta = AR.to_dev(t, v.dtype).reshape(v.shape)
        L.call("psb_fidprox", L.dcode(v.dtype), L.ptr(v), 0.0, L.ptr(ta), L.ptr(b), L.ptr(out),
               v.numel(), L.stream())
    return out


def recip_floor(x, floor):
    """1 / max(x, floor) elementwise (solvers.py:222-223)."""
    x = _dev(x)
    out = torch.empty_like(x)
    L.call("psb_recip_floor", L.dcode(x.dtype), L.ptr(x), float(floor), L.ptr(out), x.numel(),
           L.stream())
    return out
