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


def grad_forward(u):
    """Neumann forward differences, (2, H, W) (operators.py:44-57)."""
    return AR.like(grad_dev(AR.to_dev(u, _fdtype(u))), u)


def divergence(q):
    """Discrete divergence = -grad^T (operators.py:60-71)."""
    return AR.like(div_dev(AR.to_dev(q, _fdtype(q))), q)


grad_forward.device_fn = grad_dev
divergence.device_fn = div_dev


def _absgrad_dev(u):
    H, W = u.shape
    g = torch.empty((2, H, W), dtype=u.dtype, device="cuda")
    L.call("psb_absgrad2d", L.dcode(u.dtype), L.ptr(u), L.ptr(g), H, W, L.stream())
    return g


def _absdiv_dev(q):
    H, W = q.shape[1:]
    d = torch.empty((H, W), dtype=q.dtype, device="cuda")
    L.call("psb_absdiv2d", L.dcode(q.dtype), L.ptr(q), L.ptr(d), H, W, L.stream())
    return d


def grad_map(shape, norm_sq_estimate=None):
    """LinearMap of grad_forward on a fixed grid with its entrywise-absolute
    maps for diagonal preconditioning (operators.py:74-104)."""
    h, w = shape
    return LinearMap(
        domain_shape=(h, w), range_shape=(2, h, w), forward=grad_forward,
        adjoint=_wrap(lambda q: T.lincomb(-1.0, div_dev(q))),
        norm_sq_estimate=norm_sq_estimate, abs_forward=_wrap(_absgrad_dev),
        abs_adjoint=_wrap(_absdiv_dev), kind="grad")


# -- periodic blur (operators.py:109-184) ---------------------------------------

@dataclass
class BlurKernel:
    """Odd square kernel, nonnegative weights summing to 1 (operators.py:109-128).

    ``factor`` is the 1-D factor when the kernel is separable (w = f f^T, as
    for Gaussians); the production gradient kernel then runs 2k instead of
    k^2 MACs per pixel.
    """

    weights: np.ndarray
    factor: Optional[np.ndarray] = None

    def __post_init__(self):
        self.weights = np.asarray(self.weights, dtype=np.float64)
        s = self.weights.shape
        if len(s) != 2 or s[0] != s[1] or s[0] % 2 == 0:
            raise ValueError(f"BlurKernel: weights must be odd and square, got {s}")
        if np.any(self.weights < 0):
            raise ValueError("BlurKernel: negative weights")
        total = float(self.weights.sum())
        if abs(total - 1.0) > 1e-12:
            raise ValueError(f"BlurKernel: weights sum to {total}, expected 1")
        if self.factor is None:
            f = np.sqrt(np.diag(self.weights))
            if np.max(np.abs(np.outer(f, f) - self.weights)) <= 1e-15:
                self.factor = f
        if s[0] > 15:
            raise ValueError("BlurKernel: kernels up to 15x15 are supported on the device")

    @property
    def size(self):
        return self.weights.shape[0]


def gaussian_kernel(size, sigma):
    """Normalised truncated Gaussian (operators.py:131-137); exact 1-D factor kept."""
    if size % 2 == 0 or size < 1:
        raise ValueError(f"gaussian_kernel: size must be odd, got {size}")
    ax = np.arange(size) - size // 2
    g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sigma ** 2))
    e = np.exp(-(ax ** 2) / (2.0 * sigma ** 2))
    return BlurKernel(g / g.sum(), factor=e / e.sum())


def _taps(kernel):
    w2 = np.ascontiguousarray(kernel.weights, dtype=np.float64)
    return w2, w2.ctypes.data_as(L.C.c_void_p)


def _blur_dev(t, kernel, adjoint):
    if t.dim() != 2:
        raise ValueError(f"blur: expected 2-D image, got shape {tuple(t.shape)}")
    if kernel.size > min(t.shape):
        raise ValueError(f"blur: kernel size {kernel.size} exceeds image {tuple(t.shape)}")
    out = torch.empty_like(t)
    w2, wp = _taps(kernel)
    L.call("psb_blur2d", L.dcode(t.dtype), L.ptr(t), L.ptr(out), 1, t.shape[0], t.shape[1], wp,
           kernel.size, int(adjoint), L.stream())
    return out


def blur_forward(u, kernel):
    """Circular 2-D convolution (operators.py:149-158), reference tap order."""
    return _wrap(lambda t: _blur_dev(t, kernel, False))(u)


def blur_adjoint(r, kernel):
    """Circular correlation, the adjoint (operators.py:161-172)."""
    return _wrap(lambda t: _blur_dev(t, kernel, True))(r)


def blur_grad_dev(u, b, kernel, separable=True, out=None):
    """g = A^T (A u - b) in one fused kernel (separable) or the exact tap order."""
    H, W = u.shape
    g = torch.empty_like(u) if out is None else out
    w2, wp = _taps(kernel)
    sep = separable and kernel.factor is not None
    f = np.ascontiguousarray(kernel.factor if sep else np.zeros(1), dtype=np.float64)
    scratch = None if sep else torch.empty_like(u)
    L.call("psb_blur_grad2d", L.dcode(u.dtype), L.ptr(u), L.ptr(b), L.ptr(g), H, W, wp,
           f.ctypes.data_as(L.C.c_void_p), kernel.size, int(sep), L.ptr(scratch), L.stream())
    return g


def blur_map(kernel, shape):
    """LinearMap of the periodic blur (operators.py:175-184); |A| = A."""
    fwd = _wrap(lambda t: _blur_dev(t, kernel, False))
    adj = _wrap(lambda t: _blur_dev(t, kernel, True))
    return LinearMap(tuple(shape), tuple(shape), fwd, adj, abs_forward=fwd, abs_adjoint=adj,
                     kind="blur", params=kernel)


# -- parallel-beam Radon transform (operators.py:189-292) ---------------------

@dataclass
class RadonGeometry:
    """Parallel-beam geometry on a square image (operators.py:189-215)."""

    image_side: int
    n_angles: int
    n_bins: int
    bin_spacing: float = 1.0
    angles: np.ndarray = field(default=None)

    def __post_init__(self):
        if self.image_side < 2 or self.n_angles < 1:
            raise ValueError("RadonGeometry: need image_side >= 2 and n_angles >= 1")
        if self.n_bins < self.image_side:
            raise ValueError(f"RadonGeometry: n_bins {self.n_bins} < image_side {self.image_side}")
        if self.angles is None:
            self.angles = np.arange(self.n_angles) * (np.pi / self.n_angles)
        else:
            self.angles = np.asarray(self.angles, dtype=np.float64)
            if np.any(np.diff(self.angles) <= 0):
                raise ValueError("RadonGeometry: angles must be strictly increasing")
        self._dev = None

    def device(self):
        """(ctypes psb_radon_geom, device tables) -- the ray-sample lattice of
        radon_system_matrix (operators.py:224-229) computed with numpy as the
        reference does, so device sample positions are bit-identical."""
        if self._dev is None:
            n = self.image_side
            center = (n - 1) / 2.0
            half_span = n / np.sqrt(2.0)
            n_steps = int(np.ceil(2.0 * half_span)) + 1
            steps = np.linspace(-half_span, half_span, n_steps)
            offsets = (np.arange(self.n_bins) - (self.n_bins - 1) / 2.0) * self.bin_spacing
            # per-angle scalar cos/sin exactly as the reference loop evaluates them
            cs = np.array([np.cos(t) for t in self.angles])
            sn = np.array([np.sin(t) for t in self.angles])
            tab = np.concatenate([offsets, steps, cs, sn])
            tdev = AR.to_dev(tab, torch.float64)
            g = L.RadonGeom(n, len(self.angles), self.n_bins, n_steps, center, half_span,
                            2.0 * half_span / (n_steps - 1), float(self.bin_spacing),
                            tdev.data_ptr())
            self._dev = (g, tdev)
        return self._dev

    @property
    def sinogram_shape(self):
        return (len(self.angles), self.n_bins)


def _radon_dev(geom, t, adjoint):
    g, _ = geom.device()
    n = geom.image_side
    if adjoint:
        if tuple(t.shape) != geom.sinogram_shape:
            raise ValueError(f"radon adjoint: expected {geom.sinogram_shape}, got {tuple(t.shape)}")
        out = torch.empty((n, n), dtype=t.dtype, device="cuda")
        L.call("psb_radon_adj", L.dcode(t.dtype), L.C.byref(g), L.ptr(t), L.ptr(out), L.stream())
    else:
        if tuple(t.shape) != (n, n):
            raise ValueError(f"radon forward: expected {(n, n)}, got {tuple(t.shape)}")
        out = torch.empty(geom.sinogram_shape, dtype=t.dtype, device="cuda")
        L.call("psb_radon_fwd", L.dcode(t.dtype), L.C.byref(g), L.ptr(t), L.ptr(out), L.stream())
    return out


def radon_map(geom):
    """Matrix-free projector pair with the reference's ray-driven bilinear
    weights (operators.py:266-292); |A| = A (weights are nonnegative)."""
    n = geom.image_side
    fwd = _wrap(lambda t: _radon_dev(geom, t, False))
    adj = _wrap(lambda t: _radon_dev(geom, t, True))
    return LinearMap((n, n), geom.sinogram_shape, fwd, adj, abs_forward=fwd, abs_adjoint=adj,
                     kind="radon", params=geom)


# -- identity (operators.py:297-307) ------------------------------------------

def identity_map(shape):
    shape = tuple(shape)
    copy = _wrap(lambda t: t.clone())
    return LinearMap(shape, shape, copy, copy, norm_sq_estimate=1.0,
                     abs_forward=copy, abs_adjoint=copy, kind="identity")


def diagonal_map(diag):
    """Elementwise multiplication by a fixed array (operators.py:310-320)."""
    dd = AR.to_dev(diag, torch.float64)
    ad = T.lincomb(1.0, dd)
    ad = torch.where(ad < 0, -ad, ad)  # |diag| (setup, once)
    mul = _wrap(lambda t: T.axpy_arr(torch.zeros_like(t), 1, dd.to(t.dtype), t))
    amul = _wrap(lambda t: T.axpy_arr(torch.zeros_like(t), 1, ad.to(t.dtype), t))
    return LinearMap(tuple(dd.shape), tuple(dd.shape), mul, mul,
                     norm_sq_estimate=float(np.max(np.abs(np.asarray(AR.to_host(dd))))) ** 2,
                     abs_forward=amul, abs_adjoint=amul, kind="diagonal")


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

    abs_fwd = abs_adj = None
    if a.abs_forward is not None and d.abs_forward is not None:
        def afwd(x):
            return torch.cat([_dev_apply(a.abs_forward, x).reshape(-1),
                              _dev_apply(d.abs_forward, x).reshape(-1)])

        def aadj(y):
            ya = y[:na].reshape(a.range_shape)
            yd = y[na:].reshape(d.range_shape)
            return T.lincomb(1.0, _dev_apply(a.abs_adjoint, ya), 1.0, _dev_apply(d.abs_adjoint, yd))

        abs_fwd, abs_adj = _wrap(afwd), _wrap(aadj)
    return LinearMap(tuple(a.domain_shape), (na + nd,), _wrap(fwd), _wrap(adj),
                     abs_forward=abs_fwd, abs_adjoint=abs_adj, kind="stack", params=(a, d))


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
