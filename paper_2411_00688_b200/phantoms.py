"""Seeded synthetic inputs for the BASELINE configs.

The reference ships only two fixed phantoms (phantoms.py:6-54); BASELINE asks
for seeded random shapes.  These host-side generators produce them with
numpy ``default_rng`` and reuse the reference's noise convention
``u + sigma * default_rng(seed).standard_normal(u.shape)`` (phantoms.py:57-65).
They are input generation, shared by the tests, the oracle runs and the
benchmark -- not part of the solver path.
"""

from __future__ import annotations

import numpy as np


def add_noise(u, sigma, seed):
    """i.i.d. N(0, sigma^2) noise (phantoms.py:57-65 convention)."""
    if sigma < 0:
        raise ValueError(f"add_noise: sigma must be nonnegative, got {sigma}")
    u = np.asarray(u, dtype=np.float64)
    if sigma == 0.0:
        return u.copy()
    return u + sigma * np.random.default_rng(seed).standard_normal(u.shape)


def random_shapes(shape, n_shapes, rng, *, rects=True, value_range=(0.0, 1.0)):
    """Piecewise-constant 2-D phantom: ``n_shapes`` random ellipses (and, with
    ``rects``, axis-aligned rectangles) painted in order with U[value_range]
    intensities on a zero background."""
    H, W = shape
    u = np.zeros((H, W))
    rr = (np.arange(H)[:, None] + 0.5) / H
    cc = (np.arange(W)[None, :] + 0.5) / W
    lo, hi = value_range
    for _ in range(n_shapes):
        kind = rng.integers(2) if rects else 0
        cy, cx = rng.uniform(0.15, 0.85, size=2)
        ry, rx = rng.uniform(0.05, 0.3, size=2)
        val = rng.uniform(lo, hi)
        if kind == 0:
            th = rng.uniform(0.0, np.pi)
            c, s = np.cos(th), np.sin(th)
            dy, dx = rr - cy, cc - cx
            a = (dx * c + dy * s) / rx
            b = (-dx * s + dy * c) / ry
            u[a * a + b * b <= 1.0] = val
        else:
            u[(np.abs(rr - cy) <= ry) & (np.abs(cc - cx) <= rx)] = val
    return u


def shepp_like(n, n_ellipses, rng):
    """Shepp-Logan-style CT phantom: a body ellipse plus ``n_ellipses - 1``
    seeded inner ellipses with additive U[-0.3, 0.5] densities, clipped to
    [0, 1] (config 3)."""
    u = np.zeros((n, n))
    yy = (np.arange(n)[:, None] + 0.5) / n * 2.0 - 1.0
    xx = (np.arange(n)[None, :] + 0.5) / n * 2.0 - 1.0
    u[(xx / 0.69) ** 2 + (yy / 0.92) ** 2 <= 1.0] = 1.0
    for _ in range(n_ellipses - 1):
        cy, cx = rng.uniform(-0.5, 0.5, size=2)
        ry, rx = rng.uniform(0.04, 0.3, size=2)
        th = rng.uniform(0.0, np.pi)
        c, s = np.cos(th), np.sin(th)
        a = ((xx - cx) * c + (yy - cy) * s) / rx
        b = (-(xx - cx) * s + (yy - cy) * c) / ry
        u[a * a + b * b <= 1.0] += rng.uniform(-0.3, 0.5)
    return np.clip(u, 0.0, 1.0)


def random_ellipsoids(shape, n, rng, value_range=(0.0, 1.0)):
    """3-D volume of ``n`` seeded ellipsoids with U[value_range] intensities (config 5)."""
    D, H, W = shape
    u = np.zeros(shape, dtype=np.float32)
    zz = ((np.arange(D) + 0.5) / D)[:, None, None].astype(np.float32)
    yy = ((np.arange(H) + 0.5) / H)[None, :, None].astype(np.float32)
    xx = ((np.arange(W) + 0.5) / W)[None, None, :].astype(np.float32)
    for _ in range(n):
        c = rng.uniform(0.15, 0.85, size=3)
        r = rng.uniform(0.04, 0.25, size=3)
        val = rng.uniform(*value_range)
        z0, z1 = max(0, int((c[0] - r[0]) * D) - 1), min(D, int((c[0] + r[0]) * D) + 2)
        sub = (((zz[z0:z1] - c[0]) / r[0]) ** 2 + ((yy - c[1]) / r[1]) ** 2
               + ((xx - c[2]) / r[2]) ** 2) <= 1.0
        u[z0:z1][sub] = val
    return u


# -- BASELINE config inputs -----------------------------------------------------

def config1_data(seed=0, n=256):
    """256^2, 10 random ellipses/rectangles, noise 0.1."""
    truth = random_shapes((n, n), 10, np.random.default_rng(seed))
    return truth, add_noise(truth, 0.1, seed)


def config4_problem(i, n=256):
    """Problem i of the batch: its own rng draws phantom, sigma ~ U[0.05, 0.15] and noise."""
    rng = np.random.default_rng(i)
    truth = random_shapes((n, n), 10, rng)
    sigma = rng.uniform(0.05, 0.15)
    return truth, truth + sigma * rng.standard_normal(truth.shape), sigma


def config4_batch(indices, n=256, dtype=np.float32):
    out = np.empty((len(indices), n, n), dtype=dtype)
    for j, i in enumerate(indices):
        out[j] = config4_problem(int(i), n)[1]
    return out


def config2_data(seed=0, n=512):
    """512^2 deblurring: 10 seeded random ellipses, 9x9 sigma=2 periodic blur
    (D2), noise 0.01.  Returns (truth, blurred-noisy b, kernel weights)."""
    truth = random_shapes((n, n), 10, np.random.default_rng(seed), rects=False)
    w = _gaussian_weights(9, 2.0)
    return truth, add_noise(_conv_periodic(truth, w), 0.01, seed), w


def config3_phantom(seed=0, n=512):
    """512^2 Shepp-Logan-style CT phantom of 10 seeded ellipses (config 3)."""
    return shepp_like(n, 10, np.random.default_rng(seed))


def config3_noisy(sino, seed=0):
    """Config-3 sinogram noise: sigma = 1 % of max(A u_true) (D10)."""
    return add_noise(sino, 0.01 * float(np.max(sino)), seed)


def _gaussian_weights(size, sigma):
    """Normalised size x size Gaussian (the reference's gaussian_kernel,
    operators.py:131-137)."""
    ax = np.arange(size) - size // 2
    g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sigma**2))
    return g / g.sum()


def _conv_periodic(u, w):
    """Periodic 2-D convolution in the reference's tap order
    (operators.py:149-158): out = sum_a sum_b w[a,b] roll(u, (a-c, b-c))."""
    c = w.shape[0] // 2
    out = np.zeros_like(u)
    for a in range(w.shape[0]):
        for b in range(w.shape[1]):
            if w[a, b] != 0.0:
                out += w[a, b] * np.roll(u, (a - c, b - c), axis=(0, 1))
    return out


def config5_volume(side=1024, seed=0, device="cuda"):
    """Config-5 input generated on the device (a 1024^3 volume is 4.3 GB):
    50 seeded ellipsoids with U[0,1] intensities (numpy ``default_rng(seed)``
    draws the shapes, as random_ellipsoids) plus N(0, 0.1^2) noise from a
    seeded torch generator.  Returns a float32 CUDA tensor (D, H, W)."""
    import torch
    D = H = W = side
    vol = torch.zeros((D, H, W), dtype=torch.float32, device=device)
    rng = np.random.default_rng(seed)
    ax = (torch.arange(side, device=device, dtype=torch.float32) + 0.5) / side
    for _ in range(50):
        c = rng.uniform(0.15, 0.85, size=3)
        r = rng.uniform(0.04, 0.25, size=3)
        val = float(rng.uniform(0, 1))
        z0, z1 = max(0, int((c[0] - r[0]) * D) - 1), min(D, int((c[0] + r[0]) * D) + 2)
        yy = ((ax - float(c[1])) / float(r[1])) ** 2
        xx = ((ax - float(c[2])) / float(r[2])) ** 2
        zz = ((ax[z0:z1] - float(c[0])) / float(r[0])) ** 2
        m = zz[:, None, None] + yy[None, :, None] + xx[None, None, :] <= 1.0
        vol[z0:z1][m] = val
    g = torch.Generator(device=device).manual_seed(seed)
    vol.add_(torch.randn((D, H, W), generator=g, device=device), alpha=0.1)
    return vol
