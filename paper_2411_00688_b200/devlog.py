"""Device-side IterationLog and the harness CSV.

The reference observes every iteration synchronously (solvers.py:61-104):
rel_error against the reference solution and the objective are evaluated on
the host after each step.  Here a log whose observations are all
device-computable -- a reference solution, ``device_objective(recon)`` as the
objective, an optional ``tol`` and ``inner_counter`` but no ``callback`` /
``transform`` -- keeps the whole run inside the native drivers: they copy the
iterate of every outer iteration into a device history buffer (the drivers'
``x_hist`` argument), the metrics of a chunk of iterations are computed with
batched fp64 reductions (csrc/reduce.cu: psb_sumsq_bcast, psb_tv2d,
psb_count_below) and brought to the host with one copy per chunk.

``tol`` keeps the reference's semantics exactly: the first iteration whose
rel_error drops below tol is the last one recorded, and the returned iterate
and the TvProxState are those of that iteration (the chunk is replayed from a
snapshot up to it -- the drivers are deterministic).

``emit_csv`` writes the harness CSV (harness.py:447-466) byte for byte.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from . import tensor as T
from .errors import DivergenceError
from .operators import apply_forward

HIST_BYTES = 256 << 20  # iterate history per chunk

CSV_HEADER = "iter,elapsed_s,prox_count,inner_iters,rel_error,objective,prox_applied"


def _fmt(value):
    return "" if value is None else f"{value:.17g}"


def emit_csv(records, path):
    """One row per logged iteration; reals carry 17 significant digits (harness.py:447-466)."""
    try:
        with open(path, "w", encoding="utf-8", newline="\n") as f:
            f.write(CSV_HEADER + "\n")
            for r in records:
                f.write(f"{r.iteration},{_fmt(r.elapsed_s)},{r.prox_count},"
                        f"{r.inner_iter_count},{_fmt(r.l2_rel_error)},{_fmt(r.objective)},"
                        f"{'true' if r.prox_applied else 'false'}\n")
    except OSError as exc:
        raise OSError(f"emit_csv: cannot write {path}: {exc}") from exc


class DeviceObjective:
    """``objective_tv(u, recon)`` (problems.py:187-192) that the fused drivers
    can evaluate on a batch of device iterates.  Calling it on one image is
    ``problems.objective_tv`` (so it also works as a plain ``objective_fn``)."""

    def __init__(self, recon, guarded=True):
        self.recon = recon
        self.guarded = guarded

    def __call__(self, u):
        from .problems import objective_tv
        return objective_tv(u, self.recon, guarded=self.guarded)

    def batch(self, hist, out):
        """Fill out[0] = sum (A x_j - b)^2, out[1] = TV(x_j), out[2] = #(x_j < -1e-12)
        for each iterate x_j of ``hist`` (m, H, W); device, no host sync."""
        r = self.recon
        m, H, W = hist.shape
        dc = L.dcode(hist.dtype)
        if r.A.kind == "identity":
            b = AR.to_dev(r.b, hist.dtype)
            L.call("psb_sumsq_bcast", dc, L.ptr(hist), L.ptr(b), m, H * W, L.ptr(out[0]), L.stream())
        else:
            b = AR.to_dev(r.b, torch.float64)
            for j in range(m):
                ax = apply_forward(r.A, hist[j]).double()
                L.call("psb_sumsq", L.dcode(torch.float64), L.ptr(ax), L.ptr(b), 1, b.numel(),
                       L.ptr(out[0, j:]), L.stream())
        L.call("psb_tv2d", dc, L.ptr(hist), m, H, W, L.ptr(out[1]), L.stream())
        if self.guarded and r.nonneg:
            L.call("psb_count_below", dc, L.ptr(hist), m, H * W, -1e-12, L.ptr(out[2]), L.stream())
        else:
            out[2].zero_()

    def values(self, host_row_fid, host_row_tv, host_row_below):
        a = self.recon.alpha
        return [math.inf if nb > 0 else 0.5 * f + a * t
                for f, t, nb in zip(host_row_fid, host_row_tv, host_row_below)]


def device_objective(recon, guarded=True):
    """Objective of ``recon`` for an IterationLog that the fused drivers can
    evaluate on the device (see the module docstring)."""
    return DeviceObjective(recon, guarded)


def device_loggable(log):
    """True when every observation of ``log`` can be made on the device."""
    return (log.callback is None and log.transform is None
            and (log.objective_fn is None or isinstance(log.objective_fn, DeviceObjective))
            and (log.reference is not None or log.objective_fn is not None))


def run_logged(log, iters, coins, shape, dtype, run_chunk, snapshot, restore, inner_per_prox,
               base_inner):
    """Drive ``run_chunk(k0, coins_chunk, hist)`` (returns per-iteration device
    elapsed seconds relative to the chunk start, raises DivergenceError with the
    global iteration) over ``iters`` iterations and fill ``log.records``.
    Returns the number of executed iterations."""
    from .solvers import RunRecord
    shape = tuple(shape)
    HW = int(np.prod(shape))
    item = 4 if dtype == torch.float32 else 8
    M = int(max(1, min(iters, HIST_BYTES // max(1, HW * item))))
    hist = torch.empty((M,) + shape, dtype=dtype, device="cuda")
    metrics = torch.zeros((4, M), dtype=torch.float64, device="cuda")
    ref = None
    ref_norm = None
    if log.reference is not None:
        ref = AR.to_dev(log.reference, torch.float64)
        if tuple(ref.shape) != shape:
            raise ValueError(f"rel_error: shape mismatch {shape} vs {tuple(ref.shape)}")
        ref_norm = math.sqrt(float(T.reduce_sumsq(ref)))
        if ref_norm == 0.0:
            raise ZeroDivisionError("rel_error: zero reference")
    obj = log.objective_fn
    counts = np.cumsum(coins[:iters].astype(np.int64))
    t_off = 0.0
    for k0 in range(0, iters, M):
        m = min(M, iters - k0)
        snap = snapshot() if log.tol is not None else None
        err_exc = None
        try:
            el = run_chunk(k0, coins[k0:k0 + m], hist[:m])
        except DivergenceError as exc:  # record the iterations before the divergent one
            err_exc = exc
            m = max(0, int(exc.iteration) - k0)
            el = np.full(m, np.nan)
        if m > 0:
            h64 = hist[:m] if dtype == torch.float64 else hist[:m].double()
            if ref is not None:
                L.call("psb_sumsq_bcast", L.dcode(torch.float64), L.ptr(h64), L.ptr(ref), m, HW,
                       L.ptr(metrics[3]), L.stream())
            if obj is not None:
                obj.batch(hist[:m], metrics[:3, :m])
            host = metrics[:, :m].cpu().numpy()
            objs = obj.values(host[0], host[1], host[2]) if obj is not None else [None] * m
        for j in range(m):
            k = k0 + j
            err = math.sqrt(float(host[3, j])) / ref_norm if ref is not None else None
            inner = base_inner + inner_per_prox * int(counts[k]) if log.inner_counter is not None else 0
            log.records.append(RunRecord(k + 1, t_off + float(el[j]), int(counts[k]), inner, err,
                                         objs[j], bool(coins[k])))
            if log.tol is not None and err is not None and err < log.tol:
                if j < m - 1:  # land exactly on iteration k (deterministic replay)
                    restore(snap)
                    run_chunk(k0, coins[k0:k0 + j + 1], None)
                return k + 1
        if err_exc is not None:
            raise err_exc
        t_off += float(el[m - 1])
    return iters
