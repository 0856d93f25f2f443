"""Batched ProxSkip TV denoising (BASELINE config 4).

The reference has no batch API: config 4 is 4096 independent
``build_tv_recon(identity_map, b_i, alpha, inner_budget=50)`` +
``run_proxskip(..., SkipConfig(p, seed_i), K)`` problems.  Here they live in
one set of device buffers -- x, h, b, z: (N, H, W); dual slots (N, 3, 2, H, W).
For 256 x 256 problems with an fp32 FGP (config 4) one native call runs the
whole K-iteration segment of every problem in ONE launch of the cluster run
kernel (csrc/fgp_cluster8.cu: an 8-CTA cluster takes one problem at a time
and executes all of its coin-fired prox calls back to back, FGP state in
registers and tensor memory; fp64 outer state: the 16-CTA form,
csrc/fgp_cluster.cu) plus the SM-worker kernel on the SMs the clusters leave
(csrc/fgp2d.cu), both claiming problems from one device work queue.  Other
shapes / precisions advance all problems together per outer iteration: one
fused pre kernel over the batch, the FGP inner iterations over the compacted
list of coin-fired problems only, one post kernel over that list.
Per-problem semantics (own Philox coin stream, warm starts, last_weight
re-projection, inner-iteration counters) equal N separate reference runs;
tests/test_gpu_fullsize.py checks 32 config-4 problems at the full 300 x 50
schedule against fixtures produced by the reference.  Multi-GPU: problems are
sharded across ranks with no collective (``shard_balanced`` by known work,
``shard_indices`` contiguous).
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import _arrays as AR
from . import _lib as L
from .errors import DivergenceError
from .skip import INT32_MAX, SkipConfig
from .tv import PRECISIONS


def shard_indices(n_total, rank, world):
    """Contiguous block of problem indices owned by ``rank`` (weak-free, no exchange)."""
    per = (n_total + world - 1) // world
    lo = min(n_total, rank * per)
    return np.arange(lo, min(n_total, lo + per))


def shard_balanced(costs, rank, world):
    """Problem indices owned by ``rank`` when the per-problem work is known up
    front (config 4: the prox calls of each problem's coin stream): problems
    sorted by cost, longest first, and dealt to the ranks in snake order, so
    every rank gets the same count (+-1) and nearly the same total work.  Every
    rank computes the same partition on its own -- still no exchange.  Returns
    ascending indices."""
    costs = np.asarray(costs).reshape(-1)
    order = np.argsort(-costs, kind="stable")
    pos = np.arange(order.size)
    lap, slot = pos // world, pos % world
    owner = np.where(lap % 2 == 0, slot, world - 1 - slot)
    return np.sort(order[owner == rank])


def coin_table(p, seeds, iters):
    """(iters, N) uint8: column i is SkipConfig(p, seeds[i]).coins(iters), i.e.
    Generator(Philox(seed)).random() < p per draw (skip.py:27-28) -- generated
    on the device (psb_coin_table), bit-identical to the numpy stream."""
    if not 0.0 < p <= 1.0:
        raise ValueError(f"SkipConfig: p must be in (0, 1], got {p}")
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64).reshape(-1))
    out = np.empty((int(iters), seeds.size), dtype=np.uint8)
    if out.size:
        L.call("psb_coin_table", seeds.ctypes.data_as(L.C.c_void_p), seeds.size, int(iters),
               float(p), out.ctypes.data_as(L.C.c_void_p), L.stream())
    return out


class BatchedTvDenoise:
    """N independent 0.5||u - b_i||^2 + alpha TV(u) problems on one GPU."""

    def __init__(self, b, alpha, inner_budget=50, *, precision="fp32", accelerated=True,
                 nonneg=False, cold_buffers=True):
        if alpha <= 0:
            raise ValueError("alpha must be positive")
        if inner_budget < 1:
            raise ValueError("inner_budget must be >= 1")
        dto, dtf = PRECISIONS[precision]
        self.b = AR.to_dev(b, dto)
        if self.b.dim() != 3:
            raise ValueError(f"expected (N, H, W) data, got {tuple(self.b.shape)}")
        self.n, self.H, self.W = self.b.shape
        self.alpha = alpha
        self.inner_iters = inner_budget
        self.accelerated = accelerated
        self.nonneg = nonneg
        self.dto, self.dtf = dto, dtf
        # cold_buffers=False leaves x, h and the dual slots uninitialised (only
        # for the streamed run, whose kernels imply a cold start)
        alloc = torch.zeros if cold_buffers else torch.empty
        self.x = alloc(self.b.shape, dtype=self.b.dtype, device="cuda")
        self.h = alloc(self.b.shape, dtype=self.b.dtype, device="cuda")
        self.z = torch.empty((self.n, self.H, self.W), dtype=dtf, device="cuda")
        self.slots = alloc((self.n, 3, 2, self.H, self.W), dtype=dtf, device="cuda")
        self.last_weight = np.full(self.n, np.nan)
        self.prox_count = np.zeros(self.n, dtype=np.int64)
        self.bad = torch.full((self.n,), INT32_MAX, dtype=torch.int32, device="cuda")
        self.elapsed = None

    def reset(self, x0=None, h0=None):
        """Cold start: zero warm starts and counters (harness.py:283-286 semantics)."""
        if x0 is None:
            self.x.zero_()
        else:
            self.x.copy_(AR.to_dev(x0, self.dto))
        if h0 is None:
            self.h.zero_()
        else:
            self.h.copy_(AR.to_dev(h0, self.dto))
        self.slots.zero_()
        self.last_weight[:] = np.nan
        self.prox_count[:] = 0
        self.bad.fill_(INT32_MAX)

    @property
    def total_inner_iterations(self):
        return self.prox_count * self.inner_iters

    def run_proxskip(self, coins, gamma=1.0, p=0.1, *, use_graph=False, record_elapsed=False,
                     fgp_time=None, lo=0, hi=None, stream=None):
        """K outer iterations; ``coins`` is the (K, N) table of ``coin_table``.
        ``lo``/``hi`` restrict the call to problems lo..hi-1 (``coins`` then
        has hi - lo columns); ``stream`` is a torch CUDA stream (default: the
        current one)."""
        hi = self.n if hi is None else hi
        if not 0 <= lo <= hi <= self.n:
            raise ValueError("problem range out of bounds")
        coins = np.ascontiguousarray(coins, dtype=np.uint8)
        K = coins.shape[0]
        if coins.shape[1] != hi - lo:
            raise ValueError("coin table does not match the batch")
        self.elapsed = np.zeros(max(K, 1)) if record_elapsed else None
        if hi == lo:
            return self.x
        HW = self.H * self.W
        off = lambda t, per: L.C.c_void_p(t.data_ptr() + lo * per * t.element_size())  # noqa: E731
        L.call("psb_proxskip_denoise_run", L.dcode(self.dto), L.dcode(self.dtf), off(self.x, HW),
               off(self.b, HW), off(self.h, HW), off(self.z, HW), off(self.slots, 6 * HW),
               hi - lo, self.H, self.W, coins.ctypes.data_as(L.C.c_void_p), K, float(gamma),
               float(p), float(self.alpha), self.inner_iters, int(self.accelerated),
               int(self.nonneg), self.last_weight[lo:hi].ctypes.data_as(L.C.c_void_p),
               self.prox_count[lo:hi].ctypes.data_as(L.C.c_void_p), off(self.bad, 1),
               int(bool(use_graph)),
               self.elapsed.ctypes.data_as(L.C.c_void_p) if record_elapsed else None,
               fgp_time.ctypes.data_as(L.C.c_void_p) if fgp_time is not None else None,
               None, 0, None,
               L.C.c_void_p(stream.cuda_stream) if stream is not None else L.stream())
        return self.x

    def check_finite(self):
        bad = self.bad.cpu().numpy()
        hit = np.nonzero(bad != INT32_MAX)[0]
        if hit.size:
            raise DivergenceError(int(bad[hit].min()), f"proxskip[problem {int(hit[0])}]")


def _memops():
    if not hasattr(_memops, "ok"):
        v = L.C.c_int(0)
        L.call("psb_stream_memops_supported", L.C.byref(v))
        _memops.ok = bool(v.value)
    return _memops.ok


def run_proxskip_batched(b, alpha, p, seeds, iters, inner_budget=50, *, gamma=1.0,
                         precision="fp32", use_graph=False, chunk=None, out=None):
    """Config-4 entry point: returns (x, prox_counts) as the input currency.

    ``out`` (optional, host input only): a contiguous float32 CPU tensor of
    b's shape that receives x -- page-locked, the results go straight from
    the device into it by DMA (no staging, no page faults inside the call).

    Host input on the cluster path is streamed: every chunk's host->device
    copy (``chunk`` problems) is enqueued on a copy stream, each announced by
    a stream memory write; the run kernels, launched next, wait per problem
    for its chunk's flag; each chunk's result goes back to the host as soon as
    its problems are done (stream memory wait on a device counter) while later
    chunks still compute.  Same arithmetic and results as the resident run."""
    seeds = np.asarray(seeds).reshape(-1)
    n = int(seeds.size)
    if chunk is None:
        chunk = 256  # the middle chunks; the streamed path ramps up to and down from it
    shape = tuple(b.shape) if hasattr(b, "shape") else np.shape(b)
    # (streamed only for float32 host data: a dtype conversion would need a
    # kernel on the copy stream, which cannot run while the waiting run
    # kernels hold every SM)
    f32 = (b.dtype == torch.float32) if isinstance(b, torch.Tensor) else (
        getattr(b, "dtype", None) == np.float32)
    if (AR.is_host(b) and f32 and not use_graph and precision == "fp32" and chunk and n > chunk
            and len(shape) == 3 and shape[1:] == (256, 256) and _memops()
            and os.environ.get("PSB_NO_CLUSTER", "0") != "1"):
        return _run_streamed(b, alpha, p, seeds, iters, inner_budget, gamma, chunk, out)
    solver = BatchedTvDenoise(b, alpha, inner_budget, precision=precision)
    solver.run_proxskip(coin_table(p, seeds, iters), gamma, p, use_graph=use_graph)
    solver.check_finite()
    if out is not None:
        AR.download_into(out, solver.x.to(out.dtype))
        return (out if isinstance(b, torch.Tensor) else out.numpy()), solver.prox_count.copy()
    return AR.like(solver.x, b), solver.prox_count.copy()


def _chunk_edges(n, chunk):
    """Chunk boundaries of a streamed batch: sizes ramp up 16, 32, ... to
    ``chunk`` and back down at the end, so the first input arrives and the
    last result leaves in a fraction of a millisecond while the middle of the
    batch moves in few large copies."""
    ramp = []
    c = 16
    while c < chunk:
        ramp.append(c)
        c *= 2
    sizes_lo, sizes_hi, total = [], [], 0
    for c in ramp:  # leading and trailing ramps, while the batch allows
        if total + 2 * c > n:
            break
        sizes_lo.append(c)
        sizes_hi.append(c)
        total += 2 * c
    mid = n - total
    sizes = sizes_lo + [chunk] * (mid // chunk) + ([mid % chunk] if mid % chunk else []) \
        + sizes_hi[::-1]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


_COPY_STREAMS = {}


def _copy_streams():
    """The two copy streams of the streamed run, one pair per device (kept
    across calls: creating a stream costs tens of microseconds)."""
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _COPY_STREAMS[dev]


def _run_streamed(b, alpha, p, seeds, iters, inner_budget, gamma, chunk, out=None):
    tensor_in = isinstance(b, torch.Tensor)
    src = b.detach().contiguous() if tensor_in else torch.from_numpy(np.ascontiguousarray(b))
    n, H, W = src.shape
    if n != seeds.size:
        raise ValueError("one seed per problem")
    # (validated before anything is launched: the run kernels wait for input)
    if out is None:
        out = torch.empty((n, H, W), dtype=torch.float32)
    elif (not isinstance(out, torch.Tensor) or tuple(out.shape) != (n, H, W)
          or out.dtype != torch.float32 or out.is_cuda or not out.is_contiguous()):
        raise ValueError("run_proxskip_batched: out must be a contiguous float32 CPU tensor "
                         "of b's shape")
    dbg = os.environ.get("PSB_DEBUG_E2E") == "1"
    t0 = time.perf_counter() if dbg else 0.0
    # the streamed run starts cold (the kernels imply x = h = 0 and a zero warm
    # start): no 10 GB of zero-fills inside the call
    solver = BatchedTvDenoise(torch.empty((n, H, W), dtype=torch.float32, device="cuda"), alpha,
                              inner_budget, precision="fp32", cold_buffers=False)
    t1 = time.perf_counter() if dbg else 0.0
    edges = _chunk_edges(n, chunk)
    bounds = list(zip(edges[:-1], edges[1:]))
    nc = len(bounds)
    edges_h = np.ascontiguousarray(edges, dtype=np.int64)
    flags = torch.zeros(2 * nc + 1, dtype=torch.int32, device="cuda")  # ready[nc + 1], done[nc]
    ready, done = flags[:nc + 1], flags[nc + 1:]
    main = torch.cuda.current_stream()
    start = torch.cuda.Event(enable_timing=dbg)
    start.record(main)  # buffers allocated and zeroed
    h2d, d2h = _copy_streams()
    h2d.wait_event(start)
    d2h.wait_event(start)
    item = H * W * 4
    # 1) inputs, chunk by chunk, each announced to the run kernels by a fenced
    #    stream write -- all enqueued BEFORE the run, so the copies never depend
    #    on the run kernels making progress (serialised execution under
    #    CUDA_LAUNCH_BLOCKING=1, compute-sanitizer or ncu stays correct)
    if src.is_pinned():  # one native call enqueues every chunk (DMA, no kernels)
        L.call("psb_chunked_h2d", L.ptr(solver.b), L.C.c_void_p(src.data_ptr()), item,
               edges_h.ctypes.data_as(L.C.c_void_p), nc, L.ptr(ready), L.C.c_void_p(h2d.cuda_stream))
    else:
        cs = L.C.c_void_p(h2d.cuda_stream)
        with torch.cuda.stream(h2d):
            for c, (lo, hi) in enumerate(bounds):
                solver.b[lo:hi].copy_(src[lo:hi])  # float32 H2D: a DMA, no kernel on this stream
                L.call("psb_stream_write_u32", cs, L.C.c_void_p(ready.data_ptr() + 4 * c), 1)
    # (the coin streams are drawn while the first chunks are already on their way)
    coins = coin_table(p, seeds, iters)
    # 2) the run: its kernels wait per problem for the chunk flags above
    L.call("psb_proxskip_denoise_run_streamed", L.dcode(solver.dto), L.dcode(solver.dtf),
           L.ptr(solver.x), L.ptr(solver.b), L.ptr(solver.h), L.ptr(solver.z),
           L.ptr(solver.slots), n, H, W, coins.ctypes.data_as(L.C.c_void_p), coins.shape[0],
           float(gamma), float(p), float(alpha), inner_budget, 1, 0,
           solver.last_weight.ctypes.data_as(L.C.c_void_p),
           solver.prox_count.ctypes.data_as(L.C.c_void_p), L.ptr(solver.bad), L.ptr(ready),
           L.ptr(done), edges_h.ctypes.data_as(L.C.c_void_p), nc, L.stream())
    # 3) results on their own stream, chunk by chunk, as soon as the chunk's
    #    problems are done (stream wait on the device counter): they leave
    #    while later inputs still arrive
    pinned = out.is_pinned()
    if pinned:
        L.call("psb_chunked_d2h", L.C.c_void_p(out.data_ptr()), L.ptr(solver.x), item,
               edges_h.ctypes.data_as(L.C.c_void_p), nc, L.ptr(done), 16,
               L.C.c_void_p(d2h.cuda_stream))
    else:
        cs = L.C.c_void_p(d2h.cuda_stream)
        with torch.cuda.stream(d2h):
            for c, (lo, hi) in enumerate(bounds):
                L.call("psb_stream_wait_geq_u32", cs, L.C.c_void_p(done.data_ptr() + 4 * c),
                       16 * (hi - lo))
                AR.download_into(out[lo:hi], solver.x[lo:hi])
    t2 = time.perf_counter() if dbg else 0.0
    main.wait_stream(h2d)
    main.wait_stream(d2h)
    if pinned:
        d2h.synchronize()
    if dbg:
        end = torch.cuda.Event(enable_timing=True)
        end.record(main)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"[psb e2e] setup {1e3 * (t1 - t0):.1f} ms, enqueue {1e3 * (t2 - t1):.1f} ms, "
              f"run {1e3 * (t3 - t2):.1f} ms, device {start.elapsed_time(end):.1f} ms "
              f"({nc} chunks, sizes {np.diff(edges).tolist()})", flush=True)
    if int(ready[nc].item()) != 0:
        raise RuntimeError("streamed run: an input chunk never arrived (device wait timed out)")
    solver.check_finite()
    return (out if tensor_in else out.numpy()), solver.prox_count.copy()
