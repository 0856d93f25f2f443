"""Host <-> device array plumbing.

The public API accepts numpy arrays (the reference's currency) or CUDA torch
tensors.  Numpy inputs are uploaded once and results are handed back as
numpy float64, so reference call sites keep working unchanged; CUDA tensors
stay on the device end to end.  torch is used here only for device memory.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def is_host(a):
    return not isinstance(a, torch.Tensor) or a.device.type == "cpu"


# Large host<->device copies go through two pinned staging buffers: a copy
# from / to pageable memory runs at ~2 GB/s on the GPU hosts, the staged
# pipeline (DMA into one pinned buffer while the CPU moves the other) at
# 20-25 GB/s.
STAGE_BYTES = 32 << 20
_STAGES = {}


def _stages():
    dev = torch.cuda.current_device()
    st = _STAGES.get(dev)
    if st is None:
        st = ([torch.empty(STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
              [torch.cuda.Event() for _ in range(2)])
        _STAGES[dev] = st
    return st


def _staged(n, dma, cpu):
    """Run the two-buffer pipeline over ``n`` bytes in STAGE_BYTES chunks:
    dma(buf, lo, hi) enqueues the device side, cpu(buf, lo, hi) the host side."""
    bufs, evs = _stages()
    pend = None
    k = 0
    for lo in range(0, n, STAGE_BYTES):
        hi = min(n, lo + STAGE_BYTES)
        dma(bufs[k], lo, hi)
        evs[k].record()
        if pend is not None:
            pk, plo, phi = pend
            evs[pk].synchronize()
            cpu(bufs[pk], plo, phi)
        pend = (k, lo, hi)
        k ^= 1
    if pend is not None:
        pk, plo, phi = pend
        evs[pk].synchronize()
        cpu(bufs[pk], plo, phi)


def download_into(dst, src):
    """Copy CUDA tensor ``src`` into the contiguous CPU tensor ``dst`` (same dtype)."""
    src = src.detach().contiguous()
    n = src.numel() * src.element_size()
    if n < 2 * STAGE_BYTES or dst.is_pinned():
        dst.copy_(src)
        return dst
    sb = src.view(-1).view(torch.uint8)
    db = dst.view(-1).view(torch.uint8)
    _staged(n, lambda buf, lo, hi: buf[:hi - lo].copy_(sb[lo:hi], non_blocking=True),
            lambda buf, lo, hi: db[lo:hi].copy_(buf[:hi - lo]))
    return dst


def upload(src, dtype):
    """CPU tensor -> new CUDA tensor of ``dtype`` (staged when large and pageable)."""
    src = src.detach().contiguous()
    n = src.numel() * src.element_size()
    if n < 2 * STAGE_BYTES or src.is_pinned():
        return src.to(device="cuda", dtype=dtype)
    out = torch.empty(src.shape, dtype=src.dtype, device="cuda")
    sb = src.view(-1).view(torch.uint8)
    ob = out.view(-1).view(torch.uint8)
    bufs, evs = _stages()
    # host side first (fill the pinned buffer), then the DMA; reuse waits on the event
    k = 0
    busy = [False, False]
    for lo in range(0, n, STAGE_BYTES):
        hi = min(n, lo + STAGE_BYTES)
        if busy[k]:
            evs[k].synchronize()
        bufs[k][:hi - lo].copy_(sb[lo:hi])
        ob[lo:hi].copy_(bufs[k][:hi - lo], non_blocking=True)
        evs[k].record()
        busy[k] = True
        k ^= 1
    torch.cuda.current_stream().synchronize()  # staging buffers may be reused by the caller
    return out if out.dtype == dtype else out.to(dtype)


def to_dev(a, dtype=torch.float64):
    """Device tensor of ``dtype`` (contiguous) holding ``a``."""
    _lib.require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.device.type != "cuda":
            return upload(t, dtype)
        if t.dtype != dtype or not t.is_contiguous():
            t = t.to(dtype=dtype).contiguous()
        return t
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return upload(torch.from_numpy(arr), dtype)


def to_host(t):
    t = t.detach()
    if t.device.type != "cuda":
        return t.to(torch.float64).numpy()
    t = t.to(torch.float64)
    out = np.empty(tuple(t.shape), dtype=np.float64)
    download_into(torch.from_numpy(out), t)
    return out


def like(t, ref):
    """Return device tensor ``t`` in the currency of ``ref``: numpy in -> numpy
    float64 out, CPU tensor in -> CPU tensor of the same dtype, CUDA in -> CUDA."""
    if isinstance(ref, torch.Tensor):
        if ref.device.type == "cpu":
            out = torch.empty(tuple(t.shape), dtype=ref.dtype)
            return download_into(out, t.to(ref.dtype))
        return t
    return to_host(t)


def empty(shape, dtype):
    _lib.require_cuda()
    return torch.empty(tuple(shape), dtype=dtype, device="cuda")


def zeros(shape, dtype):
    _lib.require_cuda()
    return torch.zeros(tuple(shape), dtype=dtype, device="cuda")


def shape_of(a):
    return tuple(a.shape)
