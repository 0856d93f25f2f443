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


def to_dev(a, dtype=torch.float64):
    """Device tensor of ``dtype`` (contiguous) holding ``a``."""
    _lib.require_cuda()
    if isinstance(a, torch.Tensor):
        t = a.detach()
        if t.device.type != "cuda" or t.dtype != dtype or not t.is_contiguous():
            t = t.to(device="cuda", dtype=dtype).contiguous()
        return t
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    t = torch.from_numpy(arr)
    if dtype != torch.float64:
        t = t.to(dtype)
    return t.to("cuda", non_blocking=False)


def to_host(t):
    return t.detach().to("cpu", torch.float64).numpy()


def like(t, ref):
    """Return device tensor ``t`` in the currency of ``ref``: numpy in -> numpy
    float64 out, CPU tensor in -> CPU tensor of the same dtype, CUDA in -> CUDA."""
    if isinstance(ref, torch.Tensor):
        if ref.device.type == "cpu":
            return t.detach().to(device="cpu", dtype=ref.dtype)
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
