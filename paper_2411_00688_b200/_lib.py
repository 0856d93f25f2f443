"""ctypes binding of libpsb200.so (the C ABI declared in include/psb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2411_00688_b200.build``).  There is no fallback: every
compute entry point of this package goes through this module, and importing
it without the built library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .errors import DivergenceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PSB_LIB_PATH") or os.path.join(_HERE, "libpsb200.so")

PSB_OK, PSB_ERR_VALUE, PSB_ERR_CUDA, PSB_ERR_DIVERGED = 0, 1, 2, 3
F32, F64 = 0, 1

_vp, _i32, _i64, _dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double


class RadonGeom(C.Structure):
    """Mirror of psb_radon_geom (include/psb200.h)."""

    _fields_ = [("n", C.c_int), ("n_angles", C.c_int), ("n_bins", C.c_int),
                ("n_steps", C.c_int), ("center", C.c_double), ("half_span", C.c_double),
                ("step_spacing", C.c_double), ("bin_spacing", C.c_double),
                ("tables", C.c_void_p)]


_geo = C.POINTER(RadonGeom)

# name -> argtypes, mirroring include/psb200.h one for one.
SIGNATURES = {
    "psb_ctx_create": [_i32, _vp],
    "psb_ctx_destroy": [_vp],
    "psb_ctx_stream": [_vp],
    "psb_ctx_sync": [_vp],
    "psb_buf_alloc": [_vp, _i64, _vp],
    "psb_buf_free": [_vp, _vp],
    "psb_upload": [_vp, _vp, _vp, _i64],
    "psb_download": [_vp, _vp, _vp, _i64],
    "psb_coin_table": [_vp, _i64, _i32, _dbl, _vp, _vp],
    "psb_abi_version": [],
    "psb_last_error": [],
    "psb_device_sm_count": [_vp],
    "psb_grad2d": [_i32, _vp, _vp, _i64, _i32, _i32, _vp],
    "psb_div2d": [_i32, _vp, _vp, _i64, _i32, _i32, _vp],
    "psb_project_ball2d": [_i32, _vp, _vp, _i64, _i64, _dbl, _vp],
    "psb_project_nonneg": [_i32, _vp, _vp, _i64, _vp],
    "psb_lincomb": [_i32, _dbl, _vp, _dbl, _vp, _vp, _i64, _vp],
    "psb_axpy_arr": [_i32, _vp, _i32, _vp, _vp, _vp, _i64, _vp],
    "psb_fidprox": [_i32, _vp, _dbl, _vp, _vp, _vp, _i64, _vp],
    "psb_recip_floor": [_i32, _vp, _dbl, _vp, _i64, _vp],
    "psb_prox_l2_fidelity": [_i32, _vp, _dbl, _vp, _vp, _vp, _i64, _vp],
    "psb_mark_nonfinite": [_i32, _vp, _i64, _vp, _vp, _vp],
    "psb_counter_add": [_vp, _i32, _vp],
    "psb_absgrad2d": [_i32, _vp, _vp, _i32, _i32, _vp],
    "psb_absdiv2d": [_i32, _vp, _vp, _i32, _i32, _vp],
    "psb_fgp2d_iter": [_i32, _vp, _i64, _vp, _i64, _vp, _i32, _dbl, _vp, _i32, _vp, _i32, _i32,
                       _i32, _dbl, _dbl, _i32, _vp],
    "psb_fgp2d_finalize": [_i32, _vp, _i64, _vp, _i64, _vp, _i32, _i32, _i32, _i32, _i32, _vp,
                           _i64, _vp],
    "psb_aprojgd_dual_rof": [_i32, _vp, _vp, _i32, _i32, _dbl, _dbl, _i32, _vp, _vp],
    "psb_dual_rof_run": [_i32, _i32, _vp, _vp, _vp, _vp, _i32, _i32, _dbl, _dbl, _dbl, _dbl, _vp,
                         _i32, _vp, _i32, _vp, _vp, _vp],
    "psb_tv_prox2d": [_i32, _vp, _i64, _vp, _i64, _vp, _i32, _dbl, _vp, _i32, _vp, _i32, _i32,
                      _i32, _i32, _i32, _dbl, _vp, _i64, _vp],
    "psb_sumsq": [_i32, _vp, _vp, _i64, _i64, _vp, _vp],
    "psb_dot": [_i32, _vp, _vp, _i64, _i64, _vp, _vp],
    "psb_tv2d": [_i32, _vp, _i64, _i32, _i32, _vp, _vp],
    "psb_sumsq_bcast": [_i32, _vp, _vp, _i64, _i64, _vp, _vp],
    "psb_count_below": [_i32, _vp, _i64, _i64, _dbl, _vp, _vp],
    "psb_queue_stats": [_vp],
    "psb_count_outside_ball": [_i32, _vp, _i64, _dbl, _vp, _vp],
    "psb_count_nonfinite": [_i32, _vp, _i64, _vp, _vp],
    "psb_proxskip_pre": [_i32, _i32, _vp, _vp, _i32, _vp, _vp, _i64, _i64, _vp, _dbl, _dbl, _vp,
                         _i32, _vp],
    "psb_proxskip_post": [_i32, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _i64, _vp, _i32, _i32, _i32,
                          _i32, _i32, _dbl, _dbl, _vp, _i32, _vp],
    "psb_proxskip_denoise_run": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp,
                                 _i32, _dbl, _dbl, _dbl, _i32, _i32, _i32, _vp, _vp, _vp, _i32,
                                 _vp, _vp, _vp, _i32, _vp, _vp],
    "psb_proxskip_denoise_run_streamed": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32,
                                          _vp, _i32, _dbl, _dbl, _dbl, _i32, _i32, _i32, _vp,
                                          _vp, _vp, _vp, _vp, _vp, _i32, _vp],
    "psb_stream_memops_supported": [_vp],
    "psb_stream_write_u32": [_vp, _vp, C.c_uint32],
    "psb_stream_wait_geq_u32": [_vp, _vp, C.c_uint32],
    "psb_chunked_h2d": [_vp, _vp, _i64, _vp, _i32, _vp, _vp],
    "psb_chunked_d2h": [_vp, _vp, _i64, _vp, _i32, _vp, C.c_uint32, _vp],
    "psb_cluster_max_active": [_vp],
    "psb_copy_async": [_vp, _vp, _i64, _vp],
    "psb_ipc_handle_size": [],
    "psb_ipc_get_handle": [_vp, _vp, _vp],
    "psb_ipc_open_handle": [_vp, _vp],
    "psb_ipc_close": [_vp],
    "psb_fgp3d_iter": [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _dbl, _dbl, _dbl, _i32,
                       _i32, _vp, _vp, _vp, _vp, _vp, _i32, _vp],
    "psb_fgp3d_iter_part": [_i32, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _dbl, _dbl, _dbl,
                            _i32, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp],
    "psb_proxskip_post3d": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _i32,
                            _i32, _i32, _i32, _dbl, _dbl, _i32, _vp, _i32, _vp],
    "psb_skip_chain": [_i32, _i32, _vp, _vp, _vp, _vp, _i64, _i32, _dbl, _dbl, _vp, _i32, _vp],
    "psb_radon_fwd": [_i32, _geo, _vp, _vp, _vp],
    "psb_radon_adj": [_i32, _geo, _vp, _vp, _vp],
    "psb_pdhg_step": [_i32, _geo, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _dbl, _dbl, _dbl, _dbl,
                      _dbl, _i32, _vp],
    "psb_pdhg_run": [_i32, _geo, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _dbl, _dbl, _vp, _vp, _dbl,
                     _dbl, _i32, _i32, _dbl, _vp, _i32, _vp, _vp, _vp],
    "psb_ct_implicit_run": [_i32, _i32, _geo, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _dbl,
                            _dbl, _dbl, _dbl, _i32, _i32, _i32, _vp, _vp, _vp, _i32, _vp, _vp, _vp],
    "psb_blur2d": [_i32, _vp, _vp, _i64, _i32, _i32, _vp, _i32, _i32, _vp],
    "psb_blur_grad2d": [_i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _vp],
    "psb_proxskip_deblur_run": [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _vp,
                                _vp, _i32, _i32, _vp, _i32, _dbl, _dbl, _dbl, _i32, _i32, _i32,
                                _vp, _vp, _vp, _i32, _vp, _vp, _vp, _i32, _vp, _vp],
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = (C.c_char_p if name == "psb_last_error" else
                      C.c_void_p if name == "psb_ctx_stream" else C.c_int)
    return lib


LIB = _load()


def check(status, what=""):
    if status == PSB_OK:
        return
    msg = LIB.psb_last_error().decode(errors="replace")
    if status == PSB_ERR_VALUE:
        raise ValueError(msg)
    if status == PSB_ERR_DIVERGED:
        raise DivergenceError(-1, what)
    raise RuntimeError(f"libpsb200 {what}: {msg}")


def call(name, *args):
    check(getattr(LIB, name)(*args), name)


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2411_00688_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def stream():
    """Raw handle of torch's current CUDA stream (plumbing only)."""
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def dcode(dtype):
    if dtype == torch.float32:
        return F32
    if dtype == torch.float64:
        return F64
    raise ValueError(f"unsupported dtype {dtype}")
