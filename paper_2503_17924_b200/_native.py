"""ctypes binding of libwlbcp.so, the C ABI declared in include/wlbcp.h.

This replaces the reference's `balsim._kernels` dispatch module
(`_kernels/__init__.py:1-61`): there is exactly ONE backend (sm_100a), no pure
fallback and no environment switch.  If the library is missing, or no
compute-capability-10 device is visible, compute entry points raise
`NativeError` -- they never fall back to the CPU.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeError

# WLB_LIB_PATH selects an alternative build of the SAME library (A/B experiments).
_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libwlbcp.so")
LIB_PATH = os.environ.get("WLB_LIB_PATH", _DEFAULT_LIB)

WLB_OK, WLB_EINVAL, WLB_ENODEV, WLB_ECUDA = 0, 22, 19, 1000
WLB_BWD_DKV_BF16 = 1
WLB_BWD_COVERED_ONLY = 2
WLB_PULL_OUT_BF16 = 4

_p, _i32, _i64, _f64, _f32, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_float, C.c_size_t


class WlbCpSync(C.Structure):
    """`WlbCpSync` of wlbcp.h: in-kernel CP synchronisation on arrival flags."""
    _fields_ = [("wait_flags", C.c_void_p), ("signal_bases", C.c_void_p),
                ("signal_off", C.c_int64), ("counters", C.c_void_p), ("cp", C.c_int32),
                ("kv_per_group", C.c_int32), ("epoch", C.c_int32), ("pad_", C.c_int32)]

# name -> (restype, argtypes); must match include/wlbcp.h
SIGNATURES = {
    "wlb_abi_version": (_i32, []),
    "wlb_last_error": (C.c_char_p, []),
    "wlb_device_check": (C.c_int, []),
    "wlb_heuristic_fill": (C.c_int, [_p, _i64, _i32, _i64, _f64, _f64, _p]),
    "wlb_shard_plan": (C.c_int, [_i32, _p, _p, _p, _i32, _i32, _i64, _p, _p, _i32, _f64, _i32,
                                 _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "wlb_shard_plan_measured": (C.c_int, [_i32, _p, _p, _p, _i32, _i32, _p, _i32, _i32, _p, _p,
                                          _p, _p, _p, _p, _p, _p, _p, _p]),
    "wlb_kernel_latency_sum": (C.c_int, [_p, _p, _i64, _i64, _p, _p, _i32, _f64, _p, _p]),
    "wlb_attn_tiles": (C.c_int, [_i32, _p, _p, _p, _i32, _i32, _p, _p, _p]),
    "wlb_attn_fwd": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _i32, _i32, _i32,
                               _i32, _f32, _p]),
    "wlb_attn_fwd_heads": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _i32, _i32, _i32,
                                     _i32, _f32, _i32, _i32, _p]),
    "wlb_attn_bwd_heads": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32,
                                     _i32, _i32, _i32, _i32, _f32, _p, _i32, _i32, _i32, _p]),
    "wlb_attn_fwd_sync": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _i32, _i32, _i32,
                                    _i32, _f32, C.POINTER(WlbCpSync), _p]),
    "wlb_attn_bwd_sync": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32,
                                    _i32, _i32, _i32, _i32, _f32, _p, _i32, C.POINTER(WlbCpSync),
                                    _p]),
    "wlb_attn_bwd_workspace": (_sz, [_i32, _i32, _i32, _i32, _i32, _i32]),
    "wlb_attn_bwd_ex": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32,
                                  _i32, _i32, _i32, _i32, _f32, _p, _i32, _p]),
    "wlb_attn_bwd_select": (_i32, [_i32]),
    "wlb_attn_bwd_pairs": (_i32, [_i32]),
    "wlb_attn_bwd_persistent": (_i32, [_i32]),
    "wlb_attn_bwd_reserve_sms": (_i32, [_i32]),
    "wlb_attn_bwd_l2_prefetch": (_i32, [_i32]),
    "wlb_qkv_rope": (C.c_int, [_p, _p, _p, _p, _p, _i32, _i32, _i32, _i32, _f32, _p]),
    "wlb_attn_bwd": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i32, _p, _i32, _i32,
                               _i32, _i32, _i32, _f32, _p, _p]),
    "wlb_qkv_proj_rope": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _i32, _i32, _i32, _i32, _i32,
                                    _f32, _p]),
    "wlb_rows_scatter": (C.c_int, [_p, _p, _p, _i64, _i64, _p]),
    "wlb_rows_gather": (C.c_int, [_p, _p, _p, _i64, _i64, _p]),
    "wlb_cp_kv_push": (C.c_int, [_p, _p, _p, _i64, _i64, _p, _i64, _i64, _i32, _p]),
    "wlb_cp_dkv_pull": (C.c_int, [_p, _i64, _i64, _p, _i64, _i64, _p, _p, _i32, _p]),
    "wlb_cp_dkv_pull_ex": (C.c_int, [_p, _i64, _i64, _p, _i64, _i64, _p, _p, _i32, _i32, _p]),
    "wlb_cp_kv_push_cov": (C.c_int, [_p, _p, _p, _i64, _i64, _p, _i64, _i64, _i32,
                                     _p, _i32, _p, _p, _i32, _p]),
    "wlb_cp_kv_push_part": (C.c_int, [_p, _p, _p, _i64, _i64, _i64, _i64, _p, _i64, _i64, _i32,
                                      _p, _i32, _p, _p, _i32, _p]),
    "wlb_cp_dkv_pull_part": (C.c_int, [_p, _i64, _i64, _p, _i64, _i64, _i64, _i64, _p, _p, _i32,
                                       _i32, _p, _i32, _p, _p, _i32, _p]),
    "wlb_cp_kv_push_dma": (C.c_int, [_p, _p, _p, _i32, _i64, _i64, _i64, _p, _i64, _i64, _i32,
                                     _p]),
    "wlb_cp_signal": (C.c_int, [_p, _i64, _i32, _i32, _p]),
    "wlb_cp_wait": (C.c_int, [_p, _i32, _i32, _p]),
    "wlb_cp_signal_memop": (C.c_int, [_p, _i64, _i32, _i32, _p]),
    "wlb_cp_wait_memop": (C.c_int, [_p, _i32, _i32, _p]),
    "wlb_cp_dkv_pull_cov": (C.c_int, [_p, _i64, _i64, _p, _i64, _i64, _p, _p, _i32, _i32,
                                      _p, _i32, _p, _p, _i32, _p]),
}

_lib = None
_device_ok = None


def lib():
    """Load the library once (host entry points work without a GPU)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: run `python -m paper_2503_17924_b200.build`")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(handle, name) and LIB_PATH != _DEFAULT_LIB:
                continue      # an older build under WLB_LIB_PATH (A/B runs)
            fn = getattr(handle, name)
            fn.restype, fn.argtypes = res, args
        _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc == WLB_OK:
        return
    msg = lib().wlb_last_error().decode(errors="replace")
    if rc == WLB_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed ({rc}): {msg}")


def require_device() -> None:
    """Raise NativeError unless an sm_100 device is usable from torch and the library."""
    global _device_ok
    if _device_ok is None:
        import torch
        if not torch.cuda.is_available():
            raise NativeError("no CUDA device: the sm_100a path has no CPU fallback")
        torch.cuda.init()
        check(lib().wlb_device_check(), "wlb_device_check")
        _device_ok = True


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def to_device(values, dtype, device):
    """Host list -> device tensor WITHOUT a host sync (pinned staging + async
    copy; torch's caching host allocator keeps the staging buffer alive until
    the copy has run).  torch.tensor(..., device=cuda) would block the host
    until all queued GPU work drained."""
    import torch
    host = torch.tensor(values, dtype=dtype, pin_memory=True)
    return host.to(device, non_blocking=True)


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
