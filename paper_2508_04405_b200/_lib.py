"""ctypes binding of the C ABI in include/flexq.h (libflexq_sm100a.so).

The product path has no CPU fallback: if the in-tree library is missing or no
sm_100 GPU is present, every compute call raises DeviceError.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigError, DeviceError, FormatError, InvalidInputError, ShapeError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLEXQ_LIB") or os.path.join(_PKG, "_lib", "libflexq_sm100a.so")

OK, ERR_INVALID, ERR_SHAPE, ERR_CONFIG, ERR_FORMAT, ERR_CUDA = 0, -1, -2, -3, -4, -5
FLAG_NONFINITE, FLAG_NONPOS_SCALE, FLAG_KV_OVERFLOW = 1, 2, 4
DT_F16, DT_BF16, DT_F32, DT_F64 = 0, 1, 2, 3
OUT_F16, OUT_F32 = 0, 1
KERNEL_GEMV, KERNEL_TC_I8, KERNEL_TC16, KERNEL_MMA_SYNC = 0, 1, 2, 3

_EXC = {ERR_INVALID: InvalidInputError, ERR_SHAPE: ShapeError, ERR_CONFIG: ConfigError,
        ERR_FORMAT: FormatError, ERR_CUDA: DeviceError}

i64, i32, vp, cstr = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_char_p

# name -> (restype, argtypes); every symbol declared in include/flexq.h
SIGNATURES = {
    "flexq_last_error": (cstr, []),
    "flexq_tuning": (cstr, []),
    "flexq_version": (i32, []),
    "flexq_device_check": (i32, []),
    "flexq_quantize": (i32, [vp, i32, i64, i64, i32, i64, i32, vp, vp, vp, vp, vp, i64, vp, vp]),
    "flexq_planes_bytes": (i64, [i64, i64, i32, i32]),
    "flexq_pack_planes": (i32, [vp, i64, i64, i32, i32, vp, vp]),
    "flexq_unpack_planes": (i32, [vp, i64, i64, i32, i32, vp, vp]),
    "flexq_t6_bytes": (i64, [i64, i64, i64]),
    "flexq_pack_t6": (i32, [vp, vp, i64, i64, i64, i32, vp, vp, vp]),
    "flexq_act_frag_bytes": (i64, [i64, i64, i64]),
    "flexq_act_m_pad": (i64, [i64]),
    "flexq_pack_act_t6": (i32, [vp, vp, i64, i64, i64, i64, vp, vp, vp, vp]),
    "flexq_gemm_workspace_bytes": (i64, [i64, i64, i64, i64, i32]),
    "flexq_gemm_t6": (i32, [vp, vp, i32, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, i32, vp, i32, vp]),
    "flexq_gemm_t6_ex": (i32, [vp, vp, i32, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, i32, vp, i32,
                               vp, vp]),
    "flexq_gemm_bitserial": (i32, [vp, vp, vp, vp, i64, i64, i64, i32, i32, i64, i32, i32, vp, vp, i32, vp, i32, vp]),
    "flexq_group_epilogue_f64": (i32, [vp, vp, vp, i64, i64, i64, vp, vp, vp]),
    "flexq_popcount_and": (i32, [vp, vp, i64, vp, vp]),
    "flexq_act_buf_bytes": (i64, [i64, i64, i64]),
    "flexq_linear_forward": (i32, [vp, vp, i32, i32, vp, i64, i64, i64, i64, vp, vp, vp, vp, vp]),
    "flexq_linear_forward_ex": (i32, [vp, vp, i32, i32, vp, i64, i64, i64, i64, vp, i32, vp, vp, vp,
                                      vp, vp]),
    "flexq_linear_kernel": (i32, [i64, i64, i64, i64, i32]),
    "flexq_set_tc16_route": (i32, [i32]),
    "flexq_gemm_tc16": (i32, [vp, vp, vp, i64, i64, i64, vp, i32, vp, vp, vp]),
    "flexq_act_f16_operand": (vp, [vp, i64, i64, i64]),
    "flexq_rmsnorm_quantize": (i32, [vp, i64, vp, ctypes.c_float, i64, i64, i32, i64, vp, vp, vp,
                                     i64, vp, vp, vp]),
    "flexq_silu_mul_quantize": (i32, [vp, i64, i64, i64, i32, i64, vp, vp, vp, i64, vp, vp, vp]),
    "flexq_rope_kv_append": (i32, [vp, vp, vp, vp, vp, i64, i32, i32, i64, ctypes.c_float, vp]),
    "flexq_attn_decode": (i32, [vp, vp, vp, vp, vp, i64, i32, i32, i64, vp]),
    "flexq_attn_block": (i32, [vp, vp, vp, vp, vp, i64, i32, i32, i64, ctypes.c_float, i32, i64,
                               vp, vp, vp, i64, vp, vp]),
}

_lib = None
_lock = threading.Lock()
_device_ok = False


def load(check_device: bool = False):
    """Load the library (no GPU needed for loading); optionally verify an sm_100 device."""
    global _lib, _device_ok
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2508_04405_b200._build` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    if check_device and not _device_ok:
        require_device()
    return _lib


def require_device():
    global _device_ok
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the W6Ax path runs only on an sm_100 (B200) GPU; "
                          "there is no CPU fallback")
    torch.cuda.init()
    rc = _lib.flexq_device_check()
    if rc != OK:
        raise DeviceError(_lib.flexq_last_error().decode())
    _device_ok = True


def lib():
    return load(check_device=True)


def check(rc: int, prefix: str = "") -> None:
    if rc == OK:
        return
    msg = _lib.flexq_last_error().decode()
    raise _EXC.get(rc, DeviceError)(prefix + msg)


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream(device_index: int | None = None) -> int:
    """The current CUDA stream (raw cudaStream_t) of ``device_index`` (default: the current
    device).  torch's raw-stream accessor costs ~0.3 us where building a torch.cuda.Stream
    costs ~3 us -- per-call overhead the e2e path pays twice per forward."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is None:  # pragma: no cover - older torch
        return torch.cuda.current_stream(device_index).cuda_stream
    return raw(torch.cuda.current_device() if device_index is None else device_index)
