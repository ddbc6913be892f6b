"""ctypes binding of oracle/_build/liboracle.so -- TEST INFRASTRUCTURE ONLY.

See oracle/flexq_oracle.c for the reference file:line each routine restates.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        for fn in ("oracle_quantize_f64", "oracle_quantize_f32", "oracle_quantize_f16"):
            getattr(L, fn).argtypes = [vp, i64, i64, ci, i64, ci, vp, vp]
            getattr(L, fn).restype = ci
        L.oracle_int_matmul.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, vp, vp, ci]
        L.oracle_int_matmul.restype = ci
        L.oracle_pack_planes.argtypes = [vp, i64, i64, ci, ci, vp]
        L.oracle_pack_planes.restype = ci
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def quantize(x: np.ndarray, bits: int, group_size: int = 128, fp16_scales: bool = False):
    """-> (codes int8 [rows, cols], scales float64 [rows, G]); ValueError like quantize.py."""
    x = np.ascontiguousarray(x)
    rows, cols = x.shape
    ng = -(-cols // group_size)
    codes = np.empty((rows, cols), np.int8)
    scales = np.empty((rows, ng), np.float64)
    fn = {np.dtype(np.float64): "oracle_quantize_f64", np.dtype(np.float32): "oracle_quantize_f32",
          np.dtype(np.float16): "oracle_quantize_f16"}[x.dtype]
    rc = getattr(lib(), fn)(_p(x), rows, cols, bits, group_size, int(fp16_scales), _p(codes), _p(scales))
    if rc == -1:
        raise ValueError("input contains non-finite values")
    if rc == -2:
        raise ValueError("all scales must be strictly positive")
    if rc != 0:
        raise ValueError(f"oracle_quantize failed rc={rc}")
    return codes, scales


def int_matmul(wcodes, xcodes, wscales, xscales, group_size: int, trace: bool = False,
               threads: int | None = None):
    """-> (Y float64 [M, N], partials int32 [G, M, N] | None)."""
    w = np.ascontiguousarray(wcodes, dtype=np.int8)
    x = np.ascontiguousarray(xcodes, dtype=np.int8)
    ws = np.ascontiguousarray(wscales, dtype=np.float64)
    xs = np.ascontiguousarray(xscales, dtype=np.float64)
    m, k = x.shape
    n = w.shape[0]
    ng = -(-k // group_size)
    y = np.empty((m, n), np.float64)
    parts = np.empty((ng, m, n), np.int32) if trace else None
    rc = lib().oracle_int_matmul(_p(w), _p(x), _p(ws), _p(xs), m, n, k, group_size, _p(y),
                                 _p(parts) if trace else None, threads or os.cpu_count() or 1)
    if rc != 0:
        raise ValueError(f"oracle_int_matmul failed rc={rc}")
    return y, parts


def pack_planes(codes: np.ndarray, bits: int, chunk_m: int) -> np.ndarray:
    """FLXQ-P words as <u8 [KC, RC, bits, chunk_m, 2]."""
    c = np.ascontiguousarray(codes, dtype=np.int8)
    rows, cols = c.shape
    rc, kc = -(-rows // chunk_m), -(-cols // 128)
    out = np.empty(kc * rc * bits * chunk_m * 16, np.uint8)
    rcode = lib().oracle_pack_planes(_p(c), rows, cols, bits, chunk_m, _p(out))
    if rcode != 0:
        raise ValueError(f"oracle_pack_planes failed rc={rcode}")
    return out.view("<u8").reshape(kc, rc, bits, chunk_m, 2)
