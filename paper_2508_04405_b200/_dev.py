"""Array plumbing between the drop-in API and device memory.

Array-in / array-out: numpy inputs give numpy results (the reference's
contract, so callers such as sensitivity.layer_error keep working), torch CUDA
tensors give torch CUDA tensors.  Either way all compute happens in the
sm_100a library; numpy arrays are uploaded once and the device copy is cached
on the returned objects.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DeviceError


def torch():
    import torch as _t

    return _t


def is_torch(a) -> bool:
    t = torch()
    return isinstance(a, t.Tensor)


def device():
    _lib.lib()  # loads the library and verifies an sm_100 device (raises otherwise)
    return torch().device("cuda", torch().cuda.current_device())


_NP2T = None


def _np2t():
    global _NP2T
    if _NP2T is None:
        t = torch()
        _NP2T = {np.dtype(np.float16): t.float16, np.dtype(np.float32): t.float32,
                 np.dtype(np.float64): t.float64, np.dtype(np.int8): t.int8,
                 np.dtype(np.int16): t.int16, np.dtype(np.int32): t.int32,
                 np.dtype(np.int64): t.int64, np.dtype(np.uint8): t.uint8}
    return _NP2T


def to_device(a, dtype=None):
    """numpy / torch / array-like -> contiguous torch CUDA tensor (optionally cast)."""
    t = torch()
    dev = device()
    if is_torch(a):
        x = a.to(dev)
    else:
        arr = np.ascontiguousarray(np.asarray(a))
        if arr.dtype not in _np2t():
            arr = arr.astype(np.float64 if arr.dtype.kind == "f" else np.int64)
        x = t.from_numpy(arr).to(dev)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x.contiguous()


def to_host(x) -> np.ndarray:
    return x.detach().cpu().numpy()


def like_input(x, template):
    """Return device tensor x as numpy when the user handed us numpy."""
    return x if is_torch(template) else to_host(x)


def float_dtype_code(x) -> int:
    t = torch()
    codes = {t.float16: _lib.DT_F16, t.bfloat16: _lib.DT_BF16, t.float32: _lib.DT_F32,
             t.float64: _lib.DT_F64}
    if x.dtype not in codes:
        raise DeviceError(f"unsupported float dtype {x.dtype}")
    return codes[x.dtype]


def shape_of(a):
    return tuple(a.shape)
