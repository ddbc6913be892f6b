"""The C-ABI library: loads without a GPU, exports every symbol include/flexq.h
declares, its pure-host size helpers agree with the documented layouts, and the
product path fails loudly (DeviceError) when no sm_100 GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2508_04405_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flexq.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(flexq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding binds exactly the declared set
    assert set(_lib.SIGNATURES) == set(names)


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_size_helpers():
    L = _lib.load()
    assert L.flexq_version() == 100
    # FLXQ-P bytes: [KC, RC, bits, chunk_m, 16 B] (packing.py:79-129)
    assert L.flexq_planes_bytes(8, 256, 6, 8) == 2 * 1 * 6 * 8 * 16
    assert L.flexq_planes_bytes(1, 512, 6, 1) == 4 * 1 * 6 * 1 * 16
    # T6: rows padded to 64, k padded per group to 32-slot steps, 4 k-steps per block
    assert L.flexq_t6_bytes(4096, 4096, 128) == 64 * 32 * 6144
    assert L.flexq_t6_bytes(8192, 28672, 128) == 128 * 224 * 6144
    assert L.flexq_t6_bytes(100, 300, 128) == 2 * 3 * 6144          # 3 groups x 4 steps
    assert L.flexq_t6_bytes(10, 300, 999) == 1 * 3 * 6144           # 1 group of 300 -> 10 steps
    # 6 bits per weight exactly when everything is aligned
    assert L.flexq_t6_bytes(8192, 8192, 128) * 8 == 8192 * 8192 * 6
    assert L.flexq_act_frag_bytes(8, 4096, 128) == 32 * 1024
    assert L.flexq_gemm_workspace_bytes(1, 8192, 8192, 128, 0) > 0
    assert L.flexq_act_buf_bytes(1, 8192, 128) >= L.flexq_act_frag_bytes(8, 8192, 128)


def test_device_check_fails_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = _lib.load()
    assert L.flexq_device_check() == _lib.ERR_CUDA
    assert L.flexq_last_error()  # message recorded


def test_product_path_has_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2508_04405_b200 as fq

    with pytest.raises(fq.DeviceError):
        fq.quantize(np.ones((2, 128)), 6)
    with pytest.raises(fq.DeviceError):
        fq.quantized_linear(np.ones((8, 128)), np.ones((1, 128)))


def test_tc16_route_rule_and_override():
    """The kind::f16 batched route: measured size rule by default (>= 8192 units; for 128 < M
    <= 256 also any layer of >= 8192 rows), a process-wide override for A/B runs and tests."""
    L = _lib.load()  # host-only: routing needs no device
    assert L.flexq_set_tc16_route(5) == -2  # invalid mode: rejected, state unchanged
    prev = L.flexq_set_tc16_route(-1)
    try:
        assert L.flexq_linear_kernel(64, 28672, 8192, 128, 1) == _lib.KERNEL_TC16   # 70B gate
        assert L.flexq_linear_kernel(256, 28672, 8192, 128, 1) == _lib.KERNEL_TC16  # wide
        assert L.flexq_linear_kernel(256, 8192, 28672, 128, 1) == _lib.KERNEL_TC16  # long
        assert L.flexq_linear_kernel(256, 11008, 4096, 128, 1) == _lib.KERNEL_TC16  # wide, M > 128
        assert L.flexq_linear_kernel(128, 11008, 4096, 128, 1) != _lib.KERNEL_TC16  # same, M <= 128
        assert L.flexq_linear_kernel(256, 4096, 11008, 128, 1) != _lib.KERNEL_TC16  # narrow
        assert L.flexq_linear_kernel(64, 4096, 4096, 128, 0) != _lib.KERNEL_TC16    # fp32 scales
        assert L.flexq_set_tc16_route(1) == -1
        assert L.flexq_linear_kernel(64, 4096, 4096, 128, 1) == _lib.KERNEL_TC16    # forced
        assert L.flexq_linear_kernel(64, 4096, 4096, 64, 1) != _lib.KERNEL_TC16     # unsupported
        assert L.flexq_set_tc16_route(-1) == 1
    finally:
        L.flexq_set_tc16_route(prev)
