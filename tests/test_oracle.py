"""Pin the CPU oracle (numpy + C restatements) to the reference's golden vectors.

The golden vectors were produced by the real reference (tests/golden/make_golden.py);
every comparison here is exact (bit-for-bit), matching the reference's own
zero-tolerance oracle tests (test_acceptance.py:32-63, test_engine.py:108-161).
"""
import numpy as np
import pytest

from oracle import c_oracle, np_oracle


def test_quantize_numpy_and_c_match_reference(golden):
    for name in golden.names("q"):
        x = golden[f"q/{name}/x"]
        bits, gs, fp16 = (int(v) for v in golden[f"q/{name}/meta"])
        for impl in (np_oracle.quantize, c_oracle.quantize):
            codes, scales = impl(x, bits, gs, bool(fp16))
            assert np.array_equal(codes, golden[f"q/{name}/values"]), (name, impl)
            assert np.array_equal(scales, golden[f"q/{name}/scales"]), (name, impl)
        if fp16:  # fp16-valued inputs: the C oracle's fp16 loader must agree too
            codes, scales = c_oracle.quantize(x.astype(np.float16), bits, gs, True)
            assert np.array_equal(codes, golden[f"q/{name}/values"])
            assert np.array_equal(scales, golden[f"q/{name}/scales"])


def test_pack_numpy_and_c_match_reference(golden):
    for name in golden.names("p"):
        vals = golden[f"p/{name}/values"]
        rows, cols, bits, cm = (int(v) for v in golden[f"p/{name}/meta"])
        ref = golden[f"p/{name}/words"]
        got_np = np_oracle.pack_planes(np_oracle.bit_planes(vals, bits), cm)
        got_c = c_oracle.pack_planes(vals, bits, cm)
        assert got_np.tobytes() == ref.tobytes(), name
        assert got_c.tobytes() == ref.tobytes(), name
        back = np_oracle.recompose(np_oracle.unpack_planes(ref, bits, rows, cols), bits)
        assert np.array_equal(back, vals.astype(np.int64))


def test_gemm_oracles_bit_identical_to_reference(golden):
    for name in golden.names("g"):
        m, n, k, p, q, gs, passes = (int(v) for v in golden[f"g/{name}/meta"])
        wv, ws = golden[f"g/{name}/wv"], golden[f"g/{name}/ws"]
        xv, xs = golden[f"g/{name}/xv"], golden[f"g/{name}/xs"]
        y_ref, p_ref = golden[f"g/{name}/y"], golden[f"g/{name}/partials"]
        y, parts = np_oracle.int_matmul(wv, xv, ws, xs, gs, trace=True)
        assert np.array_equal(y, y_ref) and np.array_equal(parts, p_ref), name
        y, parts = c_oracle.int_matmul(wv, xv, ws, xs, gs, trace=True, threads=3)
        assert np.array_equal(y, y_ref) and np.array_equal(parts, p_ref), name
        ww = np_oracle.pack_planes(np_oracle.bit_planes(wv, p), 8)
        xw = np_oracle.pack_planes(np_oracle.bit_planes(xv, q), np_oracle.activation_chunk_m(m))
        y, parts, npass = np_oracle.bitserial_matmul(ww, xw, ws, xs, m, n, k, p, q, gs, trace=True)
        assert np.array_equal(y, y_ref) and np.array_equal(parts, p_ref), name
        assert npass == passes == np_oracle.bmma_passes(m, n, k, p, q, gs), name


def test_quantized_linear_oracle_matches_reference(golden):
    for name in golden.names("l"):
        w, x = golden[f"l/{name}/w"], golden[f"l/{name}/x"]
        p, q, gs, passes = (int(v) for v in golden[f"l/{name}/meta"])
        y, parts, npass = np_oracle.quantized_linear(w, x, p, q, gs, trace=True)
        assert np.array_equal(y, golden[f"l/{name}/y"]), name
        assert np.array_equal(parts, golden[f"l/{name}/partials"]), name
        assert npass == passes


def test_reference_kats_restated():
    # test_quantize.py:42-45, 87-91; test_engine.py:171-176
    c, s = np_oracle.quantize(np.array([[1.0, -1.0]]), 6, 2)
    assert c.tolist() == [[31, -31]] and s[0, 0] == pytest.approx(1 / 31)
    c, s = np_oracle.quantize(np.array([[2.5, -2.5, 31.0]]), 6, 3)
    assert c.tolist() == [[3, -3, 31]] and s[0, 0] == 1.0
    y, _, _ = np_oracle.quantized_linear(np.ones((1, 256)), np.ones((1, 256)), 6, 6, 128)
    assert y[0, 0] == pytest.approx(256.0)
    with pytest.raises(ValueError):
        c_oracle.quantize(np.array([[np.inf, 1.0]]), 6, 2)
