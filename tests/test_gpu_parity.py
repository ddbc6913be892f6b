"""GPU parity: the sm_100a library against the reference's golden vectors and the
CPU oracle.  Integer work (codes, packed words, INT32 group partials) must be
bit-exact; the drop-in float64 outputs are bit-exact too (exact epilogue); the
fp16 fast path must satisfy max|y - y_ref| <= 1e-3 * max|y_ref| against the
float64 oracle (the reference's own metric style, test_engine.py:163-169;
SURVEY.md sec. 8(a)).  Every reference test restated here cites its file:line.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU hosts, skipped there
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2508_04405_b200 as fq  # noqa: E402
from oracle import c_oracle, np_oracle  # noqa: E402
from paper_2508_04405_b200 import _lib  # noqa: E402
from paper_2508_04405_b200.engine import t6_pack_activations, t6_pack_weights  # noqa: E402

FP16_TOL = 1e-3


def max_rel(y, ref):
    return float(np.max(np.abs(np.asarray(y, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-300))


# ---------------------------------------------------------------- quantizer
def test_quantize_matches_reference_golden(golden):
    for name in golden.names("q"):
        x = golden[f"q/{name}/x"]
        bits, gs, fp16 = (int(v) for v in golden[f"q/{name}/meta"])
        q = fq.quantize(x, bits, gs, bool(fp16))
        assert isinstance(q.values, np.ndarray)
        assert np.array_equal(q.values, golden[f"q/{name}/values"]), name
        assert np.array_equal(q.scales, golden[f"q/{name}/scales"]), name
        if fp16:  # fp16 CUDA tensor in -> torch out, same codes (the hot-path dtype)
            qt = fq.quantize(torch.from_numpy(x.astype(np.float16)).cuda(), bits, gs, True)
            assert np.array_equal(qt.values.cpu().numpy(), golden[f"q/{name}/values"]), name
            assert np.array_equal(qt.scales.cpu().numpy(), golden[f"q/{name}/scales"]), name


def test_quantize_kats():  # test_quantize.py:22-91
    q = fq.quantize(np.array([[1.0, -1.0]]), 6, group_size=2)
    assert q.values.tolist() == [[31, -31]] and q.scales[0, 0] == pytest.approx(1 / 31)
    q = fq.quantize(np.array([[2.5, -2.5, 31.0]]), 6, group_size=3)
    assert q.values.tolist() == [[3, -3, 31]] and q.scales[0, 0] == 1.0
    q = fq.quantize(np.zeros((3, 8)), 6, group_size=4)
    assert not q.values.any() and np.all(q.scales == 1.0)
    assert fq.compute_group_scale(np.array([1.0, -1.0]), 6) == pytest.approx(1 / 31)
    assert fq.compute_group_scale(np.array([2.0, -0.5]), 8) == pytest.approx(2 / 127)
    assert fq.compute_group_scale(np.array([0.0, 0.0]), 6) == 1.0


def test_quantize_errors():  # test_quantize.py:31-35, 93-95; quantize.py:71-72, 132-140
    with pytest.raises(fq.InvalidInputError, match="non-finite"):
        fq.quantize(np.array([[np.inf, 1.0]]), 6, 2)
    with pytest.raises(fq.InvalidInputError, match="non-finite"):
        fq.compute_group_scale(np.array([1.0, np.nan]), 6)
    with pytest.raises(fq.InvalidInputError):
        fq.compute_group_scale(np.array([]), 6)
    with pytest.raises(fq.InvalidInputError):
        fq.quantize(np.ones((2, 4)), 9)
    with pytest.raises(fq.InvalidInputError):
        fq.quantize(np.ones(4), 6)
    # fp16 scale underflow -> non-positive scale, rejected like the reference's QuantTensor
    with pytest.raises(fq.InvalidInputError, match="strictly positive"):
        fq.quantize(np.full((1, 4), 1e-12), 6, 4, fp16_scales=True)


def test_quantize_round_trip_bound():  # test_acceptance.py:112-135 (criterion 4)
    rng = np.random.default_rng(7)
    for _ in range(5):
        x = rng.standard_normal((20, 20 * 128)) * rng.uniform(1e-3, 1e3, size=(20, 1))
        bits = int(rng.choice([6, 8]))
        q = fq.quantize(x, bits, 128)
        err = np.abs(x - fq.dequantize(q))
        per = np.repeat(q.scales, 128, axis=1)
        assert np.all(err <= per / 2 + 4 * np.spacing(np.abs(x)))
        assert q.values.min() >= -(2 ** (bits - 1) - 1)


def test_quantize_large_random_vs_c_oracle():
    rng = np.random.default_rng(11)
    for (rows, cols, bits, gs) in ((8, 28672, 8, 128), (3, 8192, 6, 8192), (64, 5120, 6, 64)):
        x = (rng.standard_normal((rows, cols)) * 3).astype(np.float16)
        x[:, 5] *= 60
        q = fq.quantize(torch.from_numpy(x).cuda(), bits, gs, True)
        codes, scales = c_oracle.quantize(x, bits, gs, True)
        assert np.array_equal(q.values.cpu().numpy(), codes)
        assert np.array_equal(q.scales.cpu().numpy(), scales)


# ---------------------------------------------------------------- packing
def test_pack_matches_reference_golden(golden):
    for name in golden.names("p"):
        vals = golden[f"p/{name}/values"]
        rows, cols, bits, cm = (int(v) for v in golden[f"p/{name}/meta"])
        for wb in (64, 32):
            cfg = fq.PackConfig(chunk_m=cm, word_bits=wb)
            p = fq.pack(fq.bit_planes(vals, bits), cfg)
            assert p.words.dtype == np.dtype("<u8" if wb == 64 else "<u4")
            assert p.words.tobytes() == golden[f"p/{name}/words"].tobytes(), (name, wb)
            back = fq.recompose(fq.unpack(p, cfg))
            assert np.array_equal(back, vals.astype(np.int64)), name


def test_pack_kats():  # test_packing.py:44-123
    rng = np.random.default_rng(0)
    q = fq.QuantTensor(rng.integers(-31, 32, (8, 256)).astype(np.int8), np.ones((8, 2)), 6, 128)
    p = fq.pack(fq.decompose(q), fq.weight_pack_config())
    assert p.words.shape == (2, 1, 6, 8, 2) and p.words.size == 192
    for col in (0, 1, 63, 64, 100, 127):  # LSB-first bit order
        planes = np.zeros((1, 1, 128), dtype=np.uint8)
        planes[0, 0, col] = 1
        bp = fq.BitPlaneSet(planes=planes, coeffs=np.array([1]), bits=1, signed=False)
        w = fq.pack(bp, fq.PackConfig(chunk_m=1)).words.ravel()
        assert w[col // 64] == np.uint64(1) << np.uint64(col % 64)
    with pytest.raises(fq.FormatError):
        fq.unpack(p, fq.PackConfig(chunk_m=4))
    # word_index is ravel order (test_packing.py:58-73)
    q = fq.QuantTensor(rng.integers(-3, 4, (9, 300)).astype(np.int8), np.ones((9, 3)), 3, 128)
    p = fq.pack(fq.decompose(q), fq.activation_pack_config(9))
    idx = [p.word_index(kc, rc, s, r, w) for kc in range(p.n_kchunks) for rc in range(p.n_rchunks)
           for s in range(p.bits) for r in range(p.config.chunk_m)
           for w in range(p.config.words_per_chunk)]
    assert idx == list(range(p.words.size))


def test_pack_large_vs_c_oracle():
    rng = np.random.default_rng(3)
    codes = rng.integers(-31, 32, (1000, 4100)).astype(np.int8)
    p = fq.pack(fq.bit_planes(codes, 6), fq.weight_pack_config())
    assert p.words.tobytes() == c_oracle.pack_planes(codes, 6, 8).tobytes()


def test_bit_planes_range_and_recompose():  # test_bitplane.py:36-73
    bp = fq.bit_planes(np.array([[-1]]), 6)
    assert bp.planes[:, 0, 0].tolist() == [1] * 6
    vals = np.arange(-32, 32).reshape(1, -1)
    assert np.array_equal(fq.recompose(fq.bit_planes(vals, 6)), vals)
    with pytest.raises(fq.InvalidInputError):
        fq.bit_planes(np.array([[-33]]), 6)
    with pytest.raises(fq.InvalidInputError):
        fq.bit_planes(np.array([[0.5]]), 6)


# ---------------------------------------------------------------- engine (drop-in, exact)
def _golden_case(golden, name):
    m, n, k, p, q, gs, passes = (int(v) for v in golden[f"g/{name}/meta"])
    wq = fq.QuantTensor(golden[f"g/{name}/wv"], golden[f"g/{name}/ws"], p, gs)
    xq = fq.QuantTensor(golden[f"g/{name}/xv"], golden[f"g/{name}/xs"], q, gs)
    cfg = fq.GemmConfig(m=m, n=n, k=k, weight_bits=p, activation_bits=q, group_size=gs)
    return wq, xq, cfg, passes


def test_group_matmul_fused_bit_identical_to_reference(golden):
    """Bit-serial AND+popcount kernel + exact epilogue (engine.py:290-334)."""
    for name in golden.names("g"):
        wq, xq, cfg, passes = _golden_case(golden, name)
        for wb in (64, 32):
            wp = fq.pack(fq.decompose(wq), fq.weight_pack_config(wb))
            xp = fq.pack(fq.decompose(xq), fq.activation_pack_config(cfg.m, wb))
            out = fq.group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg, trace=True)
            assert np.array_equal(out.data, golden[f"g/{name}/y"]), name
            assert np.array_equal(out.group_partials, golden[f"g/{name}/partials"]), name
            assert out.bmma_passes == passes


def test_int_matmul_reference_bit_identical(golden):
    """T6 tensor-core kernel + exact epilogue (engine.py:337-365)."""
    for name in golden.names("g"):
        wq, xq, cfg, _ = _golden_case(golden, name)
        out = fq.int_matmul_reference(wq, xq, cfg, trace=True)
        assert np.array_equal(out.data, golden[f"g/{name}/y"]), name
        assert np.array_equal(out.group_partials, golden[f"g/{name}/partials"]), name


def test_quantized_linear_bit_identical(golden):  # engine.py:487-513
    for name in golden.names("l"):
        p, q, gs, passes = (int(v) for v in golden[f"l/{name}/meta"])
        out = fq.quantized_linear(golden[f"l/{name}/w"], golden[f"l/{name}/x"], p, q, gs, trace=True)
        assert np.array_equal(out.data, golden[f"l/{name}/y"]), name
        assert np.array_equal(out.group_partials, golden[f"l/{name}/partials"]), name
        assert out.bmma_passes == passes


def test_engine_kats():  # test_engine.py:43-50, 171-197
    ones = np.full(2, 0xFFFFFFFFFFFFFFFF, dtype=np.uint64)
    assert fq.bmma_chunk(ones, ones) == 128
    a = np.full(2, 0xAAAAAAAAAAAAAAAA, dtype=np.uint64)
    b = np.full(2, 0x5555555555555555, dtype=np.uint64)
    assert fq.bmma_chunk(a, b) == 0
    with pytest.raises(fq.ShapeError):
        fq.bmma_chunk(np.zeros(2, np.uint64), np.zeros(3, np.uint64))
    assert fq.quantized_linear(np.ones((1, 256)), np.ones((1, 256)), 6, 6, 128).data[0, 0] == \
        pytest.approx(256.0)
    one = fq.QuantTensor(np.ones((1, 128), np.int8), np.ones((1, 1)), 6, 128)
    assert fq.int_matmul_reference(one, one, fq.GemmConfig(m=1, n=1, k=128)).data[0, 0] == 128.0
    rng = np.random.default_rng(13)
    wq = fq.QuantTensor(rng.integers(-31, 32, (16, 256)).astype(np.int8),
                        rng.uniform(0.25, 4, (16, 2)), 6, 128)
    xq = fq.quantize(np.zeros((4, 256)), 6, 128)
    cfg = fq.GemmConfig(m=4, n=16, k=256)
    out = fq.group_matmul_fused(fq.pack(fq.decompose(wq), fq.weight_pack_config()),
                                fq.pack(fq.decompose(xq), fq.activation_pack_config(4)),
                                wq.scales, xq.scales, cfg)
    assert not out.data.any()


def test_reduce_bits_and_fold():  # test_engine.py:64-101, 200-238; test_acceptance.py:66-88, 212-231
    s_vals = np.arange(-32, 32)
    ps = fq.bit_planes(s_vals[None, :], 6).planes[:, 0, :].astype(np.int64)
    grid = np.einsum("si,tj->stij", ps, ps)
    assert np.array_equal(fq.reduce_bits(grid, 6, 6), np.outer(s_vals, s_vals))
    a = np.arange(4)
    b = np.arange(16)
    pa = fq.bit_planes(a[None, :], 2, signed=False).planes[:, 0, :].astype(np.int64)
    pb = fq.bit_planes(b[None, :], 4, signed=False).planes[:, 0, :].astype(np.int64)
    assert np.array_equal(fq.reduce_bits(np.einsum("si,tj->stij", pa, pb), 2, 4, signed=False),
                          np.outer(a, b))
    rng = np.random.default_rng(1)
    wq = fq.QuantTensor(rng.integers(-15, 16, (6, 64)).astype(np.int8), np.ones((6, 1)), 5, 64)
    xq = fq.QuantTensor(rng.integers(-7, 8, (3, 64)).astype(np.int8), np.ones((3, 1)), 4, 64)
    got = fq.reduce_bits(fq.bit_product_grid(fq.decompose(wq), fq.decompose(xq)), 5, 4)
    assert np.array_equal(got, xq.values.astype(np.int64) @ wq.values.astype(np.int64).T)
    for mma_m in (1, 2, 4, 8):
        for chunk_m in (1, 2, 4, 8):
            if chunk_m > mma_m:
                continue
            lanes = rng.integers(-10**6, 10**6, size=(mma_m, 4, 3))
            folded, rounds = fq.fold_chunk_level(lanes, chunk_m, mma_m)
            assert rounds == mma_m.bit_length() - chunk_m.bit_length()
            for r in range(chunk_m):
                assert np.array_equal(folded[r], lanes[r::chunk_m].sum(axis=0))


def test_execute_tiled_determinism_and_validation():  # test_acceptance.py:159-189; test_engine.py:286-326
    rng = np.random.default_rng(20)
    wq = fq.QuantTensor(rng.integers(-31, 32, (32, 1024)).astype(np.int8),
                        rng.uniform(0.25, 4, (32, 8)), 6, 128)
    xq = fq.QuantTensor(rng.integers(-127, 128, (8, 1024)).astype(np.int8),
                        rng.uniform(0.25, 4, (8, 8)), 8, 128)
    wp = fq.pack(fq.decompose(wq), fq.weight_pack_config())
    xp = fq.pack(fq.decompose(xq), fq.activation_pack_config(8))
    base = fq.group_matmul_fused(wp, xp, wq.scales, xq.scales,
                                 fq.GemmConfig(m=8, n=32, k=1024, activation_bits=8)).data
    for stages in (1, 2, 4):
        for workers in (1, 2, 8):
            cfg = fq.GemmConfig(m=8, n=32, k=1024, activation_bits=8, bm=8, bn=16, bk=256,
                                pipeline_stages=stages, worker_count=workers)
            assert np.array_equal(fq.execute_tiled(wp, xp, wq.scales, xq.scales, cfg).data, base)
    with pytest.raises(fq.ConfigError):
        fq.execute_tiled(wp, xp, wq.scales, xq.scales,
                         fq.GemmConfig(m=8, n=32, k=1024, activation_bits=8, bk=200))
    with pytest.raises(fq.ShapeError):
        fq.group_matmul_fused(wp, xp, wq.scales[:, :1], xq.scales,
                              fq.GemmConfig(m=8, n=32, k=1024, activation_bits=8))


def test_criterion1_random_cases_vs_oracle():  # test_acceptance.py:32-63 (scaled to 150 cases)
    rng = np.random.default_rng(20240801)
    for _ in range(150):
        m = int(rng.choice([1, 4, 8, 16]))
        n = int(rng.integers(8, 257))
        k = int(rng.integers(128, 4097))
        p, q = (6, 6) if rng.integers(2) else (6, 8)
        wq = fq.QuantTensor(rng.integers(-31, 32, (n, k)).astype(np.int8),
                            rng.uniform(0.25, 4, (n, -(-k // 128))), p, 128)
        xq = fq.QuantTensor(rng.integers(-(2 ** (q - 1) - 1), 2 ** (q - 1), (m, k)).astype(np.int8),
                            rng.uniform(0.25, 4, (m, -(-k // 128))), q, 128)
        cfg = fq.GemmConfig(m=m, n=n, k=k, weight_bits=p, activation_bits=q)
        y_ref, p_ref = c_oracle.int_matmul(wq.values, xq.values, wq.scales, xq.scales, 128, trace=True)
        out = fq.int_matmul_reference(wq, xq, cfg, trace=True)
        assert np.array_equal(out.data, y_ref) and np.array_equal(out.group_partials, p_ref)
        wp = fq.pack(fq.decompose(wq), fq.weight_pack_config())
        xp = fq.pack(fq.decompose(xq), fq.activation_pack_config(m))
        out = fq.group_matmul_fused(wp, xp, wq.scales, xq.scales, cfg, trace=True)
        assert np.array_equal(out.data, y_ref) and np.array_equal(out.group_partials, p_ref)


# ---------------------------------------------------------------- production fast path
def _fast_case(m, n, k, q, gs, seed=0, outlier=True):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((n, k)).astype(np.float16)
    x = rng.standard_normal((m, k)).astype(np.float16)
    if outlier:
        x[:, 3] *= 60  # an outlier channel (sensitivity.py:189-190 style)
    wc, wsc = c_oracle.quantize(w, 6, gs, True)
    xc, xsc = c_oracle.quantize(x, q, gs, True)
    y_ref, p_ref = c_oracle.int_matmul(wc, xc, wsc, xsc, gs, trace=True)
    return w, x, (wc, wsc, xc, xsc), y_ref, p_ref


def _run_t6(codes, m, n, k, gs, trace=True, ksplit=0):
    wc, wsc, xc, xsc = codes
    L = _lib.lib()
    t6, wsp = t6_pack_weights(torch.from_numpy(wc).cuda(), torch.from_numpy(wsc).cuda(), k, gs, True)
    frag, xs, corr, m_pad = t6_pack_activations(torch.from_numpy(xc).cuda(),
                                                torch.from_numpy(xsc).cuda(), k, gs)
    ng = -(-k // gs)
    parts = torch.zeros((ng, m, n), dtype=torch.int32, device="cuda") if trace else None
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    ws = torch.zeros(L.flexq_gemm_workspace_bytes(m, n, k, gs, ksplit), dtype=torch.uint8,
                     device="cuda")
    _lib.check(L.flexq_gemm_t6(_lib.ptr(t6), _lib.ptr(wsp), 1, _lib.ptr(frag), _lib.ptr(xs),
                               _lib.ptr(corr), m, m_pad, n, k, gs, _lib.ptr(parts), _lib.ptr(y),
                               _lib.OUT_F16, _lib.ptr(ws), ksplit, _lib.stream()))
    torch.cuda.synchronize()
    return y.float().cpu().numpy(), (parts.cpu().numpy() if trace else None)


LLAMA = [  # (m, n, k, q): LLaMA-2 7B/13B/70B linear shapes
    (1, 4096, 4096, 8), (8, 11008, 4096, 6), (4, 4096, 11008, 8), (1, 15360, 5120, 6),
    (8, 5120, 13824, 8), (1, 10240, 8192, 6), (2, 28672, 8192, 6), (1, 8192, 28672, 8),
    (8, 8192, 28672, 8), (16, 8192, 8192, 6),
    (32, 28672, 8192, 6), (24, 8192, 28672, 8), (17, 4096, 11008, 8),  # streaming GEMV, MT = 4
]


@pytest.mark.parametrize("m,n,k,q", LLAMA)
def test_t6_fast_path_llama_shapes(m, n, k, q):
    """Exact INT32 partials through the fast kernel + fp16 within tolerance at full size."""
    _, _, codes, y_ref, p_ref = _fast_case(m, n, k, q, 128, seed=m * n + k)
    y, parts = _run_t6(codes, m, n, k, 128)
    assert np.array_equal(parts, p_ref)
    assert max_rel(y, y_ref) <= FP16_TOL


@pytest.mark.parametrize("m,n,k,q,gs", [
    (1, 1000, 1024, 6, 32), (3, 200, 1024, 8, 64), (5, 256, 2048, 6, 256), (2, 512, 4096, 8, 4096),
    (16, 384, 896, 6, 128), (12, 130, 640, 8, 100), (9, 1024, 1536, 6, 512), (1, 64, 128, 6, 128),
    (20, 96, 1024, 8, 128), (64, 128, 512, 6, 128), (100, 72, 384, 8, 128), (1, 8, 300, 6, 128),
    (25, 136, 1024, 6, 128), (32, 8, 300, 8, 128), (31, 1000, 4096, 6, 128),  # MT = 4 stream
])
def test_t6_group_sizes_and_batches(m, n, k, q, gs):
    _, _, codes, y_ref, p_ref = _fast_case(m, n, k, q, gs, seed=gs + m)
    # 16 < M <= 32 at group 128: force the streaming GEMV (automatic only for large layers)
    y, parts = _run_t6(codes, m, n, k, gs, ksplit=-3 if 16 < m <= 32 and gs == 128 else 0)
    assert np.array_equal(parts, p_ref)
    assert max_rel(y, y_ref) <= FP16_TOL


@pytest.mark.parametrize("m", [1, 4, 8, 13, 16, 28, 33])
def test_flexq_linear_public_api(m):
    """FlexQLinear (fused quantizer + GEMM from fp16 x) vs the oracle on fp16 inputs."""
    n, k = 2048, 4096
    w, x, _, y_ref, _ = _fast_case(m, n, k, 8, 128, seed=m)
    lin = fq.FlexQLinear(w, activation_bits=8)
    y = lin(torch.from_numpy(x).cuda()).float().cpu().numpy()
    assert max_rel(y, y_ref) <= FP16_TOL
    y2 = lin(torch.from_numpy(x).cuda()).float().cpu().numpy()
    assert np.array_equal(y, y2)  # deterministic run to run
    lin.check_errors()


def test_flexq_linear_policy_and_errors():
    w = np.random.default_rng(0).standard_normal((256, 512)).astype(np.float16)
    assert fq.FlexQLinear(w, layer_kind="down_proj").activation_bits == 8
    assert fq.FlexQLinear(w, layer_kind="o_proj").activation_bits == 6
    lin = fq.FlexQLinear(w)
    x = torch.ones((2, 512), dtype=torch.float16, device="cuda")
    x[0, 7] = float("nan")
    lin(x)
    with pytest.raises(fq.InvalidInputError, match="non-finite"):
        lin.check_errors()
    with pytest.raises(fq.ShapeError):
        lin(torch.ones((2, 256), dtype=torch.float16, device="cuda"))


def test_bitserial_fast_epilogue():
    """The BTC-equivalent kernel's own fp32 epilogue (the bench's bitserial leg)."""
    m, n, k, q = 4, 1024, 4096, 8
    _, _, (wc, wsc, xc, xsc), y_ref, _ = _fast_case(m, n, k, q, 128)
    L = _lib.lib()
    wp = fq.pack(fq.bit_planes(wc, 6), fq.weight_pack_config())
    xp = fq.pack(fq.bit_planes(xc, q), fq.activation_pack_config(m))
    y = torch.empty((m, n), dtype=torch.float32, device="cuda")
    ws = torch.zeros(L.flexq_gemm_workspace_bytes(m, n, k, 128, 0), dtype=torch.uint8, device="cuda")
    wsd, xsd = torch.from_numpy(wsc).float().cuda(), torch.from_numpy(xsc).float().cuda()
    _lib.check(L.flexq_gemm_bitserial(
        _lib.ptr(wp.device_bytes()), _lib.ptr(xp.device_bytes()), _lib.ptr(wsd), _lib.ptr(xsd),
        m, n, k, 6, q, 128, 8, m, None, _lib.ptr(y), _lib.OUT_F32, _lib.ptr(ws), 0, _lib.stream()))
    torch.cuda.synchronize()
    assert max_rel(y.cpu().numpy(), y_ref) <= FP16_TOL


def test_exact_epilogue_fp16_is_correctly_rounded():
    """flexq_group_epilogue_f64's fp16 output == fp16(reference float64 y)."""
    m, n, k = 3, 512, 2048
    _, _, (wc, wsc, xc, xsc), y_ref, p_ref = _fast_case(m, n, k, 6, 128)
    L = _lib.lib()
    parts = torch.from_numpy(p_ref).cuda()
    wsd, xsd = torch.from_numpy(wsc).cuda(), torch.from_numpy(xsc).cuda()  # keep alive
    y = torch.empty((m, n), dtype=torch.float64, device="cuda")
    y16 = torch.empty((m, n), dtype=torch.float16, device="cuda")
    _lib.check(L.flexq_group_epilogue_f64(_lib.ptr(parts), _lib.ptr(wsd), _lib.ptr(xsd), m, n, 16,
                                          _lib.ptr(y), _lib.ptr(y16), _lib.stream()))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), y_ref)
    assert np.array_equal(y16.cpu().numpy(), y_ref.astype(np.float16))


def test_70b_down_proj_full_size_properties():
    """70B down_proj (N=8192, K=28672, W6A8) at M=8 through FlexQLinear: tolerance vs the
    oracle, plus linearity in x's scale (power-of-two scaling is exact in the codes)."""
    m, n, k = 8, 8192, 28672
    w, x, _, y_ref, _ = _fast_case(m, n, k, 8, 128, seed=70)
    lin = fq.FlexQLinear(w, layer_kind="down_proj")
    xt = torch.from_numpy(x).cuda()
    y = lin(xt).float().cpu().numpy()
    assert max_rel(y, y_ref) <= FP16_TOL
    y4 = lin(xt * 4).float().cpu().numpy()  # codes identical, activation scales exactly x4
    assert np.array_equal(y4, 4 * y)


def test_quantizer_fast_path_matches_generic():
    """fp16 / group-128 fast kernel == the generic float64 kernel (fed the same values as
    fp32) on every output, including exact ties, zeros, subnormals and an all-zero group."""
    L = _lib.lib()
    g = torch.Generator(device="cuda").manual_seed(11)
    m, k = 5, 1024
    x = (torch.randn((m, k), generator=g, device="cuda") * 3).half()
    x[0, :128] = 0                                              # all-zero group -> scale 1
    x[1, 128:256] = torch.arange(128, device="cuda").half() * 0.5  # many exact half-step ties
    x[2, 256:260] = torch.tensor([6e-8, -6e-8, 1e-5, 65504.0]).half()
    x[3, 512:640] = torch.linspace(-31, 31, 128, device="cuda").half()
    outs = []
    for dt, src in ((_lib.DT_F16, x), (_lib.DT_F32, x.float())):
        for bits in (6, 8):
            m_pad = L.flexq_act_m_pad(m)
            codes = torch.zeros((m, k), dtype=torch.int8, device="cuda")
            scales = torch.zeros((m, k // 128), dtype=torch.float64, device="cuda")
            frag = torch.zeros(L.flexq_act_frag_bytes(m_pad, k, 128) // 4, dtype=torch.int32,
                               device="cuda")
            xs = torch.zeros((k // 128, m_pad), dtype=torch.float32, device="cuda")
            corr = torch.zeros((k // 128, m_pad), dtype=torch.int32, device="cuda")
            flag = torch.zeros(1, dtype=torch.int32, device="cuda")
            _lib.check(L.flexq_quantize(_lib.ptr(src), dt, m, k, bits, 128, 1, _lib.ptr(codes),
                                        _lib.ptr(scales), _lib.ptr(frag), _lib.ptr(xs),
                                        _lib.ptr(corr), m_pad, _lib.ptr(flag), _lib.stream()))
            outs.append((codes, scales, frag, xs, corr))
    torch.cuda.synchronize()
    for a, b in zip(outs[:2], outs[2:]):
        for ta, tb in zip(a, b):
            assert torch.equal(ta, tb)
    # and against the reference restatement on the host
    xc, xsc = c_oracle.quantize(x.cpu().numpy(), 6, 128, True)
    assert np.array_equal(outs[0][0].cpu().numpy(), xc)
    assert np.array_equal(outs[0][1].cpu().numpy(), xsc)
