"""GPU parity of the batched (M > 16) tcgen05.mma kind::i8 GEMM (csrc/gemm_tc.cu).

Same bar as the decode kernels: INT32 group partials bit-exact against the CPU
oracle's int_matmul_reference restatement (engine.py:337-365), fp16 y within
max|y - y_ref| <= 1e-3 * max|y_ref| of the float64 oracle, identical partials to
the mma.sync kernel, and run-to-run bit-identical outputs (the stream-K fixup
combines split tiles in a fixed CTA order).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU hosts, skipped there
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2508_04405_b200 as fq  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_2508_04405_b200 import _lib  # noqa: E402
from paper_2508_04405_b200.engine import t6_pack_activations, t6_pack_weights  # noqa: E402

FP16_TOL = 1e-3
# ksplit: 0 = auto (streaming GEMV up to M = 32 at group 128, tcgen05 above), -1 = the
# mma.sync kernel, -2 = tcgen05 whenever it supports the shape (M > 16)
AUTO, LEGACY, TC, STREAM = 0, -1, -2, -3


def max_rel(y, ref):
    return float(np.max(np.abs(np.asarray(y, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-300))


def case(m, n, k, q, gs, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((n, k)).astype(np.float16)
    x = rng.standard_normal((m, k)).astype(np.float16)
    x[:, 5] *= 80  # outlier channel: full-range A8 codes
    wc, wsc = c_oracle.quantize(w, 6, gs, True)
    xc, xsc = c_oracle.quantize(x, q, gs, True)
    y_ref, p_ref = c_oracle.int_matmul(wc, xc, wsc, xsc, gs, trace=True)
    return w, x, (wc, wsc, xc, xsc), y_ref, p_ref


def run(codes, m, n, k, gs, ksplit=TC, trace=True, fast=True):
    wc, wsc, xc, xsc = codes
    L = _lib.lib()
    t6, wsp = t6_pack_weights(torch.from_numpy(wc).cuda(), torch.from_numpy(wsc).cuda(), k, gs, True)
    frag, xs, corr, m_pad = t6_pack_activations(torch.from_numpy(xc).cuda(),
                                                torch.from_numpy(xsc).cuda(), k, gs)
    ng = -(-k // gs)
    parts = torch.zeros((ng, m, n), dtype=torch.int32, device="cuda") if trace else None
    y = torch.empty((m, n), dtype=torch.float16, device="cuda") if fast else None
    ws = torch.zeros(L.flexq_gemm_workspace_bytes(m, n, k, gs, ksplit), dtype=torch.uint8,
                     device="cuda")
    _lib.check(L.flexq_gemm_t6(_lib.ptr(t6), _lib.ptr(wsp), 1, _lib.ptr(frag), _lib.ptr(xs),
                               _lib.ptr(corr), m, m_pad, n, k, gs, _lib.ptr(parts), _lib.ptr(y),
                               _lib.OUT_F16, _lib.ptr(ws), ksplit, _lib.stream()))
    torch.cuda.synchronize()
    return (y.float().cpu().numpy() if fast else None), (parts.cpu().numpy() if trace else None)


def test_act_m_pad():
    L = _lib.lib()
    assert [L.flexq_act_m_pad(m) for m in (1, 8, 9, 16, 17, 32, 33, 64, 65, 128, 129, 256)] == \
        [8, 8, 16, 16, 32, 32, 64, 64, 128, 128, 256, 256]


@pytest.mark.parametrize("m,n,k,q,gs", [
    (17, 128, 256, 6, 128),     # smallest tcgen05 batch, one tile
    (32, 384, 1024, 8, 128),    # TN = 32
    (48, 136, 1024, 6, 128),    # odd number of 64-row groups: half-empty last tile
    (64, 1000, 2048, 8, 128),   # TN = 64, N not a multiple of 128
    (65, 256, 1024, 6, 256),    # TN = 128, two k-blocks per group
    (128, 512, 1536, 8, 384),   # three k-blocks per group
    (129, 384, 1024, 6, 128),   # two token tiles
    (200, 640, 2048, 8, 1024),  # long group: drained every 512 k, correction once per group
    (256, 256, 2048, 6, 2048),  # per-channel (group = K)
    (32, 128, 8192, 8, 128),    # one tile split across 64 CTAs: deep stream-K fixup
])
def test_tc_partials_and_fast_path(m, n, k, q, gs):
    _, _, codes, y_ref, p_ref = case(m, n, k, q, gs, seed=m * 7 + n + gs)
    y, parts = run(codes, m, n, k, gs)
    assert np.array_equal(parts, p_ref)
    assert max_rel(y, y_ref) <= FP16_TOL
    y2, _ = run(codes, m, n, k, gs, trace=False)
    assert np.array_equal(y, y2)  # trace on/off and run to run: identical fp16 output


@pytest.mark.parametrize("m,n,k,q", [(64, 5120, 5120, 6), (256, 5120, 5120, 6), (96, 13824, 5120, 6),
                                     (48, 5120, 13824, 8)])
def test_tc_llama13b_shapes(m, n, k, q):
    """LLaMA-2-13B linear shapes across the GEMV-to-GEMM crossover (BASELINE config 3)."""
    _, _, codes, y_ref, p_ref = case(m, n, k, q, 128, seed=m + n)
    y, parts = run(codes, m, n, k, 128)
    assert np.array_equal(parts, p_ref)
    assert max_rel(y, y_ref) <= FP16_TOL


LLAMA70B = {  # name: (N, K, q) -- the shapes the bench step serves (bench.py)
    "qkv_proj": (10240, 8192, 6),
    "o_proj": (8192, 8192, 6),
    "gate_proj": (28672, 8192, 6),
    "down_proj": (8192, 28672, 8),  # 224 k-blocks: deepest stream-K split
}
_CASES70 = {}


def _case70(name, m):
    key = (name, m)
    if key not in _CASES70:
        _CASES70.clear()  # one live case at a time: partials at M = 256 are ~2 GB
        n, k, q = LLAMA70B[name]
        _CASES70[key] = (n, k, case(m, n, k, q, 128, seed=m + n + k)[2:])
    return _CASES70[key]


@pytest.mark.parametrize("name", list(LLAMA70B))
@pytest.mark.parametrize("m", [33, 64, 128, 256])
@pytest.mark.parametrize("ksplit", [AUTO, TC])
def test_tc_llama70b_shapes(name, m, ksplit):
    """LLaMA-2-70B layers at the batches the tcgen05 route serves automatically (M > 32):
    INT32 partials bit-exact against int_matmul_reference(trace=True) (engine.py:337-365),
    fp16 y in tolerance, the automatic route identical to the forced tcgen05 route."""
    n, k, (codes, y_ref, p_ref) = _case70(name, m)
    y, parts = run(codes, m, n, k, 128, ksplit=ksplit)
    assert np.array_equal(parts, p_ref)
    del parts
    assert max_rel(y, y_ref) <= FP16_TOL


@pytest.mark.parametrize("name,m", [("gate_proj", 64), ("gate_proj", 128), ("down_proj", 64),
                                    ("down_proj", 128)])
def test_linear_llama70b_batched(name, m):
    """FlexQLinear (fused quantizer -> tcgen05 GEMM, fp16 in/out) on the 70B layers."""
    n, k, q = LLAMA70B[name]
    w, x, _, y_ref, _ = case(m, n, k, q, 128, seed=5 * m + n)
    lin = fq.FlexQLinear(w, activation_bits=q)
    y = lin(torch.from_numpy(x).cuda()).float().cpu().numpy()
    assert max_rel(y, y_ref) <= FP16_TOL
    lin.check_errors()


def test_tc_matches_mma_sync_kernel():
    m, n, k, q, gs = 80, 768, 3072, 8, 128
    _, _, codes, y_ref, p_ref = case(m, n, k, q, gs, seed=3)
    y_tc, p_tc = run(codes, m, n, k, gs, TC)
    y_ms, p_ms = run(codes, m, n, k, gs, LEGACY)
    assert np.array_equal(p_tc, p_ref) and np.array_equal(p_ms, p_ref)
    assert max_rel(y_tc, y_ref) <= FP16_TOL and max_rel(y_ms, y_ref) <= FP16_TOL


@pytest.mark.parametrize("m", [17, 32])
def test_stream_and_tc_agree_at_small_batches(m):
    """M in (16, 32] at group 128: the streaming GEMV (MT = 4; automatic for layers of >= 8192
    units) and the tcgen05 kernel give identical INT32 partials and fp16 outputs in tolerance."""
    n, k, gs = 640, 2048, 128
    _, _, codes, y_ref, p_ref = case(m, n, k, 8, gs, seed=11 * m)
    y_a, p_a = run(codes, m, n, k, gs, STREAM)
    y_t, p_t = run(codes, m, n, k, gs, TC)
    assert np.array_equal(p_a, p_ref) and np.array_equal(p_t, p_ref)
    assert max_rel(y_a, y_ref) <= FP16_TOL and max_rel(y_t, y_ref) <= FP16_TOL


@pytest.mark.parametrize("m", [24, 100, 256])
def test_tc_public_api(m):
    """FlexQLinear.__call__ at batched M: fused quantizer -> tcgen05 GEMM."""
    n, k = 1536, 4096
    w, x, _, y_ref, _ = case(m, n, k, 6, 128, seed=m)
    lin = fq.FlexQLinear(w, activation_bits=6)
    y = lin(torch.from_numpy(x).cuda()).float().cpu().numpy()
    assert max_rel(y, y_ref) <= FP16_TOL
    lin.check_errors()


@pytest.mark.parametrize("m", [1, 8, 33, 100])
def test_fused_residual_epilogue(m):
    """y = x W^T + r in the GEMM epilogue (GEMV for M <= 16, tcgen05 above), r aliasing y."""
    n, k = 1024, 2048
    g = torch.Generator(device="cuda").manual_seed(m)
    lin = fq.FlexQLinear(torch.randn((n, k), generator=g, device="cuda").half(), activation_bits=6)
    x = torch.randn((m, k), generator=g, device="cuda").half()
    r = torch.randn((m, n), generator=g, device="cuda").half()
    y0 = lin(x).float()
    y = r.clone()
    lin.forward(x, out=y, residual=y)  # in place: y <- x W^T + y
    ref = y0 + r.float()
    assert torch.allclose(y.float(), ref, atol=1e-2, rtol=2e-3)
    y2 = torch.empty_like(r)
    lin.forward(x, out=y2, residual=r)  # separate residual buffer
    assert torch.equal(y2, y)


@pytest.mark.parametrize("m,n,k,q", [
    (33, 256, 1024, 6),       # smallest tile-64 batch
    (48, 136, 2048, 8),       # odd row count: half-empty last 128-row tile
    (64, 1000, 4096, 6),      # N not a multiple of 128, split tiles
    (100, 640, 8192, 8),      # tile 128, deep stream-K
    (128, 384, 28672, 8),     # down_proj K: 224 k-blocks
    (129, 8200, 8192, 6),     # 256-token tile (single accumulator); >= 8192 units to take it
    (256, 8192, 8192, 8),     # M = 256
])
def test_tc16_fast_path(m, n, k, q):
    """The batched fast path (csrc/gemm_tc16.cu: tcgen05 kind::f16 over fp16(w*ws) and
    fp16(code*xs), fp32 accumulation): the same quantizer codes and scales as the reference,
    fp16 y within max|y - y_ref| <= 1e-3 * max|y_ref| of int_matmul_reference (engine.py:
    337-365); gemm_only replays the identical output; run to run bit-identical."""
    L = _lib.lib()
    prev = L.flexq_set_tc16_route(1)  # small shapes: the size rule would pick kind::i8
    try:
        _tc16_case(L, m, n, k, q)
    finally:
        L.flexq_set_tc16_route(prev)


def _tc16_case(L, m, n, k, q):
    assert L.flexq_linear_kernel(m, n, k, 128, 1) == _lib.KERNEL_TC16
    w, x, _, y_ref, _ = case(m, n, k, q, 128, seed=17 * m + n)
    lin = fq.FlexQLinear(w, activation_bits=q)
    xd = torch.from_numpy(x).cuda()
    y = lin(xd)
    assert max_rel(y.float().cpu().numpy(), y_ref) <= FP16_TOL
    y2 = lin(xd)
    assert torch.equal(y, y2)
    y3 = torch.empty_like(y)
    lin.gemm_only(m, y3)
    assert torch.equal(y, y3)
    r = torch.randn_like(y)
    y4 = r.clone()
    lin.forward(xd, out=y4, residual=y4)
    assert torch.allclose(y4.float(), y.float() + r.float(), atol=1e-2, rtol=2e-3)
    lin.check_errors()
