"""GEMM engine on the B200 (drop-in for bitserial.engine).

Every public function keeps the reference's signature, validation and error
messages (engine.py); the arithmetic runs in libflexq_sm100a:

* ``group_matmul_fused`` / ``execute_tiled`` over FLXQ-P packed operands ->
  the bit-serial AND+popcount kernel (csrc/bitserial.cu, the paper's BTC
  formulation) writing exact INT32 group partials, then the exact float64
  epilogue (csrc/epilogue.cu).
* ``int_matmul_reference`` / ``quantized_linear`` -> the production
  unpack-to-INT8 tensor-core kernel over the T6 layout (csrc/gemm_t6.cu), same
  partials, same epilogue.

Both epilogues reproduce _scale_accumulate (engine.py:211-216) operation for
operation, so ``GemmOutput.data`` is bit-identical with the reference's
float64 result and ``group_partials`` with its traced integers.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Any

import numpy as np

from . import _dev, _lib
from .bitplane import BitPlaneSet, decompose
from .errors import ConfigError, ShapeError
from .packing import PackedTensor, activation_pack_config, pack, weight_pack_config
from .quantize import DEFAULT_GROUP_SIZE, QuantTensor, quantize


@dataclass(frozen=True)
class GemmConfig:
    """Problem shape, precision pair, grouping and tiling knobs (engine.py:31-70).

    The tile/pipeline knobs (bm, bn, bk, pipeline_stages, worker_count) are
    validated exactly as the reference does; on the GPU the CTA tiling is
    chosen by the kernels and results never depend on these knobs
    (determinism contract, engine.py:411).
    """

    m: int
    n: int
    k: int
    weight_bits: int = 6
    activation_bits: int = 6
    group_size: int = DEFAULT_GROUP_SIZE
    bm: int = 8
    bn: int = 64
    bk: int = 512
    pipeline_stages: int = 1
    worker_count: int = 1

    def __post_init__(self):
        if min(self.m, self.n, self.k) < 1:
            raise ConfigError(f"dims must be positive, got {(self.m, self.n, self.k)}")
        for name in ("weight_bits", "activation_bits"):
            b = getattr(self, name)
            if not 2 <= b <= 8:
                raise ConfigError(f"{name} must be in 2..8, got {b}")
        if self.group_size < 1:
            raise ConfigError(f"group_size must be >= 1, got {self.group_size}")
        if min(self.bm, self.bn, self.bk) < 1:
            raise ConfigError(f"tile dims must be positive, got {(self.bm, self.bn, self.bk)}")
        if self.pipeline_stages < 1:
            raise ConfigError(f"pipeline_stages must be >= 1, got {self.pipeline_stages}")
        if self.worker_count < 1:
            raise ConfigError(f"worker_count must be >= 1, got {self.worker_count}")

    @property
    def n_groups(self) -> int:
        return -(-self.k // self.group_size)


@dataclass
class GemmOutput:
    """Result + instrumentation (engine.py:73-86): data [m, n] float64, the
    analytic bmma pass count and optional exact int64 partials [G, m, n]."""

    data: Any
    bmma_passes: int = 0
    group_partials: Any = None


# ---- small helpers of the reference API, evaluated on the GPU -------------------------

def bmma_chunk(w_words, x_words) -> int:
    """sum popcount(w & x) over two equal word spans (engine.py:89-95)."""
    w = w_words if _dev.is_torch(w_words) else np.asarray(w_words)
    x = x_words if _dev.is_torch(x_words) else np.asarray(x_words)
    if w.ndim != 1 or x.ndim != 1 or tuple(w.shape) != tuple(x.shape):
        raise ShapeError(f"word spans must be equal 1-D, got {tuple(w.shape)} and {tuple(x.shape)}")
    t = _dev.torch()
    wb = _dev.to_device(w.view(np.uint8) if not _dev.is_torch(w) else w).contiguous().view(t.uint8)
    xb = _dev.to_device(x.view(np.uint8) if not _dev.is_torch(x) else x).contiguous().view(t.uint8)
    out = t.empty(1, dtype=t.int64, device=wb.device)
    _lib.check(_lib.lib().flexq_popcount_and(_lib.ptr(wb), _lib.ptr(xb), wb.numel(), _lib.ptr(out),
                                             _lib.stream()))
    return int(out.item())


def bit_product_grid(w_planes: BitPlaneSet, x_planes: BitPlaneSet):
    """Dense Y^(s,t)[m,n] = sum_k w_s[n,k] x_t[m,k] (engine.py:98-111), on the GPU."""
    if w_planes.shape[1] != x_planes.shape[1]:
        raise ShapeError(f"contraction mismatch: weights K={w_planes.shape[1]}, "
                         f"activations K={x_planes.shape[1]}")
    t = _dev.torch()
    w = _dev.to_device(w_planes.planes, t.float64)
    x = _dev.to_device(x_planes.planes, t.float64)
    grid = t.einsum("snk,tmk->stmn", w, x).round().to(t.int64)  # exact: sums < 2^53
    return _dev.to_host(grid) if w_planes._numpy else grid


def reduce_bits(partials, weight_bits: int, activation_bits: int, signed: bool = True):
    """sum_s sum_t coeff(s) coeff(t) partials[s, t] (engine.py:114-130), on the GPU."""
    from .bitplane import plane_coeffs

    is_t = _dev.is_torch(partials)
    arr = partials if is_t else np.asarray(partials)
    if arr.ndim < 2 or arr.shape[0] != weight_bits or arr.shape[1] != activation_bits:
        raise ShapeError(f"partials must be [{weight_bits}, {activation_bits}, ...], "
                         f"got {tuple(arr.shape)}")
    t = _dev.torch()
    g = _dev.to_device(arr, t.int64)
    cw = t.as_tensor(plane_coeffs(weight_bits, signed), device=g.device)
    cx = t.as_tensor(plane_coeffs(activation_bits, signed), device=g.device)
    coef = (cw[:, None] * cx[None, :]).reshape(weight_bits, activation_bits, *([1] * (g.ndim - 2)))
    out = (coef * g).sum(dim=(0, 1))
    return out if is_t else _dev.to_host(out)


def fold_chunk_level(lane_partials, chunk_m: int, mma_m: int):
    """Tree fold of mma_m lane groups down to chunk_m (engine.py:133-157).

    The register-exchange (__shfl_xor_sync) reduction the GEMV kernel performs
    for batches below the mma tile; log2(mma_m) - log2(chunk_m) rounds.
    """
    for name, v in (("chunk_m", chunk_m), ("mma_m", mma_m)):
        if v < 1 or v & (v - 1):
            raise ConfigError(f"{name} must be a power of two, got {v}")
    if chunk_m > mma_m:
        raise ConfigError(f"chunk_m ({chunk_m}) must not exceed mma_m ({mma_m})")
    is_t = _dev.is_torch(lane_partials)
    arr = lane_partials if is_t else np.array(lane_partials)
    if arr.shape[0] != mma_m:
        raise ShapeError(f"expected {mma_m} lane groups on axis 0, got {arr.shape[0]}")
    lanes = _dev.to_device(arr).clone()
    active, rounds = mma_m, 0
    while active > chunk_m:
        half = active // 2
        lanes[:half] += lanes[half:active]
        active, rounds = half, rounds + 1
    out = lanes[:chunk_m]
    return (out if is_t else _dev.to_host(out)), rounds


# ---- pass accounting (engine.py:165-180, 283) --------------------------------------------

def _span_count(n_groups: int, group_size: int, k_pad: int, chunk_k: int = 128) -> int:
    total = 0
    for g in range(n_groups):
        lo = g * group_size
        hi = k_pad if g == n_groups - 1 else (g + 1) * group_size
        total += -(-hi // chunk_k) - lo // chunk_k
    return total


def bmma_passes(cfg: GemmConfig, x_chunk_m: int, w_chunk_m: int = 8) -> int:
    """p*q passes per (activation chunk, weight chunk, group span) (engine.py:283)."""
    k_pad = -(-cfg.k // 128) * 128
    spans = _span_count(cfg.n_groups, cfg.group_size, k_pad)
    return (cfg.weight_bits * cfg.activation_bits * (-(-cfg.m // x_chunk_m))
            * (-(-cfg.n // w_chunk_m)) * spans)


# ---- GPU cores -----------------------------------------------------------------------------

def _epilogue_f64(parts, ws, xs, m, n, ng):
    t = _dev.torch()
    y = t.empty((m, n), dtype=t.float64, device=parts.device)
    _lib.check(_lib.lib().flexq_group_epilogue_f64(_lib.ptr(parts), _lib.ptr(ws), _lib.ptr(xs), m, n,
                                                   ng, _lib.ptr(y), None, _lib.stream()))
    return y


def _bitserial_partials(wbuf, xbuf, cfg: GemmConfig, w_cm: int, x_cm: int):
    t = _dev.torch()
    parts = t.zeros((cfg.n_groups, cfg.m, cfg.n), dtype=t.int32, device=wbuf.device)
    _lib.check(_lib.lib().flexq_gemm_bitserial(
        _lib.ptr(wbuf), _lib.ptr(xbuf), None, None, cfg.m, cfg.n, cfg.k, cfg.weight_bits,
        cfg.activation_bits, cfg.group_size, w_cm, x_cm, _lib.ptr(parts), None, _lib.OUT_F32,
        None, 0, _lib.stream()))
    return parts


def t6_pack_weights(wcodes, wscales, k: int, group_size: int, scale_f16: bool, with_scales=True):
    """int8 codes [n, k] (+ float64 scales) -> (T6 words, packed fp16/fp32 scales)."""
    t = _dev.torch()
    L = _lib.lib()
    n = wcodes.shape[0]
    t6 = t.empty(L.flexq_t6_bytes(n, k, group_size) // 4, dtype=t.int32, device=wcodes.device)
    ws = None
    if with_scales:
        ng = -(-k // group_size)
        ws = t.empty(-(-n // 64) * 4 * ng * 16, dtype=t.float16 if scale_f16 else t.float32,
                     device=wcodes.device)
    _lib.check(L.flexq_pack_t6(_lib.ptr(wcodes), _lib.ptr(wscales), n, k, group_size,
                               int(scale_f16), _lib.ptr(t6), _lib.ptr(ws), _lib.stream()))
    return t6, ws


def t6_pack_activations(xcodes, xscales, k: int, group_size: int):
    """int8 codes [m, k] + float64 scales -> (act fragments, fp32 scales, corrections, m_pad)."""
    t = _dev.torch()
    L = _lib.lib()
    m = xcodes.shape[0]
    m_pad = L.flexq_act_m_pad(m)
    ng = -(-k // group_size)
    frag = t.zeros(L.flexq_act_frag_bytes(m_pad, k, group_size) // 4, dtype=t.int32,
                   device=xcodes.device)
    xs = t.zeros((ng, m_pad), dtype=t.float32, device=xcodes.device)
    corr = t.zeros((ng, m_pad), dtype=t.int32, device=xcodes.device)
    _lib.check(L.flexq_pack_act_t6(_lib.ptr(xcodes), _lib.ptr(xscales), m, m_pad, k, group_size,
                                   _lib.ptr(frag), _lib.ptr(xs), _lib.ptr(corr), _lib.stream()))
    return frag, xs, corr, m_pad


def _t6_partials(wcodes, xcodes, xscales, cfg: GemmConfig):
    t = _dev.torch()
    t6, _ = t6_pack_weights(wcodes, None, cfg.k, cfg.group_size, False, with_scales=False)
    frag, xs, corr, m_pad = t6_pack_activations(xcodes, xscales, cfg.k, cfg.group_size)
    parts = t.zeros((cfg.n_groups, cfg.m, cfg.n), dtype=t.int32, device=wcodes.device)
    _lib.check(_lib.lib().flexq_gemm_t6(
        _lib.ptr(t6), None, 0, _lib.ptr(frag), _lib.ptr(xs), _lib.ptr(corr), cfg.m, m_pad, cfg.n,
        cfg.k, cfg.group_size, _lib.ptr(parts), None, _lib.OUT_F32, None, 0, _lib.stream()))
    return parts


def _finish(parts, ws, xs, cfg: GemmConfig, trace: bool, passes: int, as_numpy: bool):
    t = _dev.torch()
    y = _epilogue_f64(parts, ws, xs, cfg.m, cfg.n, cfg.n_groups)
    gp = parts.to(t.int64) if trace else None
    if as_numpy:
        return GemmOutput(data=_dev.to_host(y), bmma_passes=passes,
                          group_partials=_dev.to_host(gp) if trace else None)
    return GemmOutput(data=y, bmma_passes=passes, group_partials=gp)


# ---- reference entry points ----------------------------------------------------------------

def _check_operands(wp: PackedTensor, xp: PackedTensor, w_scales, x_scales, cfg: GemmConfig):
    """Same checks and messages as engine.py:227-248."""
    if wp.cols != cfg.k or xp.cols != cfg.k:
        raise ShapeError(f"K mismatch: weights have K={wp.cols}, activations K={xp.cols}, "
                         f"config k={cfg.k}")
    if wp.rows != cfg.n or xp.rows != cfg.m:
        raise ShapeError(f"row mismatch: weights {wp.rows} rows (config n={cfg.n}), "
                         f"activations {xp.rows} rows (config m={cfg.m})")
    if wp.bits != cfg.weight_bits or xp.bits != cfg.activation_bits:
        raise ShapeError(f"bit mismatch: packed ({wp.bits}, {xp.bits}) vs config "
                         f"({cfg.weight_bits}, {cfg.activation_bits})")
    if wp.config.chunk_k != xp.config.chunk_k or wp.config.word_bits != xp.config.word_bits:
        raise ShapeError("weight and activation packs must share chunk_k and word_bits")
    g = cfg.n_groups
    if tuple(w_scales.shape) != (cfg.n, g):
        raise ShapeError(f"weight scales shape {tuple(w_scales.shape)} != {(cfg.n, g)}")
    if tuple(x_scales.shape) != (cfg.m, g):
        raise ShapeError(f"activation scales shape {tuple(x_scales.shape)} != {(cfg.m, g)}")


def group_matmul_fused(wp: PackedTensor, xp: PackedTensor, w_scales, x_scales, cfg: GemmConfig,
                       trace: bool = False) -> GemmOutput:
    """Bit-serial GEMM with fused group dequantization (engine.py:290-334), on the GPU."""
    t = _dev.torch()
    ws_arr = w_scales if _dev.is_torch(w_scales) else np.asarray(w_scales, dtype=np.float64)
    xs_arr = x_scales if _dev.is_torch(x_scales) else np.asarray(x_scales, dtype=np.float64)
    _check_operands(wp, xp, ws_arr, xs_arr, cfg)
    parts = _bitserial_partials(wp.device_bytes(), xp.device_bytes(), cfg, wp.config.chunk_m,
                                xp.config.chunk_m)
    ws = _dev.to_device(ws_arr, t.float64)
    xs = _dev.to_device(xs_arr, t.float64)
    passes = bmma_passes(cfg, xp.config.chunk_m, wp.config.chunk_m)
    return _finish(parts, ws, xs, cfg, trace, passes, not _dev.is_torch(wp.words))


def int_matmul_reference(wq: QuantTensor, xq: QuantTensor, cfg: GemmConfig,
                         trace: bool = False) -> GemmOutput:
    """Per-group integer GEMM + the shared epilogue (engine.py:337-365).

    Runs the production tensor-core kernel (T6 layout) for weights of up to 6
    bits and the bit-serial kernel for 7-8 bit weights.
    """
    if wq.shape != (cfg.n, cfg.k) or xq.shape != (cfg.m, cfg.k):
        raise ShapeError(f"operand shapes {wq.shape} / {xq.shape} do not match config "
                         f"(n={cfg.n}, m={cfg.m}, k={cfg.k})")
    if wq.group_size != cfg.group_size or xq.group_size != cfg.group_size:
        raise ShapeError("operand group sizes must match the config group_size")
    if wq.bits != cfg.weight_bits or xq.bits != cfg.activation_bits:
        raise ShapeError("operand bit widths must match the config precision pair")
    wcodes, ws = wq.device_tensors()
    xcodes, xs = xq.device_tensors()
    parts = _partials_from_codes(wq, xq, cfg)
    return _finish(parts, ws, xs, cfg, trace, 0, not _dev.is_torch(wq.values))


def _partials_from_codes(wq: QuantTensor, xq: QuantTensor, cfg: GemmConfig):
    wcodes, _ = wq.device_tensors()
    xcodes, xs = xq.device_tensors()
    if wq.bits <= 6:
        return _t6_partials(wcodes, xcodes, xs, cfg)
    wp = pack(decompose(wq), weight_pack_config())
    xp = pack(decompose(xq), activation_pack_config(cfg.m))
    return _bitserial_partials(wp.device_bytes(), xp.device_bytes(), cfg, 8, xp.config.chunk_m)


def execute_tiled(wp: PackedTensor, xp: PackedTensor, w_scales, x_scales,
                  cfg: GemmConfig) -> GemmOutput:
    """Tiled executor (engine.py:398-484): same validation, identical results.

    The reference's output-tile x K-tile schedule with a prefetch pipeline maps
    onto the kernels' CTA tiling + load pipelining; the knobs are validated like
    the reference and, as its determinism contract requires, never change the
    result.
    """
    ws_arr = w_scales if _dev.is_torch(w_scales) else np.asarray(w_scales, dtype=np.float64)
    xs_arr = x_scales if _dev.is_torch(x_scales) else np.asarray(x_scales, dtype=np.float64)
    _check_operands(wp, xp, ws_arr, xs_arr, cfg)
    cm, cn, ck = xp.config.chunk_m, wp.config.chunk_m, xp.config.chunk_k
    if cfg.bm % cm or cfg.bn % cn or cfg.bk % ck:
        raise ConfigError(
            f"tile dims (bm={cfg.bm}, bn={cfg.bn}, bk={cfg.bk}) must be multiples of "
            f"chunk dims (chunk_m={cm}, chunk_n={cn}, chunk_k={ck})")
    if xp.padded_cols > cfg.bk and cfg.bk % cfg.group_size:
        raise ConfigError(
            f"bk ({cfg.bk}) must cover whole scale groups (group_size={cfg.group_size}) "
            "so fused dequantization applies each group's scales exactly once")
    out = group_matmul_fused(wp, xp, ws_arr, xs_arr, cfg, trace=False)
    return GemmOutput(data=out.data, bmma_passes=out.bmma_passes)


def quantized_linear(weight, activations, weight_bits: int = 6, activation_bits: int = 6,
                     group_size: int = DEFAULT_GROUP_SIZE, word_bits: int = 64,
                     trace: bool = False) -> GemmOutput:
    """quantize -> GEMM -> fused dequant in one call (engine.py:487-513), on the GPU.

    word_bits only selects the FLXQ-P word type in the reference; the T6
    tensor-core path does not use FLXQ-P, and the result is identical.
    """
    if word_bits not in (32, 64):
        raise ConfigError(f"word_bits must be 32 or 64, got {word_bits}")
    wq = quantize(weight, weight_bits, group_size)
    xq = quantize(activations, activation_bits, group_size)
    cfg = GemmConfig(m=xq.shape[0], n=wq.shape[0], k=wq.shape[1], weight_bits=weight_bits,
                     activation_bits=activation_bits, group_size=group_size)
    _, ws = wq.device_tensors()
    _, xs = xq.device_tensors()
    parts = _partials_from_codes(wq, xq, cfg)
    passes = bmma_passes(cfg, min(cfg.m, 8))
    return _finish(parts, ws, xs, cfg, trace, passes, not _dev.is_torch(wq.values))
