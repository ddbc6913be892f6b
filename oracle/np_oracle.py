"""CPU oracle (numpy restatement) of the reference's W6Ax quantized-linear path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(``paper_2508_04405_b200``) may import this module; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` leg use it, and only as the checker or the timed CPU baseline.

Every function restates the algorithm of the reference package ``bitserial``
(``/root/reference/pkg/src/bitserial``) and cites the file:line it follows.
Parity of this restatement is pinned against golden vectors produced by the
real reference (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).

Conventions (reference ``engine.py:3``): W is ``[N, K]`` (rows = output
features), X is ``[M, K]``; groups of ``group_size`` run along K.
"""

from __future__ import annotations

import numpy as np

CHUNK_K = 128          # packing.py:27  MMA_K
WEIGHT_CHUNK_M = 8     # packing.py:74-76 weight_pack_config -> chunk_m = MMA_N = 8
MMA_M = 8              # packing.py:25


def qmax(bits: int) -> int:
    """Symmetric range limit 2^(b-1)-1 (quantize.py:34-36)."""
    return (1 << (bits - 1)) - 1


def n_groups(k: int, group_size: int) -> int:
    return -(-k // group_size)


def round_half_away(v: np.ndarray) -> np.ndarray:
    """sign(v)*floor(|v|+0.5) (quantize.py:29-31)."""
    return np.sign(v) * np.floor(np.abs(v) + 0.5)


def group_scales(data: np.ndarray, bits: int, group_size: int) -> np.ndarray:
    """Per-(row, group) max|x|/qmax, 1.0 for all-zero groups (quantize.py:99-110).

    The last group may be partial; padding with zeros does not change a max of
    absolute values.
    """
    rows, cols = data.shape
    g = n_groups(cols, group_size)
    mags = np.zeros((rows, g * group_size), dtype=np.float64)
    mags[:, :cols] = np.abs(data)
    peak = mags.reshape(rows, g, group_size).max(axis=2)
    out = np.ones_like(peak)
    nz = peak > 0.0
    out[nz] = peak[nz] / qmax(bits)
    return out


def quantize(data, bits: int, group_size: int = 128, fp16_scales: bool = False):
    """Symmetric group quantizer (quantize.py:118-148).

    Returns (codes int8 [rows, cols], scales float64 [rows, G]).  Raises
    ValueError on non-finite input (quantize.py:135-136) and on a
    non-positive scale, which the reference's QuantTensor rejects
    (quantize.py:71-72) -- e.g. an fp16 scale that underflowed to zero.
    """
    x = np.asarray(data, dtype=np.float64)
    if x.ndim != 2:
        raise ValueError(f"expected a 2-D tensor, got shape {x.shape}")
    if not np.isfinite(x).all():
        raise ValueError("input contains non-finite values")
    s = group_scales(x, bits, group_size)
    if fp16_scales:
        s = s.astype(np.float16).astype(np.float64)
    if not (s > 0).all():
        raise ValueError("all scales must be strictly positive")
    per_elem = np.repeat(s, group_size, axis=1)[:, : x.shape[1]]
    lim = qmax(bits)
    codes = np.clip(round_half_away(x / per_elem), -lim, lim).astype(np.int8)
    return codes, s


def dequantize(codes: np.ndarray, scales: np.ndarray, group_size: int) -> np.ndarray:
    """codes * expanded scales (quantize.py:151-154)."""
    per_elem = np.repeat(scales, group_size, axis=1)[:, : codes.shape[1]]
    return codes.astype(np.float64) * per_elem


def plane_coeffs(bits: int, signed: bool = True) -> np.ndarray:
    """2^s, with -2^(b-1) for the signed MSB (bitplane.py:23-34)."""
    c = np.array([1 << s for s in range(bits)], dtype=np.int64)
    if signed:
        c[-1] = -c[-1]
    return c


def bit_planes(codes: np.ndarray, bits: int) -> np.ndarray:
    """Two's-complement planes uint8 [bits, rows, cols] (bitplane.py:55-79)."""
    enc = codes.astype(np.int64) & ((1 << bits) - 1)
    return np.stack([((enc >> s) & 1).astype(np.uint8) for s in range(bits)])


def recompose(planes: np.ndarray, bits: int) -> np.ndarray:
    """sum_s coeff_s * plane_s (bitplane.py:87-89)."""
    c = plane_coeffs(bits)
    return np.tensordot(c, planes.astype(np.int64), axes=(0, 0))


def pack_planes(planes: np.ndarray, chunk_m: int, word_bits: int = 64) -> np.ndarray:
    """FLXQ-P chunked layout (packing.py:132-147, docs/format.md:47-84).

    planes uint8 [bits, R, K] -> words [KC, RC, bits, chunk_m, 128/word_bits],
    LSB-first within little-endian words, zero padded to chunk multiples.
    """
    bits, rows, cols = planes.shape
    rc = -(-rows // chunk_m)
    kc = -(-cols // CHUNK_K)
    full = np.zeros((bits, rc * chunk_m, kc * CHUNK_K), dtype=np.uint8)
    full[:, :rows, :cols] = planes
    # axes (s, rc, r, kc, j) -> (kc, rc, s, r, j)
    blocks = full.reshape(bits, rc, chunk_m, kc, CHUNK_K).transpose(3, 1, 0, 2, 4)
    as_bytes = np.packbits(np.ascontiguousarray(blocks), axis=-1, bitorder="little")
    dt = np.dtype("<u8") if word_bits == 64 else np.dtype("<u4")
    return np.ascontiguousarray(as_bytes).view(dt)


def unpack_planes(words: np.ndarray, bits: int, rows: int, cols: int) -> np.ndarray:
    """Inverse of pack_planes over the unpadded region (packing.py:150-165)."""
    kc, rc, b, cm, _ = words.shape
    assert b == bits
    raw = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), axis=-1, bitorder="little")
    planes = raw.transpose(2, 1, 3, 0, 4).reshape(bits, rc * cm, kc * CHUNK_K)
    return np.ascontiguousarray(planes[:, :rows, :cols])


def activation_chunk_m(m: int) -> int:
    """min(M, MMA_M) (packing.py:69-71)."""
    return min(m, MMA_M)


def scale_accumulate(acc: np.ndarray, xs_g: np.ndarray, ws_g: np.ndarray, partial: np.ndarray):
    """acc += (xs (x) ws) * partial, float64 (engine.py:211-216).

    The association (xs*ws first, then * partial, then +=) is part of the
    contract: the reference's two paths are bit-identical only because both
    funnel through this one expression in ascending group order.
    """
    acc += (xs_g[:, None] * ws_g[None, :]) * partial.astype(np.float64)


def int_matmul(wcodes, xcodes, wscales, xscales, group_size: int, trace: bool = False):
    """Per-group int64 dot products + f64 epilogue (engine.py:337-365).

    Returns (Y float64 [M, N], partials int64 [G, M, N] or None).
    """
    m, k = xcodes.shape
    n = wcodes.shape[0]
    g_total = n_groups(k, group_size)
    w = wcodes.astype(np.int64)
    x = xcodes.astype(np.int64)
    acc = np.zeros((m, n), dtype=np.float64)
    parts = np.zeros((g_total, m, n), dtype=np.int64) if trace else None
    for g in range(g_total):
        lo, hi = g * group_size, min((g + 1) * group_size, k)
        p = x[:, lo:hi] @ w[:, lo:hi].T
        if trace:
            parts[g] = p
        scale_accumulate(acc, xscales[:, g], wscales[:, g], p)
    return acc, parts


def _segments(g_total: int, group_size: int, k_pad: int):
    """Group -> list of (kchunk, lo, hi) bit spans (engine.py:165-180).

    The last group runs through the zero padding.
    """
    out = []
    for g in range(g_total):
        lo = g * group_size
        hi = k_pad if g == g_total - 1 else (g + 1) * group_size
        spans = []
        kc = lo // CHUNK_K
        while kc * CHUNK_K < hi:
            base = kc * CHUNK_K
            spans.append((kc, max(lo, base) - base, min(hi, base + CHUNK_K) - base))
            kc += 1
        out.append(spans)
    return out


def _span_mask128(lo: int, hi: int) -> np.ndarray:
    """Two u64 words selecting chunk bits [lo, hi) (engine.py:183-193)."""
    m = np.zeros(2, dtype=np.uint64)
    for w in range(2):
        a, b = max(lo, 64 * w), min(hi, 64 * (w + 1))
        if a < b:
            m[w] = np.uint64(((1 << (b - a)) - 1) << (a - 64 * w))
    return m


def bitserial_matmul(wwords, xwords, wscales, xscales, m, n, k, p, q, group_size,
                     trace: bool = False):
    """AND+popcount bit-serial GEMM with fused dequant (engine.py:251-334).

    wwords/xwords are FLXQ-P u64 word arrays [KC, RC, bits, chunk_m, 2].
    For every group and k-chunk span: popcount(w_plane_s & x_plane_t) for all
    (s, t), weighted by coeff_s*coeff_t (engine.py:114-130, 196-208), summed
    exactly, then the same scale_accumulate as int_matmul.
    """
    cw, cx = plane_coeffs(p), plane_coeffs(q)
    pair_w = np.outer(cx, cw)  # [t, s]
    kc_n, rc_x, _, cm, _ = xwords.shape
    _, rc_w, _, cn, _ = wwords.shape
    g_total = n_groups(k, group_size)
    m_pad, n_pad = rc_x * cm, rc_w * cn
    ws = np.ones((n_pad, g_total)); ws[:n] = wscales
    xs = np.ones((m_pad, g_total)); xs[:m] = xscales
    acc = np.zeros((m_pad, n_pad), dtype=np.float64)
    parts = np.zeros((g_total, m_pad, n_pad), dtype=np.int64) if trace else None
    passes = 0
    for g, spans in enumerate(_segments(g_total, group_size, kc_n * CHUNK_K)):
        part = np.zeros((rc_x, cm, rc_w, cn), dtype=np.int64)
        for kc, lo, hi in spans:
            wblk = wwords[kc]  # [rc_w, p, cn, 2]
            xblk = xwords[kc]  # [rc_x, q, cm, 2]
            if (lo, hi) != (0, CHUNK_K):
                msk = _span_mask128(lo, hi)
                wblk = wblk & msk
            # [rc_x, q, cm, 1, 1, 1, 2] & [1, 1, 1, rc_w, p, cn, 2]
            anded = xblk[:, :, :, None, None, None, :] & wblk[None, None, None, :, :, :, :]
            cnt = np.bitwise_count(anded).sum(axis=-1, dtype=np.int64)  # [rcx,q,cm,rcw,p,cn]
            part += np.einsum("ts,atbcsd->abcd", pair_w, cnt)
            passes += p * q * rc_x * rc_w
        p2 = part.reshape(m_pad, n_pad)
        if trace:
            parts[g] = p2
        scale_accumulate(acc, xs[:, g], ws[:, g], p2)
    y = acc[:m, :n]
    return y, (parts[:, :m, :n] if trace else None), passes


def bmma_passes(m: int, n: int, k: int, p: int, q: int, group_size: int) -> int:
    """Analytic pass count: p*q per (activation chunk, weight chunk, span) (engine.py:283)."""
    cm = activation_chunk_m(m)
    rc_x, rc_w = -(-m // cm), -(-n // WEIGHT_CHUNK_M)
    kc_n = -(-k // CHUNK_K)
    spans = sum(len(s) for s in _segments(n_groups(k, group_size), group_size, kc_n * CHUNK_K))
    return p * q * rc_x * rc_w * spans


def quantized_linear(weight, acts, p=6, q=6, group_size=128, fp16_scales=False, trace=False):
    """quantize -> planes -> pack -> bit-serial GEMM (engine.py:487-513)."""
    wc, wsc = quantize(weight, p, group_size, fp16_scales)
    xc, xsc = quantize(acts, q, group_size, fp16_scales)
    m, k = xc.shape
    n = wc.shape[0]
    ww = pack_planes(bit_planes(wc, p), WEIGHT_CHUNK_M)
    xw = pack_planes(bit_planes(xc, q), activation_chunk_m(m))
    return bitserial_matmul(ww, xw, wsc, xsc, m, n, k, p, q, group_size, trace)
