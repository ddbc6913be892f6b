// Decode-regime (M <= 16) T6 GEMV/GEMM: persistent, TMA-bulk-fed, warp-streamed.
//
// Same math as gemm_t6_kernel (unpack-to-INT8 + mma.sync m16n8k32, exact INT32
// group partials, fused fp32 dequant: engine.py:251-365, 211-216), organised
// for HBM bandwidth:
//
//  * The T6 weights are a sequence of 6 KB units u = rg*KB + kb (64 rows x 128
//    k-slots).  The launch is persistent (CTAs resident on every SM) and every
//    warp owns one contiguous unit range [u0, u1) of equal size -> the weight
//    bytes are balanced to within one unit across all warps of the GPU, for
//    every layer shape (no wave quantisation, no tail).
//  * Each warp streams its range through an S-stage shared-memory ring filled
//    by cp.async.bulk (the TMA engine: one elected lane issues, an mbarrier
//    counts the bytes), with an L2 evict_first hint on the weights (PAPER.md
//    sec. 4.3.2).  Each stage carries the unit's weights, activation
//    fragments, weight scales, activation scales and corrections, so no
//    global load sits on a warp's critical path.  2 stages x 7.4 KB x 12
//    warps keeps ~180 KB per SM in flight (Little's law asks ~45 KB at
//    6.5 TB/s; tools/probe/stream.cu measured 6.6-7.0 TB/s for this ring).
//  * The 4 row tiles of a unit are interleaved per k-step (4 independent mma
//    accumulator chains) so a warp is never serialised on mma latency.
//  * One unit feeds 4 row tiles x 4 k-steps of mma; the activation B
//    fragments (1 KB per 8 tokens per unit, also bulk-copied) are reused by
//    the 4 row tiles.
//  * Warp partial sums of a row group that is split between warps are
//    combined deterministically: every contributor writes its fp32 partial to
//    slot (rg + warp_id) of the workspace; the last to arrive (atomic counter)
//    sums the slots in warp order and stores y.  Results never depend on
//    timing.
#include "common.cuh"

namespace flexq {

constexpr int kSWarps = 4;  // warps per CTA in the default launch (independent pipelines)
// Warps per CTA are a launch parameter (blockDim): the default packs 4-warp CTAs several to
// an SM; FLEXQ_GEMV_WIDE=1 launches one CTA per SM holding all of that SM's warps.
constexpr int kMaxWarpsMT1 = 12, kMaxWarpsMT2 = 8, kMaxWarpsMT4 = 8;
template <int MT>
constexpr int max_warps() { return MT == 1 ? kMaxWarpsMT1 : MT == 2 ? kMaxWarpsMT2 : kMaxWarpsMT4; }
constexpr int kMinUnitsPerWarp = 6;
#ifndef FLEXQ_GEMV_FB1
#define FLEXQ_GEMV_FB1 8  // split-fixup slots loaded per L2 round trip at M = 1
#endif

struct StreamParams {
  const uint8_t* t6;
  const void* wscale;
  const uint8_t* act;
  const float* xs;
  const int32_t* corr;
  int64_t m, m_pad, n, ng, spg, ks, kb, rg, units, nw;
  T6Geom geo;
  int32_t* partials;
  void* y;
  float* ws_part;
  unsigned* counters;
  const void* res;  // optional residual added at the store (same dtype/shape as y)
  int rev;
  long long* dbg;  // FLEXQ_TRACE event buffer (debug)
  long long dbg_tag;
  long long* tl;  // debug timeline (FLEXQ_GEMV_TIMELINE): per warp [start, init, prologue, pdl done, first data, loop done, smid, end]
};

__device__ __forceinline__ long long gv_timer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Stage layout: [T6 weights 6 KB][B fragments MT x 1 KB][weight-scale slice][xs slice][corr slice]
// A unit touches NGR groups at most: 4 when spg in {1,2} (MODE 1), otherwise 1.
template <int MT, int MODE, bool SF16>
struct StageLayout {
  static constexpr int kNgr = MODE == 1 ? 4 : 1;
  static constexpr int kWs = kNgr * kRowGroup * 8 * (SF16 ? 4 : 8);
  static constexpr int kVec = kNgr * (MT <= 2 ? 16 : 8 * MT) * 4;  // m_pad tokens x 4 B
  static constexpr int kOffB = kUnitBytes;
  static constexpr int kOffWs = kOffB + MT * 1024;
  static constexpr int kOffXs = kOffWs + kWs;
  static constexpr int kOffCorr = kOffXs + kVec;
  static constexpr int kBytes = kOffCorr + kVec;
};

__device__ __forceinline__ int64_t unit_owner(int64_t u, int64_t nw, int64_t units) {
  return ((u + 1) * nw - 1) / units;  // largest warp whose range start <= u
}

template <int OUT>
__device__ __forceinline__ void store_out(void* y, int64_t i, float v) {
  if constexpr (OUT == FLEXQ_OUT_F16)
    reinterpret_cast<__half*>(y)[i] = __float2half_rn(v);
  else
    reinterpret_cast<float*>(y)[i] = v;
}

// MODE 0: spg == 4 (group = k-block, e.g. group_size 128)
// MODE 1: spg in {1, 2} (several groups per k-block)
// MODE 2: spg % 4 == 0, spg > 4 (a group spans k-blocks: per-channel / large groups)
// ONE: m == 1 (decode GEMV) -- only accumulator column 0 (c0, c2) is live, so the
// dequant, the split fixup and the stores touch half the values.
template <int MT, int MODE, bool SF16, bool TRACE, bool FAST, int OUT, int S, bool ONE>
__global__ void __launch_bounds__(max_warps<MT>() * 32, 1)
    gemv_t6_stream_kernel(StreamParams p) {
  static_assert(!ONE || MT == 1, "ONE implies a single token tile");
  constexpr bool ROUT = MT >= 4;  // row-tile-outer unit loop (M <= 32, MODE 0 only)
  static_assert(!ROUT || MODE == 0, "MT = 4 needs one group per k-block");
  using L = StageLayout<MT, MODE, SF16>;
  constexpr int UB = L::kBytes;
  constexpr int SB = SF16 ? 4 : 8;  // bytes of one weight-scale pair
  extern __shared__ __align__(128) uint8_t smem[];
  const int nwc = blockDim.x >> 5;  // warps in this CTA
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * nwc + warp;
  if (gw >= p.nw) return;  // warp-uniform; no CTA-wide barriers below
  const long long dt0 = p.dbg ? dbg_now() : 0;
  long long dt1 = 0;
  if (p.tl && lane == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.tl[gw * 8 + 0] = gv_timer();
    p.tl[gw * 8 + 6] = smid;
  }
  uint8_t* ring = smem + warp * (S * UB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + nwc * (S * UB)) + warp * S;
  const int64_t gr = p.rev ? p.nw - 1 - gw : gw;  // debug: reversed range assignment
  const int64_t u0 = gr * p.units / p.nw, u1 = (gr + 1) * p.units / p.nw;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol_w = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
  if (p.tl && lane == 0) p.tl[gw * 8 + 1] = gv_timer();

  // No integer division on the per-unit path: (row group, k-block, group) advance
  // incrementally.  spu = k-blocks per group (MODE 2), gshift = log2 groups per k-block (MODE 1).
  const int kbn = (int)p.kb, ngi = (int)p.ng;
  const int spu = MODE == 2 ? (int)(p.spg / 4) : 1;
  const int gshift = MODE == 1 ? (p.spg == 1 ? 2 : 1) : 0;
  auto group_lo = [&](int kb, int gdiv) -> int {  // first group touched by k-block kb
    if constexpr (MODE == 0) return kb;
    else if constexpr (MODE == 1) return kb << gshift;
    else return gdiv;
  };
  auto group_cnt = [&](int kb, int g_lo) -> int {  // groups touched by k-block kb
    if constexpr (MODE == 1) {
      const int hi = min((kb << gshift) + (1 << gshift) - 1, ngi - 1);
      return hi - g_lo + 1;
    } else {
      return 1;
    }
  };
  // part 0: weights + weight scales (offline data, may run before pdl_wait);
  // part 1: activation fragments, scales, corrections (written by the quantizer)
  auto issue = [&](int64_t u, int rg, int kb, int g_lo, int s, int part) {
    const int ngr = group_cnt(kb, g_lo);
    const uint32_t wsb = FAST ? (uint32_t)(ngr * kRowGroup * 8 * SB) : 0u;
    const uint32_t xsb = FAST ? (uint32_t)(ngr * p.m_pad * 4) : 0u;
    const uint32_t cb = (uint32_t)(ngr * p.m_pad * 4);
    uint8_t* dst = ring + s * UB;
    if (part == 0) {
      mbar_expect_tx(&bar[s], kUnitBytes + MT * 1024 + wsb + xsb + cb);
      bulk_g2s(dst, p.t6 + u * (int64_t)kUnitBytes, kUnitBytes, &bar[s], pol_w);
      if (FAST)
        bulk_g2s(dst + L::kOffWs,
                 reinterpret_cast<const uint8_t*>(p.wscale) +
                     p.geo.scale_index(rg * kRowGroup, g_lo, 0) * SB,
                 wsb, &bar[s], pol_w);
    } else {
      bulk_g2s(dst + L::kOffB, p.act + (int64_t)kb * (p.m_pad >> 3) * 1024, MT * 1024, &bar[s],
               pol_a);
      if (FAST) bulk_g2s(dst + L::kOffXs, p.xs + g_lo * p.m_pad, xsb, &bar[s], pol_a);
      bulk_g2s(dst + L::kOffCorr, p.corr + g_lo * p.m_pad, cb, &bar[s], pol_a);
    }
  };
  // issue cursor (lane 0 only): next unit to fetch
  int64_t iu = u0;
  int irg = (int)(u0 / p.kb), ikb = (int)(u0 - (int64_t)irg * p.kb);
  int ig = MODE == 2 ? ikb / spu : 0, irem = MODE == 2 ? ikb - ig * spu : 0;
  auto issue_next = [&](int s) {
    issue(iu, irg, ikb, group_lo(ikb, ig), s, 0);
    issue(iu, irg, ikb, group_lo(ikb, ig), s, 1);
    iu++;
    if (++ikb == kbn) { ikb = 0; irg++; ig = 0; irem = 0; }
    else if (MODE == 2 && ++irem == spu) { irem = 0; ig++; }
  };
  // Prologue: start the weight stream, then wait for the quantizer (PDL) before the
  // activation side of the same stages.
  int pro = 0;
  if (lane == 0) {
    int64_t pu = iu;
    int prg = irg, pkb = ikb, pg = ig, prem = irem;
    for (; pro < S && pu < u1; pro++) {
      issue(pu, prg, pkb, group_lo(pkb, pg), pro, 0);
      pu++;
      if (++pkb == kbn) { pkb = 0; prg++; pg = 0; prem = 0; }
      else if (MODE == 2 && ++prem == spu) { prem = 0; pg++; }
    }
  }
  if (p.tl && lane == 0) p.tl[gw * 8 + 2] = gv_timer();
  pdl_wait();
  pdl_launch_dependents();
  if (p.tl && lane == 0) p.tl[gw * 8 + 3] = gv_timer();
  if (lane == 0) {
    for (int s = 0; s < pro; s++) {
      issue(iu, irg, ikb, group_lo(ikb, ig), s, 1);
      iu++;
      if (++ikb == kbn) { ikb = 0; irg++; ig = 0; irem = 0; }
      else if (MODE == 2 && ++irem == spu) { irem = 0; ig++; }
    }
  }

  float acc[4][MT][4];
  int P[4][MT][4];
  int2 corr0[MT];  // MODE 0: this unit's corrections, applied at drain
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) { acc[r][mt][i] = 0.f; P[r][mt][i] = 0; }

  // ---- group bookkeeping over the stage's slices (dg = group - g_lo of the unit) ----
  auto init_groups = [&](const uint8_t* st, int64_t dg) {
#pragma unroll
    for (int mt = 0; mt < MT; mt++) {
      int2 cr = reinterpret_cast<const int2*>(st + L::kOffCorr)[(dg * p.m_pad + mt * kTokTile) / 2 + t];
      cr.x -= kCorrBias; cr.y -= kCorrBias;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        P[r][mt][0] = -cr.x; P[r][mt][1] = -cr.y; P[r][mt][2] = -cr.x; P[r][mt][3] = -cr.y;
      }
    }
  };
  // drain all 4 row tiles of group g: trace (exact ints) and/or fused fp32 dequant
  auto drain_groups = [&](int64_t rg, int64_t g, const float2* sw, const float2* sx) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      if constexpr (MODE == 0) {  // the group's mma chain started from zero: apply -32*sum(x) now
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          P[r][mt][0] -= corr0[mt].x; P[r][mt][2] -= corr0[mt].x;
          if (!ONE) { P[r][mt][1] -= corr0[mt].y; P[r][mt][3] -= corr0[mt].y; }
        }
      }
      const int64_t row0 = (rg * kRowGroup + r) * kRowTile + gq, row1 = row0 + 8;
      if constexpr (TRACE) {
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) {
            if (ONE && (i & 1)) continue;
            const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
            if (tok < p.m && row < p.n)
              atomicAdd(&p.partials[(g * p.m + tok) * p.n + row], P[r][mt][i]);
          }
      }
      if constexpr (FAST && MODE != 2) {
        // |P| < 2^22 for groups <= 128: convert without I2F (0x4B400000 + P read as an fp32 is
        // 12582912 + P exactly) and dequantise with packed FADD2/FMUL2/FFMA2 -- the same
        // IEEE operations as fmaf(sw * sx, (float)P, acc)
        const float2 c2 = make_float2(12582912.f, 12582912.f);
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          if (ONE) {
            const float2 f = f2_sub(make_float2(__int_as_float(P[r][mt][0] + kCorrBias),
                                                __int_as_float(P[r][mt][2] + kCorrBias)), c2);
            const float2 sc = f2_mul(sw[r], make_float2(sx[mt].x, sx[mt].x));
            const float2 a = f2_fma(sc, f, make_float2(acc[r][mt][0], acc[r][mt][2]));
            acc[r][mt][0] = a.x; acc[r][mt][2] = a.y;
          } else {
            const float2 f01 = f2_sub(make_float2(__int_as_float(P[r][mt][0] + kCorrBias),
                                                  __int_as_float(P[r][mt][1] + kCorrBias)), c2);
            const float2 f23 = f2_sub(make_float2(__int_as_float(P[r][mt][2] + kCorrBias),
                                                  __int_as_float(P[r][mt][3] + kCorrBias)), c2);
            const float2 s01 = f2_mul(make_float2(sw[r].x, sw[r].x), sx[mt]);
            const float2 s23 = f2_mul(make_float2(sw[r].y, sw[r].y), sx[mt]);
            const float2 a01 = f2_fma(s01, f01, make_float2(acc[r][mt][0], acc[r][mt][1]));
            const float2 a23 = f2_fma(s23, f23, make_float2(acc[r][mt][2], acc[r][mt][3]));
            acc[r][mt][0] = a01.x; acc[r][mt][1] = a01.y; acc[r][mt][2] = a23.x; acc[r][mt][3] = a23.y;
          }
        }
      } else if constexpr (FAST) {
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          acc[r][mt][0] = fmaf(sw[r].x * sx[mt].x, (float)P[r][mt][0], acc[r][mt][0]);
          acc[r][mt][2] = fmaf(sw[r].y * sx[mt].x, (float)P[r][mt][2], acc[r][mt][2]);
          if (!ONE) {
            acc[r][mt][1] = fmaf(sw[r].x * sx[mt].y, (float)P[r][mt][1], acc[r][mt][1]);
            acc[r][mt][3] = fmaf(sw[r].y * sx[mt].y, (float)P[r][mt][3], acc[r][mt][3]);
          }
        }
      }
    }
  };
  auto stage_scales = [&](const uint8_t* st, int64_t dg, float2* sw, float2* sx) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int64_t idx = (dg * kRowGroup + r) * 8 + gq;
      if constexpr (SF16) sw[r] = __half22float2(reinterpret_cast<const __half2*>(st + L::kOffWs)[idx]);
      else sw[r] = reinterpret_cast<const float2*>(st + L::kOffWs)[idx];
    }
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
      sx[mt] = reinterpret_cast<const float2*>(st + L::kOffXs)[(dg * p.m_pad + mt * kTokTile) / 2 + t];
  };

  // publish a finished row group's sums: direct store, or the deterministic split fixup
  auto flush = [&](int64_t rg) {
    if constexpr (!FAST) return;
    const int64_t first = unit_owner(rg * p.kb, p.nw, p.units);
    const int64_t last = unit_owner(rg * p.kb + p.kb - 1, p.nw, p.units);
    constexpr int kSlot = 4 * MT * 4 * 32;
    if (first != last) {
      float* slot = p.ws_part + (rg + gr) * (int64_t)kSlot + lane;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++)
            if (!(ONE && (i & 1))) slot[((r * MT + mt) * 4 + i) * 32] = acc[r][mt][i];
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0) prev = atom_add_acq_rel_gpu(&p.counters[rg], 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != (unsigned)(last - first)) return;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
      // fixed order; FB contributors' slots in flight per L2 round trip
      constexpr int FB = ONE ? FLEXQ_GEMV_FB1 : (MT == 1 ? 4 : MT == 2 ? 2 : 1);  // measured best (tools/sweep.py)
      for (int64_t w = first; w <= last; w += FB) {
        float v[FB][4][MT][4];
#pragma unroll
        for (int f = 0; f < FB; f++) {
          const float* src = p.ws_part + (rg + w + f) * (int64_t)kSlot + lane;
#pragma unroll
          for (int r = 0; r < 4; r++)
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
              for (int i = 0; i < 4; i++)
                v[f][r][mt][i] = ((ONE && (i & 1)) || w + f > last)
                                     ? 0.f : __ldcg(src + ((r * MT + mt) * 4 + i) * 32);
        }
#pragma unroll
        for (int f = 0; f < FB; f++)
#pragma unroll
          for (int r = 0; r < 4; r++)
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
              for (int i = 0; i < 4; i++) acc[r][mt][i] += v[f][r][mt][i];
      }
      if (lane == 0) p.counters[rg] = 0u;
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int64_t row0 = (rg * kRowGroup + r) * kRowTile + gq;
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if (ONE && (i & 1)) continue;
          const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = row0 + ((i & 2) ? 8 : 0);
          if (tok < p.m && row < p.n)
            store_out<OUT>(p.y, tok * p.n + row, acc[r][mt][i] + residual_at<OUT>(p.res, tok * p.n + row));
        }
    }
  };

  int rg = (int)(u0 / p.kb), kb = (int)(u0 - (int64_t)rg * p.kb);
  int gdiv = MODE == 2 ? kb / spu : 0, grem = MODE == 2 ? kb - gdiv * spu : 0;
  const int cur_rg0 = rg;
  int s = 0;
  uint32_t parity = 0;
  for (int64_t u = u0; u < u1; u++) {
    const int g_lo = group_lo(kb, gdiv);
    mbar_wait(&bar[s], parity);
    if (p.tl && lane == 0 && u == u0) p.tl[gw * 8 + 4] = gv_timer();
    if (p.dbg && u == u0) dt1 = dbg_now();
    const uint8_t* st = ring + s * UB;
    if constexpr (ROUT) {
      // MT = 4 (M <= 32), one group per k-block: row tile outermost, so only one row
      // tile's weights and INT32 partials are live (MT independent mma chains per k-step)
      uint4 bv[MT][2];
      int2 cz[MT], cb[MT];  // corrections; cb = 0x4B400000 - corr (the fp32 conversion bias)
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        bv[mt][0] = lds128(st + L::kOffB + mt * 1024 + (2 * t) * 128 + gq * 16);
        bv[mt][1] = lds128(st + L::kOffB + mt * 1024 + (2 * t + 1) * 128 + gq * 16);
        cz[mt] = reinterpret_cast<const int2*>(st + L::kOffCorr)[(mt * kTokTile) / 2 + t];
        cz[mt].x -= kCorrBias; cz[mt].y -= kCorrBias;
        cb[mt] = make_int2(kCorrBias - cz[mt].x, kCorrBias - cz[mt].y);
      }
      float2 sw[4], sx[MT];
      if constexpr (FAST) stage_scales(st, 0, sw, sx);
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const uint4 w0 = lds128(st + (r * 3 + 0) * 512 + lane * 16);
        const uint4 w1 = lds128(st + (r * 3 + 1) * 512 + lane * 16);
        const uint4 w2 = lds128(st + (r * 3 + 2) * 512 + lane * 16);
        int Pr[MT][4];
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          uint32_t a[4];
          unpack_t6(u4get(w0, jj), u4get(w1, jj), u4get(w2, jj), a);
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            if (jj == 0) mma_u8s8_zc(Pr[mt], a, bv[mt][0].x, bv[mt][1].x);
            else mma_u8s8(Pr[mt], a, u4get(bv[mt][0], jj), u4get(bv[mt][1], jj));
          }
        }
        const int64_t row0 = ((int64_t)rg * kRowGroup + r) * kRowTile + gq, row1 = row0 + 8;
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          if constexpr (TRACE) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
              if (tok < p.m && row < p.n)
                atomicAdd(&p.partials[((int64_t)kb * p.m + tok) * p.n + row], Pr[mt][i] - (i & 1 ? cz[mt].y : cz[mt].x));
            }
          }
          if constexpr (FAST) {
            // P = Pr - corr (|P| < 2^22 for a 128-k group) as an fp32 without I2F: the bits
            // 0x4B400000 + P read as 12582912 + P, exactly; packed FADD2/FMUL2/FFMA2
            const float2 c2 = make_float2(12582912.f, 12582912.f);
            const float2 f01 = f2_sub(make_float2(__int_as_float(Pr[mt][0] + cb[mt].x), __int_as_float(Pr[mt][1] + cb[mt].y)), c2);
            const float2 f23 = f2_sub(make_float2(__int_as_float(Pr[mt][2] + cb[mt].x), __int_as_float(Pr[mt][3] + cb[mt].y)), c2);
            const float2 s01 = f2_mul(make_float2(sw[r].x, sw[r].x), sx[mt]);
            const float2 s23 = f2_mul(make_float2(sw[r].y, sw[r].y), sx[mt]);
            const float2 a01 = f2_fma(s01, f01, make_float2(acc[r][mt][0], acc[r][mt][1]));
            const float2 a23 = f2_fma(s23, f23, make_float2(acc[r][mt][2], acc[r][mt][3]));
            acc[r][mt][0] = a01.x; acc[r][mt][1] = a01.y; acc[r][mt][2] = a23.x; acc[r][mt][3] = a23.y;
          }
        }
      }
    } else {
    uint4 bv[MT][2], w[4][3];
#pragma unroll
    for (int mt = 0; mt < MT; mt++) {
      bv[mt][0] = lds128(st + L::kOffB + mt * 1024 + (2 * t) * 128 + gq * 16);
      bv[mt][1] = lds128(st + L::kOffB + mt * 1024 + (2 * t + 1) * 128 + gq * 16);
    }
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int v = 0; v < 3; v++) w[r][v] = lds128(st + (r * 3 + v) * 512 + lane * 16);
    if constexpr (MODE == 0) {
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
      {
        corr0[mt] = reinterpret_cast<const int2*>(st + L::kOffCorr)[(mt * kTokTile) / 2 + t];
        corr0[mt].x -= kCorrBias; corr0[mt].y -= kCorrBias;
      }
    }
    if constexpr (MODE == 2) {
      if (grem == 0) init_groups(st, 0);  // this warp owns the group's first k-step
    }
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      const int ks = kb * 4 + jj;
      if (ks < p.ks) {  // k-steps past K pad the last unit of a row group
        int g = g_lo;
        if constexpr (MODE == 1) {
          g = ks >> (2 - gshift);  // spg = 1 or 2
          if ((ks & ((1 << (2 - gshift)) - 1)) == 0) init_groups(st, g - g_lo);
        }
#pragma unroll
        for (int r = 0; r < 4; r++) {  // 4 independent accumulator chains
          uint32_t a[4];
          unpack_t6(u4get(w[r][0], jj), u4get(w[r][1], jj), u4get(w[r][2], jj), a);
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            if (MODE == 0 && jj == 0)
              mma_u8s8_zc(P[r][mt], a, bv[mt][0].x, bv[mt][1].x);
            else
              mma_u8s8(P[r][mt], a, u4get(bv[mt][0], jj), u4get(bv[mt][1], jj));
          }
        }
        bool gend;
        if constexpr (MODE == 0) gend = (jj == 3);
        else if constexpr (MODE == 1) gend = (((ks + 1) & ((1 << (2 - gshift)) - 1)) == 0) || ks + 1 == p.ks;
        else gend = (jj == 3 && grem == spu - 1) || ks + 1 == p.ks;
        if (gend) {
          float2 sw[4], sx[MT];
          if constexpr (FAST) stage_scales(st, g - g_lo, sw, sx);
          drain_groups(rg, g, sw, sx);
        }
      }
    }
    }  // !ROUT
    __syncwarp();
    if (lane == 0 && iu < u1) {
      fence_proxy_async_smem();
      issue_next(s);
    }
    if (++s == S) { s = 0; parity ^= 1u; }
    // advance the consumer cursor; a finished row group is published
    if (++kb == kbn) {
      flush(rg);
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) { acc[r][mt][i] = 0.f; P[r][mt][i] = 0; }
      kb = 0; rg++; gdiv = 0; grem = 0;
    } else if (MODE == 2 && ++grem == spu) {
      grem = 0; gdiv++;
    }
  }
  (void)cur_rg0;
  const int64_t cur_rg = kb == 0 ? rg - 1 : rg;  // row group of the last unit processed
  if constexpr (MODE == 2) {
    // the range ended inside a group: drain the partial group (the correction was
    // applied by the warp that owns the group's first k-step)
    const int64_t ks_end = (u1 - cur_rg * p.kb) * 4;  // k-steps of cur_rg consumed
    if (kb != 0 && ks_end < p.ks && ks_end % p.spg != 0) {
      const int64_t g = (ks_end - 1) / p.spg;
      float2 sw[4], sx[MT];
      if constexpr (FAST) {
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
          sx[mt] = *reinterpret_cast<const float2*>(&p.xs[g * p.m_pad + mt * kTokTile + 2 * t]);
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int64_t idx = p.geo.scale_index(cur_rg * kRowGroup + r, g, gq);
          if constexpr (SF16) sw[r] = __half22float2(reinterpret_cast<const __half2*>(p.wscale)[idx]);
          else sw[r] = reinterpret_cast<const float2*>(p.wscale)[idx];
        }
      }
      drain_groups(cur_rg, g, sw, sx);
    }
  }
  if (p.tl && lane == 0) p.tl[gw * 8 + 5] = gv_timer();
  if (kb != 0) flush(cur_rg);  // (kb == 0: the last row group was already published)
  if (p.tl && lane == 0) p.tl[gw * 8 + 7] = gv_timer();
  if (p.dbg && lane == 0) dbg_record(p.dbg, p.dbg_tag | (gw << 40), dt0, dt1, dbg_now());
}

// ---- host side ------------------------------------------------------------------------------
static int stream_mode(int64_t spg) {
  if (spg == 4) return 0;
  if (spg == 1 || spg == 2) return 1;
  if (spg % 4 == 0) return 2;
  return -1;
}

static long long* g_gemv_tl = nullptr;
extern "C" int flexq_debug_gemv_timeline(long long* host, int max_entries) {
  const int n = 148 * 16 * 8;
  if (!g_gemv_tl || max_entries < n) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_gemv_tl, n * sizeof(long long), cudaMemcpyDeviceToHost);
  return n;
}

// M <= 16 for every group layout; 16 < M <= 32 (MT = 4) for one group per k-block, where the
// mma.sync stream beats the tcgen05 kernel (FLEXQ_STREAM_MAX_M = 16 turns it off)
static int64_t stream_max_m() { return tuning().stream_max_m; }
// M in (16, 32] only for layers of >= 8192 units (48 MB of T6 weights): smaller layers have
// too few units per warp to hide the MT = 4 split fixup, and tcgen05 is faster there
// (LLaMA-2-7B shapes, tools/sweep.py r01)
bool gemv_stream_supported(int64_t m, int64_t spg, int64_t units) {
  if (m > stream_max_m()) return false;
  if (m <= 16) return stream_mode(spg) >= 0;
  return m <= 32 && stream_mode(spg) == 0 && units >= 8192;
}

static int stream_stages() { return tuning().stream_stages; }  // -1: automatic (A/B knob)

template <int MT, int MODE, bool SF16, bool TRACE, bool FAST, int OUT, int S>
static int launch_stream_inst(StreamParams p, int num_sms, cudaStream_t st) {
  auto kern = (MT == 1 && p.m == 1) ? gemv_t6_stream_kernel<MT, MODE, SF16, TRACE, FAST, OUT, S, MT == 1>
                                    : gemv_t6_stream_kernel<MT, MODE, SF16, TRACE, FAST, OUT, S, false>;
  constexpr int UB = StageLayout<MT, MODE, SF16>::kBytes;
  constexpr int kMaxW = max_warps<MT>();
  const bool wide = tuning().gemv_wide;
  {  // once per (device, instantiation)
    const int cap = kMaxW * S * (UB + 8) < 227 * 1024 ? kMaxW * S * (UB + 8) : 227 * 1024;
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), cap);
    if (e != cudaSuccess) return cuda_status(e, "gemv_stream attribute");
  }
  int wpc = kSWarps, per_sm = 0;  // warps per CTA, CTAs per SM
  if (wide) {  // one CTA per SM with as many warps as the SM's shared memory holds
    wpc = (int)(227 * 1024 / (S * (UB + 8)));
    if (wpc > kMaxW) wpc = kMaxW;
    per_sm = 1;
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSWarps * 32,
                                                  kSWarps * S * (UB + 8));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 4) per_sm = 4;  // workspace slots are sized for <= 16 warps per SM
  }
  const int smem = wpc * S * (UB + 8);
  int64_t warps = (int64_t)num_sms * per_sm * wpc;
  // bounds the fixup fan-in; deep rings (small layers) spread the units thinner so that a
  // warp's whole range is in flight at once
  const int min_deep = tuning().min_units;  // units per warp with 4-stage rings
  const int64_t by_units = cdiv(p.units, S >= 4 ? min_deep : kMinUnitsPerWarp);
  if (warps > by_units) warps = by_units;
  p.nw = warps;
  const unsigned ctas = (unsigned)cdiv(warps, wpc);
  cudaError_t e = launch_pdl(kern, dim3(ctas), dim3(wpc * 32), (size_t)smem, st, p);
  if (e != cudaSuccess) return cuda_status(e, "gemv_t6_stream launch");
  return FLEXQ_OK;
}

template <int MT, int MODE, int S>
static int dispatch_stream_flags(const StreamParams& p, bool sf16, bool trace, bool fast, int out,
                                 int sms, cudaStream_t st) {
#define FLEXQ_SC(SF, TR, FA, OU)                                         \
  if (sf16 == SF && trace == TR && fast == FA && (!FA || out == OU))    \
    return launch_stream_inst<MT, MODE, SF, TR, FA, OU, S>(p, sms, st);
  FLEXQ_SC(true, false, true, FLEXQ_OUT_F16)
  FLEXQ_SC(true, false, true, FLEXQ_OUT_F32)
  FLEXQ_SC(false, false, true, FLEXQ_OUT_F16)
  FLEXQ_SC(false, false, true, FLEXQ_OUT_F32)
  FLEXQ_SC(true, true, true, FLEXQ_OUT_F16)
  FLEXQ_SC(false, true, true, FLEXQ_OUT_F16)
  FLEXQ_SC(true, true, true, FLEXQ_OUT_F32)
  FLEXQ_SC(false, true, true, FLEXQ_OUT_F32)
  FLEXQ_SC(false, true, false, FLEXQ_OUT_F16)
  FLEXQ_SC(true, true, false, FLEXQ_OUT_F16)
#undef FLEXQ_SC
  set_error("gemv_stream: unsupported flag combination");
  return FLEXQ_ERR_CONFIG;
}

static int64_t stream_slots(int64_t rg) { return rg + 148 * 16 + 16; }

int64_t gemv_stream_workspace(int64_t m, int64_t n, int64_t k, int64_t gs) {
  T6Geom G(n, k, gs);
  const int64_t mt = m <= 8 ? 1 : m <= 16 ? 2 : 4;
  return cdiv(stream_slots(G.rg) * 4 * mt * 4 * 32 * 4, 256) * 256 + cdiv(G.rg * 4, 256) * 256;
}

int gemv_stream_launch(const uint32_t* t6, const void* wscale, int scale_f16,
                       const uint32_t* act_frag, const float* xs, const int32_t* corr, int64_t m,
                       int64_t m_pad, int64_t n, int64_t k, int64_t gs, int32_t* partials, void* y,
                       int out_dtype, void* workspace, const void* residual, cudaStream_t st) {
  T6Geom G(n, k, gs);
  const int mode = stream_mode(G.spg);
  if (m > 32 || mode < 0 || (m > 16 && mode != 0)) {  // (the unit threshold is a routing choice)
    set_error("gemv_stream: unsupported m=%lld / group_size=%lld", (long long)m, (long long)gs);
    return FLEXQ_ERR_CONFIG;
  }
  if (y && !workspace) {
    set_error("gemv_stream: workspace required");
    return FLEXQ_ERR_CONFIG;
  }
  const int sms = device_sms();
  StreamParams p{};
  p.t6 = reinterpret_cast<const uint8_t*>(t6);
  p.wscale = wscale;
  p.act = reinterpret_cast<const uint8_t*>(act_frag);
  p.xs = xs;
  p.corr = corr;
  p.m = m; p.m_pad = m_pad; p.n = n;
  p.ng = G.ng; p.spg = G.spg; p.ks = G.ks; p.kb = G.kb; p.rg = G.rg;
  p.units = G.rg * G.kb;
  p.geo = G;
  p.partials = partials;
  p.y = y;
  p.res = residual;
  if (tuning().gemv_rev) p.rev = 1;
  p.dbg = dbg_trace_buf();
  if (p.dbg) p.dbg_tag = dbg_next_launch() << 8 | 2;
  if (tuning().gemv_timeline) {
    static long long* tlbuf = nullptr;
    if (!tlbuf) cudaMalloc(&tlbuf, 148 * 16 * 8 * sizeof(long long));
    cudaMemsetAsync(tlbuf, 0, 148 * 16 * 8 * sizeof(long long), st);
    p.tl = tlbuf;
    g_gemv_tl = tlbuf;
  }
  const int mt = m <= 8 ? 1 : m <= 16 ? 2 : 4;
  if (workspace) {
    p.ws_part = reinterpret_cast<float*>(workspace);
    p.counters = reinterpret_cast<unsigned*>(
        reinterpret_cast<char*>(workspace) +
        cdiv(stream_slots(G.rg) * 4 * (int64_t)mt * 4 * 32 * 4, 256) * 256);
  }
  const bool trace = partials != nullptr, fast = y != nullptr;
  const bool sf16 = scale_f16 != 0;
  // small layers (fewer than ~6 units per warp at full occupancy): 4-stage rings
  const int forced = stream_stages();
  // ring depth by layer size (measured on B200, tools/sweep.py): small layers are latency-
  // bound and want every unit of a warp in flight; large ones want more warps per SM
  // MT = 4 stages are 10.6 KB: two per warp keep 8 warps (two CTAs) per SM in shared memory
  const int S = forced > 0 ? forced : mt == 4 ? 2 : (p.units <= 4096 ? 4 : p.units <= 12288 ? 3 : 2);
#define FLEXQ_SM(MT_, MODE_, S_)                                                          \
  if (mt == MT_ && mode == MODE_ && S == S_)                                              \
    return dispatch_stream_flags<MT_, MODE_, S_>(p, sf16, trace, fast, out_dtype, sms, st);
  FLEXQ_SM(1, 0, 2) FLEXQ_SM(1, 1, 2) FLEXQ_SM(1, 2, 2)
  FLEXQ_SM(2, 0, 2) FLEXQ_SM(2, 1, 2) FLEXQ_SM(2, 2, 2)
  FLEXQ_SM(1, 0, 3) FLEXQ_SM(2, 0, 3)
  FLEXQ_SM(1, 0, 4) FLEXQ_SM(2, 0, 4)
  FLEXQ_SM(4, 0, 2) FLEXQ_SM(4, 0, 3) FLEXQ_SM(4, 0, 4)
#undef FLEXQ_SM
  if (S >= 3) {  // only MODE 0 has 3/4-stage instances; others use 2
#define FLEXQ_SM2(MT_, MODE_)                                                             \
  if (mt == MT_ && mode == MODE_)                                                         \
    return dispatch_stream_flags<MT_, MODE_, 2>(p, sf16, trace, fast, out_dtype, sms, st);
    FLEXQ_SM2(1, 1) FLEXQ_SM2(1, 2) FLEXQ_SM2(2, 1) FLEXQ_SM2(2, 2)
#undef FLEXQ_SM2
  }
  set_error("gemv_stream: no kernel instance");
  return FLEXQ_ERR_CONFIG;
}

}  // namespace flexq
