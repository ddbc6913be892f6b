// Production GEMV/GEMM core: unpack-to-INT8 on the tensor cores.
//
// Replaces the numerics of group_matmul_fused / int_matmul_reference
// (engine.py:251-365): per (token m, row n, scale group g) the exact integer
//   P[g,m,n] = sum_{k in g} x[m,k] * w[n,k]
// followed by the fused dequant y[m,n] = sum_g (xs[m,g]*ws[n,g]) * P
// (engine.py:211-216).
//
// Why not the bit-serial BMMA of the paper on B200: sm_100a has no binary
// tensor core (mma .b1 lowers to IMMA + MOVM emulation) and POPC issues at
// 16/clk/SM (measured, tools/probe/rates.cu), so AND+popcount caps a W6A8 GEMV
// at ~35% of HBM roofline.  Unpacking the 6-bit codes costs ~0.75 ALU op per
// weight and feeds mma.sync.m16n8k32 (IMMA, measured 1.15 POPS), which keeps
// the layer HBM-bound for the decode batches this kernel serves.
//
// Operands:
//   T6 weights   u32 [RT][KB][3][32 lanes][4]: per lane per k-step three words
//                L0/L1 (low nibbles) and H (2-bit highs) of 16 offset-binary
//                codes u = w + 32 -> the four A registers of one mma.
//   act fragments u32 [MT][KB][32 lanes][8]: per lane per k-step the two B
//                registers (int8 codes).
//   Because A holds u = w + 32, the group partial is sum u*x - 32*sum x; the
//   second term (act_corr) seeds the accumulator of the group's first k-step.
//
// Work split: CTA = (16-row tile, K range); its 4 warps take interleaved
// k-blocks (128 k-slots, 3 x LDG.128 per lane).  A warp's fp32 partial sums
// are reduced across warps in fixed order, then across K-split CTAs by the
// last-arriving CTA in fixed order -> deterministic output.
#include <cstdint>
#include "common.cuh"

namespace flexq {

struct T6Params {
  const uint4* __restrict__ t6;
  const void* __restrict__ wscale;
  const uint4* __restrict__ act;
  const float* __restrict__ xs;
  const int32_t* __restrict__ corr;
  int64_t m, m_pad, n;          // m: valid tokens of this chunk; m_pad: stride of xs/corr
  int64_t m_total, tok0;        // trace / output token indexing
  int64_t ws_mstride;           // token stride of the split-K workspace
  int64_t ng, spg, ks, kb, rt;
  int64_t act_mp8;              // token octets per k-block row of the activation operand
  T6Geom geo;
  int32_t* partials;
  void* y;
  float* ws_part;
  unsigned* counters;
  const void* res;  // optional residual added at the store
  int ksplit;
};

// Weights are read exactly once: bypass L1 and mark the L2 lines evict-first
// (the paper's evict_first hint) so the L2-resident
// activation fragments and scales are not displaced.
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

template <bool SF16>
__device__ __forceinline__ float2 load_wscale(const void* ws, int64_t idx) {
  if constexpr (SF16) {
    __half2 h = reinterpret_cast<const __half2*>(ws)[idx];
    return __half22float2(h);
  } else {
    return reinterpret_cast<const float2*>(ws)[idx];
  }
}

template <int OUT>
__device__ __forceinline__ void store_y(void* y, int64_t i, float v) {
  if constexpr (OUT == FLEXQ_OUT_F16)
    reinterpret_cast<__half*>(y)[i] = __float2half_rn(v);
  else
    reinterpret_cast<float*>(y)[i] = v;
}

constexpr int kT6Warps = 4;

template <int MT, bool SF16, bool TRACE, bool FAST, int OUT>
__global__ void __launch_bounds__(kT6Warps * 32) gemm_t6_kernel(T6Params p) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int64_t rt = blockIdx.x, split = blockIdx.y;
  const int64_t kb0 = split * p.kb / p.ksplit, kb1 = (split + 1) * p.kb / p.ksplit;
  const int64_t row0 = rt * kRowTile + gq, row1 = row0 + 8;

  float acc[MT][4];
  int P[MT][4];
#pragma unroll
  for (int mt = 0; mt < MT; mt++)
#pragma unroll
    for (int i = 0; i < 4; i++) { acc[mt][i] = 0.f; P[mt][i] = 0; }
  int64_t cur = -1;

  auto drain = [&](int64_t g) {
    if constexpr (TRACE) {
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        const int64_t tok0 = mt * kTokTile + 2 * t;
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t tok = tok0 + (i & 1), row = (i & 2) ? row1 : row0;
          if (tok < p.m && row < p.n)
            atomicAdd(&p.partials[(g * p.m_total + p.tok0 + tok) * p.n + row], P[mt][i]);
        }
      }
    }
    if constexpr (FAST) {
      const float2 sw = load_wscale<SF16>(p.wscale, p.geo.scale_index(rt, g, gq));
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        float2 sx = make_float2(0.f, 0.f);  // token tiles past the chunk are never stored
        if (mt * kTokTile < p.ws_mstride)
          sx = *reinterpret_cast<const float2*>(&p.xs[g * p.m_pad + mt * kTokTile + 2 * t]);
        acc[mt][0] = fmaf(sw.x * sx.x, (float)P[mt][0], acc[mt][0]);
        acc[mt][1] = fmaf(sw.x * sx.y, (float)P[mt][1], acc[mt][1]);
        acc[mt][2] = fmaf(sw.y * sx.x, (float)P[mt][2], acc[mt][2]);
        acc[mt][3] = fmaf(sw.y * sx.y, (float)P[mt][3], acc[mt][3]);
      }
    }
  };

  const uint4* wbase = p.t6 + p.geo.vec_index(rt, 0, 0, lane);
  const uint64_t pol = evict_first_policy();
  int64_t kb = kb0 + warp;
  uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0, w2 = w0;
  if (kb < kb1) {
    const uint4* q = wbase + kb * (kRowGroup * 96);
    w0 = ld_stream(q, pol); w1 = ld_stream(q + 32, pol); w2 = ld_stream(q + 64, pol);
  }
  for (; kb < kb1; kb += kT6Warps) {
    // prefetch the next k-block of this warp while the current one computes
    uint4 n0 = make_uint4(0, 0, 0, 0), n1 = n0, n2 = n0;
    const int64_t kbn = kb + kT6Warps;
    if (kbn < kb1) {
      const uint4* q = wbase + kbn * (kRowGroup * 96);
      n0 = ld_stream(q, pol); n1 = ld_stream(q + 32, pol); n2 = ld_stream(q + 64, pol);
    }
    uint4 b[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; mt++) {
      if (mt * kTokTile + gq < p.m) {
        const uint4* q = p.act + (kb * p.act_mp8 + mt) * 64 + (2 * t) * 8 + gq;
        b[mt][0] = __ldg(q); b[mt][1] = __ldg(q + 8);
      } else {
        b[mt][0] = make_uint4(0, 0, 0, 0); b[mt][1] = b[mt][0];
      }
    }
#pragma unroll
    for (int jj = 0; jj < 4; jj++) {
      const int64_t ks = kb * 4 + jj;
      if (ks >= p.ks) break;
      const int64_t g = ks / p.spg;
      if (g != cur) {
        if (cur >= 0) drain(cur);
        cur = g;
        const bool first = (ks == g * p.spg);
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          int2 cr = make_int2(0, 0);
          if (first && mt * kTokTile < p.ws_mstride)
            cr = *reinterpret_cast<const int2*>(&p.corr[g * p.m_pad + mt * kTokTile + 2 * t]);
          if (first) { cr.x -= kCorrBias; cr.y -= kCorrBias; }
          P[mt][0] = -cr.x; P[mt][1] = -cr.y; P[mt][2] = -cr.x; P[mt][3] = -cr.y;
        }
      }
      uint32_t a[4];
      unpack_t6(u4get(w0, jj), u4get(w1, jj), u4get(w2, jj), a);
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        mma_u8s8(P[mt], a, u4get(b[mt][0], jj), u4get(b[mt][1], jj));
      }
    }
    w0 = n0; w1 = n1; w2 = n2;
  }
  if (cur >= 0) drain(cur);

  if constexpr (FAST) {
    __shared__ float red[kT6Warps][MT][4][32];
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) red[warp][mt][i][lane] = acc[mt][i];
    __syncthreads();
    if (warp != 0) return;
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) {
        float s = red[0][mt][i][lane];
#pragma unroll
        for (int w = 1; w < kT6Warps; w++) s += red[w][mt][i][lane];
        acc[mt][i] = s;
      }
    const int64_t n_pad = p.rt * kRowTile;
    if (p.ksplit > 1) {
      // publish this CTA's partial; the last CTA of the row tile reduces in split order
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
          if (tok < p.ws_mstride)  // token tiles past this chunk's padding are not stored
            p.ws_part[(split * p.ws_mstride + tok) * n_pad + row] = acc[mt][i];
        }
      __threadfence();
      unsigned prev = 0;
      if (lane == 0) prev = atomicAdd(&p.counters[rt], 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != (unsigned)p.ksplit - 1) return;
      __threadfence();
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
          float s = 0.f;
          if (tok < p.ws_mstride)
            for (int sp = 0; sp < p.ksplit; sp++)
            s += __ldcg(&p.ws_part[(sp * p.ws_mstride + tok) * n_pad + row]);
          acc[mt][i] = s;
        }
      if (lane == 0) p.counters[rt] = 0u;
    }
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
        if (tok < p.m && row < p.n)
          store_y<OUT>(p.y, (p.tok0 + tok) * p.n + row,
                       acc[mt][i] + residual_at<OUT>(p.res, (p.tok0 + tok) * p.n + row));
      }
  }
}

int auto_ksplit_t6(int64_t rt, int64_t kb) {
  // aim for ~6 CTAs of 4 warps per SM (148 SMs) while keeping >= 2 k-blocks per warp
  int64_t want = cdiv(148 * 6, rt);
  int64_t cap = kb / (2 * kT6Warps);
  if (cap < 1) cap = 1;
  if (want > cap) want = cap;
  if (want > 16) want = 16;
  return (int)(want < 1 ? 1 : want);
}

template <int MT, bool SF16, bool TRACE, bool FAST, int OUT>
static void launch_t6(const T6Params& p, cudaStream_t st) {
  dim3 grid((unsigned)p.rt, (unsigned)p.ksplit);
  gemm_t6_kernel<MT, SF16, TRACE, FAST, OUT><<<grid, kT6Warps * 32, 0, st>>>(p);
}

template <int MT>
static void dispatch_t6(const T6Params& p, bool sf16, bool trace, bool fast, int out,
                        cudaStream_t st) {
#define FLEXQ_T6_CASE(SF, TR, FA, OU)                                   \
  if (sf16 == SF && trace == TR && fast == FA && (!FA || out == OU)) { \
    launch_t6<MT, SF, TR, FA, OU>(p, st);                              \
    return;                                                            \
  }
  FLEXQ_T6_CASE(true, false, true, FLEXQ_OUT_F16)
  FLEXQ_T6_CASE(true, false, true, FLEXQ_OUT_F32)
  FLEXQ_T6_CASE(false, false, true, FLEXQ_OUT_F16)
  FLEXQ_T6_CASE(false, false, true, FLEXQ_OUT_F32)
  FLEXQ_T6_CASE(true, true, true, FLEXQ_OUT_F16)
  FLEXQ_T6_CASE(true, true, true, FLEXQ_OUT_F32)
  FLEXQ_T6_CASE(false, true, true, FLEXQ_OUT_F16)
  FLEXQ_T6_CASE(false, true, true, FLEXQ_OUT_F32)
  FLEXQ_T6_CASE(true, true, false, 0)
  FLEXQ_T6_CASE(false, true, false, 0)
#undef FLEXQ_T6_CASE
}

constexpr int64_t kT6TokChunk = 64;  // 8 mma n-tiles per launch

// Counters sit after the fp32 split partials of one token chunk.  Sized and located from the
// token count m alone (never from a caller's m_pad, which may be a whole tcgen05 tile), so
// gemm_t6_workspace and gemm_t6_launch agree for every caller.
static int64_t ws_counters_offset(int64_t ksplit, int64_t m, int64_t rt) {
  const int64_t m8 = cdiv(m, kTokTile) * kTokTile;
  const int64_t mc = m8 < kT6TokChunk ? m8 : kT6TokChunk;
  return cdiv(ksplit * mc * rt * kRowTile * 4, 256) * 256;
}

bool gemv_stream_supported(int64_t m, int64_t spg, int64_t units);
int64_t gemv_stream_workspace(int64_t m, int64_t n, int64_t k, int64_t gs);
int gemv_stream_launch(const uint32_t*, const void*, int, const uint32_t*, const float*,
                       const int32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int32_t*, void*,
                       int, void*, const void*, cudaStream_t);

int64_t tc_act_m_pad(int64_t m);
bool gemm_tc_supported(int64_t m, int64_t m_pad, int64_t spg);
int64_t gemm_tc16_workspace(int64_t m, int64_t n);
int64_t gemm_tc_workspace(int64_t m, int64_t n, int64_t k, int64_t gs);
int gemm_tc_launch(const uint32_t*, const void*, int, const uint32_t*, const float*,
                   const int32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int32_t*, void*, int,
                   void*, const void*, cudaStream_t);

// FLEXQ_DISABLE_TC=1 routes M > 16 to the mma.sync kernel (A/B runs; read once, tuning())
static bool tc_enabled() { return !tuning().disable_tc; }

int64_t gemm_t6_workspace(int64_t m, int64_t n, int64_t k, int64_t gs, int ksplit) {
  T6Geom G(n, k, gs);
  const int ks_eff = ksplit <= 0 ? auto_ksplit_t6(G.rt, G.kb) : ksplit;
  int64_t bytes = ws_counters_offset(ks_eff, m, G.rt) + cdiv(G.rt * 4, 256) * 256;
  if ((ksplit == -3 && gemv_stream_supported(m, G.spg, INT64_MAX)) ||
      (ksplit <= 0 && (ksplit == 0 || m <= 16) && gemv_stream_supported(m, G.spg, G.rg * G.kb))) {
    const int64_t b2 = gemv_stream_workspace(m, n, k, gs);
    if (b2 > bytes) bytes = b2;
  }
  if ((ksplit == 0 || ksplit == -2) && gemm_tc_supported(m, tc_act_m_pad(m), G.spg)) {
    const int64_t b3 = gemm_tc_workspace(m, n, k, gs);
    if (b3 > bytes) bytes = b3;
  }
  if (ksplit == 0 && m > 32 && m <= 256 && gs == 128) {  // the kind::f16 batched forward
    const int64_t b6 = gemm_tc16_workspace(m, n);
    if (b6 > bytes) bytes = b6;
  }
  return bytes;
}

int gemm_t6_launch(const uint32_t* t6, const void* wscale, int scale_f16,
                   const uint32_t* act_frag, const float* act_scale, const int32_t* act_corr,
                   int64_t m, int64_t m_pad, int64_t n, int64_t k, int64_t gs, int32_t* partials,
                   void* y, int out_dtype, void* workspace, int ksplit, const void* residual,
                   cudaStream_t st) {
  if (m < 1 || n < 1 || k < 1 || gs < 1) {
    set_error("gemm_t6: dims must be positive, got m=%lld n=%lld k=%lld group=%lld",
              (long long)m, (long long)n, (long long)k, (long long)gs);
    return FLEXQ_ERR_CONFIG;
  }
  if (m_pad < m || m_pad % kTokTile) {
    set_error("gemm_t6: m_pad (%lld) must be a multiple of 8 >= m (%lld)", (long long)m_pad,
              (long long)m);
    return FLEXQ_ERR_SHAPE;
  }
  if (out_dtype != FLEXQ_OUT_F16 && out_dtype != FLEXQ_OUT_F32) {
    set_error("gemm_t6: unknown out_dtype %d", out_dtype);
    return FLEXQ_ERR_CONFIG;
  }
  const bool fast = y != nullptr, trace = partials != nullptr;
  if (!fast && !trace) {
    set_error("gemm_t6: nothing to compute (y and partials are both NULL)");
    return FLEXQ_ERR_CONFIG;
  }
  T6Geom G(n, k, gs);
  // ksplit = -2: the tcgen05 kernel even where the streaming GEMV would be chosen (tests, A/B)
  const bool force_tc = ksplit == -2;
  if (force_tc) {
    if (!gemm_tc_supported(m, m_pad, G.spg)) {
      set_error("gemm_t6: ksplit=-2 (tcgen05) unsupported for m=%lld", (long long)m);
      return FLEXQ_ERR_CONFIG;
    }
    return gemm_tc_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k, gs,
                          partials, y, out_dtype, workspace, residual, st);
  }
  // ksplit = -3: the streaming GEMV whenever it supports the shape (tests, A/B)
  if (ksplit == -3) {
    if (!gemv_stream_supported(m, G.spg, INT64_MAX) || (fast && !workspace)) {
      set_error("gemm_t6: ksplit=-3 (streaming GEMV) unsupported for m=%lld", (long long)m);
      return FLEXQ_ERR_CONFIG;
    }
    return gemv_stream_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k,
                              gs, partials, y, out_dtype, workspace, residual, st);
  }
  // decode regime: the persistent TMA-fed streaming kernel (gemv_stream.cu)
  if (ksplit <= 0 && (ksplit == 0 || m <= 16) && gemv_stream_supported(m, G.spg, G.rg * G.kb) && (workspace || !fast))
    return gemv_stream_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k,
                              gs, partials, y, out_dtype, workspace, residual, st);
  // batched regime: tcgen05.mma kind::i8 with TMEM accumulators (gemm_tc.cu)
  if (ksplit == 0 && tc_enabled() && gemm_tc_supported(m, m_pad, G.spg) && (workspace || !fast))
    return gemm_tc_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k, gs,
                          partials, y, out_dtype, workspace, residual, st);
  if (ksplit <= 0) ksplit = auto_ksplit_t6(G.rt, G.kb);
  if (ksplit > 65535) ksplit = 65535;
  if (ksplit > 1 && fast && !workspace) {
    set_error("gemm_t6: workspace required for ksplit=%d", ksplit);
    return FLEXQ_ERR_CONFIG;
  }
  for (int64_t m0 = 0; m0 < m; m0 += kT6TokChunk) {
    const int64_t mc = (m - m0) < kT6TokChunk ? (m - m0) : kT6TokChunk;
    T6Params p{};
    p.geo = G;
    p.t6 = reinterpret_cast<const uint4*>(t6);
    p.wscale = wscale;
    p.act = reinterpret_cast<const uint4*>(act_frag) + (m0 / kTokTile) * 64;
    p.act_mp8 = m_pad / kTokTile;
    p.xs = act_scale + m0;
    p.corr = act_corr + m0;
    p.m = mc;
    p.m_pad = m_pad;
    p.n = n;
    p.m_total = m;
    p.tok0 = m0;
    p.ws_mstride = cdiv(mc, kTokTile) * kTokTile;
    p.ng = G.ng; p.spg = G.spg; p.ks = G.ks; p.kb = G.kb; p.rt = G.rt;
    p.partials = partials;
    p.y = y;
    p.ws_part = reinterpret_cast<float*>(workspace);
    p.counters = workspace ? reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) +
                                                         ws_counters_offset(ksplit, m, G.rt))
                           : nullptr;
    p.ksplit = ksplit;
    p.res = residual;
    const int mtiles = (int)cdiv(mc, kTokTile);
    if (mtiles <= 1) dispatch_t6<1>(p, scale_f16, trace, fast, out_dtype, st);
    else if (mtiles <= 2) dispatch_t6<2>(p, scale_f16, trace, fast, out_dtype, st);
    else if (mtiles <= 4) dispatch_t6<4>(p, scale_f16, trace, fast, out_dtype, st);
    else dispatch_t6<8>(p, scale_f16, trace, fast, out_dtype, st);
    FLEXQ_LAUNCH_CHECK("gemm_t6");
  }
  return FLEXQ_OK;
}

}  // namespace flexq
