// EXPERIMENT (not built into libflexq_sm100a.so) -- round 2, DESIGN.md sec. 4.1.
// Paired-warp stream for 16 < M <= 32: two warps share each TMA stage and split the 32 tokens.
// Bit-exact (tests passed), 134 registers -> 12-16 warps per SM instead of 8, but no faster:
// 70B gate_proj M = 32 59.8-61 us vs 55 us for the MT = 4 stream (qkv / o equal).  The
// duplicated unpack and weight LDS per unit cost what the extra occupancy buys.
// Streaming GEMV for 16 < M <= 32 with warp PAIRS (group 128, one group per k-block).
//
// Same math as gemv_stream.cu's MT = 4 path (unpack-to-INT8 + mma.sync m16n8k32, exact INT32
// group partials, fused fp32 dequant: engine.py:251-365, 211-216) and the same TMA-bulk unit
// stream, but two warps consume every stage: the leader issues the copies of a unit (6 KB of
// T6 weights + the activation operand of all 32 tokens + scales), both warps unpack the same
// weights and each multiplies them with HALF of the tokens (two 8-token tiles).  A warp then
// holds half the accumulators of the MT = 4 kernel (32 instead of 64 fp32 per thread), so the
// register footprint drops from 237 to ~130 and twice as many warps fit on an SM -- the MT = 4
// stream was latency-bound at two warps per SMSP (ncu at M = 32).  The
// stage is consumed by both warps before the leader refills it (an "empty" mbarrier with two
// arrivals).  Split row groups are combined deterministically as in gemv_stream.cu (slot per
// contributor and token half, the last arrival sums in contributor order).
#include "common.cuh"

namespace flexq {

constexpr int kPairWarps = 4;   // 2 pairs per CTA

__device__ __forceinline__ void pair_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
constexpr int kPairMinUnits = 6;

struct PairParams {
  const uint8_t* t6;
  const void* wscale;
  const uint8_t* act;
  const float* xs;
  const int32_t* corr;
  int64_t m, m_pad, n, kb, rg, units, np;  // np: pairs in the launch
  T6Geom geo;
  int32_t* partials;
  void* y;
  float* ws_part;
  unsigned* counters;  // [rg][2]
  const void* res;
};

template <bool SF16>
struct PairStage {
  static constexpr int kOffB = kUnitBytes;           // 4 token tiles x 1 KB
  static constexpr int kOffWs = kOffB + 4 * 1024;
  static constexpr int kWs = kRowGroup * 8 * (SF16 ? 4 : 8);
  static constexpr int kOffXs = kOffWs + kWs;        // 32 tokens x 4 B
  static constexpr int kOffCorr = kOffXs + 128;
  static constexpr int kBytes = kOffCorr + 128;
};

template <int OUT>
__device__ __forceinline__ void pair_store(void* y, int64_t i, float v) {
  if constexpr (OUT == FLEXQ_OUT_F16)
    reinterpret_cast<__half*>(y)[i] = __float2half_rn(v);
  else
    reinterpret_cast<float*>(y)[i] = v;
}

template <bool SF16, bool TRACE, bool FAST, int OUT, int S>
__global__ void __launch_bounds__(kPairWarps * 32, 4) gemv_pair_kernel(PairParams p) {
  using L = PairStage<SF16>;
  constexpr int UB = L::kBytes;
  constexpr int SB = SF16 ? 4 : 8;
  constexpr int MT = 2;  // token tiles per warp
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int half = warp & 1;  // 0: leader (issues the copies), tokens 0-15; 1: tokens 16-31
  const int64_t gp = (int64_t)blockIdx.x * (kPairWarps / 2) + (warp >> 1);
  if (gp >= p.np) return;  // pair-uniform; no CTA-wide barriers below
  uint8_t* ring = smem + (warp >> 1) * (S * UB);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (kPairWarps / 2) * (S * UB)) + (warp >> 1) * 2 * S;
  uint64_t* empty = full + S;
  const int64_t u0 = gp * p.units / p.np, u1 = (gp + 1) * p.units / p.np;
  const bool leader = half == 0 && lane == 0;
  if (leader) {
#pragma unroll
    for (int s = 0; s < S; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
    }
    fence_mbar_init();
  }
  // both warps of the pair see the barriers initialised: a named barrier per pair
  asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
  const uint64_t pol_w = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
  const int64_t kbn = p.kb;
  // part 0: weights + weight scales (offline data, before the PDL wait); part 1: activations
  auto issue = [&](int64_t u, int s, int part) {
    const int64_t rg = u / kbn, kb = u - rg * kbn;
    uint8_t* dst = ring + s * UB;
    const uint32_t vb = (uint32_t)(p.m_pad * 4);
    if (part == 0) {
      mbar_expect_tx(&full[s], kUnitBytes + 4 * 1024 + kRowGroup * 8 * SB + (FAST ? vb : 0) + vb);
      bulk_g2s(dst, p.t6 + u * (int64_t)kUnitBytes, kUnitBytes, &full[s], pol_w);
      bulk_g2s(dst + L::kOffWs, reinterpret_cast<const uint8_t*>(p.wscale) +
                                    p.geo.scale_index(rg * kRowGroup, kb, 0) * SB,
               kRowGroup * 8 * SB, &full[s], pol_w);
    } else {
      bulk_g2s(dst + L::kOffB, p.act + kb * (p.m_pad >> 3) * 1024, 4 * 1024, &full[s], pol_a);
      if (FAST) bulk_g2s(dst + L::kOffXs, p.xs + kb * p.m_pad, vb, &full[s], pol_a);
      bulk_g2s(dst + L::kOffCorr, p.corr + kb * p.m_pad, vb, &full[s], pol_a);
    }
  };
  int pro = 0;
  if (leader)
    for (; pro < S && u0 + pro < u1; pro++) issue(u0 + pro, pro, 0);
  pdl_wait();
  pdl_launch_dependents();
  if (leader)
    for (int s = 0; s < pro; s++) issue(u0 + s, s, 1);

  float acc[4][MT][4];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;

  // publish a finished row group: direct store, or the deterministic split fixup over the
  // contributing pairs (slot per pair and token half)
  auto flush = [&](int64_t rg) {
    if constexpr (!FAST) return;
    const int64_t first = ((rg * kbn + 1) * p.np - 1) / p.units;
    const int64_t last = ((rg * kbn + kbn) * p.np - 1) / p.units;
    constexpr int kSlot = 4 * MT * 4 * 32;
    if (first != last) {
      float* slot = p.ws_part + ((rg + gp) * 2 + half) * (int64_t)kSlot + lane;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) slot[((r * MT + mt) * 4 + i) * 32] = acc[r][mt][i];
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0) prev = atom_add_acq_rel_gpu(&p.counters[rg * 2 + half], 1u);
      prev = __shfl_sync(0xffffffffu, prev, 0);
      if (prev != (unsigned)(last - first)) return;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
      constexpr int FB = 2;  // contributors' slots in flight per L2 round trip
      for (int64_t w = first; w <= last; w += FB) {
        float v[FB][4][MT][4];
#pragma unroll
        for (int f = 0; f < FB; f++) {
          const float* src = p.ws_part + ((rg + w + f) * 2 + half) * (int64_t)kSlot + lane;
#pragma unroll
          for (int r = 0; r < 4; r++)
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
              for (int i = 0; i < 4; i++)
                v[f][r][mt][i] = w + f > last ? 0.f : __ldcg(src + ((r * MT + mt) * 4 + i) * 32);
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
      if (lane == 0) p.counters[rg * 2 + half] = 0u;
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int64_t row0 = (rg * kRowGroup + r) * kRowTile + gq;
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int64_t tok = (2 * half + mt) * kTokTile + 2 * t + (i & 1);
          const int64_t row = row0 + ((i & 2) ? 8 : 0);
          if (tok < p.m && row < p.n)
            pair_store<OUT>(p.y, tok * p.n + row, acc[r][mt][i] + residual_at<OUT>(p.res, tok * p.n + row));
        }
    }
  };

  int64_t rg = u0 / kbn, kb = u0 - rg * kbn;
  int s = 0;
  uint32_t parity = 0;
  for (int64_t u = u0; u < u1; u++) {
    mbar_wait(&full[s], parity);
    const uint8_t* st = ring + s * UB;
    // this warp's two token tiles: 2 * half, 2 * half + 1 of the stage's four
    uint4 bv[MT][2];
    int2 cz[MT], cb[MT];  // corrections; cb = 0x4B400000 - corr (the fp32 conversion bias)
#pragma unroll
    for (int mt = 0; mt < MT; mt++) {
      const int tt = 2 * half + mt;
      bv[mt][0] = lds128(st + L::kOffB + tt * 1024 + (2 * t) * 128 + gq * 16);
      bv[mt][1] = lds128(st + L::kOffB + tt * 1024 + (2 * t + 1) * 128 + gq * 16);
      cz[mt] = reinterpret_cast<const int2*>(st + L::kOffCorr)[(tt * kTokTile) / 2 + t];
      cz[mt].x -= kCorrBias; cz[mt].y -= kCorrBias;
      cb[mt] = make_int2(kCorrBias - cz[mt].x, kCorrBias - cz[mt].y);
    }
    float2 sw[4], sx[MT];
    if constexpr (FAST) {
#pragma unroll
      for (int r = 0; r < 4; r++) {
        if constexpr (SF16) sw[r] = __half22float2(reinterpret_cast<const __half2*>(st + L::kOffWs)[r * 8 + gq]);
        else sw[r] = reinterpret_cast<const float2*>(st + L::kOffWs)[r * 8 + gq];
      }
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
        sx[mt] = reinterpret_cast<const float2*>(st + L::kOffXs)[((2 * half + mt) * kTokTile) / 2 + t];
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {  // row tile outermost: one tile's weights and partials live
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
      const int64_t row0 = (rg * kRowGroup + r) * kRowTile + gq, row1 = row0 + 8;
#pragma unroll
      for (int mt = 0; mt < MT; mt++) {
        if constexpr (TRACE) {
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int64_t tok = (2 * half + mt) * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
            if (tok < p.m && row < p.n)
              atomicAdd(&p.partials[(kb * p.m + tok) * p.n + row], Pr[mt][i] - (i & 1 ? cz[mt].y : cz[mt].x));
          }
        }
        if constexpr (FAST) {
          // P = Pr - corr (|P| < 2^22 for a 128-k group) read as an fp32 without I2F, packed math
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
    // this warp is done with the stage; the leader refills it once its partner is too
    __syncwarp();
    if (lane == 0) pair_arrive(&empty[s]);
    if (leader && u + S < u1) {
      mbar_wait(&empty[s], parity);
      fence_proxy_async_smem();
      issue(u + S, s, 0);
      issue(u + S, s, 1);
    }
    if (++s == S) { s = 0; parity ^= 1u; }
    if (++kb == kbn) {
      flush(rg);
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
          for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
      kb = 0;
      rg++;
    }
  }
  if (kb != 0) flush(rg);
}

// ---- host side ------------------------------------------------------------------------------
bool gemv_pair_supported(int64_t m, int64_t spg) { return m > 16 && m <= 32 && spg == 4; }

static int64_t pair_slots(int64_t rg) { return rg + 148 * 8 + 16; }

int64_t gemv_pair_workspace(int64_t m, int64_t n, int64_t k, int64_t gs) {
  (void)m;
  T6Geom G(n, k, gs);
  return cdiv(pair_slots(G.rg) * 2 * 4 * 2 * 4 * 32 * 4, 256) * 256 + cdiv(G.rg * 2 * 4, 256) * 256;
}

template <bool SF16, bool TRACE, bool FAST, int OUT, int S>
static int launch_pair_inst(PairParams p, cudaStream_t st) {
  auto kern = gemv_pair_kernel<SF16, TRACE, FAST, OUT, S>;
  constexpr int UB = PairStage<SF16>::kBytes;
  const int smem = (kPairWarps / 2) * S * (UB + 16);
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return cuda_status(e, "gemv_pair attribute");
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kPairWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;  // slots are sized for <= 8 pairs per SM
  int64_t pairs = (int64_t)device_sms() * per_sm * (kPairWarps / 2);
  const int64_t by_units = cdiv(p.units, kPairMinUnits);
  if (pairs > by_units) pairs = by_units;
  p.np = pairs;
  const unsigned ctas = (unsigned)cdiv(pairs, kPairWarps / 2);
  e = launch_pdl(kern, dim3(ctas), dim3(kPairWarps * 32), (size_t)smem, st, p);
  if (e != cudaSuccess) return cuda_status(e, "gemv_pair launch");
  return FLEXQ_OK;
}

int gemv_pair_launch(const uint32_t* t6, const void* wscale, int scale_f16,
                     const uint32_t* act_frag, const float* xs, const int32_t* corr, int64_t m,
                     int64_t m_pad, int64_t n, int64_t k, int64_t gs, int32_t* partials, void* y,
                     int out_dtype, void* workspace, const void* residual, cudaStream_t st) {
  T6Geom G(n, k, gs);
  if (!gemv_pair_supported(m, G.spg) || m_pad < 32) {
    set_error("gemv_pair: needs 16 < m <= 32 (m_pad >= 32) and group_size 128, got m=%lld", (long long)m);
    return FLEXQ_ERR_CONFIG;
  }
  if (y && !workspace) {
    set_error("gemv_pair: workspace required");
    return FLEXQ_ERR_CONFIG;
  }
  PairParams p{};
  p.t6 = reinterpret_cast<const uint8_t*>(t6);
  p.wscale = wscale;
  p.act = reinterpret_cast<const uint8_t*>(act_frag);
  p.xs = xs;
  p.corr = corr;
  p.m = m; p.m_pad = m_pad; p.n = n;
  p.kb = G.kb; p.rg = G.rg; p.units = G.rg * G.kb;
  p.geo = G;
  p.partials = partials;
  p.y = y;
  p.res = residual;
  if (workspace) {
    p.ws_part = reinterpret_cast<float*>(workspace);
    p.counters = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) +
                                             cdiv(pair_slots(G.rg) * 2 * 4 * 2 * 4 * 32 * 4, 256) * 256);
  }
  const bool trace = partials != nullptr, fast = y != nullptr, sf16 = scale_f16 != 0;
  const int S = p.units <= 12288 ? 3 : 2;
#define FLEXQ_PC(SF, TR, FA, OU, SS)                                                        \
  if (sf16 == SF && trace == TR && fast == FA && (!FA || out_dtype == OU) && S == SS)      \
    return launch_pair_inst<SF, TR, FA, OU, SS>(p, st);
#define FLEXQ_PC_S(SF, TR, FA, OU) FLEXQ_PC(SF, TR, FA, OU, 2) FLEXQ_PC(SF, TR, FA, OU, 3)
  FLEXQ_PC_S(true, false, true, FLEXQ_OUT_F16)
  FLEXQ_PC_S(true, false, true, FLEXQ_OUT_F32)
  FLEXQ_PC_S(false, false, true, FLEXQ_OUT_F16)
  FLEXQ_PC_S(false, false, true, FLEXQ_OUT_F32)
  FLEXQ_PC_S(true, true, true, FLEXQ_OUT_F16)
  FLEXQ_PC_S(false, true, true, FLEXQ_OUT_F16)
  FLEXQ_PC_S(true, true, true, FLEXQ_OUT_F32)
  FLEXQ_PC_S(false, true, true, FLEXQ_OUT_F32)
  FLEXQ_PC_S(true, true, false, FLEXQ_OUT_F16)
  FLEXQ_PC_S(false, true, false, FLEXQ_OUT_F16)
#undef FLEXQ_PC_S
#undef FLEXQ_PC
  set_error("gemv_pair: unsupported flag combination");
  return FLEXQ_ERR_CONFIG;
}

}  // namespace flexq
