// EXPERIMENT (not built into libflexq_sm100a.so) -- kept with its measurement, DESIGN.md sec. 4.1.
// Round 2: the five LLaMA-2-70B decode linears as one persistent "chain" launch (grid
// barriers between links, next-link weight prefetch during the tail) were bit-identical to
// per-linear launches but SLOWER: 174 us vs 143.7 us per M=1 step (profiles/
// r02_bench_chain_experiment.json).  The per-CTA timeline (profiles/r02_chain_timeline.txt,
// tools/experiments/chain_timeline.py) shows why: each grid barrier costs ~2 us (444
// same-address arrivals serialise in L2) and the in-kernel quantizer phase ~2.5 us, so a
// link boundary costs ~7 us -- more than the ~2.8 us a PDL-overlapped per-linear launch pays.
// It compiled against an older C ABI (FlexQChainLink in flexq.h), which was removed with it.
// A chain of decode-regime W6Ax linears in ONE persistent launch (M <= 16, group 128).
//
// Each link is the online half of the reference's quantized_linear (engine.py:487-513):
// quantize the fp16 activations x_j (quantize.py:118-148, fp16 scales) and run the T6 GEMV
// with the fused group-dequant epilogue (engine.py:251-287, 211-216) -- exactly what
// flexq_linear_forward does per call, with the same per-warp streaming pipeline as
// gemv_stream.cu (MODE 0).  What the single launch removes is the per-linear fixed cost
// measured in DESIGN.md sec. 4.1 (launch and CTA ramp of every GEMV, the streaming tail of
// every layer, the quantizer kernel in between):
//
//   * every warp owns a contiguous unit range of EVERY link (static split, per link);
//   * the moment a warp has consumed its range of link j it issues the weight half of the
//     first S stages of its link-(j+1) range -- the weight stream of the next layer starts
//     during this layer's tail, not after it;
//   * grid barrier A (only if link j+1 depends on link j's output): every warp of the grid
//     has finished link j, so y_j is complete (fixups included);
//   * the quantizer phase: warp w quantizes (row, group) items w, w + W, ... of x_{j+1} into
//     link j+1's activation operand (quantize_g128_lane: bit-identical to the quantizer
//     kernel);
//   * grid barrier B: the operand is complete; each warp issues the activation half of its
//     prefetched stages and streams on.
//
// Results are identical to a flexq_linear_forward per link (same split of every link over
// the same number of warps -> same fixed-order fixups): the chain changes the schedule, not
// the arithmetic.  The grid is sized to the occupancy (all CTAs co-resident), so the
// barriers cannot deadlock.
#include <algorithm>

#include "common.cuh"
#include "quant_math.cuh"

namespace flexq {

constexpr int kChainMax = 16;
constexpr int kChainWarps = 4;  // warps per CTA (several CTAs per SM)

struct ChainLinkDev {
  const uint8_t* t6;
  const uint8_t* wscale;
  const __half* x;
  uint8_t* act;   // operand [kb][m_pad/8][8][8][16 B]
  float* xs;      // [G][m_pad]
  int32_t* corr;  // [G][m_pad]
  void* y;
  const void* res;
  int64_t n, k, kb, rg, units, nw;
  int bits, dep;
};

struct ChainParams {
  ChainLinkDev L[kChainMax];
  int nl;
  int64_t m, m_pad;
  int64_t tw;          // warps in the grid
  float* ws_part;      // split-fixup slots (shared by the links: they run one after another)
  unsigned* counters;  // per row group (max over links), zero between links
  unsigned* gbar;      // [0] arrival counter, [32] epoch (own 128 B lines)
  uint32_t* flag;
  long long* tl;       // debug timeline (FLEXQ_CHAIN_TIMELINE), normally NULL:
                       // per CTA [start, then per link: barrier A in/out, B out, loop done]
};
constexpr int kChainTlPerCta = 1 + 4 * kChainMax;

template <int MT, bool SF16>
struct ChainStage {
  static constexpr int kOffB = kUnitBytes;
  static constexpr int kOffWs = kOffB + MT * 1024;
  static constexpr int kWs = kRowGroup * 8 * (SF16 ? 4 : 8);
  static constexpr int kOffXs = kOffWs + kWs;
  static constexpr int kVec = 16 * 4;  // m_pad <= 16 tokens x 4 B
  static constexpr int kOffCorr = kOffXs + kVec;
  static constexpr int kBytes = kOffCorr + kVec;
};

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Sense-reversal grid barrier over all CTAs (every warp of every CTA calls it).  The epoch is
// read before arriving; the last arriver resets the counter and bumps the epoch.
__device__ __forceinline__ void grid_barrier(unsigned* gbar, unsigned nctas) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* cnt = gbar;
    unsigned* epoch = gbar + 32;
    const unsigned e = ld_acquire_gpu(epoch);
    __threadfence();
    const unsigned old = atomicAdd(cnt, 1u);
    if (old == nctas - 1) {
      atomicExch(cnt, 0u);
      __threadfence();
      st_release_gpu(epoch, e + 1);
    } else {
      while (ld_acquire_gpu(epoch) == e) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int MT, bool SF16, int S, bool ONE>
__global__ void __launch_bounds__(kChainWarps * 32) gemv_chain_kernel(const __grid_constant__ ChainParams p) {
  using L = ChainStage<MT, SF16>;
  constexpr int UB = L::kBytes;
  constexpr int SB = SF16 ? 4 : 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  // warps interleaved over the CTAs: a link that uses fewer than all warps spreads its
  // warps over every SM
  const int64_t gw = (int64_t)warp * gridDim.x + blockIdx.x;
  uint8_t* ring = smem + warp * (S * UB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kChainWarps * (S * UB)) + warp * S;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol_w = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
  const int64_t m = p.m, m_pad = p.m_pad;

  int s = 0;            // ring position (continues across links)
  uint32_t parity = 0;
  // issue one stage: part 0 = weights + weight scales (offline data), part 1 = activation
  // operand, scales, corrections (written by the quantizer phase)
  auto issue = [&](const ChainLinkDev& l, int64_t u, int st, int part) {
    const int64_t rgu = u / l.kb, kb = u - rgu * l.kb;  // group g = kb (group 128)
    uint8_t* dst = ring + st * UB;
    const uint32_t vb = (uint32_t)(m_pad * 4);
    if (part == 0) {
      mbar_expect_tx(&bar[st], kUnitBytes + MT * 1024 + kRowGroup * 8 * SB + 2 * vb);
      bulk_g2s(dst, l.t6 + u * (int64_t)kUnitBytes, kUnitBytes, &bar[st], pol_w);
      bulk_g2s(dst + L::kOffWs, l.wscale + ((rgu * l.kb + kb) * kRowGroup * 8) * SB,
               kRowGroup * 8 * SB, &bar[st], pol_w);
    } else {
      bulk_g2s(dst + L::kOffB, l.act + kb * (m_pad >> 3) * 1024, MT * 1024, &bar[st], pol_a);
      bulk_g2s(dst + L::kOffXs, l.xs + kb * m_pad, vb, &bar[st], pol_a);
      bulk_g2s(dst + L::kOffCorr, l.corr + kb * m_pad, vb, &bar[st], pol_a);
    }
  };

  float acc[4][MT][4];
  int P[4][MT][4];
  auto zero_acc = [&]() {
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
  };

  // publish a finished row group (same fixed-order split fixup as gemv_stream.cu)
  auto flush = [&](const ChainLinkDev& l, int64_t rg, int64_t gr) {
    const int64_t first = ((rg * l.kb + 1) * l.nw - 1) / l.units;
    const int64_t last = ((rg * l.kb + l.kb) * l.nw - 1) / l.units;
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
      zero_acc();
      constexpr int FB = ONE ? 8 : (MT == 1 ? 4 : 2);
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
          if (tok < m && row < l.n) {
            const float v = acc[r][mt][i] + residual_at<FLEXQ_OUT_F16>(l.res, tok * l.n + row);
            reinterpret_cast<__half*>(l.y)[tok * l.n + row] = __float2half_rn(v);
          }
        }
    }
  };

  // ---- link 0's weight prologue runs before the PDL wait (weights are offline data) ----
  int pro = 0;
  auto prefetch_weights = [&](const ChainLinkDev& l) {
    pro = 0;
    if (gw >= l.nw) return;
    const int64_t u0 = gw * l.units / l.nw, u1 = (gw + 1) * l.units / l.nw;
    if (lane == 0)
      for (int i = 0; i < S && u0 + i < u1; i++) issue(l, u0 + i, (s + i) % S, 0);
    pro = (int)(u1 - u0 < S ? u1 - u0 : S);
  };
  auto mark = [&](int slot) {
    if (p.tl && threadIdx.x == 0) p.tl[blockIdx.x * kChainTlPerCta + slot] = dbg_now();
  };
  mark(0);
  prefetch_weights(p.L[0]);
  pdl_wait();

  for (int j = 0; j < p.nl; j++) {
    const ChainLinkDev& l = p.L[j];
    mark(1 + 4 * j);
    if (j > 0 && l.dep) grid_barrier(p.gbar, gridDim.x);  // y_{j-1} complete
    mark(2 + 4 * j);
    // ---- quantizer phase: (row, group) items of x_j over all warps of the grid ----
    {
      const int64_t ng = l.kb, items = m * ng;
      for (int64_t it = gw; it < items; it += p.tw) {
        const int64_t r = it / ng, g = it - r * ng;
        const uint2 raw = *reinterpret_cast<const uint2*>(l.x + r * l.k + g * 128 + lane * 4);
        uint32_t word;
        int csum;
        const double sc = quantize_g128_lane(raw, l.bits, 1, p.flag, lane, word, csum);
        *reinterpret_cast<uint32_t*>(l.act + operand_word_offset(g, r, m_pad, lane)) = word;
        if (lane == 0) {
          l.xs[g * m_pad + r] = (float)sc;
          l.corr[g * m_pad + r] = kCorrBias + 32 * csum;
        }
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");  // read back by TMA after B
    }
    grid_barrier(p.gbar, gridDim.x);  // x_j's operand complete
    mark(3 + 4 * j);
    if (j == p.nl - 1) pdl_launch_dependents();
    if (gw < l.nw) {
      const int64_t u0 = gw * l.units / l.nw, u1 = (gw + 1) * l.units / l.nw;
      if (lane == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> TMA reads
        for (int i = 0; i < pro; i++) issue(l, u0 + i, (s + i) % S, 1);
      }
      int64_t iu = u0 + pro;  // next unit to fetch
      int64_t rg = u0 / l.kb, kb = u0 - rg * l.kb;
      zero_acc();
      for (int64_t u = u0; u < u1; u++) {
        mbar_wait(&bar[s], parity);
        const uint8_t* st = ring + s * UB;
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
        int2 corr0[MT];
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          corr0[mt] = reinterpret_cast<const int2*>(st + L::kOffCorr)[(mt * kTokTile) / 2 + t];
          corr0[mt].x -= kCorrBias;
          corr0[mt].y -= kCorrBias;
        }
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
#pragma unroll
          for (int r = 0; r < 4; r++) {  // 4 independent accumulator chains
            uint32_t a[4];
            unpack_t6(u4get(w[r][0], jj), u4get(w[r][1], jj), u4get(w[r][2], jj), a);
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
              if (jj == 0) mma_u8s8_zc(P[r][mt], a, bv[mt][0].x, bv[mt][1].x);
              else mma_u8s8(P[r][mt], a, u4get(bv[mt][0], jj), u4get(bv[mt][1], jj));
            }
          }
        }
        // drain the unit's group: P - 32 * sum(x) read as fp32 without I2F, packed dequant
        float2 sw[4], sx[MT];
#pragma unroll
        for (int r = 0; r < 4; r++) {
          if constexpr (SF16) sw[r] = __half22float2(reinterpret_cast<const __half2*>(st + L::kOffWs)[r * 8 + gq]);
          else sw[r] = reinterpret_cast<const float2*>(st + L::kOffWs)[r * 8 + gq];
        }
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
          sx[mt] = reinterpret_cast<const float2*>(st + L::kOffXs)[(mt * kTokTile) / 2 + t];
        const float2 c2 = make_float2(12582912.f, 12582912.f);
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            const int cb0 = kCorrBias - corr0[mt].x, cb1 = kCorrBias - corr0[mt].y;
            if (ONE) {
              const float2 f = f2_sub(make_float2(__int_as_float(P[r][mt][0] + cb0),
                                                  __int_as_float(P[r][mt][2] + cb0)), c2);
              const float2 sc = f2_mul(sw[r], make_float2(sx[mt].x, sx[mt].x));
              const float2 a = f2_fma(sc, f, make_float2(acc[r][mt][0], acc[r][mt][2]));
              acc[r][mt][0] = a.x; acc[r][mt][2] = a.y;
            } else {
              const float2 f01 = f2_sub(make_float2(__int_as_float(P[r][mt][0] + cb0),
                                                    __int_as_float(P[r][mt][1] + cb1)), c2);
              const float2 f23 = f2_sub(make_float2(__int_as_float(P[r][mt][2] + cb0),
                                                    __int_as_float(P[r][mt][3] + cb1)), c2);
              const float2 s01 = f2_mul(make_float2(sw[r].x, sw[r].x), sx[mt]);
              const float2 s23 = f2_mul(make_float2(sw[r].y, sw[r].y), sx[mt]);
              const float2 a01 = f2_fma(s01, f01, make_float2(acc[r][mt][0], acc[r][mt][1]));
              const float2 a23 = f2_fma(s23, f23, make_float2(acc[r][mt][2], acc[r][mt][3]));
              acc[r][mt][0] = a01.x; acc[r][mt][1] = a01.y;
              acc[r][mt][2] = a23.x; acc[r][mt][3] = a23.y;
            }
          }
        __syncwarp();
        if (lane == 0 && iu < u1) {
          fence_proxy_async_smem();
          issue(l, iu, s, 0);
          issue(l, iu, s, 1);
        }
        iu++;
        if (++s == S) { s = 0; parity ^= 1u; }
        if (++kb == l.kb) {
          flush(l, rg, gw);
          zero_acc();
          kb = 0;
          rg++;
        }
      }
      if (kb != 0) flush(l, rg, gw);
    }
    __syncwarp();
    if (p.tl) {  // (debug) CTA-level loop end = its slowest warp
      __syncthreads();
      mark(4 + 4 * j);
    }
    // the next link's weight stream starts now, during this link's tail
    if (j + 1 < p.nl) prefetch_weights(p.L[j + 1]);
  }
}

// ---- host side ------------------------------------------------------------------------------
int64_t gemv_stream_plan_warps(int64_t m, int64_t n, int64_t k, int64_t gs, int scale_f16);
static long long* g_chain_tl = nullptr;
static int g_chain_ctas = 0;
extern "C" int flexq_debug_chain_timeline(long long* host, int max_entries) {
  const int n = g_chain_ctas * kChainTlPerCta;
  if (!g_chain_tl || max_entries < n) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_chain_tl, n * sizeof(long long), cudaMemcpyDeviceToHost);
  return g_chain_ctas;
}

int64_t chain_workspace(const FlexQChainLink* links, int nl, int64_t m) {
  int64_t rg_max = 0;
  for (int i = 0; i < nl; i++) rg_max = std::max<int64_t>(rg_max, cdiv(links[i].n, 64));
  const int64_t mt = m <= 8 ? 1 : 2;
  const int64_t slots = rg_max + 148 * 16 + 16;
  return cdiv(slots * 4 * mt * 4 * 32 * 4, 256) * 256 + cdiv(rg_max * 4, 256) * 256 + 256;
}

struct ChainDevCache {
  int dev = -1, sms = 0;
  bool configured[8] = {};
};
static thread_local ChainDevCache g_chain_cache[16];

template <int MT, bool SF16, int S, bool ONE>
static int chain_launch_inst(ChainParams& p, int dev, cudaStream_t st) {
  auto kern = gemv_chain_kernel<MT, SF16, S, ONE>;
  constexpr int UB = ChainStage<MT, SF16>::kBytes;
  const int smem = kChainWarps * S * (UB + 8);
  ChainDevCache& c = g_chain_cache[dev & 15];
  if (c.dev != dev) {
    c = ChainDevCache{};
    c.dev = dev;
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int ci = (MT == 1 ? 0 : 4) + (SF16 ? 0 : 2) + (ONE ? 1 : 0);
  if (!c.configured[ci]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "gemv_chain attribute");
    c.configured[ci] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kChainWarps * 32, smem);
  if (per_sm < 1) {
    set_error("gemv_chain: kernel does not fit on an SM");
    return FLEXQ_ERR_CUDA;
  }
  if (per_sm > 4) per_sm = 4;  // fixup slots are sized for <= 16 warps per SM
  const int ctas = c.sms * per_sm;
  g_chain_ctas = ctas;
  p.tw = (int64_t)ctas * kChainWarps;
  for (int i = 0; i < p.nl; i++) {
    ChainLinkDev& l = p.L[i];
    // split every link over exactly the warps of its per-linear launch (gemv_stream.cu), so
    // the fixed-order fixups -- and the outputs -- are identical to flexq_linear_forward
    const int64_t nw = gemv_stream_plan_warps(p.m, l.n, l.k, 128, SF16 ? 1 : 0);
    if (nw < 1) {
      set_error("gemv_chain: link %d is not a streaming-GEMV shape", i);
      return FLEXQ_ERR_CONFIG;
    }
    l.nw = std::min<int64_t>(p.tw, nw);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ctas);
  cfg.blockDim = dim3(kChainWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeCooperative;  // co-residency of every CTA (grid barriers)
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  if (e != cudaSuccess) return cuda_status(e, "gemv_chain launch");
  return FLEXQ_OK;
}

int chain_launch(const FlexQChainLink* links, int nl, int64_t m, int scale_f16, void* workspace,
                 int64_t workspace_bytes, uint32_t* flag, cudaStream_t st) {
  if (nl < 1 || nl > kChainMax) {
    set_error("chain_forward: 1..%d links, got %d", kChainMax, nl);
    return FLEXQ_ERR_CONFIG;
  }
  if (m < 1 || m > 16) {
    set_error("chain_forward: decode batches only (1 <= m <= 16), got m=%lld", (long long)m);
    return FLEXQ_ERR_CONFIG;
  }
  if (!workspace || !flag) {
    set_error("chain_forward: workspace and flag are required");
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (workspace_bytes < chain_workspace(links, nl, m)) {
    set_error("chain_forward: workspace of %lld bytes, need %lld", (long long)workspace_bytes,
              (long long)chain_workspace(links, nl, m));
    return FLEXQ_ERR_SHAPE;
  }
  ChainParams p{};
  p.nl = nl;
  p.m = m;
  p.m_pad = cdiv(m, kTokTile) * kTokTile;
  for (int i = 0; i < nl; i++) {
    const FlexQChainLink& a = links[i];
    if (a.group_size != 128 || a.k % 128 || a.n < 1 || a.k < 128) {
      set_error("chain_forward: link %d needs group_size 128 and K a multiple of 128 "
                "(got n=%lld k=%lld group=%lld)", i, (long long)a.n, (long long)a.k,
                (long long)a.group_size);
      return FLEXQ_ERR_CONFIG;
    }
    if (a.xbits < 2 || a.xbits > 8) {
      set_error("chain_forward: link %d: bits must be in 2..8, got %d", i, a.xbits);
      return FLEXQ_ERR_INVALID_INPUT;
    }
    if (!a.t6 || !a.wscale || !a.x || !a.act_buf || !a.y) {
      set_error("chain_forward: link %d: t6, wscale, x, act_buf and y are required", i);
      return FLEXQ_ERR_INVALID_INPUT;
    }
    if (reinterpret_cast<uintptr_t>(a.x) % 8) {
      set_error("chain_forward: link %d: x must be 8-byte aligned", i);
      return FLEXQ_ERR_INVALID_INPUT;
    }
    T6Geom G(a.n, a.k, 128);
    ChainLinkDev& l = p.L[i];
    l.t6 = reinterpret_cast<const uint8_t*>(a.t6);
    l.wscale = reinterpret_cast<const uint8_t*>(a.wscale);
    l.x = reinterpret_cast<const __half*>(a.x);
    // act_buf: the flexq_linear_forward layout (flexq_act_buf_bytes)
    char* base = reinterpret_cast<char*>(a.act_buf);
    const int64_t frag = cdiv(cdiv(p.m_pad, kTokTile) * G.kb * 32 * 32, 256) * 256;
    const int64_t vec = cdiv(G.ng * p.m_pad * 4, 256) * 256;
    l.act = reinterpret_cast<uint8_t*>(base);
    l.xs = reinterpret_cast<float*>(base + frag);
    l.corr = reinterpret_cast<int32_t*>(base + frag + vec);
    l.y = a.y;
    l.res = a.residual;
    l.n = a.n;
    l.k = a.k;
    l.kb = G.kb;
    l.rg = G.rg;
    l.units = G.rg * G.kb;
    l.bits = a.xbits;
    l.dep = a.depends_on_prev ? 1 : 0;
  }
  char* ws = reinterpret_cast<char*>(workspace);
  int64_t rg_max = 0;
  for (int i = 0; i < nl; i++) rg_max = std::max<int64_t>(rg_max, p.L[i].rg);
  const int64_t mt = m <= 8 ? 1 : 2;
  const int64_t slot_bytes = cdiv((rg_max + 148 * 16 + 16) * 4 * mt * 4 * 32 * 4, 256) * 256;
  p.ws_part = reinterpret_cast<float*>(ws);
  p.counters = reinterpret_cast<unsigned*>(ws + slot_bytes);
  p.gbar = reinterpret_cast<unsigned*>(ws + slot_bytes + cdiv(rg_max * 4, 256) * 256);
  p.flag = flag;
  static long long* tlbuf = nullptr;
  if (getenv("FLEXQ_CHAIN_TIMELINE")) {  // debug only (tools/chain_timeline.py)
    if (!tlbuf) cudaMalloc(&tlbuf, 148 * 16 * kChainTlPerCta * sizeof(long long));
    cudaMemsetAsync(tlbuf, 0, 148 * 16 * kChainTlPerCta * sizeof(long long), st);
    p.tl = tlbuf;
    g_chain_tl = tlbuf;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const bool sf16 = scale_f16 != 0;
  int rc;
  if (m == 1) rc = sf16 ? chain_launch_inst<1, true, 2, true>(p, dev, st)
                        : chain_launch_inst<1, false, 2, true>(p, dev, st);
  else if (m <= 8) rc = sf16 ? chain_launch_inst<1, true, 2, false>(p, dev, st)
                             : chain_launch_inst<1, false, 2, false>(p, dev, st);
  else rc = sf16 ? chain_launch_inst<2, true, 2, false>(p, dev, st)
                 : chain_launch_inst<2, false, 2, false>(p, dev, st);
  return rc;
}

}  // namespace flexq
