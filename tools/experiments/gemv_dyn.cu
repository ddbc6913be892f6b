// EXPERIMENT (not built into libflexq_sm100a.so; round 1, opt-in FLEXQ_GEMV_DYN=1 until round 2):
// dynamically scheduled GEMV pieces.  Removed the per-warp spread but its claim / fixup
// atomics cost more than they saved (70B gate M=1: 34.1 -> 42.6 us), DESIGN.md sec. 4.1.
// Kept for the record; it compiled against the round-1 gemm_t6.cu dispatch.
// Decode-regime T6 GEMV with dynamic piece scheduling (group = one k-block, e.g. g = 128).
//
// Same math, stage layout and TMA ring as gemv_stream.cu, but the work is cut into fixed
// pieces (row group rg, k-block range j) that warps take from a global queue: every warp
// starts with its own piece (so the weight stream begins before griddepcontrol.wait) and
// then claims the next free one with one atomicAdd, issued a whole piece ahead so its
// latency stays off the stream.  Measured on B200 (tools/gemv_timeline.py) a static equal
// split leaves the slowest warps ~25 % behind the median on 70B layers; claiming pieces lets
// fast warps absorb that -- but the claim/fixup atomics cost more than they save, so this
// kernel is opt-in (FLEXQ_GEMV_DYN=1) and kept for A/B runs.  The result stays deterministic: a piece's fp32 partial always
// goes to slot (rg, j), and the last piece of a row group to finish (atomic counter) sums
// the slots in j order -- the reduction order never depends on which warp ran which piece.
#include "common.cuh"

namespace flexq {

constexpr int kDWarps = 4;

struct DynParams {
  const uint8_t* t6;
  const void* wscale;
  const uint8_t* act;
  const float* xs;
  const int32_t* corr;
  int64_t m, m_pad, n, kb, rg;
  int pk, ppr;          // k-blocks per piece, pieces per row group
  int64_t np, nw;       // pieces, warps
  T6Geom geo;
  int32_t* partials;
  void* y;
  float* slots;         // [rg][ppr][4][MT][4][32] fp32 piece partials
  unsigned* counters;   // [rg] pieces finished (left zeroed)
  unsigned* queue;      // [2]: next dynamic piece - nw, finished warps (left zeroed)
  const void* res;      // optional residual added at the store
};

template <int MT, bool SF16>
struct DynStage {
  static constexpr int kWs = kRowGroup * 8 * (SF16 ? 4 : 8);
  static constexpr int kOffB = kUnitBytes;
  static constexpr int kOffWs = kOffB + MT * 1024;
  static constexpr int kOffXs = kOffWs + kWs;
  static constexpr int kOffCorr = kOffXs + 16 * 4;
  static constexpr int kBytes = kOffCorr + 16 * 4;
};

template <int OUT>
__device__ __forceinline__ void dyn_store(void* y, int64_t i, float v) {
  if constexpr (OUT == FLEXQ_OUT_F16)
    reinterpret_cast<__half*>(y)[i] = __float2half_rn(v);
  else
    reinterpret_cast<float*>(y)[i] = v;
}

template <int MT, bool SF16, bool TRACE, bool FAST, int OUT, int S, bool ONE>
__global__ void __launch_bounds__(kDWarps * 32, MT == 1 ? 3 : 2) gemv_t6_dyn_kernel(DynParams p) {
  using L = DynStage<MT, SF16>;
  constexpr int UB = L::kBytes;
  constexpr int SB = SF16 ? 4 : 8;
  constexpr int kSlot = 4 * MT * 4 * 32;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kDWarps][S];
  __shared__ int pq[kDWarps][8];  // piece ids in flight (issue side -> compute side)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gq = lane >> 2, t = lane & 3;
  const int64_t gw = (int64_t)blockIdx.x * kDWarps + warp;
  if (gw >= p.nw) return;
  uint8_t* ring = smem + warp * (S * UB);
  uint64_t* bar = bars[warp];
  int* q = pq[warp];
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol_w = l2_policy_evict_first(), pol_a = l2_policy_evict_last();
  const int kbn = (int)p.kb;

  auto issue = [&](int rg, int kb, int s, int part) {
    const uint32_t wsb = FAST ? (uint32_t)(kRowGroup * 8 * SB) : 0u;
    const uint32_t xsb = FAST ? (uint32_t)(p.m_pad * 4) : 0u;
    const uint32_t cb = (uint32_t)(p.m_pad * 4);
    uint8_t* dst = ring + s * UB;
    if (part == 0) {
      mbar_expect_tx(&bar[s], kUnitBytes + MT * 1024 + wsb + xsb + cb);
      bulk_g2s(dst, p.t6 + ((int64_t)rg * kbn + kb) * kUnitBytes, kUnitBytes, &bar[s], pol_w);
      if (FAST)
        bulk_g2s(dst + L::kOffWs,
                 reinterpret_cast<const uint8_t*>(p.wscale) +
                     p.geo.scale_index((int64_t)rg * kRowGroup, kb, 0) * SB,
                 wsb, &bar[s], pol_w);
    } else {
      bulk_g2s(dst + L::kOffB, p.act + (int64_t)kb * (p.m_pad >> 3) * 1024, MT * 1024, &bar[s],
               pol_a);
      if (FAST) bulk_g2s(dst + L::kOffXs, p.xs + (int64_t)kb * p.m_pad, xsb, &bar[s], pol_a);
      bulk_g2s(dst + L::kOffCorr, p.corr + (int64_t)kb * p.m_pad, cb, &bar[s], pol_a);
    }
  };

  // ---- issue cursor (lane 0): walks pieces; q[] hands their ids to the compute side ----
  int ip = (int)gw;            // piece being issued
  int ikb = 0, ikb1 = 0, irg = 0;
  int qhead = 0;               // next q[] slot to fill
  unsigned claimed = 0;        // next dynamic piece (claimed one piece ahead)
  bool issue_done = false;
  auto start_piece = [&](int piece) {
    if (piece >= p.np) { issue_done = true; return; }
    irg = piece / p.ppr;
    const int j = piece - irg * p.ppr;
    ikb = j * p.pk;
    ikb1 = min(ikb + p.pk, kbn);
    q[qhead & 7] = piece;
    qhead++;
  };
  // unit number iss (issue order) always goes to stage iss % S, the order the compute side
  // consumes them in; the piece after the current one is claimed as soon as it starts
  int iss = 0;
  auto next_unit = [&]() {
    iss++;
    if (++ikb == ikb1) {
      const int next = (int)claimed;
      claimed = (unsigned)p.nw + atomicAdd(&p.queue[0], 1u);
      start_piece(next);
    }
  };
  int pro = 0;
  if (lane == 0) {
    start_piece(ip);
    // before griddepcontrol.wait: only this warp's own first piece, and only its weights
    for (int pkb = ikb; pro < S && pkb < ikb1; pro++, pkb++) issue(irg, pkb, pro, 0);
  }
  pdl_wait();
  pdl_launch_dependents();
  if (lane == 0) {
    claimed = (unsigned)p.nw + atomicAdd(&p.queue[0], 1u);
    for (int s = 0; s < pro; s++) {
      issue(irg, ikb, s, 1);
      next_unit();
    }
    while (iss < S && !issue_done) {  // top the ring up across the piece boundary
      issue(irg, ikb, iss % S, 0);
      issue(irg, ikb, iss % S, 1);
      next_unit();
    }
  }
  __syncwarp();

  float acc[4][MT][4];
  int P[4][MT][4];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int mt = 0; mt < MT; mt++)
#pragma unroll
      for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;

  auto store_rows = [&](int rg) {
#pragma unroll
    for (int r = 0; r < 4; r++) {
      const int64_t row0 = ((int64_t)rg * kRowGroup + r) * kRowTile + gq;
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if (ONE && (i & 1)) continue;
          const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = row0 + ((i & 2) ? 8 : 0);
          if (tok < p.m && row < p.n)
            dyn_store<OUT>(p.y, tok * p.n + row, acc[r][mt][i] + residual_at<OUT>(p.res, tok * p.n + row));
        }
    }
  };
  // a finished piece: direct store, or its slot + the in-order sum by the row group's last piece
  auto flush_piece = [&](int rg, int j) {
    if constexpr (!FAST) return;
    if (p.ppr == 1) { store_rows(rg); return; }
    float* slot = p.slots + ((int64_t)rg * p.ppr + j) * kSlot + lane;
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
    if (prev != (unsigned)(p.ppr - 1)) return;
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
    constexpr int FB = ONE ? 4 : 2;
    for (int j0 = 0; j0 < p.ppr; j0 += FB) {  // fixed slot order: deterministic
      float v[FB][4][MT][4];
#pragma unroll
      for (int f = 0; f < FB; f++) {
        const float* src = p.slots + ((int64_t)rg * p.ppr + j0 + f) * kSlot + lane;
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int i = 0; i < 4; i++)
              v[f][r][mt][i] = ((ONE && (i & 1)) || j0 + f >= p.ppr)
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
    store_rows(rg);
    if (lane == 0) p.counters[rg] = 0u;
  };

  // ---- compute cursor ----
  int qtail = 0, s = 0;
  uint32_t parity = 0;
  while (true) {
    const int piece = __shfl_sync(0xffffffffu, qtail < qhead ? q[qtail & 7] : -1, 0);
    // (lane 0 owns qhead; its q[] writes precede the __syncwarp at the end of each unit)
    if (piece < 0) break;
    qtail++;
    const int rg = piece / p.ppr, j = piece - rg * p.ppr;
    const int kb0 = j * p.pk, kb1 = min(kb0 + p.pk, kbn);
    for (int kb = kb0; kb < kb1; kb++) {
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
        corr0[mt].x -= kCorrBias; corr0[mt].y -= kCorrBias;
      }
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
          uint32_t a[4];
          unpack_t6(u4get(w[r][0], jj), u4get(w[r][1], jj), u4get(w[r][2], jj), a);
#pragma unroll
          for (int mt = 0; mt < MT; mt++) {
            if (jj == 0) mma_u8s8_zc(P[r][mt], a, bv[mt][0].x, bv[mt][1].x);
            else mma_u8s8(P[r][mt], a, u4get(bv[mt][0], jj), u4get(bv[mt][1], jj));
          }
        }
      }
      // drain the group (= this k-block)
      float2 sw[4], sx[MT];
      if constexpr (FAST) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int idx = r * 8 + gq;
          if constexpr (SF16) sw[r] = __half22float2(reinterpret_cast<const __half2*>(st + L::kOffWs)[idx]);
          else sw[r] = reinterpret_cast<const float2*>(st + L::kOffWs)[idx];
        }
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
          sx[mt] = reinterpret_cast<const float2*>(st + L::kOffXs)[(mt * kTokTile) / 2 + t];
      }
#pragma unroll
      for (int r = 0; r < 4; r++) {
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
          P[r][mt][0] -= corr0[mt].x; P[r][mt][2] -= corr0[mt].x;
          if (!ONE) { P[r][mt][1] -= corr0[mt].y; P[r][mt][3] -= corr0[mt].y; }
        }
        const int64_t row0 = ((int64_t)rg * kRowGroup + r) * kRowTile + gq, row1 = row0 + 8;
        if constexpr (TRACE) {
#pragma unroll
          for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int i = 0; i < 4; i++) {
              if (ONE && (i & 1)) continue;
              const int64_t tok = mt * kTokTile + 2 * t + (i & 1), row = (i & 2) ? row1 : row0;
              if (tok < p.m && row < p.n)
                atomicAdd(&p.partials[((int64_t)kb * p.m + tok) * p.n + row], P[r][mt][i]);
            }
        }
        if constexpr (FAST) {
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
      __syncwarp();
      if (lane == 0 && !issue_done) {  // refill the freed stage with the next unit in issue order
        fence_proxy_async_smem();
        issue(irg, ikb, iss % S, 0);
        issue(irg, ikb, iss % S, 1);
        next_unit();
      }
      __syncwarp();
      if (++s == S) { s = 0; parity ^= 1u; }
    }
    flush_piece(rg, j);
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
      for (int mt = 0; mt < MT; mt++)
#pragma unroll
        for (int i = 0; i < 4; i++) acc[r][mt][i] = 0.f;
    qhead = __shfl_sync(0xffffffffu, qhead, 0);
  }
  // the last warp out resets the queue for the next launch on this workspace
  if (lane == 0) {
    const unsigned fin = atom_add_acq_rel_gpu(&p.queue[1], 1u);
    if (fin == (unsigned)(p.nw - 1)) { p.queue[0] = 0u; p.queue[1] = 0u; }
  }
}

// ---- host side ------------------------------------------------------------------------------
static int dyn_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// pieces per row group: about 4 pieces per warp at full occupancy, whole k-blocks each
static void dyn_geometry(int64_t rg, int64_t kb, int64_t warps, int stages, int* pk, int* ppr) {
  int64_t want = cdiv(4 * warps, rg);  // pieces per row group
  if (want < 1) want = 1;
  if (want > kb / stages) want = kb / stages > 0 ? kb / stages : 1;  // a piece fills the ring
  if (want > 16) want = 16;              // bounds the in-order fan-in of the fixup
  *pk = (int)cdiv(kb, want);
  *ppr = (int)cdiv(kb, *pk);
}

bool gemv_dyn_supported(int64_t m, int64_t spg) {
  static int en = -1;
  if (en < 0) {
    // opt-in (FLEXQ_GEMV_DYN=1): measured slower than the static split on B200 -- the per-
    // piece claim and fixup atomics (~1 us each on the warp's critical path) cost more than
    // the ~25 % warp imbalance they remove (70B gate_proj M=1: 34.1 -> 42.6 us)
    const char* e = getenv("FLEXQ_GEMV_DYN");
    en = (e && atoi(e) == 1) ? 1 : 0;
  }
  return en == 1 && m <= 16 && spg == 4;
}

int64_t gemv_dyn_workspace(int64_t m, int64_t n, int64_t k, int64_t gs) {
  T6Geom G(n, k, gs);
  const int mt = m <= 8 ? 1 : 2;
  return cdiv(G.rg * 16 * 4 * mt * 4 * 32 * 4, 256) * 256 + cdiv(G.rg * 4, 256) * 256 + 256;
}

template <int MT, bool SF16, bool TRACE, bool FAST, int OUT, int S>
static int launch_dyn(DynParams p, cudaStream_t st) {
  const bool one = MT == 1 && p.m == 1;
  auto kern = one ? gemv_t6_dyn_kernel<MT, SF16, TRACE, FAST, OUT, S, MT == 1>
                  : gemv_t6_dyn_kernel<MT, SF16, TRACE, FAST, OUT, S, false>;
  const int smem = kDWarps * S * DynStage<MT, SF16>::kBytes;
  static bool configured[2] = {false, false};
  if (!configured[one]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "gemv_dyn attribute");
    configured[one] = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kDWarps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 4) per_sm = 4;
  int64_t warps = (int64_t)dyn_sms() * per_sm * kDWarps;
  int pk, ppr;
  dyn_geometry(p.rg, p.kb, warps, S, &pk, &ppr);
  p.pk = pk;
  p.ppr = ppr;
  p.np = p.rg * ppr;
  if (warps > p.np) warps = p.np;
  p.nw = warps;
  cudaError_t e = launch_pdl(kern, dim3((unsigned)cdiv(warps, kDWarps)), dim3(kDWarps * 32),
                             (size_t)smem, st, p);
  if (e != cudaSuccess) return cuda_status(e, "gemv_dyn launch");
  return FLEXQ_OK;
}

template <int MT, int S>
static int dispatch_dyn(const DynParams& p, bool sf16, bool trace, bool fast, int out,
                        cudaStream_t st) {
#define FLEXQ_DC(SF, TR, FA, OU) \
  if (sf16 == SF && trace == TR && fast == FA && (!FA || out == OU)) return launch_dyn<MT, SF, TR, FA, OU, S>(p, st);
  FLEXQ_DC(true, false, true, FLEXQ_OUT_F16)
  FLEXQ_DC(true, false, true, FLEXQ_OUT_F32)
  FLEXQ_DC(false, false, true, FLEXQ_OUT_F16)
  FLEXQ_DC(false, false, true, FLEXQ_OUT_F32)
  FLEXQ_DC(true, true, true, FLEXQ_OUT_F16)
  FLEXQ_DC(false, true, true, FLEXQ_OUT_F16)
  FLEXQ_DC(true, true, true, FLEXQ_OUT_F32)
  FLEXQ_DC(false, true, true, FLEXQ_OUT_F32)
  FLEXQ_DC(false, true, false, FLEXQ_OUT_F16)
  FLEXQ_DC(true, true, false, FLEXQ_OUT_F16)
#undef FLEXQ_DC
  set_error("gemv_dyn: unsupported flag combination");
  return FLEXQ_ERR_CONFIG;
}

int gemv_dyn_launch(const uint32_t* t6, const void* wscale, int scale_f16, const uint32_t* act_frag,
                    const float* xs, const int32_t* corr, int64_t m, int64_t m_pad, int64_t n,
                    int64_t k, int64_t gs, int32_t* partials, void* y, int out_dtype,
                    void* workspace, const void* residual, cudaStream_t st) {
  T6Geom G(n, k, gs);
  if (!gemv_dyn_supported(m, G.spg) || !workspace) {
    set_error("gemv_dyn: unsupported m=%lld group_size=%lld (or no workspace)", (long long)m,
              (long long)gs);
    return FLEXQ_ERR_CONFIG;
  }
  DynParams p{};
  p.t6 = reinterpret_cast<const uint8_t*>(t6);
  p.wscale = wscale;
  p.act = reinterpret_cast<const uint8_t*>(act_frag);
  p.xs = xs;
  p.corr = corr;
  p.m = m; p.m_pad = m_pad; p.n = n; p.kb = G.kb; p.rg = G.rg;
  p.geo = G;
  p.partials = partials;
  p.y = y;
  p.res = residual;
  const int mt = m <= 8 ? 1 : 2;
  char* ws = reinterpret_cast<char*>(workspace);
  p.slots = reinterpret_cast<float*>(ws);
  const int64_t slot_bytes = cdiv(G.rg * 16 * 4 * mt * 4 * 32 * 4, 256) * 256;
  p.counters = reinterpret_cast<unsigned*>(ws + slot_bytes);
  p.queue = reinterpret_cast<unsigned*>(ws + slot_bytes + cdiv(G.rg * 4, 256) * 256);
  const bool trace = partials != nullptr, fast = y != nullptr, sf16 = scale_f16 != 0;
  const int64_t units = G.rg * G.kb;
  const int S = units <= 4096 ? 4 : units <= 12288 ? 3 : 2;
  if (mt == 1) {
    if (S == 4) return dispatch_dyn<1, 4>(p, sf16, trace, fast, out_dtype, st);
    if (S == 3) return dispatch_dyn<1, 3>(p, sf16, trace, fast, out_dtype, st);
    return dispatch_dyn<1, 2>(p, sf16, trace, fast, out_dtype, st);
  }
  if (S == 4) return dispatch_dyn<2, 4>(p, sf16, trace, fast, out_dtype, st);
  if (S == 3) return dispatch_dyn<2, 3>(p, sf16, trace, fast, out_dtype, st);
  return dispatch_dyn<2, 2>(p, sf16, trace, fast, out_dtype, st);
}

}  // namespace flexq
