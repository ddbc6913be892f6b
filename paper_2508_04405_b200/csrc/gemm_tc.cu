// Batched (M > 16) T6 GEMM on the 5th-generation tensor cores: tcgen05.mma kind::i8.
//
// Same math as the decode kernels (engine.py:251-365 numerics): per (token m, row n,
// scale group g) the exact integer partial P[g,m,n] = sum_{k in g} x[m,k] * w[n,k],
// then y[m,n] = sum_g (xs[m,g] * ws[n,g]) * P (engine.py:211-216) in fp32, or the
// exact INT32 partials themselves (trace mode).
//
// Data flow per CTA (one persistent CTA per SM, warp-specialised, all hand-off
// through mbarriers):
//   warp 4   weight producer: cp.async.bulk of the two 6 KB T6 units (128 weight
//            rows x one 128-slot k-block) into a 6-deep raw ring.  Weights are
//            offline data, so it starts before griddepcontrol.wait (PDL).
//   warps 0-3 converters: unpack the 6-bit offset-binary codes (unpack_t6) and store
//            them as a K-major, no-swizzle UMMA A tile (128 rows x 128 B, 8x16 B core
//            matrices) -- four STS.128 per lane per 16-row tile.
//   warp 6   activation producer: cp.async.bulk of the B tile (TN tokens x 128 B, the
//            quantizer already wrote it in the UMMA layout) and, per drain event, the
//            column table {-(2^23 + 2^22 + corr), xs} in shared memory.
//   warp 5   MMA issuer (one thread): four tcgen05.mma.kind::i8 (M=128, N=TN, K=32,
//            A u8, B s8, D s32 in TMEM) per k-block; tcgen05.commit frees the stage
//            and, at the end of a scale group, hands the TMEM buffer to the epilogue.
//   warps 7-14 epilogue: tcgen05.ld the INT32 group partial, dequantise into fp32
//            registers, re-seed the TMEM buffer, flush the tile (direct fp16 store or a
//            deterministic stream-K fixup through the workspace).
//
// The TMEM accumulator of every group starts at the integer 0x4B400000 instead of 0
// (re-seeded by the epilogue with one tcgen05.st per 32 columns), so after the group
// D = 0x4B400000 + sum u*x, which read as an fp32 is exactly 12582912 + sum u*x while
// |sum u*x| < 2^22 (any group <= 512 elements; longer groups are drained every 512).
// The dequant is then one FADD (which also removes the offset-binary correction),
// one FMUL and one FFMA per element, and the exact integer is D - 0x4B400000.
//
// Work split (stream-K): units u = tile * KB + kb over (128-row x TN-token tiles,
// k-blocks); CTA c owns units [c*U/P, (c+1)*U/P), so every CTA streams the same number
// of weight bytes for every shape.  A tile split across CTAs is combined in CTA order
// by the last contributor (atomic counter) -- deterministic, as in gemv_stream.cu.
#include "common.cuh"

namespace flexq {

// ---- tcgen05 / TMEM primitives (sm_100a) -------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::i8 (A u8, B s8, D s32), M=128, N=TN, K=32
__device__ __forceinline__ void tc_mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
// every column of this thread's lane in [addr, addr + 16) <- c
__device__ __forceinline__ void tmem_fill16(uint32_t addr, uint32_t c) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1};" ::"r"(addr),
      "r"(c)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sts128(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// K-major, no-swizzle canonical layout: 8-row x 16 B core matrices, LBO = 128 B between
// k-adjacent cores, SBO = 1024 B between 8-row groups (sm_100 descriptor version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}

constexpr int kTcRows = 128;                 // weight rows per tile (UMMA M)
constexpr int kTcConvWarps = 4;              // warps 0-3
constexpr int kTcWarpProdW = 4, kTcWarpMma = 5, kTcWarpProdA = 6, kTcWarpEpi0 = 7;
constexpr int kTcEpiWarps = 8;               // warps 7-14
constexpr int kTcThreads = (kTcWarpEpi0 + kTcEpiWarps) * 32;
constexpr uint32_t kSeed = 0x4B400000u;      // fp32 bits of 12582912 = 1.5 * 2^23
constexpr int kMaxDrainKb = 4;               // exact fp32 reinterpretation needs <= 512 k per drain

template <int TN>
struct TcCfg {
  static constexpr int SW = 6;                     // raw weight ring (12 KB stages)
  static constexpr int SA = TN == 128 ? 3 : 4;     // A/B ring
  static constexpr int NB = 2;                     // TMEM drain buffers
  static constexpr int SS = 4;                     // column-table ring
  static constexpr int kRaw = 2 * kUnitBytes;
  static constexpr int kA = kTcRows * 128;
  static constexpr int kB = TN * 128;
  static constexpr int kTab = TN * 12;             // negC[TN] f32, sx[TN] f32, corr[TN] i32
  static constexpr int kOffRaw = 0;
  static constexpr int kOffA = kOffRaw + SW * kRaw;
  static constexpr int kOffB = kOffA + SA * kA;
  static constexpr int kOffTab = kOffB + SA * kB;
  static constexpr int kOffBar = kOffTab + SS * kTab;
  static constexpr int kNumBars = 2 * SW + 3 * SA + 2 * NB + 2 * SS;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  // NB drain buffers + the fp32 tile accumulator
  static constexpr uint32_t kTmemCols = (NB + 1) * TN <= 64 ? 64 : (NB + 1) * TN <= 128 ? 128 : (NB + 1) * TN <= 256 ? 256 : 512;
  static constexpr int CH = TN / 2;                // columns per epilogue thread
  // instruction descriptor: D s32 (bits 4-5 = 2), A u8 (7-9 = 0), B s8 (10-12 = 1),
  // both K-major, N >> 3 at bit 17, M >> 4 at bit 24
  static constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(TN >> 3) << 17) |
                                     ((uint32_t)(kTcRows >> 4) << 24);
};

struct TcParams {
  const uint8_t* t6;
  const void* wscale;
  const uint8_t* act;
  const float* xs;
  const int32_t* corr;
  int64_t m, m_pad, n;
  int kbn;        // k-blocks per row
  int kpg;        // k-blocks per scale group
  int rg;         // T6 row groups (64 rows)
  int tt;         // token tiles
  int64_t units;  // tiles * kbn
  int nctas;
  T6Geom geo;
  int32_t* partials;
  void* y;
  float* ws_part;
  unsigned* counters;
};

__device__ __forceinline__ int64_t tc_unit_start(int64_t c, int64_t units, int64_t P) {
  return c * units / P;
}
__device__ __forceinline__ int64_t tc_owner(int64_t u, int64_t units, int64_t P) {
  return ((u + 1) * P - 1) / units;
}

// a drain event ends after k-block kb of a tile when the scale group ends, 4 k-blocks of
// a long group have accumulated, the tile's K ends, or the CTA's range ends
__device__ __forceinline__ bool tc_drain_end(int kb, int kbn, int kpg, bool range_end) {
  const int kg = kb % kpg;
  return range_end || kb == kbn - 1 || kg == kpg - 1 || (kg % kMaxDrainKb) == kMaxDrainKb - 1;
}

template <int TN, bool SF16, bool TRACE, bool FAST, int OUT>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(TcParams p) {
  using C = TcCfg<TN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* wfull = bars;
  uint64_t* wempty = wfull + C::SW;
  uint64_t* bfull = wempty + C::SW;
  uint64_t* afull = bfull + C::SA;
  uint64_t* abempty = afull + C::SA;
  uint64_t* dfull = abempty + C::SA;
  uint64_t* dempty = dfull + C::NB;
  uint64_t* sfull = dempty + C::NB;
  uint64_t* sempty = sfull + C::SS;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + C::SS);
  volatile int* flush_flag = reinterpret_cast<volatile int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cta = blockIdx.x, P = p.nctas, U = p.units;
  const int64_t u0 = tc_unit_start(cta, U, P), u1 = tc_unit_start(cta + 1, U, P);
  const int kbn = p.kbn, kpg = p.kpg;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::SW; i++) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], kTcConvWarps); }
    for (int i = 0; i < C::SA; i++) {
      mbar_init(&bfull[i], 1); mbar_init(&afull[i], kTcConvWarps); mbar_init(&abempty[i], 1);
    }
    for (int i = 0; i < C::NB; i++) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], kTcEpiWarps); }
    for (int i = 0; i < C::SS; i++) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], kTcEpiWarps); }
    fence_mbar_init();
  }
  if (warp == kTcWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_launch_dependents();

  if (warp < kTcConvWarps) {
    // ===== converters: T6 unit -> u8 UMMA A tile =====
    const int gq = lane >> 2, t = lane & 3;
    const int rgl = warp >> 1;
    int wi = 0, ai = 0;
    uint32_t wph = 0, aph = 0;
    for (int64_t u = u0; u < u1; u++) {
      mbar_wait(&wfull[wi], wph);
      mbar_wait(&abempty[ai], aph ^ 1u);
      const uint8_t* raw = smem + C::kOffRaw + wi * C::kRaw + rgl * kUnitBytes;
      uint8_t* A = smem + C::kOffA + ai * C::kA;
#pragma unroll
      for (int rr = 0; rr < 2; rr++) {
        const int r = 2 * (warp & 1) + rr;
        const uint4 w0 = lds128(raw + (r * 3 + 0) * 512 + lane * 16);
        const uint4 w1 = lds128(raw + (r * 3 + 1) * 512 + lane * 16);
        const uint4 w2 = lds128(raw + (r * 3 + 2) * 512 + lane * 16);
        uint32_t a[4][4];  // [jj][reg]
#pragma unroll
        for (int jj = 0; jj < 4; jj++) unpack_t6(u4get(w0, jj), u4get(w1, jj), u4get(w2, jj), a[jj]);
        const int r8 = 8 * rgl + 2 * r;  // 8-row group of rows 16r + gq (+8 -> r8 + 1)
        sts128(A + ((r8 + 0) * 8 + 2 * t + 0) * 128 + gq * 16, a[0][0], a[1][0], a[2][0], a[3][0]);
        sts128(A + ((r8 + 1) * 8 + 2 * t + 0) * 128 + gq * 16, a[0][1], a[1][1], a[2][1], a[3][1]);
        sts128(A + ((r8 + 0) * 8 + 2 * t + 1) * 128 + gq * 16, a[0][2], a[1][2], a[2][2], a[3][2]);
        sts128(A + ((r8 + 1) * 8 + 2 * t + 1) * 128 + gq * 16, a[0][3], a[1][3], a[2][3], a[3][3]);
      }
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core
      __syncwarp();
      if (lane == 0) { mbar_arrive(&wempty[wi]); mbar_arrive(&afull[ai]); }
      if (++wi == C::SW) { wi = 0; wph ^= 1u; }
      if (++ai == C::SA) { ai = 0; aph ^= 1u; }
    }
  } else if (warp == kTcWarpProdW) {
    // ===== weight producer =====
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int wi = 0;
      uint32_t wph = 0;
      for (int64_t u = u0; u < u1; u++) {
        const int64_t tile = u / kbn;
        const int kb = (int)(u - tile * kbn);
        const int rg0 = (int)(tile / p.tt) * 2;
        const int nu = rg0 + 1 < p.rg ? 2 : 1;
        mbar_wait(&wempty[wi], wph ^ 1u);
        mbar_expect_tx(&wfull[wi], nu * kUnitBytes);
        uint8_t* dst = smem + C::kOffRaw + wi * C::kRaw;
        bulk_g2s(dst, p.t6 + ((int64_t)rg0 * kbn + kb) * kUnitBytes, kUnitBytes, &wfull[wi], pol);
        if (nu == 2)
          bulk_g2s(dst + kUnitBytes, p.t6 + ((int64_t)(rg0 + 1) * kbn + kb) * kUnitBytes,
                   kUnitBytes, &wfull[wi], pol);
        if (++wi == C::SW) { wi = 0; wph ^= 1u; }
      }
    }
  } else if (warp == kTcWarpProdA) {
    // ===== activation producer: B tiles + per-drain column tables =====
    pdl_wait();
    const uint64_t pol = l2_policy_evict_last();
    int bi = 0, si = 0;
    uint32_t bph = 0, sph = 0;
    int ev_kb0 = -1;  // first k-block of the current drain event
    for (int64_t u = u0; u < u1; u++) {
      const int64_t tile = u / kbn;
      const int kb = (int)(u - tile * kbn);
      const int tt = (int)(tile % p.tt);
      if (ev_kb0 < 0) ev_kb0 = kb;
      if (lane == 0) {
        mbar_wait(&abempty[bi], bph ^ 1u);
        mbar_expect_tx(&bfull[bi], C::kB);
        bulk_g2s(smem + C::kOffB + bi * C::kB,
                 p.act + ((int64_t)kb * (p.m_pad >> 3) + (int64_t)tt * (TN / 8)) * 1024, C::kB,
                 &bfull[bi], pol);
      }
      if (++bi == C::SA) { bi = 0; bph ^= 1u; }
      if (tc_drain_end(kb, kbn, kpg, u == u1 - 1)) {
        mbar_wait(&sempty[si], sph ^ 1u);
        const int g = kb / kpg;
        const bool first = (ev_kb0 % kpg) == 0;  // this event holds the group's first k-block
        float* negc = reinterpret_cast<float*>(smem + C::kOffTab + si * C::kTab);
        float* sx = negc + TN;
        int* cr = reinterpret_cast<int*>(sx + TN);
        for (int col = lane; col < TN; col += 32) {
          const int64_t idx = (int64_t)g * p.m_pad + (int64_t)tt * TN + col;
          const int c = first ? __ldg(&p.corr[idx]) : 0;
          negc[col] = -(12582912.0f + (float)c);
          sx[col] = FAST ? __ldg(&p.xs[idx]) : 0.f;
          cr[col] = c;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfull[si]);
        if (++si == C::SS) { si = 0; sph ^= 1u; }
        ev_kb0 = -1;
      }
    }
  } else if (warp == kTcWarpMma) {
    // ===== MMA issuer =====
    if (lane == 0) {
      int ai = 0, d = 0;
      uint32_t aph = 0;
      bool ev_open = false;
      for (int64_t u = u0; u < u1; u++) {
        const int64_t tile = u / kbn;
        const int kb = (int)(u - tile * kbn);
        const int b = d % C::NB;
        if (!ev_open) {
          mbar_wait(&dempty[b], ((uint32_t)(d / C::NB) & 1u) ^ 1u);
          tc_fence_after();
          ev_open = true;
        }
        mbar_wait(&bfull[ai], aph);
        mbar_wait(&afull[ai], aph);
        tc_fence_after();
        const uint64_t ad = umma_desc(smem_u32(smem + C::kOffA + ai * C::kA));
        const uint64_t bd = umma_desc(smem_u32(smem + C::kOffB + ai * C::kB));
#pragma unroll
        for (int s = 0; s < 4; s++)  // k-cores {2s, 2s+1}: +256 B per K=32 step
          tc_mma_i8(tmem + b * TN, ad + (uint64_t)(s * 16), bd + (uint64_t)(s * 16), C::kIdesc, 1u);
        tc_commit(&abempty[ai]);
        if (tc_drain_end(kb, kbn, kpg, u == u1 - 1)) {
          tc_commit(&dfull[b]);
          d++;
          ev_open = false;
        }
        if (++ai == C::SA) { ai = 0; aph ^= 1u; }
      }
    }
  } else if (warp >= kTcWarpEpi0) {
    // ===== epilogue =====
    // The fp32 accumulator of the tile lives in TMEM too (columns [NB*TN, NB*TN + TN)),
    // so the epilogue holds only 16 columns in registers at a time.
    const int e = warp - kTcWarpEpi0;
    const int q = warp & 3;    // TMEM lane quarter this warp may access
    const int hc = e >> 2;     // column half
    constexpr int CH = C::CH;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16) + hc * CH;
    const uint32_t tacc = tl + C::NB * TN;
    const int rho = 32 * q + lane;  // tile row of this thread
#pragma unroll
    for (int b = 0; b < C::NB; b++)
#pragma unroll
      for (int c0 = 0; c0 < CH; c0 += 16) tmem_fill16(tl + b * TN + c0, kSeed);
    tmem_wait_st();
    tc_fence_before();
    pdl_wait();

    // weight-scale index of this thread's row: T6 row group rg, row tile r, pair (gq, i)
    const int rgl = rho >> 6, r_in = (rho >> 4) & 3, gq = rho & 7, half8 = (rho >> 3) & 1;
    auto load_sw = [&](int64_t tile, int g) -> float {
      if constexpr (!FAST) return 0.f;
      const int64_t rg = (tile / p.tt) * 2 + rgl;
      if (rg >= p.rg) return 0.f;
      const int64_t idx = p.geo.scale_index(rg * kRowGroup + r_in, g, gq) * 2 + half8;
      if constexpr (SF16) return __half2float(reinterpret_cast<const __half*>(p.wscale)[idx]);
      else return reinterpret_cast<const float*>(p.wscale)[idx];
    };
    auto store_row = [&](int64_t tt, int64_t n_row, int c0, const float (&a)[16]) {
      if (n_row >= p.n) return;
#pragma unroll
      for (int j = 0; j < 16; j++) {
        const int64_t m = tt * TN + hc * CH + c0 + j;
        if (m < p.m) {
          if constexpr (OUT == FLEXQ_OUT_F16)
            reinterpret_cast<__half*>(p.y)[m * p.n + n_row] = __float2half_rn(a[j]);
          else
            reinterpret_cast<float*>(p.y)[m * p.n + n_row] = a[j];
        }
      }
    };

    int d = 0, si = 0;
    uint32_t sph = 0;
    int ev_kb0 = -1;
    bool acc_live = false;  // the TMEM accumulator holds this tile's earlier drains
    for (int64_t u = u0; u < u1; u++) {
      const int64_t tile = u / kbn;
      const int kb = (int)(u - tile * kbn);
      if (ev_kb0 < 0) ev_kb0 = kb;
      const bool rend = u == u1 - 1;
      if (!tc_drain_end(kb, kbn, kpg, rend)) continue;
      const int g = kb / kpg;
      const bool first = (ev_kb0 % kpg) == 0;
      const float sw = load_sw(tile, g);
      const int b = d % C::NB;
      mbar_wait(&dfull[b], (uint32_t)(d / C::NB) & 1u);
      mbar_wait(&sfull[si], sph);
      tc_fence_after();
      const float* tab = reinterpret_cast<const float*>(smem + C::kOffTab + si * C::kTab);
      const float* negc = tab + hc * CH;
      const float* sx = tab + TN + hc * CH;
      const int* cr = reinterpret_cast<const int*>(tab + 2 * TN) + hc * CH;
      const int64_t tt = tile % p.tt;
      const int64_t n_row = (tile / p.tt) * kTcRows + rho;
#pragma unroll 1
      for (int c0 = 0; c0 < CH; c0 += 16) {
        uint32_t v[32], av[32];
        tmem_ld16(tl + b * TN + c0, v);
        if (FAST && acc_live) tmem_ld16(tacc + c0, av);
        tmem_wait_ld();
        if constexpr (FAST) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 nc = *reinterpret_cast<const float4*>(negc + c0 + j);
            const float4 sv = *reinterpret_cast<const float4*>(sx + c0 + j);
            const float n4[4] = {nc.x, nc.y, nc.z, nc.w}, s4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
            for (int i = 0; i < 4; i++) {
              const float prev = acc_live ? __uint_as_float(av[j + i]) : 0.f;
              av[j + i] = __float_as_uint(fmaf(sw * s4[i], __uint_as_float(v[j + i]) + n4[i], prev));
            }
          }
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,"
              "%12,%13,%14,%15,%16};" ::"r"(tacc + c0),
              "r"(av[0]), "r"(av[1]), "r"(av[2]), "r"(av[3]), "r"(av[4]), "r"(av[5]), "r"(av[6]),
              "r"(av[7]), "r"(av[8]), "r"(av[9]), "r"(av[10]), "r"(av[11]), "r"(av[12]),
              "r"(av[13]), "r"(av[14]), "r"(av[15])
              : "memory");
        }
        if constexpr (TRACE) {
#pragma unroll
          for (int j = 0; j < 16; j++) {
            const int64_t m = tt * TN + hc * CH + c0 + j;
            if (m < p.m && n_row < p.n) {
              const int P = (int)(v[j] - kSeed) - (first ? cr[c0 + j] : 0);
              atomicAdd(&p.partials[((int64_t)g * p.m + m) * p.n + n_row], P);
            }
          }
        }
        tmem_fill16(tl + b * TN + c0, kSeed);  // re-seed for the buffer's next group
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) { mbar_arrive(&dempty[b]); mbar_arrive(&sempty[si]); }
      d++;
      if (++si == C::SS) { si = 0; sph ^= 1u; }
      ev_kb0 = -1;
      acc_live = true;

      if (FAST && (kb == kbn - 1 || rend)) {
        // ---- flush this tile: direct store, or the deterministic stream-K fixup ----
        acc_live = false;
        const int64_t first_c = tc_owner(tile * kbn, U, P);
        const int64_t last_c = tc_owner(tile * kbn + kbn - 1, U, P);
        if (first_c == last_c) {
#pragma unroll 1
          for (int c0 = 0; c0 < CH; c0 += 16) {
            uint32_t av[32];
            tmem_ld16(tacc + c0, av);
            tmem_wait_ld();
            float a[16];
#pragma unroll
            for (int j = 0; j < 16; j++) a[j] = __uint_as_float(av[j]);
            store_row(tt, n_row, c0, a);
          }
          continue;
        }
        const int which = u0 >= tile * kbn ? 0 : 1;
        float* slot = p.ws_part + ((cta * 2 + which) * TN + hc * CH) * (int64_t)kTcRows + rho;
#pragma unroll 1
        for (int c0 = 0; c0 < CH; c0 += 16) {
          uint32_t av[32];
          tmem_ld16(tacc + c0, av);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; j++) slot[(c0 + j) * kTcRows] = __uint_as_float(av[j]);
        }
        __threadfence();
        named_bar_sync(1, kTcEpiWarps * 32);
        if (e == 0 && lane == 0) {
          const unsigned prev = atom_add_acq_rel_gpu(&p.counters[tile], 1u);
          *flush_flag = prev == (unsigned)(last_c - first_c) ? 1 : 0;
        }
        named_bar_sync(1, kTcEpiWarps * 32);
        const bool last = *flush_flag != 0;
        named_bar_sync(1, kTcEpiWarps * 32);  // flag read by all before the next flush
        if (!last) continue;
        __threadfence();
#pragma unroll 1
        for (int c0 = 0; c0 < CH; c0 += 16) {
          float a[16];
#pragma unroll
          for (int j = 0; j < 16; j++) a[j] = 0.f;
          for (int64_t c = first_c; c <= last_c; c++) {  // fixed CTA order: deterministic
            const int wc = tc_unit_start(c, U, P) >= tile * kbn ? 0 : 1;
            const float* src =
                p.ws_part + ((c * 2 + wc) * TN + hc * CH + c0) * (int64_t)kTcRows + rho;
#pragma unroll
            for (int j = 0; j < 16; j++) a[j] += __ldcg(src + j * kTcRows);
          }
          store_row(tt, n_row, c0, a);
        }
        if (e == 0 && lane == 0) p.counters[tile] = 0u;
      }
    }
  }

  // ---- teardown: every role done with TMEM before the allocating warp frees it ----
  tc_fence_before();
  __syncthreads();
  if (warp == kTcWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::kTmemCols)
                 : "memory");
  }
}

// ---- host side ------------------------------------------------------------------------------
static int tc_tn(int64_t m) { return m <= 32 ? 32 : m <= 64 ? 64 : 128; }

int64_t tc_act_m_pad(int64_t m) {
  if (m <= 16) return cdiv(m, kTokTile) * kTokTile;
  const int tn = tc_tn(m);
  return cdiv(m, tn) * tn;
}

bool gemm_tc_supported(int64_t m, int64_t m_pad, int64_t spg) {
  if (m <= 16 || spg % 4 != 0) return false;
  const int tn = tc_tn(m);
  return m_pad >= cdiv(m, tn) * tn;
}

static int tc_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

static int64_t tc_ctas(int64_t units) { return units < tc_sms() ? units : tc_sms(); }

int64_t gemm_tc_workspace(int64_t m, int64_t n, int64_t k, int64_t gs) {
  T6Geom G(n, k, gs);
  const int tn = tc_tn(m);
  const int64_t tiles = cdiv(n, kTcRows) * cdiv(m, tn);
  const int64_t sms = tc_sms() > 148 ? tc_sms() : 148;  // two partial-tile slots per CTA
  return cdiv(sms * 2 * tn * kTcRows * 4, 256) * 256 + cdiv(tiles * 4, 256) * 256;
}

template <int TN, bool SF16, bool TRACE, bool FAST, int OUT>
static int launch_tc_inst(const TcParams& p, cudaStream_t st) {
  auto kern = gemm_tc_kernel<TN, SF16, TRACE, FAST, OUT>;
  constexpr int smem = TcCfg<TN>::kBytes;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "gemm_tc attribute");
    configured = true;
  }
  cudaError_t e = launch_pdl(kern, dim3((unsigned)p.nctas), dim3(kTcThreads), (size_t)smem, st, p);
  if (e != cudaSuccess) return cuda_status(e, "gemm_tc launch");
  return FLEXQ_OK;
}

template <int TN>
static int dispatch_tc(const TcParams& p, bool sf16, bool trace, bool fast, int out,
                       cudaStream_t st) {
#define FLEXQ_TC(SF, TR, FA, OU)                                      \
  if (sf16 == SF && trace == TR && fast == FA && (!FA || out == OU)) \
    return launch_tc_inst<TN, SF, TR, FA, OU>(p, st);
  FLEXQ_TC(true, false, true, FLEXQ_OUT_F16)
  FLEXQ_TC(true, false, true, FLEXQ_OUT_F32)
  FLEXQ_TC(false, false, true, FLEXQ_OUT_F16)
  FLEXQ_TC(false, false, true, FLEXQ_OUT_F32)
  FLEXQ_TC(true, true, true, FLEXQ_OUT_F16)
  FLEXQ_TC(false, true, true, FLEXQ_OUT_F16)
  FLEXQ_TC(true, true, true, FLEXQ_OUT_F32)
  FLEXQ_TC(false, true, true, FLEXQ_OUT_F32)
  FLEXQ_TC(true, true, false, FLEXQ_OUT_F16)
  FLEXQ_TC(false, true, false, FLEXQ_OUT_F16)
#undef FLEXQ_TC
  set_error("gemm_tc: unsupported flag combination");
  return FLEXQ_ERR_CONFIG;
}

int gemm_tc_launch(const uint32_t* t6, const void* wscale, int scale_f16, const uint32_t* act_frag,
                   const float* xs, const int32_t* corr, int64_t m, int64_t m_pad, int64_t n,
                   int64_t k, int64_t gs, int32_t* partials, void* y, int out_dtype,
                   void* workspace, cudaStream_t st) {
  T6Geom G(n, k, gs);
  if (!gemm_tc_supported(m, m_pad, G.spg)) {
    set_error("gemm_tc: unsupported m=%lld m_pad=%lld group_size=%lld", (long long)m,
              (long long)m_pad, (long long)gs);
    return FLEXQ_ERR_CONFIG;
  }
  const bool trace = partials != nullptr, fast = y != nullptr;
  if (fast && !workspace) {
    set_error("gemm_tc: workspace required");
    return FLEXQ_ERR_CONFIG;
  }
  const int tn = tc_tn(m);
  TcParams p{};
  p.t6 = reinterpret_cast<const uint8_t*>(t6);
  p.wscale = wscale;
  p.act = reinterpret_cast<const uint8_t*>(act_frag);
  p.xs = xs;
  p.corr = corr;
  p.m = m; p.m_pad = m_pad; p.n = n;
  p.kbn = (int)G.kb;
  p.kpg = (int)(G.spg / 4);
  p.rg = (int)G.rg;
  p.tt = (int)cdiv(m, tn);
  const int64_t tiles = cdiv(n, kTcRows) * p.tt;
  p.units = tiles * G.kb;
  p.nctas = (int)tc_ctas(p.units);
  p.geo = G;
  p.partials = partials;
  p.y = y;
  if (workspace) {
    p.ws_part = reinterpret_cast<float*>(workspace);
    const int64_t sms = tc_sms() > 148 ? tc_sms() : 148;
    p.counters = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) +
                                             cdiv(sms * 2 * tn * kTcRows * 4, 256) * 256);
  }
  const bool sf16 = scale_f16 != 0;
  switch (tn) {
    case 32: return dispatch_tc<32>(p, sf16, trace, fast, out_dtype, st);
    case 64: return dispatch_tc<64>(p, sf16, trace, fast, out_dtype, st);
    default: return dispatch_tc<128>(p, sf16, trace, fast, out_dtype, st);
  }
}

}  // namespace flexq
