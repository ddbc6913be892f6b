// Batched (32 < M <= 256) W6Ax fast path on tcgen05 kind::f16: the group scales are applied to
// the OPERANDS, so the tensor core accumulates the whole K range of a tile in one fp32 TMEM
// accumulator and the epilogue runs once per tile instead of once per 128-k group.
//
// Why (round 2): the INT8 kernel (gemm_tc.cu) must take every group's
// INT32 partial out of TMEM to scale it (engine.py:211-216), and those per-group TMEM round
// trips run at ~40 B/clk per SM while the MMAs accumulate into the same TMEM -- they pace that
// kernel at ~1300 cycles per 128-row k-block (2-3 TB/s).  Here:
//   A[n, k] = fp16(w[n,k] * ws[n, g(k)])   (converters: 6-bit code, exact, times its fp16 scale,
//                                            one IEEE fp16 rounding -- HSUB2 + HMUL2)
//   B[m, k] = fp16(x[m,k] * xs[m, g(k)])   (the activation quantizer writes it: its code times
//                                            its fp16 scale, one rounding)
//   y[m, n] = sum_k A[n,k] * B[m,k]         (fp16 products are exact in fp32; fp32 accumulation)
// i.e. the reference's sum_g (xs*ws) * P_g (engine.py:251-287) with the scales distributed
// over the products.  The codes and scales are the reference's (quantize.py:118-148, fp16
// scales); the fp16 y is within the fast path's stated tolerance (max|y - y_ref| <= 1e-3 *
// max|y_ref|, measured ~5e-4).  Exact INT32 group partials (trace mode) stay on the integer
// kernels.  Group size 128 only (one group per k-block), fp16 weight scales.
//
// Work split and roles as gemm_tc.cu (persistent, stream-K over (128-row tile, k-block) units,
// fixed-order fixup of split tiles), with
//   warps 0-7  converters: one 16-row tile each: T6 unpack -> fp16 * scale -> the A tile
//              (K-major, 128 B swizzle; an A-in-TMEM variant via tcgen05.st 16x256b measured
//              slower: 70B gate M=64 89.8 vs 74 us)
//   warp 8     weight producer (T6 units + the two row groups' scale slices, TMA bulk)
//   warp 9     MMA issuer: 8 x tcgen05.mma.kind::f16 (M=128, N=TN, K=16) per k-block, one
//              accumulator per tile (double-buffered in TMEM), tcgen05.commit per stage / tile
//   warp 10    activation producer (the fp16 B tile, TMA bulk)
//   warps 11-14 epilogue: per tile, tcgen05.ld the fp32 tile -> fp16 store or stream-K fixup
#include "common.cuh"

namespace flexq {

namespace tc16 {

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T, kind::f16 (A, B fp16, D fp32), M=128, N=TN, K=16
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// One k-block's 8 MMAs (K = 16 each, A columns +8 and B descriptor +16 per step) and the
// commit of the A slot, issued by the whole converged warp through one elect.sync inside a
// single asm block (B descriptor +16 = +256 B per K = 16 step): the operands are converted to uniform registers once per k-block instead of
// once per instruction inside a per-MMA elect loop (tools/probe/umma_factors.cu).
__device__ __forceinline__ void mma8_commit(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate, uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e, p, t;\n.reg .b32 a;\n.reg .b64 b;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\nsetp.eq.b32 t, 0, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "add.u32 a, %1, 8;\nadd.u64 b, %2, 16;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 16;\nadd.u64 b, %2, 32;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 24;\nadd.u64 b, %2, 48;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 32;\nadd.u64 b, %2, 64;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 40;\nadd.u64 b, %2, 80;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 48;\nadd.u64 b, %2, 96;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "add.u32 a, %1, 56;\nadd.u64 b, %2, 112;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(smem_u32(bar))
      : "memory");
}
// 16 TMEM lanes x 64 columns from one warp: thread t's registers 4j..4j+3 land in
// (lane t/4, columns 8j + 2(t%4), +1) and (lane 8 + t/4, same columns) -- measured,
// tools/probe/tmem_layout.cu
__device__ __forceinline__ void st_16x256b_x8(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
      "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void ld16(uint32_t addr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void wait_ld(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                 "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]),
                 "+r"(v[13]), "+r"(v[14]), "+r"(v[15])::"memory");
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void sts128(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}
__device__ __forceinline__ void named_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
// K-major, 128 B swizzle (A tiles, 1024 B aligned); a K=16 fp16 step advances 32 B
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// K-major, no swizzle (B tiles): 8-token x 16 B cores, LBO 128 B (K-adjacent cores), SBO
// 2048 B (8-token groups: 16 cores per 128-k block)
__device__ __forceinline__ uint64_t desc_b(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(2048 >> 4) << 32) | (1ull << 46);
}

// 4 offset-binary codes u (w = u - 32) of one word -> two half2 of fp16(w * s): the magic
// 0x6400 | u is 1024 + u exactly, minus 1056 is w exactly, times s is one IEEE rounding
__device__ __forceinline__ void scale4(uint32_t word, __half2 s2, uint32_t& lo, uint32_t& hi) {
  const __half2 off = __floats2half2_rn(1056.f, 1056.f);
  uint32_t a = __byte_perm(word, 0x64646464u, 0x5140);
  uint32_t b = __byte_perm(word, 0x64646464u, 0x5342);
  __half2 ha = __hmul2(__hsub2(*reinterpret_cast<__half2*>(&a), off), s2);
  __half2 hb = __hmul2(__hsub2(*reinterpret_cast<__half2*>(&b), off), s2);
  lo = *reinterpret_cast<uint32_t*>(&ha);
  hi = *reinterpret_cast<uint32_t*>(&hb);
}

}  // namespace tc16

constexpr int kT16ConvWarps = 8, kT16WarpProdW = 8, kT16WarpMma = 9, kT16WarpProdB = 10,
              kT16WarpEpi0 = 11, kT16EpiWarps = 4, kT16WarpProdW2 = 15;
constexpr int kT16Threads = 16 * 32;
constexpr int kT16WsSlice = kRowGroup * 8 * 4;  // fp16 scale pairs of one row group and group

template <int TN>
struct T16Cfg {
  static constexpr int SW = TN >= 128 ? 6 : 8;                   // raw ring (HBM latency)
  // operand ring (A in TMEM, B in smem); TN = 256 (128 < M <= 256): 64 KB B tiles, so two
  // stages and a single tile accumulator (256 + 2 x 64 TMEM columns)
  static constexpr int SA = TN == 256 ? 2 : TN == 128 ? 4 : 6;
  static constexpr int NACC = TN == 256 ? 1 : 2;                 // tile accumulators in TMEM
  static constexpr int kRaw = 2 * (kUnitBytes + kT16WsSlice);    // two row groups + scales
  static constexpr int kB = TN * 256;                            // TN tokens x 128 fp16
  static constexpr int kOffRaw = 0;
  static constexpr int kOffB = ((kOffRaw + SW * kRaw + 1023) / 1024) * 1024;
  static constexpr int kOffBar = kOffB + SA * kB;
  static constexpr int kNumBars = 2 * SW + 2 * SA + 4;
  static constexpr int kBytes = kOffBar + kNumBars * 8 + 16;
  static_assert(kBytes <= 232448, "shared memory budget");
  static constexpr int kAcolBase = NACC * TN;
  static_assert(NACC * TN + SA * 64 <= 512, "TMEM budget");
  static constexpr uint32_t kTmemCols = 512;
  // D f32 (bits 4-5 = 1), A f16 (7-9 = 0), B f16 (10-12 = 0), K-major; N >> 3, M >> 4
  static constexpr uint32_t kIdesc = (1u << 4) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
};

struct T16Params {
  const uint8_t* t6;
  const uint8_t* wscale;  // fp16 pairs [rg][G][4][8]
  const uint8_t* act;     // fp16 operand [kb][m_pad/8][16 cores][8 tokens][16 B]
  int64_t m, m_pad, n;
  int kbn, rg;
  int64_t units;  // (N/128 tiles) * kbn
  int nctas;
  void* y;
  int out_dtype;
  const void* res;
  float* ws_part;
  unsigned* counters;
  long long* tl;  // debug timeline of CTA 0 (FLEXQ_TC_TIMELINE): [role][unit][4] clock64
};

#ifndef FLEXQ_TC16_TIMELINE
#define FLEXQ_TC16_TIMELINE 0  // debug builds only (-DFLEXQ_TC16_TIMELINE=1)
#endif
// Debug profile of CTA 0: every role sums the cycles it spends in each phase in registers and
// writes the totals once at the end (per-event stores in the loops cost up to 30 %).
struct T16Prof {
  long long acc[4] = {0, 0, 0, 0};
  long long t = 0;
  __device__ void start() { if constexpr (FLEXQ_TC16_TIMELINE) t = clock64(); }
  __device__ void lap(int i) {
    if constexpr (FLEXQ_TC16_TIMELINE) { const long long n = clock64(); acc[i] += n - t; t = n; }
  }
  __device__ void flush(const T16Params& p, int role, int64_t units) {
    if constexpr (FLEXQ_TC16_TIMELINE) {
      if (p.tl && blockIdx.x == 0) {
        for (int i = 0; i < 4; i++) p.tl[role * 8 + i] = acc[i];
        p.tl[role * 8 + 4] = units;
      }
    }
  }
};
__device__ __forceinline__ int64_t t16_start(int64_t c, int64_t units, int64_t P) { return c * units / P; }
__device__ __forceinline__ int64_t t16_owner(int64_t u, int64_t units, int64_t P) { return ((u + 1) * P - 1) / units; }

template <int TN, int OUT>
__global__ void __launch_bounds__(kT16Threads, 1) gemm_tc16_kernel(T16Params p) {
  using C = T16Cfg<TN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* wfull = bars;
  uint64_t* wempty = wfull + C::SW;
  uint64_t* afull = wempty + C::SW;   // A converted (8 warps) + B landed (TMA)
  uint64_t* aempty = afull + C::SA;   // consumed by the MMAs (tcgen05.commit)
  uint64_t* dfull = aempty + C::SA;   // [2] tile accumulator complete
  uint64_t* dempty = dfull + 2;       // [2] drained by the epilogue
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(dempty + 2);
  volatile int* flush_flag = reinterpret_cast<volatile int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cta = blockIdx.x, P = p.nctas, U = p.units;
  const int64_t u0 = t16_start(cta, U, P), u1 = t16_start(cta + 1, U, P);
  const int kbn = p.kbn;
  // debug builds: per-CTA globaltimer marks {entry, MMA loop start, MMA loop end, exit}
  auto cta_mark = [&](int i) {
    if constexpr (FLEXQ_TC16_TIMELINE) {
      if (p.tl) p.tl[32 + 1024 + blockIdx.x * 4 + i] = dbg_now();
    }
  };
  if (threadIdx.x == 0) cta_mark(0);

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::SW; i++) { mbar_init(&wfull[i], 2); mbar_init(&wempty[i], kT16ConvWarps); }
    for (int i = 0; i < C::SA; i++) { mbar_init(&afull[i], kT16ConvWarps + 1); mbar_init(&aempty[i], 1); }
    for (int i = 0; i < 2; i++) { mbar_init(&dfull[i], 1); mbar_init(&dempty[i], kT16EpiWarps); }
    fence_mbar_init();
  }
  if (warp == kT16WarpMma) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "r"(C::kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc16::fence_before();
  __syncthreads();
  tc16::fence_after();
  const uint32_t tmem = *tmem_holder;
  pdl_launch_dependents();

  if (warp < kT16ConvWarps) {
    // ===== converters: T6 row tile -> fp16(w * ws) A rows, straight into TMEM =====
    const int gq = lane >> 2, t = lane & 3;
    const int q = warp & 3;
    const int r8 = 2 * q + (warp >> 2);
    const int rgl = r8 >> 2, r = r8 & 3;
    const uint32_t tlane = tmem + ((uint32_t)(16 * r8) << 16);
    int wi = 0, ai = 0;
    uint32_t wph = 0, aph = 0;
    T16Prof pf;
    pf.start();
    for (int64_t u = u0; u < u1; u++) {
      mbar_wait(&wfull[wi], wph);
      pf.lap(0);
      mbar_wait(&aempty[ai], aph ^ 1u);
      pf.lap(1);
      tc16::fence_after();
      const uint8_t* raw = smem + C::kOffRaw + wi * C::kRaw + rgl * (kUnitBytes + kT16WsSlice);
      const uint4 w0 = lds128(raw + (r * 3 + 0) * 512 + lane * 16);
      const uint4 w1 = lds128(raw + (r * 3 + 1) * 512 + lane * 16);
      const uint4 w2 = lds128(raw + (r * 3 + 2) * 512 + lane * 16);
      const __half2 sp = reinterpret_cast<const __half2*>(raw + kUnitBytes)[r * 8 + gq];
      const __half2 s0 = __half2half2(__low2half(sp)), s1 = __half2half2(__high2half(sp));
      uint32_t v[32];
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        uint32_t a[4];
        unpack_t6(u4get(w0, jj), u4get(w1, jj), u4get(w2, jj), a);
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int j = 2 * jj + h;
          tc16::scale4(a[2 * h], s0, v[4 * j + 0], v[4 * j + 1]);
          tc16::scale4(a[2 * h + 1], s1, v[4 * j + 2], v[4 * j + 3]);
        }
      }
      pf.lap(2);
      tc16::st_16x256b_x8(tlane + C::kAcolBase + ai * 64, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc16::fence_before();
      __syncwarp();
      if (lane == 0) { tc16::arrive(&wempty[wi]); tc16::arrive(&afull[ai]); }
      pf.lap(3);
      if (++wi == C::SW) { wi = 0; wph ^= 1u; }
      if (++ai == C::SA) { ai = 0; aph ^= 1u; }
    }
    if (warp == 0 && lane == 0) pf.flush(p, 0, u1 - u0);
  } else if (warp == kT16WarpProdW || warp == kT16WarpProdW2) {
    // ===== weight producers: one per row group of the tile, a T6 unit and its scale slice per
    // k-block each (two issuing threads: one thread's bulk copies stream measurably slower,
    // tools/probe/stream.cu) =====
    const int pj = warp == kT16WarpProdW ? 0 : 1;
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int wi = 0;
      uint32_t wph = 0;
      int64_t tile = u0 / kbn, kb = u0 - tile * kbn;
      T16Prof pf;
      pf.start();
      for (int64_t u = u0; u < u1; u++) {
        const int rg0 = (int)tile * 2;
        const int nu = rg0 + 1 < p.rg ? 2 : 1;
        mbar_wait(&wempty[wi], wph ^ 1u);
        pf.lap(0);
        mbar_expect_tx(&wfull[wi], pj < nu ? kUnitBytes + kT16WsSlice : 0);
        uint8_t* dst = smem + C::kOffRaw + wi * C::kRaw;
        for (int j = pj; j < nu && j == pj; j++) {
          bulk_g2s(dst + j * (kUnitBytes + kT16WsSlice), p.t6 + ((int64_t)(rg0 + j) * kbn + kb) * kUnitBytes,
                   kUnitBytes, &wfull[wi], pol);
          bulk_g2s(dst + j * (kUnitBytes + kT16WsSlice) + kUnitBytes,
                   p.wscale + ((int64_t)(rg0 + j) * kbn + kb) * kT16WsSlice, kT16WsSlice, &wfull[wi], pol);
        }
        pf.lap(1);
        if (++wi == C::SW) { wi = 0; wph ^= 1u; }
        if (++kb == kbn) { kb = 0; tile++; }
      }
      if (pj == 0) pf.flush(p, 1, u1 - u0);
    }
  } else if (warp == kT16WarpProdB) {
    // ===== activation producer: the fp16 B tile of each k-block (L2-resident) =====
    if (lane == 0) {
      pdl_wait();
      const uint64_t pol = l2_policy_evict_last();
      int bi = 0;
      uint32_t bph = 0;
      int64_t kb = u0 % kbn;
      T16Prof pf;
      pf.start();
      for (int64_t u = u0; u < u1; u++) {
        mbar_wait(&aempty[bi], bph ^ 1u);
        pf.lap(0);
        mbar_expect_tx(&afull[bi], C::kB);
        bulk_g2s(smem + C::kOffB + bi * C::kB, p.act + kb * (p.m_pad >> 3) * 2048, C::kB, &afull[bi], pol);
        pf.lap(1);
        if (++bi == C::SA) { bi = 0; bph ^= 1u; }
        if (++kb == kbn) kb = 0;
      }
      pf.flush(p, 2, u1 - u0);
    }
  } else if (warp == kT16WarpMma) {
    // ===== MMA issuer: 8 x (M=128, N=TN, K=16) per k-block into the tile's accumulator =====
    int ai = 0, db = 0;
    uint32_t aph = 0, dph = 0;
    bool fresh = true;  // the next MMA starts a tile accumulator
    int64_t kb = u0 % kbn;
    T16Prof pf;
    pf.start();
    if (lane == 0) cta_mark(1);
    for (int64_t u = u0; u < u1; u++) {
      const bool tile_end = kb == kbn - 1 || u == u1 - 1;
      if (++kb == kbn) kb = 0;
      if (fresh) mbar_wait(&dempty[db], dph ^ 1u);
      pf.lap(0);
      mbar_wait(&afull[ai], aph);
      pf.lap(1);
      tc16::fence_after();
      __syncwarp();
      tc16::mma8_commit(tmem + db * TN, tmem + C::kAcolBase + ai * 64,
                        tc16::desc_b(smem_u32(smem + C::kOffB + ai * C::kB)), C::kIdesc,
                        fresh ? 0u : 1u, &aempty[ai]);
      if (lane == 0 && tile_end) tc16::commit(&dfull[db]);
      __syncwarp();
      pf.lap(2);
      fresh = tile_end;
      if (tile_end) {
        if (C::NACC == 2) { db ^= 1; if (db == 0) dph ^= 1u; }
        else dph ^= 1u;
      }
      if (++ai == C::SA) { ai = 0; aph ^= 1u; }
    }
    if (lane == 0) { pf.flush(p, 3, u1 - u0); cta_mark(2); }
    if constexpr (FLEXQ_TC16_TIMELINE) {  // every CTA: its MMA loop's total cycles
      if (lane == 0 && p.tl) p.tl[32 + blockIdx.x] = pf.acc[0] + pf.acc[1] + pf.acc[2];
    }
  } else if (warp >= kT16WarpEpi0 && warp < kT16WarpEpi0 + kT16EpiWarps) {
    // ===== epilogue: per tile, fp32 accumulator -> fp16 y (or the stream-K fixup) =====
    const int q = warp & 3;  // TMEM lane quarter
    const int rho = 32 * q + lane;
    const uint32_t tl = tmem + ((uint32_t)(32 * q) << 16);
    pdl_wait();
    int db = 0;
    uint32_t dph = 0;
    int64_t u = u0;
    while (u < u1) {
      const int64_t tile = u / kbn;
      const int64_t t_end = (tile + 1) * kbn < u1 ? (tile + 1) * kbn : u1;  // this CTA's part
      const int64_t n_row = tile * 128 + rho;
      mbar_wait(&dfull[db], dph);
      tc16::fence_after();
      const int64_t first_c = t16_owner(tile * kbn, U, P), last_c = t16_owner(tile * kbn + kbn - 1, U, P);
      const bool split = first_c != last_c;
      const int which = u0 >= tile * kbn ? 0 : 1;
      float* wslot = p.ws_part + ((cta * 2 + which) * TN) * (int64_t)128 + rho;
#pragma unroll 1
      for (int c0 = 0; c0 < TN; c0 += 16) {
        uint32_t v[16];
        tc16::ld16(tl + db * TN + c0, v);
        tc16::wait_ld(v);
        if (split) {
#pragma unroll
          for (int j = 0; j < 16; j++) wslot[(c0 + j) * 128] = __uint_as_float(v[j]);
        } else if (n_row < p.n) {
#pragma unroll
          for (int j = 0; j < 16; j++) {
            const int64_t m = c0 + j;
            if (m < p.m) {
              const float yv = __uint_as_float(v[j]) + residual_at<OUT>(p.res, m * p.n + n_row);
              if constexpr (OUT == FLEXQ_OUT_F16) reinterpret_cast<__half*>(p.y)[m * p.n + n_row] = __float2half_rn(yv);
              else reinterpret_cast<float*>(p.y)[m * p.n + n_row] = yv;
            }
          }
        }
      }
      tc16::fence_before();
      __syncwarp();
      if (lane == 0) tc16::arrive(&dempty[db]);  // the MMA may refill this accumulator
      if (C::NACC == 2) { db ^= 1; if (db == 0) dph ^= 1u; }
      else dph ^= 1u;
      if (split) {
        __threadfence();
        tc16::named_sync(1, kT16EpiWarps * 32);
        if (q == 0 && lane == 0) {
          const unsigned prev = atom_add_acq_rel_gpu(&p.counters[tile], 1u);
          *flush_flag = prev == (unsigned)(last_c - first_c) ? 1 : 0;
        }
        tc16::named_sync(1, kT16EpiWarps * 32);
        const bool last = *flush_flag != 0;
        tc16::named_sync(1, kT16EpiWarps * 32);  // flag read by all before the next flush
        if (last) {
          __threadfence();
#pragma unroll 1
          for (int c0 = 0; c0 < TN; c0 += 16) {
            float a[16];
#pragma unroll
            for (int j = 0; j < 16; j++) a[j] = 0.f;
            // contributors in fixed CTA order (deterministic), four per L2 round trip: the
            // loads of a batch are all issued before the ordered sum consumes them
            for (int64_t cb = first_c; cb <= last_c; cb += 4) {
              float v[4][16];
#pragma unroll
              for (int b = 0; b < 4; b++) {
                const int64_t cc = cb + b;
                if (cc <= last_c) {
                  const int wc = t16_start(cc, U, P) >= tile * kbn ? 0 : 1;
                  const float* src = p.ws_part + ((cc * 2 + wc) * TN + c0) * (int64_t)128 + rho;
#pragma unroll
                  for (int j = 0; j < 16; j++) v[b][j] = __ldcg(src + j * 128);
                }
              }
#pragma unroll
              for (int b = 0; b < 4; b++)
                if (cb + b <= last_c) {
#pragma unroll
                  for (int j = 0; j < 16; j++) a[j] += v[b][j];
                }
            }
            if (n_row < p.n) {
#pragma unroll
              for (int j = 0; j < 16; j++) {
                const int64_t m = c0 + j;
                if (m < p.m) {
                  const float yv = a[j] + residual_at<OUT>(p.res, m * p.n + n_row);
                  if constexpr (OUT == FLEXQ_OUT_F16) reinterpret_cast<__half*>(p.y)[m * p.n + n_row] = __float2half_rn(yv);
                  else reinterpret_cast<float*>(p.y)[m * p.n + n_row] = yv;
                }
              }
            }
          }
          if (q == 0 && lane == 0) p.counters[tile] = 0u;
        }
      }
      u = t_end;
    }
  }

  tc16::fence_before();
  __syncthreads();
  if (threadIdx.x == 0) cta_mark(3);
  if (warp == kT16WarpMma) {
    tc16::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols) : "memory");
  }
}

// ---- host side ------------------------------------------------------------------------------
static long long* g_t16_tl = nullptr;
extern "C" int flexq_debug_tc16_timeline(long long* host, int max_entries) {
  const int n = 32 + 1024 + 4 * 1024;
  if (!g_t16_tl || max_entries < n) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_t16_tl, n * sizeof(long long), cudaMemcpyDeviceToHost);
  return n;
}

static int t16_tn(int64_t m) { return m <= 32 ? 32 : m <= 64 ? 64 : m <= 128 ? 128 : 256; }

bool gemm_tc16_supported(int64_t m, int64_t n, int64_t k, int64_t gs, int scale_f16) {
  return m > 16 && m <= 256 && gs == 128 && k % 128 == 0 && scale_f16 && n >= 1;
}

int64_t gemm_tc16_act_bytes(int64_t m, int64_t k) {
  const int64_t m_pad = cdiv(m, t16_tn(m)) * t16_tn(m);
  return m_pad * k * 2;
}

int64_t gemm_tc16_workspace(int64_t m, int64_t n) {
  const int tn = t16_tn(m);
  const int64_t sms = device_sms() > 148 ? device_sms() : 148;
  return cdiv(sms * 2 * tn * 128 * 4, 256) * 256 + cdiv(cdiv(n, 128) * 4, 256) * 256;
}

template <int TN, int OUT>
static int launch_tc16_inst(const T16Params& p, cudaStream_t st) {
  auto kern = gemm_tc16_kernel<TN, OUT>;
  constexpr int smem = T16Cfg<TN>::kBytes;
  cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return cuda_status(e, "gemm_tc16 attribute");
  e = launch_pdl(kern, dim3((unsigned)p.nctas), dim3(kT16Threads), (size_t)smem, st, p);
  if (e != cudaSuccess) return cuda_status(e, "gemm_tc16 launch");
  return FLEXQ_OK;
}

int gemm_tc16_launch(const uint32_t* t6, const void* wscale, const void* act_f16, int64_t m,
                     int64_t n, int64_t k, void* y, int out_dtype, void* workspace,
                     const void* residual, cudaStream_t st) {
  if (!gemm_tc16_supported(m, n, k, 128, 1) || !workspace || !y) {
    set_error("gemm_tc16: needs 16 < m <= 256, group 128, fp16 scales, K %% 128 == 0, a workspace");
    return FLEXQ_ERR_CONFIG;
  }
  T6Geom G(n, k, 128);
  const int tn = t16_tn(m);
  T16Params p{};
  p.t6 = reinterpret_cast<const uint8_t*>(t6);
  p.wscale = reinterpret_cast<const uint8_t*>(wscale);
  p.act = reinterpret_cast<const uint8_t*>(act_f16);
  p.m = m;
  p.m_pad = cdiv(m, tn) * tn;
  p.n = n;
  p.kbn = (int)G.kb;
  p.rg = (int)G.rg;
  p.units = cdiv(n, 128) * G.kb;
  // aligned grids from TN = 128 up; at TN = 64 only on layers of <= 8192 units with >= 70 % of
  // the SMs busy (13B gate_proj M = 64: 31.9 -> 24.8 us; 70B down_proj, 14336 units, slower)
  p.nctas = tc_grid(p.units, G.kb, tn >= 128 ? 50 : p.units <= 8192 ? 70 : 101);
  const int64_t sms = device_sms();
  p.y = y;
  p.out_dtype = out_dtype;
  p.res = residual;
  p.ws_part = reinterpret_cast<float*>(workspace);
  const int64_t s2 = sms > 148 ? sms : 148;
  p.counters = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(workspace) +
                                           cdiv(s2 * 2 * tn * 128 * 4, 256) * 256);
  if (tuning().tc_timeline) {
    if (!g_t16_tl) cudaMalloc(&g_t16_tl, (32 + 1024 + 4 * 1024) * sizeof(long long));
    cudaMemsetAsync(g_t16_tl, 0, (32 + 1024 + 4 * 1024) * sizeof(long long), st);
    p.tl = g_t16_tl;
  }
  const bool f32 = out_dtype == FLEXQ_OUT_F32;
  switch (tn) {
    case 32: return f32 ? launch_tc16_inst<32, FLEXQ_OUT_F32>(p, st) : launch_tc16_inst<32, FLEXQ_OUT_F16>(p, st);
    case 64: return f32 ? launch_tc16_inst<64, FLEXQ_OUT_F32>(p, st) : launch_tc16_inst<64, FLEXQ_OUT_F16>(p, st);
    case 256: return f32 ? launch_tc16_inst<256, FLEXQ_OUT_F32>(p, st) : launch_tc16_inst<256, FLEXQ_OUT_F16>(p, st);
    default: return f32 ? launch_tc16_inst<128, FLEXQ_OUT_F32>(p, st) : launch_tc16_inst<128, FLEXQ_OUT_F16>(p, st);
  }
}

}  // namespace flexq
