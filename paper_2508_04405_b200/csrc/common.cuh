// Shared definitions for the sm_100a W6Ax kernels.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/flexq.h"

namespace flexq {

// ---- error plumbing (host) ---------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
#define FLEXQ_LAUNCH_CHECK(where)                               \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::flexq::cuda_status(_e, where); \
  } while (0)

// ---- runtime (host): environment knobs, per-device caches ----------------------
// Every FLEXQ_* environment knob is read ONCE, at the library's first use (tuning()); the
// values are reported by flexq_tuning() so a benchmark line can record them.  The product
// path never reads the environment per launch.  The knobs are debug / A-B switches only;
// unset, the automatic routes documented in DESIGN.md sec. 4 apply.
struct Tuning {
  bool trace = false;          // FLEXQ_TRACE: kernel event trace (tools/step_trace.py)
  bool disable_tc = false;     // FLEXQ_DISABLE_TC=1: M > 16 on the mma.sync kernel
  bool gemv_wide = false;      // FLEXQ_GEMV_WIDE: one 12-warp GEMV CTA per SM
  bool gemv_rev = false;       // FLEXQ_GEMV_REV: reversed unit-range assignment
  bool gemv_timeline = false;  // FLEXQ_GEMV_TIMELINE: per-warp GEMV timeline
  bool tc_timeline = false;    // FLEXQ_TC_TIMELINE: tcgen05 CTA-0 timeline
  bool q_early = false;        // FLEXQ_Q_EARLY: quantizer triggers dependents before waiting
  bool disable_tc16 = false;   // FLEXQ_DISABLE_TC16=1: batched forwards on the INT8 tcgen05 kernel
  int stream_max_m = 32;       // FLEXQ_STREAM_MAX_M: largest M on the streaming GEMV
  int stream_stages = -1;      // FLEXQ_STREAM_STAGES: 2/3/4 forced ring depth (-1: by size)
  int min_units = 4;           // FLEXQ_MIN_UNITS: units per warp with 4-stage rings
  int tc_min_units = 1;        // FLEXQ_TC_MIN_UNITS: fewest stream-K units per tcgen05 CTA
  bool tc_align = true;        // FLEXQ_TC_ALIGN=0: plain stream-K grids (A/B)
};
// CTAs of a persistent stream-K tcgen05 launch over `units` = tiles x kbn work items: one per
// SM, or -- when that keeps at least min_pct % of the SMs busy -- the count that gives every
// CTA a whole divisor of a tile's k-blocks (ranges aligned to tile fractions)
int tc_grid(int64_t units, int64_t kbn, int min_pct);
const Tuning& tuning();
int device_sms();  // SM count of the current device (cached per device)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, bytes)
cudaError_t ensure_smem(const void* kern, int bytes);

// ---- geometry ------------------------------------------------------------------
constexpr int kChunkK = 128;   // packing.py:27 MMA_K, one FLXQ-P k-chunk
constexpr int kKStep = 32;     // mma.m16n8k32 contraction per instruction
constexpr int kStepsPerBlock = 4;  // one T6 k-block = 4 k-steps = 128 k-slots
constexpr int kRowTile = 16;   // mma M (weight rows per A fragment)
constexpr int kTokTile = 8;    // mma N (tokens per B fragment)
constexpr int kRowGroup = 4;   // row tiles per T6 unit (64 weight rows share one B fragment)
constexpr int kUnitBytes = kRowGroup * 3 * 512;  // T6 bytes per (row group, k-block) unit
// act_corr holds kCorrBias + 32 * sum(codes) per (group, token): the fp32 bit pattern of
// 12582912 + corr, which the tcgen05 epilogue subtracts from its seeded accumulator
// directly (gemm_tc.cu); the integer kernels remove the bias.
constexpr int32_t kCorrBias = 0x4B400000;

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Group-padded K geometry of the T6 layouts: every scale group occupies
// spg = ceil(group_size/32) k-steps, so a k-step never straddles two groups.
struct T6Geom {
  int64_t n, k, gs;
  int64_t ng;   // scale groups  ceil(k / gs)
  int64_t spg;  // k-steps per group
  int64_t ks;   // total k-steps = ng * spg
  int64_t kb;   // k-blocks = ceil(ks / 4)
  int64_t rg;   // row groups = ceil(n / 64)
  int64_t rt;   // row tiles = 4 * rg (rows padded to 64)
  __host__ __device__ T6Geom() : n(0), k(0), gs(1), ng(0), spg(1), ks(0), kb(0), rg(0), rt(0) {}
  __host__ __device__ T6Geom(int64_t n_, int64_t k_, int64_t gs_) : n(n_), k(k_), gs(gs_) {
    ng = cdiv(k, gs);
    spg = cdiv(gs < k ? gs : k, kKStep);  // a group holds at most min(gs, k) elements
    ks = ng * spg;
    kb = cdiv(ks, kStepsPerBlock);
    rg = cdiv(n, kRowTile * kRowGroup);
    rt = rg * kRowGroup;
  }
  // uint4 index of T6 vector v (0: L0, 1: L1, 2: H) of `lane` for (row tile, k-block):
  // layout [rg][kb][r][v][lane] x 16 B, i.e. unit u = rg*kb_total + kb is 6 KB contiguous
  __host__ __device__ int64_t vec_index(int64_t rtile, int64_t kblk, int v, int lane) const {
    const int64_t g = rtile / kRowGroup, r = rtile - g * kRowGroup;
    return (((g * kb + kblk) * kRowGroup + r) * 3 + v) * 32 + lane;
  }
  // half2/float2 index of the weight-scale pair {row 16rt+gq, row 16rt+gq+8} of group `grp`:
  // layout [rg][G][r][8] pairs (128 B of fp16 per (row group, group))
  __host__ __device__ int64_t scale_index(int64_t rtile, int64_t grp, int gq) const {
    const int64_t g = rtile / kRowGroup, r = rtile - g * kRowGroup;
    return ((g * ng + grp) * kRowGroup + r) * 8 + gq;
  }
  // u32 word index inside the activation fragment array [mt][kb][c][lane][4 words]:
  // chunk c = jj/2, word w = (jj%2)*2 + half  (half 0 = b0, 1 = b1 of k-step jj)
  __host__ __device__ static int64_t act_word(int64_t kb_total, int64_t mt, int64_t kblk, int jj,
                                             int half, int lane) {
    return ((mt * kb_total + kblk) * 2 + (jj >> 1)) * 128 + lane * 4 + (jj & 1) * 2 + half;
  }
  // padded slot of logical column kk
  __host__ __device__ int64_t slot(int64_t kk) const {
    int64_t g = kk / gs, j = kk - g * gs;
    return g * spg * kKStep + j;
  }
};

// ---- programmatic dependent launch (PDL) -------------------------------------------------
// Kernels launched with launch_pdl may start while the previous kernel on the stream is
// still running; pdl_wait() blocks until that grid has completed and its writes are
// visible (a no-op when there is no programmatic predecessor).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

// ---- debug event trace (FLEXQ_TRACE=1; tools/step_trace.py) -------------------------------
// Kernels append {tag = launch << 8 | kind, t_start, t_mid, t_end} globaltimer records so a
// multi-kernel step can be laid out on one time axis.  Off (nullptr) unless the env var is
// set; never used on a production path.
constexpr unsigned long long kDbgCap = 1 << 16;
long long* dbg_trace_buf();  // host: device buffer, or nullptr when tracing is off
long long dbg_next_launch();  // host: launch sequence number
__device__ __forceinline__ long long dbg_now() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void dbg_record(long long* buf, long long tag, long long a, long long b,
                                           long long c) {
  const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(buf), 1ull);
  if (i < kDbgCap) {
    long long* r = buf + 4 + 4 * i;
    r[0] = tag; r[1] = a; r[2] = b; r[3] = c;
  }
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- async-copy / mbarrier primitives (sm_90+ PTX, used by the TMA-fed kernels) ----------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)  // (a suspend-time hint measured +40 cycles per completed wait, tools/probe/mbar_lat.cu)
      : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// packed fp32x2 math (FADD2 / FMUL2 / FFMA2 on sm_100)
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\n"
      "sub.rn.f32x2 rd, ra, rb;\nmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\n"
      "mul.rn.f32x2 rd, ra, rb;\nmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2,%3};\nmov.b64 rb, {%4,%5};\n"
      "mov.b64 rc, {%6,%7};\nfma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
// ---- T6 unpack + IMMA -------------------------------------------------------------------
// A registers of one m16n8k32 from the three T6 words of a k-step.
// Offset-binary u = w + 32 in [1, 63] (6 bits).  Byte b of word v holds u(a_v, b) in
// bits 0-5 and, in bits 6-7, two of the six bits of u(a_3, b): bits 0-1 in W0, 2-3 in
// W1, 4-5 in W2.  a0..a2 are one AND each; a3 is reassembled with 3 shifts + 3 LOP3.
__device__ __forceinline__ void unpack_t6(uint32_t W0, uint32_t W1, uint32_t W2, uint32_t a[4]) {
  a[0] = W0 & 0x3F3F3F3Fu;
  a[1] = W1 & 0x3F3F3F3Fu;
  a[2] = W2 & 0x3F3F3F3Fu;
  const uint32_t lo = ((W0 >> 6) & 0x03030303u) | ((W1 >> 4) & 0x0C0C0C0Cu);
  a[3] = lo | ((W2 >> 2) & 0x30303030u);
}

__device__ __forceinline__ void mma_u8s8(int c[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// same with a zero accumulator input (first k-step of a group)
__device__ __forceinline__ void mma_u8s8_zc(int c[4], const uint32_t a[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0));
}

// split-K handshake: release this thread's prior writes / acquire the others'
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// optional fused residual of the output store: y[i] = acc + res[i] (res may alias y)
template <int OUT>
__device__ __forceinline__ float residual_at(const void* res, int64_t i) {
  if (!res) return 0.f;
  if constexpr (OUT == FLEXQ_OUT_F16) return __half2float(reinterpret_cast<const __half*>(res)[i]);
  else return reinterpret_cast<const float*>(res)[i];
}

__device__ __forceinline__ uint32_t u4get(const uint4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

}  // namespace flexq
