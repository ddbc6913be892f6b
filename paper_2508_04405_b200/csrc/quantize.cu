// Symmetric per-(row, group) quantizer -- the online activation quantizer of
// the hot path and the offline weight quantizer.
//
// Follows quantize.py:118-148 exactly: scale = max|x| / qmax in float64
// (1.0 for an all-zero group, quantize.py:99-110), optionally rounded to fp16
// straight from float64 (quantize.py:143-144), code = clamp(sign(v) *
// floor(|v| + 0.5), +-qmax) with v = x / scale in float64 (quantize.py:29-31,
// 147).  Every step is one correctly-rounded IEEE float64 operation, so the
// codes and scales are bit-identical with numpy for every input dtype.
//
// One warp owns one (row, group) for groups up to kWarpGroupMax elements; a
// whole CTA owns it for larger groups (per-token mode, group_size >= K).
// Besides row-major codes / float64 scales (the QuantTensor of the drop-in
// API) it can emit, fused, the i8-path activation operand: codes scattered
// into the T6 B-fragment layout, fp32 scales and the offset-binary correction
// 32 * sum(codes) per (group, token).
#include <cuda_bf16.h>

#include "common.cuh"
#include "quant_math.cuh"

namespace flexq {

template <int DT>
__device__ __forceinline__ double load_as_f64(const void* base, int64_t i) {
  if constexpr (DT == FLEXQ_DT_F16) {
    return (double)__half2float(reinterpret_cast<const __half*>(base)[i]);
  } else if constexpr (DT == FLEXQ_DT_BF16) {
    return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  } else if constexpr (DT == FLEXQ_DT_F32) {
    return (double)reinterpret_cast<const float*>(base)[i];
  } else {
    return reinterpret_cast<const double*>(base)[i];
  }
}

struct QuantArgs {
  const void* x;
  int64_t rows, cols, gs, ng;
  int bits;
  int fp16_scales;
  int8_t* codes;
  double* scales;
  uint8_t* act_frag;
  float* act_scale;
  int32_t* act_corr;
  int64_t m_pad;
  uint32_t* flag;
  // T6 geometry of the activation fragment layout
  int64_t spg, kb;
  long long* dbg = nullptr;  // FLEXQ_TRACE event buffer (debug)
  long long dbg_tag = 0;
  int early = 0;  // experiment (FLEXQ_Q_EARLY): trigger dependents before waiting
  // optional fp16 operand of the kind::f16 batched kernel (gemm_tc16.cu): fp16(code * scale)
  // at [k-block][m_pad/8][16 cores][8 tokens][16 B], position p = 16(2t+h) + 4jj + b of slot
  // 32jj + 16h + 4t + b (the same permutation as act_frag); group 128 fast path only
  __half* act_f16 = nullptr;
};

// Byte of (token m, logical column c) in the activation operand:
// [k-block][m_pad/8 token octets][8 k-cores][8 tokens][16 B] -- the K-major, no-swizzle
// canonical UMMA layout.  Inside a k-block, padded slot s = 32*jj + 16*h + 4*t + b (k-step jj)
// lives in k-core 2t+h at byte 4*jj+b, so lane (gq, t) of an mma.m16n8k32 finds its b0 / b1
// registers of all four k-steps in the 16 B rows of k-cores 2t / 2t+1, and a tcgen05.mma of
// K=32 over k-cores {2j, 2j+1} contracts the same slots as the converted weight tile.
__device__ __forceinline__ int64_t frag_byte(const QuantArgs& A, int64_t m, int64_t c) {
  const int64_t g = c / A.gs, j = c - g * A.gs;
  const int64_t kp = g * A.spg * kKStep + j;
  const int64_t ks = kp >> 5, within = kp & 31;
  const int64_t kb = ks >> 2, jj = ks & 3;
  const int64_t h = within >> 4, t = (within & 15) >> 2, byte = within & 3;
  return ((kb * (A.m_pad >> 3) + (m >> 3)) * 8 + 2 * t + h) * 128 + (m & 7) * 16 + jj * 4 + byte;
}

__device__ __forceinline__ void emit(const QuantArgs& A, int64_t r, int64_t c, int code) {
  if (A.codes) A.codes[r * A.cols + c] = (int8_t)code;
  if (A.act_frag) A.act_frag[frag_byte(A, r, c)] = (uint8_t)(int8_t)code;
}

// ---- warp per (row, group) ---------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(256) quantize_warp_kernel(QuantArgs A) {
  pdl_wait();               // x may be the previous kernel's output
  pdl_launch_dependents();  // let the GEMM launch and start streaming its weights
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= A.rows * A.ng) return;
  const int64_t r = item / A.ng, g = item - r * A.ng;
  const int64_t lo = g * A.gs, hi = min(lo + A.gs, A.cols);
  const int64_t base = r * A.cols;
  constexpr int kReg = 8;  // groups up to 256 stay in registers (single pass over x)
  double vals[kReg];
  double peak = 0.0;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < kReg; i++) {
    const int64_t c = lo + lane + 32 * i;
    vals[i] = c < hi ? load_as_f64<DT>(A.x, base + c) : 0.0;
    finite &= isfinite(vals[i]);
    peak = fmax(peak, fabs(vals[i]));
  }
  for (int64_t c = lo + lane + 32 * kReg; c < hi; c += 32) {  // larger groups: stream the rest
    double v = load_as_f64<DT>(A.x, base + c);
    finite &= isfinite(v);
    peak = fmax(peak, fabs(v));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  if (!__all_sync(0xffffffffu, finite)) {
    if (lane == 0) atomicOr(A.flag, FLEXQ_FLAG_NONFINITE);
    peak = 0.0;  // keep going deterministically; the wrapper raises
  }
  const double s = group_scale(peak, A.bits, A.fp16_scales, lane == 0 ? A.flag : nullptr);
  int csum = 0;
#pragma unroll
  for (int i = 0; i < kReg; i++) {
    const int64_t c = lo + lane + 32 * i;
    if (c < hi) {
      const int code = isfinite(vals[i]) ? quant_one(vals[i], s, A.bits) : 0;
      csum += code;
      emit(A, r, c, code);
    }
  }
  for (int64_t c = lo + lane + 32 * kReg; c < hi; c += 32) {
    double v = load_as_f64<DT>(A.x, base + c);
    int code = isfinite(v) ? quant_one(v, s, A.bits) : 0;
    csum += code;
    emit(A, r, c, code);
  }
  if (lane == 0 && A.scales) A.scales[r * A.ng + g] = s;
  if (A.act_scale || A.act_corr) {
#pragma unroll
    for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if (lane == 0) {
      if (A.act_scale) A.act_scale[g * A.m_pad + r] = (float)s;
      if (A.act_corr) A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * csum;
    }
  }
}

// ---- CTA per (row, group): large groups (per-token / per-channel mode) -------
template <int DT>
__global__ void __launch_bounds__(1024) quantize_cta_kernel(QuantArgs A) {
  pdl_wait();
  pdl_launch_dependents();
  __shared__ double red_d[32];
  __shared__ int red_i[32];
  __shared__ int red_f[32];
  const int64_t r = blockIdx.x / A.ng, g = blockIdx.x - r * A.ng;
  const int64_t lo = g * A.gs, hi = min(lo + A.gs, A.cols);
  const int64_t base = r * A.cols;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double peak = 0.0;
  int finite = 1;
  for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    double v = load_as_f64<DT>(A.x, base + c);
    finite &= isfinite(v) ? 1 : 0;
    peak = fmax(peak, fabs(v));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  finite = __all_sync(0xffffffffu, finite);
  if (lane == 0) { red_d[warp] = peak; red_f[warp] = finite; }
  __syncthreads();
  if (warp == 0) {
    peak = lane < nw ? red_d[lane] : 0.0;
    finite = lane < nw ? red_f[lane] : 1;
#pragma unroll
    for (int o = 16; o; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    finite = __all_sync(0xffffffffu, finite);
    if (lane == 0) {
      if (!finite) { atomicOr(A.flag, FLEXQ_FLAG_NONFINITE); peak = 0.0; }
      red_d[0] = group_scale(peak, A.bits, A.fp16_scales, A.flag);
    }
  }
  __syncthreads();
  const double s = red_d[0];
  int csum = 0;
  for (int64_t c = lo + threadIdx.x; c < hi; c += blockDim.x) {
    double v = load_as_f64<DT>(A.x, base + c);
    int code = isfinite(v) ? quant_one(v, s, A.bits) : 0;
    csum += code;
    emit(A, r, c, code);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  __syncthreads();
  if (lane == 0) red_i[warp] = csum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < nw; w++) tot += red_i[w];
    if (A.scales) A.scales[r * A.ng + g] = s;
    if (A.act_scale) A.act_scale[g * A.m_pad + r] = (float)s;
    if (A.act_corr) A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * tot;
  }
}

// ---- already-quantized codes -> T6 activation operand (warp per (row, group)) -----
// Used when the caller holds a QuantTensor (int_matmul_reference semantics,
// engine.py:337-365) instead of float activations.
__global__ void __launch_bounds__(256) codes_to_frag_kernel(QuantArgs A,
                                                            const int8_t* __restrict__ codes,
                                                            const double* __restrict__ scales) {
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (item >= A.rows * A.ng) return;
  const int64_t r = item / A.ng, g = item - r * A.ng;
  const int64_t lo = g * A.gs, hi = min(lo + A.gs, A.cols);
  int csum = 0;
  for (int64_t c = lo + lane; c < hi; c += 32) {
    const int code = codes[r * A.cols + c];
    csum += code;
    A.act_frag[frag_byte(A, r, c)] = (uint8_t)(int8_t)code;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  if (lane == 0) {
    A.act_scale[g * A.m_pad + r] = (float)scales[r * A.ng + g];
    A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * csum;
  }
}

int codes_to_frag_launch(const int8_t* codes, const double* scales, int64_t m, int64_t m_pad,
                         int64_t k, int64_t gs, uint32_t* act_frag, float* act_scale,
                         int32_t* act_corr, cudaStream_t st) {
  if (m < 1 || k < 1 || gs < 1 || m_pad < m || m_pad % kTokTile) {
    set_error("pack_act_t6: bad geometry m=%lld m_pad=%lld k=%lld group=%lld", (long long)m,
              (long long)m_pad, (long long)k, (long long)gs);
    return FLEXQ_ERR_SHAPE;
  }
  T6Geom geo(m_pad, k, gs);
  QuantArgs A{nullptr, m, k, gs, geo.ng, 8, 0, nullptr, nullptr,
              reinterpret_cast<uint8_t*>(act_frag), act_scale, act_corr, m_pad, nullptr,
              geo.spg, geo.kb};
  codes_to_frag_kernel<<<(unsigned)cdiv(m * geo.ng, 8), 256, 0, st>>>(A, codes, scales);
  FLEXQ_LAUNCH_CHECK("pack_act_t6");
  return FLEXQ_OK;
}

// ---- sum(popcount(a & b)) over a byte span (bmma_chunk, engine.py:89-95) ----------
__global__ void popcount_and_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                    int64_t nbytes, unsigned long long* out) {
  unsigned long long tot = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbytes;
       i += (int64_t)gridDim.x * blockDim.x)
    tot += __popc((unsigned)(a[i] & b[i]));
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(out, tot);
}

int popcount_and_launch(const uint8_t* a, const uint8_t* b, int64_t nbytes, int64_t* out,
                        cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return cuda_status(e, "popcount_and");
  if (nbytes > 0) {
    const int64_t blocks = cdiv(nbytes, 256) < 1024 ? cdiv(nbytes, 256) : 1024;
    popcount_and_kernel<<<(unsigned)blocks, 256, 0, st>>>(
        a, b, nbytes, reinterpret_cast<unsigned long long*>(out));
    FLEXQ_LAUNCH_CHECK("popcount_and");
  }
  return FLEXQ_OK;
}

// ---- fast path: fp16 input, group = 128 = one k-block, K % 128 == 0 -----------------
// One warp per (row, group); lane L owns the 4 consecutive columns 4L..4L+3, i.e. 4
// consecutive bytes of the activation operand (k-step L/8, k-core 2(L%4) + (L/4)%2), so
// every lane issues one 8 B load and one 4 B store and no address needs a 64-bit division.
// Same float64 arithmetic as quantize_warp_kernel (code_of: quant_math.cuh): bit-identical
// codes / scales.

__global__ void __launch_bounds__(256) quantize_g128_kernel(QuantArgs A) {
  const long long dt0 = A.dbg ? dbg_now() : 0;
  if (A.early) pdl_launch_dependents();
  pdl_wait();
  if (!A.early) pdl_launch_dependents();
  const long long dt1 = A.dbg ? dbg_now() : 0;
  const int lane = threadIdx.x & 31;
  const int64_t ng = A.ng, items = A.rows * ng;
  // grid-stride over (row, group) items, two per pass with both loads issued first: the
  // grid is capped at one CTA per SM so that the quantizer's CTAs never take the register
  // room a persistent GEMM CTA launched behind it (PDL) needs on an SM
  auto quantize_item = [&](int64_t r, int64_t g, uint2 raw) {
    const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
    const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
    const float f[4] = {f01.x, f01.y, f23.x, f23.y};
    bool finite = true;
    float peak = 0.f;  // max of fp16 magnitudes: exact in fp32
#pragma unroll
    for (int i = 0; i < 4; i++) {
      finite &= isfinite(f[i]);
      peak = fmaxf(peak, fabsf(f[i]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (!__all_sync(0xffffffffu, finite)) {
      if (lane == 0) atomicOr(A.flag, FLEXQ_FLAG_NONFINITE);
      peak = 0.f;
    }
    int c[4];
    double sc;
    float sc32 = 0.f;
    bool h = false;
    if (A.fp16_scales) {
      // fp16 scales (the production path): scale and codes in fp32, bit-identical to the
      // float64 steps (group_scale_h, quant_one_h; exhaustive check tools/check_f32_quant.c)
      sc32 = group_scale_h(peak, A.bits, lane == 0 ? A.flag : nullptr);
      sc = (double)sc32;
      h = sc32 > 0.f;
    } else {
      sc = group_scale((double)peak, A.bits, A.fp16_scales, lane == 0 ? A.flag : nullptr);
    }
    if (h) {
      const float lim = (float)((1 << (A.bits - 1)) - 1);
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const float q = __fdiv_rn(f[i], sc32);
        const float a = fminf(roundf(fabsf(q)), lim);
        const int ci = q < 0.f ? -(int)a : (int)a;
        c[i] = isfinite(f[i]) ? ci : 0;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; i++) c[i] = code_of((double)f[i], sc, A.bits);
    }
    const uint32_t word = (uint32_t)(c[0] & 0xff) | ((uint32_t)(c[1] & 0xff) << 8) |
                          ((uint32_t)(c[2] & 0xff) << 16) | ((uint32_t)(c[3] & 0xff) << 24);
    if (A.codes) *reinterpret_cast<uint32_t*>(A.codes + r * A.cols + g * 128 + lane * 4) = word;
    if (A.act_frag)
      *reinterpret_cast<uint32_t*>(A.act_frag + operand_word_offset(g, r, A.m_pad, lane)) = word;
    if (A.act_f16) {  // fp16(code * scale): the product is exact (fp32 for an fp16 scale), one rounding
      __half hv[4];
#pragma unroll
      for (int i = 0; i < 4; i++)
        hv[i] = h ? __float2half_rn((float)c[i] * sc32) : __double2half((double)c[i] * sc);
      // columns 4L .. 4L+3 of the group: core L / 2 (8 k each), bytes 8 (L % 2) ..
      uint8_t* dst = reinterpret_cast<uint8_t*>(A.act_f16) +
                     ((g * (A.m_pad >> 3) + (r >> 3)) * 16 + (lane >> 1)) * 128 + (r & 7) * 16 + 8 * (lane & 1);
      *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(hv);
    }
    if (A.act_corr) {
      int csum = c[0] + c[1] + c[2] + c[3];
#pragma unroll
      for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
      if (lane == 0) A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * csum;
    }
    if (lane == 0) {
      if (A.scales) A.scales[r * ng + g] = sc;
      if (A.act_scale) A.act_scale[g * A.m_pad + r] = (float)sc;
      if (A.dbg) dbg_record(A.dbg, A.dbg_tag, dt0, dt1, dbg_now());
    }
  };
  auto load = [&](int64_t r, int64_t g) {
    return *reinterpret_cast<const uint2*>(reinterpret_cast<const __half*>(A.x) + r * A.cols +
                                           g * 128 + lane * 4);
  };
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t a = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); a < items; a += 2 * stride) {
    const int64_t b = a + stride;
    const int64_t ra = a / ng, ga = a - ra * ng;
    const uint2 xa = load(ra, ga);
    const bool hb = b < items;
    const int64_t rb = hb ? b / ng : 0, gb = b - rb * ng;
    const uint2 xb = hb ? load(rb, gb) : make_uint2(0u, 0u);
    quantize_item(ra, ga, xa);
    if (hb) quantize_item(rb, gb, xb);
  }
}

constexpr int64_t kWarpGroupMax = 1024;

template <int DT>
static void launch_quantize(const QuantArgs& A, cudaStream_t st) {
  const int64_t items = A.rows * A.ng;
  if (DT == FLEXQ_DT_F16 && A.gs == 128 && A.cols % 128 == 0 &&
      reinterpret_cast<uintptr_t>(A.x) % 8 == 0) {
    const int sms = device_sms();
    // decode batches feed the persistent GEMV (3 CTAs per SM, registers nearly full): at most
    // one quantizer CTA per SM.  Larger batches keep one warp per item (one wave).
    // Larger batches: one wave of 8 CTAs per SM, every warp grid-striding over its items with
    // two loads in flight (one warp per item took 6+ waves: 70B down_proj M = 256, 57344 items)
    const int64_t ctas = (A.rows <= 16 && cdiv(items, 8) > sms) ? sms
                         : cdiv(items, 8) > 8 * (int64_t)sms ? 8 * (int64_t)sms : cdiv(items, 8);
    launch_pdl(quantize_g128_kernel, dim3((unsigned)ctas), dim3(256), 0, st, A);
    return;
  }
  if (A.gs <= kWarpGroupMax || A.cols <= kWarpGroupMax) {
    const int warps = 8;
    launch_pdl(quantize_warp_kernel<DT>, dim3((unsigned)cdiv(items, warps)), dim3(warps * 32), 0,
               st, A);
  } else {
    launch_pdl(quantize_cta_kernel<DT>, dim3((unsigned)items), dim3(1024), 0, st, A);
  }
}

// fp16 input, group 128, K % 128 == 0: codes -> the fp16 operand of gemm_tc16 only
int quantize_f16op_launch(const void* x, int64_t rows, int64_t cols, int bits, __half* act_f16,
                          int64_t m_pad, uint32_t* flag, cudaStream_t st) {
  if (rows < 1 || cols % 128 || bits < 2 || bits > 8 || !flag || !act_f16 || m_pad < rows ||
      m_pad % kTokTile || reinterpret_cast<uintptr_t>(x) % 8) {
    set_error("quantize_f16op: bad arguments (rows=%lld cols=%lld bits=%d)", (long long)rows,
              (long long)cols, bits);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  T6Geom geo(m_pad, cols, 128);
  QuantArgs A{x, rows, cols, 128, geo.ng, bits, 1, nullptr, nullptr, nullptr, nullptr, nullptr,
              m_pad, flag, geo.spg, geo.kb};
  A.act_f16 = act_f16;
  A.early = tuning().q_early ? 1 : 0;
  launch_quantize<FLEXQ_DT_F16>(A, st);
  FLEXQ_LAUNCH_CHECK("quantize_f16op");
  return FLEXQ_OK;
}

int quantize_launch(const void* x, int dtype, int64_t rows, int64_t cols, int bits, int64_t gs,
                    int fp16_scales, int8_t* codes, double* scales, uint32_t* act_frag,
                    float* act_scale, int32_t* act_corr, int64_t m_pad, uint32_t* flag,
                    cudaStream_t st) {
  if (rows < 1 || cols < 1) {
    set_error("quantize: expected a non-empty 2-D tensor, got (%lld, %lld)", (long long)rows,
              (long long)cols);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (bits < 2 || bits > 8) {
    set_error("bits must be in 2..8, got %d", bits);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (gs < 1) {
    set_error("group_size must be >= 1, got %lld", (long long)gs);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (!flag) {
    set_error("quantize: flag pointer is required");
    return FLEXQ_ERR_INVALID_INPUT;
  }
  const bool frag = act_frag || act_scale || act_corr;
  if (frag && (m_pad < rows || m_pad % kTokTile)) {
    set_error("quantize: m_pad (%lld) must be a multiple of 8 >= rows (%lld)", (long long)m_pad,
              (long long)rows);
    return FLEXQ_ERR_SHAPE;
  }
  T6Geom geo(m_pad > 0 ? m_pad : rows, cols, gs);
  QuantArgs A{x, rows, cols, gs, geo.ng, bits, fp16_scales, codes, scales,
              reinterpret_cast<uint8_t*>(act_frag), act_scale, act_corr, m_pad, flag,
              geo.spg, geo.kb};
  A.dbg = dbg_trace_buf();
  A.early = tuning().q_early ? 1 : 0;
  if (A.dbg) A.dbg_tag = dbg_next_launch() << 8 | 1;
  switch (dtype) {
    case FLEXQ_DT_F16: launch_quantize<FLEXQ_DT_F16>(A, st); break;
    case FLEXQ_DT_BF16: launch_quantize<FLEXQ_DT_BF16>(A, st); break;
    case FLEXQ_DT_F32: launch_quantize<FLEXQ_DT_F32>(A, st); break;
    case FLEXQ_DT_F64: launch_quantize<FLEXQ_DT_F64>(A, st); break;
    default:
      set_error("quantize: unknown dtype code %d", dtype);
      return FLEXQ_ERR_INVALID_INPUT;
  }
  FLEXQ_LAUNCH_CHECK("quantize");
  return FLEXQ_OK;
}

}  // namespace flexq

// ---- fused decode producers --------------------
// RMSNorm -> quantize and SiLU(gate) * up -> quantize in one kernel: each warp builds the
// fp16 intermediate h of one group in registers and quantizes it exactly as
// quantize_warp_kernel does, so the codes, scales and corrections are bit-identical to
// quantize(h) of that fp16 h.  h follows the LLaMA definitions:
//   rmsnorm: h = w * fp16(x * rsqrt(mean(x^2) + eps))      (fp32 statistics)
//   silu:    h = fp16(fp16(g / (1 + exp(-g))) * u)
namespace flexq {
struct FusedQuantArgs {
  QuantArgs q;       // rows, cols, gs, ng, bits, fp16_scales, act_*, m_pad, flag, spg, kb
  const __half* x;   // rmsnorm: [rows, x_stride]; silu: [rows, x_stride] = gate | up
  const __half* w;   // rmsnorm weight [cols]
  __half* h_out;     // optional fp16 h [rows, cols]
  int64_t x_stride;
  float eps;
  int mode;          // 0 = rmsnorm, 1 = silu * up
};

// grid (rows, ceil(G / 8)), 8 warps: warp w quantizes group blockIdx.y * 8 + w of row
// blockIdx.x.  RMSNorm: every CTA reduces the row's sum of squares itself (an L2-resident
// re-read of one row), so the row is spread over G/8 CTAs instead of one.
constexpr int kFusedWarps = 8;
__device__ __forceinline__ __half fused_h(const FusedQuantArgs& F, const __half* xr, int64_t c,
                                          float inv) {
  if (F.mode == 0) return __hmul(F.w[c], __float2half_rn(__half2float(xr[c]) * inv));
  const float g = __half2float(xr[c]);
  return __hmul(__float2half_rn(g / (1.f + __expf(-g))), xr[F.q.cols + c]);
}

__global__ void __launch_bounds__(kFusedWarps * 32) fused_quant_kernel(FusedQuantArgs F) {
  __shared__ float red[kFusedWarps];
  pdl_launch_dependents();
  pdl_wait();
  const QuantArgs& A = F.q;
  const int64_t r = blockIdx.x;
  const int K = (int)A.cols;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const __half* xr = F.x + r * F.x_stride;
  float inv = 0.f;
  if (F.mode == 0) {
    float ss = 0.f;
    for (int i = tid * 8; i < K; i += kFusedWarps * 32 * 8) {
      if (i + 8 <= K && (K & 7) == 0) {
        const uint4 raw = *reinterpret_cast<const uint4*>(xr + i);
        const __half2* h2 = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const float2 f = __half22float2(h2[j]);
          ss = fmaf(f.x, f.x, ss);
          ss = fmaf(f.y, f.y, ss);
        }
      } else {
        for (int j = i; j < i + 8 && j < K; j++) {
          const float v = __half2float(xr[j]);
          ss = fmaf(v, v, ss);
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) red[warp] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kFusedWarps; w++) tot += red[w];  // same order in every CTA
    inv = rsqrtf(tot / (float)K + F.eps);
  }
  const int64_t g = (int64_t)blockIdx.y * kFusedWarps + warp;
  if (g >= A.ng) return;
  if (A.gs == 128 && (K & 127) == 0) {
    // lane L: the 4 consecutive columns 4L..4L+3 -> 4 consecutive operand bytes, one store
    const int64_t c0 = g * 128 + lane * 4;
    float v[4];
    bool finite = true;
    float peak = 0.f;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const __half hv = fused_h(F, xr, c0 + i, inv);
      if (F.h_out) F.h_out[r * K + c0 + i] = hv;
      v[i] = __half2float(hv);
      finite &= isfinite(v[i]);
      peak = fmaxf(peak, fabsf(v[i]));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (!__all_sync(0xffffffffu, finite)) {
      if (lane == 0) atomicOr(A.flag, FLEXQ_FLAG_NONFINITE);
      peak = 0.f;
    }
    int cd[4];
    const double s = codes4_fp16(v, peak, A.bits, A.fp16_scales, lane == 0 ? A.flag : nullptr, cd);
    int csum = 0;
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
      csum += cd[i];
      word |= (uint32_t)(cd[i] & 0xff) << (8 * i);
    }
    const int jj = lane >> 3, hh = (lane >> 2) & 1, t = lane & 3;
    const int64_t off = ((g * (A.m_pad >> 3) + (r >> 3)) * 8 + 2 * t + hh) * 128 + (r & 7) * 16 + jj * 4;
    *reinterpret_cast<uint32_t*>(A.act_frag + off) = word;
#pragma unroll
    for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
    if (lane == 0) {
      A.act_scale[g * A.m_pad + r] = (float)s;
      A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * csum;
    }
    return;
  }
  const int64_t lo = g * A.gs, hi = min(lo + A.gs, A.cols);
  double peak = 0.0;
  bool finite = true;
  for (int64_t c = lo + lane; c < hi; c += 32) {
    const __half hv = fused_h(F, xr, c, inv);
    if (F.h_out) F.h_out[r * K + c] = hv;
    const double v = (double)__half2float(hv);
    finite &= isfinite(v);
    peak = fmax(peak, fabs(v));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  if (!__all_sync(0xffffffffu, finite)) {
    if (lane == 0) atomicOr(A.flag, FLEXQ_FLAG_NONFINITE);
    peak = 0.0;
  }
  const double s = group_scale(peak, A.bits, A.fp16_scales, lane == 0 ? A.flag : nullptr);
  int csum = 0;
  for (int64_t c = lo + lane; c < hi; c += 32) {
    const double v = (double)__half2float(fused_h(F, xr, c, inv));
    const int code = isfinite(v) ? quant_one(v, s, A.bits) : 0;
    csum += code;
    emit(A, r, c, code);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  if (lane == 0) {
    if (A.act_scale) A.act_scale[g * A.m_pad + r] = (float)s;
    if (A.act_corr) A.act_corr[g * A.m_pad + r] = kCorrBias + 32 * csum;
  }
}

int fused_quant_launch(int mode, const void* x, int64_t x_stride, const void* w, float eps,
                       int64_t rows, int64_t cols, int bits, int64_t gs, uint32_t* act_frag,
                       float* act_scale, int32_t* act_corr, int64_t m_pad, uint32_t* flag,
                       void* h_out, cudaStream_t st) {
  if (rows < 1 || cols < 1 || bits < 2 || bits > 8 || gs < 1 || gs > 1024 || !flag || !act_frag ||
      !act_scale || !act_corr || m_pad < rows || m_pad % kTokTile || (mode == 0 && !w)) {
    set_error("fused quantize: bad arguments (rows=%lld cols=%lld bits=%d group=%lld m_pad=%lld)",
              (long long)rows, (long long)cols, bits, (long long)gs, (long long)m_pad);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  T6Geom geo(m_pad, cols, gs);
  FusedQuantArgs F{};
  F.q = QuantArgs{nullptr, rows, cols, gs, geo.ng, bits, 1, nullptr, nullptr,
                  reinterpret_cast<uint8_t*>(act_frag), act_scale, act_corr, m_pad, flag, geo.spg,
                  geo.kb};
  F.x = reinterpret_cast<const __half*>(x);
  F.w = reinterpret_cast<const __half*>(w);
  F.h_out = reinterpret_cast<__half*>(h_out);
  F.x_stride = x_stride;
  F.eps = eps;
  F.mode = mode;
  cudaError_t e = launch_pdl(fused_quant_kernel,
                             dim3((unsigned)rows, (unsigned)cdiv(geo.ng, kFusedWarps)),
                             dim3(kFusedWarps * 32), 0, st, F);
  if (e != cudaSuccess) return cuda_status(e, "fused quantize launch");
  return FLEXQ_OK;
}
}  // namespace flexq
