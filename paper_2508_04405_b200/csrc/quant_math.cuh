// Scalar quantization math shared by every quantizer (quantize.py:29-36, 99-148):
// float64 throughout, one correctly rounded IEEE operation per step, so codes and scales
// are bit-identical with numpy.
#pragma once
#include "common.cuh"

namespace flexq {

__device__ __forceinline__ double group_scale(double peak, int bits, int fp16, uint32_t* flag) {
  const double lim = (double)((1 << (bits - 1)) - 1);
  double s = peak > 0.0 ? peak / lim : 1.0;
  if (fp16) s = (double)__half2float(__double2half(s));
  if (!(s > 0.0) && flag) atomicOr(flag, FLEXQ_FLAG_NONPOS_SCALE);
  return s;
}

__device__ __forceinline__ int quant_one(double v, double s, int bits) {
  const double lim = (double)((1 << (bits - 1)) - 1);
  double q = v / s;
  double a = floor(fabs(q) + 0.5);
  if (a > lim) a = lim;
  return q < 0.0 ? -(int)a : (int)a;
}

// group_scale(peak, bits, fp16 = 1) in fp32: fp16(fl32(peak / lim)) equals fp16(fl64(peak /
// lim)) for every positive fp16 peak and bits 2..8 (exhaustive, tools/check_f32_quant.c)
__device__ __forceinline__ float group_scale_h(float peak, int bits, uint32_t* flag) {
  const float lim = (float)((1 << (bits - 1)) - 1);
  const float s = peak > 0.f ? __half2float(__float2half_rn(__fdiv_rn(peak, lim))) : 1.f;
  if (!(s > 0.f) && flag) atomicOr(flag, FLEXQ_FLAG_NONPOS_SCALE);
  return s;
}

// The same code when v and s are both fp16 values (fp16 input, fp16 scales), in fp32: one
// correctly rounded fp32 quotient lies on the same side of every half-integer as the exact
// quotient (or on it exactly), so roundf() of it equals floor(|fl64(v / s)| + 0.5) with its
// sign -- checked exhaustively over all 2.0e9 (finite fp16 v, positive fp16 s) pairs
// (tools/check_f32_quant.c).  ~8x fewer issue slots than the float64 divide.
__device__ __forceinline__ int quant_one_h(float v, float s, int bits) {
  const float lim = (float)((1 << (bits - 1)) - 1);
  const float q = __fdiv_rn(v, s);
  const float a = fminf(roundf(fabsf(q)), lim);
  return q < 0.f ? -(int)a : (int)a;
}

// Non-finite inputs quantize to 0 (the caller raises the flag and zeroes the peak).
__device__ __forceinline__ int code_of(double v, double s, int bits) {
  return isfinite(v) ? quant_one(v, s, bits) : 0;
}

// Codes of four fp16-valued inputs of one group and the group's scale (peak = the group's
// max |v|, 0 when the group holds a non-finite value): fp32 steps for fp16 scales, float64
// otherwise -- the same results either way.
__device__ __forceinline__ double codes4_fp16(const float f[4], float peak, int bits, int fp16,
                                              uint32_t* flag, int c[4]) {
  if (fp16) {
    const float s = group_scale_h(peak, bits, flag);
    if (s > 0.f) {
#pragma unroll
      for (int i = 0; i < 4; i++) c[i] = isfinite(f[i]) ? quant_one_h(f[i], s, bits) : 0;
      return (double)s;
    }
#pragma unroll
    for (int i = 0; i < 4; i++) c[i] = code_of((double)f[i], (double)s, bits);
    return (double)s;
  }
  const double s = group_scale((double)peak, bits, 0, flag);
#pragma unroll
  for (int i = 0; i < 4; i++) c[i] = code_of((double)f[i], s, bits);
  return s;
}

// Byte offset of the 4 consecutive operand bytes holding columns 4*lane .. 4*lane+3 of
// group g (group = one 128-slot k-block) for token r.
__device__ __forceinline__ int64_t operand_word_offset(int64_t g, int64_t r, int64_t m_pad, int lane) {
  const int jj = lane >> 3, h = (lane >> 2) & 1, t = lane & 3;
  return ((g * (m_pad >> 3) + (r >> 3)) * 8 + 2 * t + h) * 128 + (r & 7) * 16 + jj * 4;
}

}  // namespace flexq
