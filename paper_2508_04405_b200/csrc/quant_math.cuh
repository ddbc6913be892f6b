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

// Non-finite inputs quantize to 0 (the caller raises the flag and zeroes the peak).
__device__ __forceinline__ int code_of(double v, double s, int bits) {
  return isfinite(v) ? quant_one(v, s, bits) : 0;
}

// One warp quantizes one fp16 group of 128 columns; lane L holds columns 4L..4L+3 (`raw`, one
// 8 B load).  Returns the group's scale; `word` gets the lane's 4 codes (byte i = column
// 4L+i) and `csum` the group's code sum (all lanes).  Shared by quantize_g128_kernel and the
// chain kernel's quantizer phase, so both emit bit-identical operands.
__device__ __forceinline__ double quantize_g128_lane(uint2 raw, int bits, int fp16_scales,
                                                     uint32_t* flag, int lane, uint32_t& word,
                                                     int& csum) {
  const float2 f01 = __half22float2(*reinterpret_cast<const __half2*>(&raw.x));
  const float2 f23 = __half22float2(*reinterpret_cast<const __half2*>(&raw.y));
  const double v[4] = {(double)f01.x, (double)f01.y, (double)f23.x, (double)f23.y};
  bool finite = true;
  float peak = 0.f;  // max of fp16 magnitudes: exact in fp32
#pragma unroll
  for (int i = 0; i < 4; i++) {
    finite &= isfinite(v[i]);
    peak = fmaxf(peak, fabsf((float)v[i]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, o));
  if (!__all_sync(0xffffffffu, finite)) {
    if (lane == 0) atomicOr(flag, FLEXQ_FLAG_NONFINITE);
    peak = 0.f;
  }
  const double sc = group_scale((double)peak, bits, fp16_scales, lane == 0 ? flag : nullptr);
  int c[4];
  csum = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    c[i] = code_of(v[i], sc, bits);
    csum += c[i];
  }
  word = (uint32_t)(c[0] & 0xff) | ((uint32_t)(c[1] & 0xff) << 8) |
         ((uint32_t)(c[2] & 0xff) << 16) | ((uint32_t)(c[3] & 0xff) << 24);
#pragma unroll
  for (int o = 16; o; o >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, o);
  return sc;
}

// Byte offset of the 4 consecutive operand bytes holding columns 4*lane .. 4*lane+3 of
// group g (group = one 128-slot k-block) for token r.
__device__ __forceinline__ int64_t operand_word_offset(int64_t g, int64_t r, int64_t m_pad, int lane) {
  const int jj = lane >> 3, h = (lane >> 2) & 1, t = lane & 3;
  return ((g * (m_pad >> 3) + (r >> 3)) * 8 + 2 * t + h) * 128 + (r & 7) * 16 + jj * 4;
}

}  // namespace flexq
