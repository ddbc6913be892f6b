// Exact float64 group epilogue over traced INT32 partials.
//
// y[m,n] = sum over g ascending of (xs[m,g] * ws[n,g]) * double(P[g,m,n]) with
// every multiply and add a separate correctly-rounded IEEE operation (no FMA
// contraction: __dmul_rn / __dadd_rn), exactly the reference's
// _scale_accumulate (engine.py:211-216) applied in its group order
// (engine.py:277-286, 359-364).  The result is bit-identical with the
// reference's float64 output; y16 is the fp16 rounding of that float64 value.
#include "common.cuh"

namespace flexq {

__global__ void group_epilogue_f64_kernel(const int32_t* __restrict__ P,
                                          const double* __restrict__ ws,
                                          const double* __restrict__ xs, int64_t m, int64_t n,
                                          int64_t ng, double* __restrict__ y,
                                          __half* __restrict__ y16) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m * n) return;
  const int64_t row = i / n, col = i - row * n;
  double acc = 0.0;
  for (int64_t g = 0; g < ng; g++) {
    const double s = __dmul_rn(xs[row * ng + g], ws[col * ng + g]);
    acc = __dadd_rn(acc, __dmul_rn(s, (double)P[(g * m + row) * n + col]));
  }
  if (y) y[i] = acc;
  if (y16) y16[i] = __double2half(acc);
}

int group_epilogue_launch(const int32_t* P, const double* ws, const double* xs, int64_t m,
                          int64_t n, int64_t ng, double* y, uint16_t* y16, cudaStream_t st) {
  if (m < 1 || n < 1 || ng < 1) {
    set_error("group_epilogue: dims must be positive, got m=%lld n=%lld groups=%lld",
              (long long)m, (long long)n, (long long)ng);
    return FLEXQ_ERR_CONFIG;
  }
  group_epilogue_f64_kernel<<<(unsigned)cdiv(m * n, 256), 256, 0, st>>>(
      P, ws, xs, m, n, ng, y, reinterpret_cast<__half*>(y16));
  FLEXQ_LAUNCH_CHECK("group_epilogue_f64");
  return FLEXQ_OK;
}

}  // namespace flexq
