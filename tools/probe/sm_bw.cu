// Aggregate HBM streaming bandwidth vs the number of active SMs (1 CTA per SM, 8 warps,
// per-warp TMA bulk ring of S x 6 KB), for a large stream and for a 12.6 MB "7B layer".
// Answers: can a CTA-per-row-group GEMV (64 CTAs for a 4096-row layer) saturate HBM?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int CH = 6144, S = 4, W = 8;

__global__ void stream(const uint8_t* src, size_t bytes, unsigned* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[W][S];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long nw = (long)gridDim.x * W, gw = (long)blockIdx.x * W + warp;
  size_t units = bytes / CH;
  size_t u0 = gw * units / nw, u1 = (gw + 1) * units / nw;
  uint8_t* ring = smem + warp * S * CH;
  uint64_t* bar = bars[warp];
  if (lane == 0) { for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](size_t u, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[s])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(sa(ring + s * CH)), "l"(src + u * CH), "r"(CH), "r"(sa(&bar[s])), "l"(pol) : "memory");
  };
  if (lane == 0) for (int s = 0; s < S && u0 + s < u1; s++) issue(u0 + s, s);
  unsigned acc = 0;
  for (size_t u = u0, it = 0; u < u1; u++, it++) {
    int s = it % S; unsigned par = (it / S) & 1;
    asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}" :: "r"(sa(&bar[s])), "r"(par) : "memory");
    const uint4* v = (const uint4*)(ring + s * CH);
    for (int i = lane; i < CH / 16; i += 32) { uint4 x = v[i]; acc ^= x.x ^ x.w; }
    __syncwarp();
    if (lane == 0 && u + S < u1) issue(u + S, s);
  }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const size_t big = (size_t)1 << 30;
  uint8_t* buf; cudaMalloc(&buf, big * 2);
  cudaMemset(buf, 1, big * 2);
  unsigned* out; cudaMalloc(&out, 64);
  const int smem = W * S * CH;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (size_t bytes : {(size_t)256 << 20, (size_t)12582912}) {
    for (int n : {16, 32, 64, 96, 128, 148}) {
      const int reps = bytes > (64u << 20) ? 5 : 40;
      for (int r = 0; r < 2; r++) stream<<<n, W * 32, smem>>>(buf + (r % 2) * big, bytes, out);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; r++) stream<<<n, W * 32, smem>>>(buf + (r % 2) * big, bytes, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double us = ms * 1e3 / reps;
      printf("bytes %7.1f MB  ctas %3d: %7.2f us  %7.0f GB/s  (%5.1f GB/s per SM)\n", bytes / 1e6, n, us,
             bytes / (us * 1e-6) / 1e9, bytes / (us * 1e-6) / 1e9 / n);
    }
  }
  return 0;
}
