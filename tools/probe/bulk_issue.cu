// cp.async.bulk (TMA 1-D bulk copy) issue cost on B200: how many cycles one thread spends
// issuing a copy, by size, with 1..4 issuing warps in the CTA, and the time to completion.
// Source is either L2-resident (a small buffer re-read) or streamed from HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_issue bulk_issue.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const uint8_t* src, int64_t src_span, int bytes, int n, int nwarps,
                      long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 4) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (warp >= nwarps || lane != 0) return;
  uint8_t* dst = sm + warp * (48 * 1024);
  int per_p2 = 1;  // destination slots per warp (power of 2)
  while (per_p2 * 2 * bytes <= 48 * 1024) per_p2 *= 2;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t base = ((int64_t)blockIdx.x * nwarps + warp) * (int64_t)n * bytes;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[warp])),
               "r"(n * bytes) : "memory");
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const uint8_t* s = src + ((base + (int64_t)i * bytes) & (src_span - 1));  // span: power of 2
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(s32(dst + (i & (per_p2 - 1)) * bytes)),
        "l"(s), "r"(bytes), "r"(s32(&bar[warp])), "l"(pol)
        : "memory");
  }
  long long t1 = clock64();
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          s32(&bar[warp]))
      : "memory");
  long long t2 = clock64();
  if (blockIdx.x == 0) {
    out[warp * 2] = t1 - t0;
    out[warp * 2 + 1] = t2 - t0;
  }
}

int main() {
  const int64_t big = 1ll << 31;  // 2 GB: streamed from HBM
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  long long* d;
  cudaMalloc(&d, 64 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 48 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int grid : {1, sms}) {
    for (int64_t span : {(int64_t)4 << 20, big}) {
      for (int bytes : {64, 512, 1024, 6144, 12288, 24576}) {
        for (int nw : {1, 2, 4}) {
          const int n = 32;
          probe<<<grid, 128, 4 * 48 * 1024>>>(buf, span, bytes, n, nw, d);
          probe<<<grid, 128, 4 * 48 * 1024>>>(buf, span, bytes, n, nw, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
          long long h[8];
          cudaMemcpy(h, d, 8 * 8, cudaMemcpyDeviceToHost);
          printf("grid %3d src %-4s %6d B x %d copies, %d issuing warps: issue %6.1f cyc/copy, "
                 "complete %7.1f cyc/copy (warp 0)\n", grid, span > (64 << 20) ? "HBM" : "L2",
                 bytes, n, nw, (double)h[0] / n, (double)h[1] / n);
        }
      }
    }
  }
  return 0;
}
