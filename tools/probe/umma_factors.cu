// What slows tcgen05.mma (B200)?  One thread issues 2000 k-blocks of 8 x kind::f16 (M=128,
// N=64, K=16) MMAs; factors: operand data (sparse 0x0101 vs fp16 1.0 vs random), block size
// (128 vs 320 threads, idle), a runtime branch around each MMA, a runtime accumulate predicate.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_none(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}

template <int BRANCH, int RTPRED>
__global__ void probe(long long* out, int iters, int fill, int flag) {
  constexpr int N = 64;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* A = sm;
  uint8_t* B = sm + 4 * 16384;
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x) {
    uint32_t v = fill == 0 ? 0x01010101u : fill == 1 ? 0x3c003c00u : (i * 2654435761u) & 0x3bff3bffu;
    reinterpret_cast<uint32_t*>(sm)[i] = v;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      const int st = it & 3;
      const uint64_t ad = desc_sw128(s32(A + st * 16384));
      const uint64_t bd = desc_none(s32(B + st * N * 128));
#pragma unroll
      for (int s = 0; s < 8; s++) {
        const uint64_t a2 = ad + (uint64_t)((s & 3) * 2), b2 = bd + (uint64_t)((s & 3) * 16);
        const uint32_t acc = RTPRED ? ((flag && s == 0) ? 0u : 1u) : 1u;
        if (BRANCH && flag > 5) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + 64), "l"(a2), "l"(b2), "r"(idesc), "r"(acc) : "memory");
        } else {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(a2), "l"(b2), "r"(idesc), "r"(acc) : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar)) : "memory");
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int BRANCH, int RTPRED>
void run(long long* d, int threads, int fill) {
  const int smem = 4 * 16384 + 4 * 64 * 128;
  cudaFuncSetAttribute(probe<BRANCH, RTPRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<BRANCH, RTPRED><<<1, threads, smem>>>(d, 2000, fill, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const char* fills[] = {"0x01 bytes", "fp16 1.0", "random fp16"};
  printf("threads %3d, data %-12s, branch %d, runtime-pred %d: %6.1f cycles per MMA\n", threads,
         fills[fill], BRANCH, RTPRED, (double)h / 2000 / 8);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int fill = 0; fill < 3; fill++) {
    run<0, 0>(d, 128, fill);
    run<0, 0>(d, 320, fill);
    run<1, 0>(d, 128, fill);
    run<0, 1>(d, 128, fill);
  }
  return 0;
}
