// tcgen05.mma kind::f16 issue cost with A from shared memory (.ss: smem descriptor) vs A from
// tensor memory (.ts: TMEM address, the layout gemm_tc16.cu uses).  One thread issues 2000
// k-blocks of 8 MMAs (M=128, K=16) into one accumulator; N = 64 / 128 / 256.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_none(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) | (1ull << 46);
}

template <int N, int TS>
__global__ void probe(long long* out, int iters, int stores) {
  __shared__ volatile int done;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* A = sm;
  uint8_t* B = sm + 4 * 16384;
  for (int i = threadIdx.x; i < (4 * 16384 + 2 * N * 256) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) & 0x3bff3bffu;
  if (threadIdx.x == 0) {
    done = 0;
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
  const uint32_t acol0 = tmem + (N == 256 ? 256 : 2 * N);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      const int st = it & 3;
      const uint64_t ad = desc_sw128(s32(A + st * 16384));
      const uint64_t bd = desc_none(s32(B + (st & 1) * N * 256));
      const uint32_t d = tmem + (N == 256 ? 0 : (it & 1) * N);
#pragma unroll
      for (int s = 0; s < 8; s++) {
        const uint64_t b2 = bd + (uint64_t)(s * 16);
        if (TS) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                       "r"(acol0 + (uint32_t)((st & 1) * 64 + 8 * s)), "l"(b2), "r"(idesc), "r"(1u) : "memory");
        } else {
          const uint64_t a2 = ad + (uint64_t)((s & 3) * 2);
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a2), "l"(b2),
                       "r"(idesc), "r"(1u) : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar)) : "memory");
    out[0] = clock64() - t0;
    done = 1;
  } else if (stores && threadIdx.x >= 32) {
    // warps 1..8: tcgen05.st.16x256b.x8 (4 KB per warp-instruction) into columns 256..511,
    // the converters' traffic in gemm_tc16.cu, until the MMA thread is done
    const int w = threadIdx.x / 32 - 1;
    const uint32_t base = tmem + ((uint32_t)((w & 3) * 32 + (w >> 2) * 16) << 16) + 256;
    long long n = 0;
    uint32_t v0 = threadIdx.x;
    while (!done) {
      asm volatile("tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
                   "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + (uint32_t)((n & 3) * 64)), "r"(v0) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      n++;
    }
    if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&out[1], (unsigned long long)n);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int TS>
void run(long long* d, int stores) {
  const int smem = 4 * 16384 + 2 * N * 256;
  cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaMemset(d, 0, 16);
  probe<N, TS><<<1, stores ? 288 : 128, smem>>>(d, 2000, stores);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("error %s\n", cudaGetErrorString(e)); return; }
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d A from %s, TMEM stores %s: %6.1f cycles per MMA; stores %.1f B/clk\n", N,
         TS ? "TMEM (.ts)" : "SMEM (.ss)", stores ? "on " : "off", (double)h[0] / 2000 / 8,
         (double)h[1] * 4096 / (double)h[0]);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int st = 0; st < 2; st++) {
    run<64, 0>(d, st); run<64, 1>(d, st);
    run<128, 0>(d, st); run<128, 1>(d, st);
    run<256, 0>(d, st); run<256, 1>(d, st);
  }
  return 0;
}
