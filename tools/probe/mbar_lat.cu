// mbarrier wait cost on an already-completed phase: try_wait (with / without suspend hint)
// vs test_wait, cycles per wait in a dependent loop (B200).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(long long* out, int mode, int iters) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&bar)));  // phase 0 complete
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    uint32_t ok;
    if (mode == 0) {
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P;}"
                   : "=r"(ok) : "r"(s32(&bar)), "r"(acc & 0));
    } else if (mode == 1) {
      asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3; selp.u32 %0, 1, 0, P;}"
                   : "=r"(ok) : "r"(s32(&bar)), "r"(acc & 0), "r"(0x989680));
    } else {
      asm volatile("{.reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.u32 %0, 1, 0, P;}"
                   : "=r"(ok) : "r"(s32(&bar)), "r"(acc & 0));
    }
    acc += ok;  // dependent chain through the parity operand
  }
  long long t1 = clock64();
  out[mode] = (t1 - t0) / iters;
  out[8 + mode] = acc;
}

int main() {
  long long* d; cudaMalloc(&d, 16 * 8);
  long long h[16];
  for (int m = 0; m < 3; m++) probe<<<1, 32>>>(d, m, 10000);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  printf("try_wait: %lld cycles, try_wait+hint: %lld, test_wait: %lld (ok counts %lld %lld %lld)\n",
         h[0], h[1], h[2], h[8], h[9], h[10]);
  return 0;
}
