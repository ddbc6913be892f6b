// TMEM access latency probe (B200): cycles per tcgen05.ld(+wait), ld+st(+waits),
// and the same with 4 / 16 warps issuing concurrently.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld16(uint32_t a, uint32_t (&v)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(a));
}
__device__ __forceinline__ void waitld(uint32_t (&v)[16]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
               "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])::"memory");
}
__device__ __forceinline__ void st16(uint32_t a, const uint32_t (&v)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
               "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
}
__device__ __forceinline__ void waitst() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void probe(long long* out, int mode, int iters) {
  __shared__ uint32_t holder;
  __shared__ float4 tab[16];
  if (threadIdx.x < 16) tab[threadIdx.x] = make_float4(1.f, 2.f, 3.f, 4.f);
  int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = holder + ((uint32_t)(32 * (warp & 3)) << 16) + (warp >> 2) * 64;
  uint32_t v[16];
  for (int i = 0; i < 16; i++) v[i] = i;
  st16(base, v); waitst();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (mode == 0) { ld16(base, v); waitld(v); }
    else if (mode == 1) { ld16(base, v); waitld(v); v[0] += 1; st16(base + 16, v); waitst(); }
    else if (mode == 2) { ld16(base, v); ld16(base + 16, v); waitld(v); }
    else if (mode == 3) { uint32_t w[16]; ld16(base, v); ld16(base + 16, w); waitld(v); waitld(w); for (int i = 0; i < 16; i++) v[i] += w[i]; st16(base + 32, v); st16(base+48, v); waitst(); }
    else if (mode == 4) {  // LDS latency alone
      float4 t = tab[(it & 7) + (int)(acc > 1e30f)]; v[0] += __float_as_uint(t.x); }
    else if (mode == 5) {  // LDS right behind two tcgen05.st (no wait)
      st16(base + 32, v); st16(base + 48, v);
      float4 t = tab[(it & 7) + (int)(acc > 1e30f)]; v[0] += __float_as_uint(t.x); }
    else if (mode == 6) {  // LDS right behind a tcgen05.ld + wait
      ld16(base, v); waitld(v);
      float4 t = tab[(it & 7) + (int)(acc > 1e30f)]; v[0] += __float_as_uint(t.x); }
    else {  // fence::after_thread_sync cost
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float4 t = tab[(it & 7) + (int)(acc > 1e30f)]; v[0] += __float_as_uint(t.x); }
    for (int i = 0; i < 16; i++) acc += __uint_as_float(v[i]);
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + warp] = (t1 - t0) / iters;
  if (acc == 12345.f) out[1000] = 1;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(holder), "r"(512));
}

int main() {
  long long* d; cudaMalloc(&d, 8192 * 8);
  long long h[64];
  const char* names[] = {"ld16+wait", "ld16+wait+st16+wait", "2x ld16 + wait", "2ld+2st round",
                         "LDS.128 alone", "2 st16 then LDS", "ld16+wait then LDS", "fence::after + LDS"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 8; mode++) {
      probe<<<1, warps * 32>>>(d, mode, 2000);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
      printf("warps=%2d %-22s cycles/iter warp0=%lld warp%d=%lld\n", warps, names[mode], h[0], warps - 1, h[warps - 1]);
    }
  }
  return 0;
}
