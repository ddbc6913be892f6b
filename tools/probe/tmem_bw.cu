// TMEM read/write bandwidth probe (B200): W warps (W/4 per lane quarter) stream tcgen05.ld
// 32x32b.x32 (4 KB per warp instruction) with one wait per X loads; reports B/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define LD32(a, v)                                                                                         \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
               "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"               \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),         \
                 "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),     \
                 "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),               \
                 "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),               \
                 "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])                \
               : "r"(a))
#define ST32(a, v)                                                                                          \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
               "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a),     \
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),       \
               "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), \
               "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),           \
               "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),           \
               "r"(v[30]), "r"(v[31])                                                                      \
               : "memory")

__global__ void probe(long long* out, int mode, int iters) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&holder)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = holder + ((uint32_t)(32 * (warp & 3)) << 16) + ((warp >> 2) & 3) * 128;
  uint32_t v[32], w[32];
  uint32_t acc = 0;
  for (int i = 0; i < 32; i++) v[i] = i + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (mode == 0) {  // 2 loads of 32 columns, one wait
      LD32(base, v); LD32(base + 32, w);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 32; i++) acc += v[i] ^ w[i];
    } else if (mode == 1) {  // 2 stores of 32 columns, one wait
      ST32(base, v); ST32(base + 32, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      v[0] += 1;
    } else {  // load 32 + store 32 (read-modify-write of an fp32 accumulator)
      LD32(base, v); LD32(base + 32, w);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 32; i++) v[i] += w[i];
      ST32(base + 64, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) out[warp] = t1 - t0;
  if (acc == 0x12345678u) out[100] = acc;
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(holder), "r"(512));
}

int main() {
  long long* d; cudaMalloc(&d, 8192);
  long long h[32];
  const char* names[] = {"ld 2x32 cols", "st 2x32 cols", "ld 2x32 + st 32"};
  const int bytes_per_iter[] = {2 * 4096, 2 * 4096, 3 * 4096};
  for (int mode = 0; mode < 3; mode++)
    for (int warps : {4, 8, 16}) {
      const int iters = 4000;
      probe<<<1, warps * 32>>>(d, mode, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < warps; i++) mx = h[i] > mx ? h[i] : mx;
      const double bpc = (double)warps * bytes_per_iter[mode] * iters / mx;
      printf("%-18s warps=%2d  %7.1f cycles/iter/warp  %6.1f B/clk/SM\n", names[mode], warps,
             (double)mx / iters, bpc);
    }
  return 0;
}
