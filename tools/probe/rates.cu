// Microbenchmarks that decide the B200 design of the W6Ax linear path:
// POPC / LOP3 / IDP4A / IMMA(mma.sync s8) / b1-mma / DFMA / I2F issue rates, and HBM read bandwidth.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
constexpr int ITERS = 4096;

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t a[8]; uint32_t acc[8];
  for (int i = 0; i < 8; i++) { a[i] = seed * (threadIdx.x + i * 77); acc[i] = 0; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) { acc[i] += __popc(a[i] ^ it); }
  }
  uint32_t s = 0; for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0xdeadbeef) out[0] = s;
}
__global__ void k_popc_only(uint32_t* out, uint32_t seed) {
  // pure POPC chain count: popc of independent regs, summed via IADD3 every 2
  uint32_t a[16]; uint32_t acc = 0;
  for (int i = 0; i < 16; i++) a[i] = seed * (threadIdx.x + i * 77);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) { acc += __popc(a[i]) + __popc(a[i+1]); a[i] += it; a[i+1] ^= it; }
  }
  if (acc == 0xdeadbeef) out[0] = acc;
}
__global__ void k_dp4a(uint32_t* out, uint32_t seed) {
  int a[8]; int acc[8];
  for (int i = 0; i < 8; i++) { a[i] = seed * (threadIdx.x + i * 77); acc[i] = 0; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) { acc[i] = __dp4a(a[i], a[(i+1)&7], acc[i]); }
  }
  int s = 0; for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x1234567) out[0] = s;
}
__global__ void k_imma(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed*threadIdx.x, a1 = a0*3, a2 = a0*5, a3 = a0*7, b0 = a0*11, b1 = a0*13;
  int c[4][4] = {};
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0; for (int j = 0; j < 4; j++) for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 0x1234567) out[0] = s;
}
__global__ void k_bmma(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed*threadIdx.x, a1 = a0*3, a2 = a0*5, a3 = a0*7, b0 = a0*11, b1 = a0*13;
  int c[4][4] = {};
  for (int it = 0; it < ITERS / 8; it++) {
#pragma unroll
    for (int j = 0; j < 4; j++)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0; for (int j = 0; j < 4; j++) for (int i = 0; i < 4; i++) s += c[j][i];
  if (s == 0x1234567) out[0] = s;
}
__global__ void k_dfma(uint32_t* out, uint32_t seed) {
  double a[8]; double x = seed * 1e-9;
  for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], x, 0.5);
  }
  double s = 0; for (int i = 0; i < 8; i++) s += a[i];
  if (s == 1.2345) out[0] = 1;
}
__global__ void k_i2f(uint32_t* out, uint32_t seed) {
  int a[8]; float acc[8];
  for (int i = 0; i < 8; i++) { a[i] = seed * (threadIdx.x + i); acc[i] = 0.f; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) { acc[i] += __int2float_rn(a[i] + it); }
  }
  float s = 0; for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 1.2345f) out[0] = 1;
}
__global__ void k_read(const int4* __restrict__ p, size_t n16, int4* out) {
  int4 acc = make_int4(0,0,0,0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2*stride), v3 = __ldcs(p + i + 3*stride);
    acc.x ^= v0.x ^ v1.x ^ v2.x ^ v3.x; acc.y ^= v0.y ^ v1.y ^ v2.y ^ v3.y;
    acc.z ^= v0.z ^ v1.z ^ v2.z ^ v3.z; acc.w ^= v0.w ^ v1.w ^ v2.w ^ v3.w;
  }
  for (; i < n16; i += stride) { int4 v = __ldcs(p + i); acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w; }
  if (acc.x == 0x12345 && acc.y == 7) out[0] = acc;
}

template <typename K>
float time_kernel(K kern, int blocks, int threads, uint32_t* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 3u);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; r++) kern<<<blocks, threads>>>(out, 3u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 3;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d l2=%d MB clock=%d MHz smem/blk optin=%zu\n", prop.name, sms, prop.l2CacheSize >> 20, clk_khz / 1000, prop.sharedMemPerBlockOptin);
  uint32_t* out; CK(cudaMalloc(&out, 64));
  int blocks = sms * 4, threads = 512;
  double thr = (double)blocks * threads;
  float ms;
  ms = time_kernel(k_popc, blocks, threads, out);
  printf("popc+xor+iadd: %.3f ms -> %.2f Tpopc/s (8 per iter)\n", ms, thr * ITERS * 8 / ms / 1e9);
  ms = time_kernel(k_popc_only, blocks, threads, out);
  printf("popc-dense   : %.3f ms -> %.2f Tpopc/s (16 per iter)\n", ms, thr * ITERS * 16 / ms / 1e9);
  ms = time_kernel(k_dp4a, blocks, threads, out);
  printf("dp4a         : %.3f ms -> %.2f Tdp4a/s = %.1f TOPS\n", ms, thr * ITERS * 8 / ms / 1e9, thr * ITERS * 8 * 8 / ms / 1e9);
  ms = time_kernel(k_imma, blocks, threads, out);
  printf("imma m16n8k32: %.3f ms -> %.1f TOPS (int8, mma.sync)\n", ms, thr / 32 * ITERS * 4 * (16.0*8*32*2) / ms / 1e9);
  ms = time_kernel(k_bmma, blocks, threads, out);
  printf("b1 m16n8k256 : %.3f ms -> %.1f T bit-ops/s (emulated)\n", ms, thr / 32 * (ITERS/8) * 4 * (16.0*8*256*2) / ms / 1e9);
  ms = time_kernel(k_dfma, blocks, threads, out);
  printf("dfma         : %.3f ms -> %.2f TFLOP/s fp64\n", ms, thr * ITERS * 8 * 2 / ms / 1e9);
  ms = time_kernel(k_i2f, blocks, threads, out);
  printf("i2f+fadd     : %.3f ms -> %.2f T i2f/s\n", ms, thr * ITERS * 8 / ms / 1e9);
  // HBM read bandwidth
  size_t bytes = (size_t)2 << 30; int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  int4* o4; CK(cudaMalloc(&o4, 64));
  for (int bpsm : {2, 4, 8}) for (int t : {256, 512}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k_read<<<sms * bpsm, t>>>(buf, bytes / 16, o4);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k_read<<<sms * bpsm, t>>>(buf, bytes / 16, o4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms2; cudaEventElapsedTime(&ms2, e0, e1);
    printf("read %d blk/sm x %d thr: %.1f GB/s\n", bpsm, t, bytes * 5.0 / ms2 / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
