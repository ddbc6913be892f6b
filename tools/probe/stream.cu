// Streaming-read microbenchmark: which load mechanism saturates B200 HBM with a
// per-warp contiguous range (the GEMV's access pattern)?
//   mode 0: per-warp TMA bulk ring (cp.async.bulk + mbarrier), S stages of CH bytes
//   mode 1: per-warp cp.async 16B (LDGSTS) ring, S stages of CH bytes
//   mode 2: plain LDG.128, U vectors in flight per lane
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int CH>
__global__ void tma_stream(const uint8_t* src, size_t bytes, int nw, unsigned* out, int wpc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[16][S];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long gw = (long)blockIdx.x * wpc + warp;
  if (gw >= nw) return;
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

template <int S, int CH, int NSMALL, int SMALL>
__global__ void tma_multi(const uint8_t* src, const uint8_t* side, size_t bytes, int nw, unsigned* out, int wpc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[16][S];
  constexpr int ST = CH + NSMALL * SMALL;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long gw = (long)blockIdx.x * wpc + warp;
  if (gw >= nw) return;
  size_t units = bytes / CH;
  size_t u0 = gw * units / nw, u1 = (gw + 1) * units / nw;
  uint8_t* ring = smem + warp * S * ST;
  uint64_t* bar = bars[warp];
  if (lane == 0) { for (int s = 0; s < S; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar[s]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](size_t u, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar[s])), "r"(ST) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(sa(ring + s * ST)), "l"(src + u * CH), "r"(CH), "r"(sa(&bar[s])), "l"(pol) : "memory");
    for (int i = 0; i < NSMALL; i++)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(sa(ring + s * ST + CH + i * SMALL)), "l"(side + ((u * 7 + i * 131) % 4096) * SMALL), "r"(SMALL), "r"(sa(&bar[s])) : "memory");
  };
  if (lane == 0) for (int s = 0; s < S && u0 + s < u1; s++) issue(u0 + s, s);
  unsigned acc = 0;
  for (size_t u = u0, it = 0; u < u1; u++, it++) {
    int s = it % S; unsigned par = (it / S) & 1;
    asm volatile("{\n.reg .pred P1;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W%=;\n}" :: "r"(sa(&bar[s])), "r"(par) : "memory");
    const uint4* v = (const uint4*)(ring + s * ST);
    for (int i = lane; i < ST / 16; i += 32) { uint4 x = v[i]; acc ^= x.x ^ x.w; }
    __syncwarp();
    if (lane == 0 && u + S < u1) issue(u + S, s);
  }
  if (acc == 0x1234567) out[0] = acc;
}

template <int S, int CH>
__global__ void ldgsts_stream(const uint8_t* src, size_t bytes, int nw, unsigned* out, int wpc) {
  extern __shared__ __align__(128) uint8_t smem[];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long gw = (long)blockIdx.x * wpc + warp;
  if (gw >= nw) return;
  size_t units = bytes / CH;
  size_t u0 = gw * units / nw, u1 = (gw + 1) * units / nw;
  uint8_t* ring = smem + warp * S * CH;
  uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](size_t u, int s) {
    for (int i = lane; i < CH / 16; i += 32)
      asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" :: "r"(sa(ring + s * CH + i * 16)), "l"(src + u * CH + i * 16), "l"(pol));
    asm volatile("cp.async.commit_group;");
  };
  for (int s = 0; s < S; s++) { if (u0 + s < u1) issue(u0 + s, s); else asm volatile("cp.async.commit_group;"); }
  unsigned acc = 0;
  for (size_t u = u0, it = 0; u < u1; u++, it++) {
    int s = it % S;
    asm volatile("cp.async.wait_group %0;" :: "n"(S - 1));
    __syncwarp();
    const uint4* v = (const uint4*)(ring + s * CH);
    for (int i = lane; i < CH / 16; i += 32) { uint4 x = v[i]; acc ^= x.x ^ x.w; }
    __syncwarp();
    if (u + S < u1) issue(u + S, s); else asm volatile("cp.async.commit_group;");
  }
  if (acc == 0x1234567) out[0] = acc;
}

template <int U>
__global__ void ldg_stream(const uint4* src, size_t n16, int nw, unsigned* out, int wpc) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long gw = (long)blockIdx.x * wpc + warp;
  if (gw >= nw) return;
  size_t per = n16 / nw / (32 * U) * (32 * U);
  size_t b0 = gw * per;
  unsigned acc = 0;
  for (size_t i = b0; i < b0 + per; i += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; j++) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(src + i + j * 32 + lane));
#pragma unroll
    for (int j = 0; j < U; j++) acc ^= v[j].x ^ v[j].w;
  }
  if (acc == 0x1234567) out[0] = acc;
}

template <typename F>
void run(const char* name, F launch, size_t bytes) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 10; r++) launch();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("%-44s %8.1f GB/s %s\n", name, bytes * 10.0 / ms / 1e6, err ? cudaGetErrorString(err) : "");
}

template <int S, int CH>
void tma_case(const uint8_t* buf, size_t bytes, unsigned* out, int wpc, int cps) {
  int smem = wpc * S * CH;
  cudaFuncSetAttribute(tma_stream<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nw = 148 * cps * wpc;
  char name[128]; snprintf(name, 128, "tma S=%d CH=%d warps/cta=%d cta/sm=%d", S, CH, wpc, cps);
  run(name, [&] { tma_stream<S, CH><<<148 * cps, wpc * 32, smem>>>(buf, bytes, nw, out, wpc); }, bytes / CH * CH);
}
template <int S, int CH>
void lgs_case(const uint8_t* buf, size_t bytes, unsigned* out, int wpc, int cps) {
  int smem = wpc * S * CH;
  cudaFuncSetAttribute(ldgsts_stream<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nw = 148 * cps * wpc;
  char name[128]; snprintf(name, 128, "ldgsts S=%d CH=%d warps/cta=%d cta/sm=%d", S, CH, wpc, cps);
  run(name, [&] { ldgsts_stream<S, CH><<<148 * cps, wpc * 32, smem>>>(buf, bytes, nw, out, wpc); }, bytes / CH * CH);
}
template <int U>
void ldg_case(const uint8_t* buf, size_t bytes, unsigned* out, int wpc, int cps) {
  int nw = 148 * cps * wpc;
  char name[128]; snprintf(name, 128, "ldg U=%d warps/cta=%d cta/sm=%d", U, wpc, cps);
  size_t n16 = bytes / 16;
  size_t per = n16 / nw / (32 * U) * (32 * U);
  run(name, [&] { ldg_stream<U><<<148 * cps, wpc * 32>>>((const uint4*)buf, n16, nw, out, wpc); }, per * nw * 16);
}

template <int S, int CH, int NS, int SM>
void multi_case(const uint8_t* buf, const uint8_t* side, size_t bytes, unsigned* out, int wpc, int cps) {
  int smem = wpc * S * (CH + NS * SM);
  cudaFuncSetAttribute(tma_multi<S, CH, NS, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nw = 148 * cps * wpc;
  char name[128]; snprintf(name, 128, "tma-multi S=%d CH=%d +%dx%d w/cta=%d cta/sm=%d", S, CH, NS, SM, wpc, cps);
  run(name, [&] { tma_multi<S, CH, NS, SM><<<148 * cps, wpc * 32, smem>>>(buf, side, bytes, nw, out, wpc); }, bytes / CH * CH);
}

int main(int argc, char** argv) {
  size_t bytes = (size_t)1 << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  unsigned* out; cudaMalloc(&out, 64);
  uint8_t* side; cudaMalloc(&side, 4096 * 1024); cudaMemset(side, 2, 4096 * 1024);
  if (argc > 1) {  // one issuing thread per SM (the tcgen05 kernels' weight producer)
    tma_case<8, 12288>(buf, bytes, out, 1, 1);
    tma_case<14, 12288>(buf, bytes, out, 1, 1);
    tma_case<7, 24576>(buf, bytes, out, 1, 1);
    tma_case<16, 6144>(buf, bytes, out, 1, 1);
    tma_case<28, 6144>(buf, bytes, out, 1, 1);
    tma_case<7, 12288>(buf, bytes, out, 2, 1);
    tma_case<4, 12288>(buf, bytes, out, 4, 1);
    tma_case<3, 6144>(buf, bytes, out, 4, 2);
    return 0;
  }
  multi_case<2, 6144, 0, 16>(buf, side, bytes, out, 4, 3);
  multi_case<2, 6144, 1, 1024>(buf, side, bytes, out, 4, 3);
  multi_case<2, 6144, 4, 32>(buf, side, bytes, out, 4, 3);
  multi_case<2, 6144, 4, 128>(buf, side, bytes, out, 4, 3);
  multi_case<2, 12288, 4, 64>(buf, side, bytes, out, 4, 2);
  multi_case<3, 6144, 4, 32>(buf, side, bytes, out, 4, 2);
  tma_case<3, 6144>(buf, bytes, out, 4, 2);
  tma_case<3, 7168>(buf, bytes, out, 4, 2);
  tma_case<4, 6144>(buf, bytes, out, 4, 2);
  tma_case<2, 12288>(buf, bytes, out, 4, 2);
  tma_case<3, 12288>(buf, bytes, out, 2, 2);
  tma_case<6, 6144>(buf, bytes, out, 2, 2);
  tma_case<4, 16384>(buf, bytes, out, 1, 3);
  tma_case<8, 8192>(buf, bytes, out, 1, 3);
  tma_case<3, 6144>(buf, bytes, out, 8, 1);
  tma_case<2, 6144>(buf, bytes, out, 16, 1);
  lgs_case<3, 6144>(buf, bytes, out, 4, 2);
  lgs_case<4, 6144>(buf, bytes, out, 4, 2);
  lgs_case<3, 6144>(buf, bytes, out, 8, 1);
  lgs_case<2, 6144>(buf, bytes, out, 16, 1);
  ldg_case<4>(buf, bytes, out, 4, 4);
  ldg_case<8>(buf, bytes, out, 4, 4);
  ldg_case<12>(buf, bytes, out, 4, 3);
  ldg_case<12>(buf, bytes, out, 8, 2);
  ldg_case<6>(buf, bytes, out, 8, 2);
  ldg_case<24>(buf, bytes, out, 4, 2);
  return 0;
}
