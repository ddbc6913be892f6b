// tcgen05.mma.cta_group::2 issue rate (B200): one thread of the leader CTA of a 2-CTA cluster
// issues k-blocks of MMAs with M = 256 (128 rows per SM), against cta_group::1 M = 128 on one
// SM.  Data are don't-care; the question is cycles per instruction and per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma2_rate umma2_rate.cu
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

template <int N, int CG, int KIND>  // KIND 0: i8 (K=32), 1: f16 (K=16)
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* A = sm;              // 4 x 16 KB
  uint8_t* B = sm + 4 * 16384;  // 4 x N*128 (per CTA: its half of N for CG = 2)
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s32(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  const int MROWS = CG == 2 ? 256 : 128;
  const uint32_t dfmt = KIND == 0 ? 2u : 1u, afmt = KIND == 0 ? 0u : 0u, bfmt = KIND == 0 ? 1u : 0u;
  const uint32_t idesc = (dfmt << 4) | (afmt << 7) | (bfmt << 10) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(MROWS >> 4) << 24);
  if (threadIdx.x == 0 && rank == 0) {
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      const int st = it & 3;
      const uint64_t ad = desc_sw128(s32(A + st * 16384));
      const uint64_t bd = desc_none(s32(B + st * N * 128));
      const int steps = KIND == 0 ? 4 : 8;
      for (int s = 0; s < steps; s++) {
        const uint64_t a2 = ad + (uint64_t)((s & 3) * 2), b2 = bd + (uint64_t)((s & 3) * 16);
        if (CG == 2) {
          if (KIND == 0)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(a2), "l"(b2), "r"(idesc) : "memory");
          else
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(a2), "l"(b2), "r"(idesc) : "memory");
        } else {
          if (KIND == 0)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(a2), "l"(b2), "r"(idesc) : "memory");
          else
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(a2), "l"(b2), "r"(idesc) : "memory");
        }
      }
    }
    if (CG == 2)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(s32(&bar)), "h"((unsigned short)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar)), "r"(ph) : "memory");
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  if (CG == 2 && rank == 1 && threadIdx.x == 0) {  // the peer waits for the multicast commit
    asm volatile("{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W2;\n}\n" ::"r"(s32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, int CG, int KIND>
void run(long long* d) {
  const int smem = 4 * 16384 + 4 * N * 128;
  auto k = probe<N, CG, KIND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int iters = 2000;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, d, iters);
  if (!e) e = cudaDeviceSynchronize();
  if (e) { printf("N=%d CG=%d kind=%s: error %s\n", N, CG, KIND ? "f16" : "i8", cudaGetErrorString(e)); return; }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const int steps = KIND == 0 ? 4 : 8;
  const double per_instr = (double)h / iters / steps;
  printf("N=%3d cta_group::%d kind::%s: %6.1f cycles per instruction, %6.1f cycles per 128-row k-block per SM\n",
         N, CG, KIND ? "f16" : "i8", per_instr, per_instr * steps / CG);
}


// kernel-like variant (cta_group::1, kind::f16, N): A from TMEM or smem, a commit per k-block,
// and optionally 8 warps storing 32 KB per k-block-equivalent into other TMEM columns
template <int N>
__global__ void probe_k(long long* out, int iters, int a_tmem, int commit_each, int stores) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ volatile int stop;
  uint8_t* A = sm;
  uint8_t* B = sm + 4 * 16384;
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    stop = 0;
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
  const int warp = threadIdx.x >> 5;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    uint32_t ph0 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
      const int st = it & 3;
      const uint64_t ad = desc_sw128(s32(A + st * 16384));
      const uint64_t bd = desc_none(s32(B + st * N * 128));
      for (int s = 0; s < 8; s++) {
        if (a_tmem)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "r"(tmem + 2 * N + 8 * s), "l"(bd + (uint64_t)((s & 3) * 16)), "r"(idesc) : "memory");
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * N), "l"(ad + (uint64_t)((s & 3) * 2)), "l"(bd + (uint64_t)((s & 3) * 16)), "r"(idesc) : "memory");
      }
      if (commit_each)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar[1])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar[0])) : "memory");
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(s32(&bar[0])), "r"(ph0) : "memory");
    long long t1 = clock64();
    out[0] = t1 - t0;
    stop = 1;
  } else if (stores && warp >= 1 && warp <= 8) {  // 8 warps x 16 lanes x 64 columns, repeated
    const int w = warp - 1;
    const uint32_t taddr = tmem + ((uint32_t)(32 * (w & 3) + 16 * (w >> 2)) << 16) + 2 * N + 64 * 4;
    uint32_t v[32];
    for (int i = 0; i < 32; i++) v[i] = i;
    while (!stop) {
      asm volatile(
          "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
          "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
          "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      __nanosleep(stores > 1 ? 0 : 400);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N>
void run_k(long long* d, int a_tmem, int commit_each, int stores) {
  const int smem = 4 * 16384 + 4 * N * 128;
  cudaFuncSetAttribute(probe_k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_k<N><<<1, 320, smem>>>(d, 2000, a_tmem, commit_each, stores);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("probe_k error %s\n", cudaGetErrorString(e)); return; }
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d f16 A from %s, commit per k-block %d, TMEM store traffic %d: %6.1f cycles per 8-MMA k-block\n",
         N, a_tmem ? "TMEM" : "smem", commit_each, stores, (double)h / 2000);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<64, 1, 0>(d); run<64, 2, 0>(d); run<128, 1, 0>(d); run<128, 2, 0>(d); run<256, 2, 0>(d);
  run<64, 1, 1>(d); run<64, 2, 1>(d); run<128, 1, 1>(d); run<128, 2, 1>(d); run<256, 2, 1>(d);
  for (int at = 0; at < 2; at++)
    for (int ce = 0; ce < 2; ce++)
      for (int stv = 0; stv < 3; stv++) { run_k<64>(d, at, ce, stv); }
  run_k<128>(d, 1, 1, 0); run_k<128>(d, 1, 1, 2);
  return 0;
}
