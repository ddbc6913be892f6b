// tcgen05.mma kind::i8 issue/throughput probe (B200): one CTA issues `iters` k-blocks of
// 4 x (M=128, N, K=32) MMAs from shared memory, with and without per-k-block commits,
// and reports cycles per k-block and the implied TOPS per SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_none(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@!P1 bra W;\n}\n" ::"r"(s32(bar)), "r"(ph), "r"(0x989680) : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 1, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(idesc) : "memory");
}

template <int N>
__global__ void probe(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[4], bar3[2], done[2];
  uint8_t* A = sm;             // 4 stages x 16 KB
  uint8_t* B = sm + 4 * 16384; // 4 stages x N*128
  for (int i = threadIdx.x; i < (4 * 16384 + 4 * N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&holder)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    for (int i = 0; i < 4; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 100000;" ::"r"(s32(&bar2[i])));
    for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 100000;" ::"r"(s32(&bar3[i])));
    for (int i = 0; i < 2; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&done[i])));
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(&done[i])));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = holder;
  const uint32_t idesc = (mode & 128)
      ? (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24)   // bf16 x bf16 -> f32
      : (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);  // u8 x s8 -> s32
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; it++) {
      const int st = it & 3;
      const uint64_t ad = (mode & 1) ? desc_sw128(s32(A + st * 16384)) : desc_none(s32(A + st * 16384));
      const uint64_t bd = desc_none(s32(B + st * N * 128));
      if (mode & 128) {  // kind::f16 (bf16): K=16 per instruction = 32 B, same byte steps as i8
        const int nk = (mode & 256) ? 4 : 8;  // 4: half a 128-k block (same bytes as 4 x i8)
        for (int s = 0; s < nk; s++) mma_f16(tmem + (it & 1) * N, ad + (s & 3) * 2, bd + (s & 3) * 16, idesc);
      } else if (mode & 96) {  // interleave C independent accumulator chains (k-blocks to distinct D)
        const int C = (mode & 32) ? 2 : 4;
        for (int s = 0; s < 4; s++)
          for (int j = 0; j < C; j++)
            mma(tmem + j * N, desc_sw128(s32(A + ((it + j) & 3) * 16384)) + s * 2,
                desc_none(s32(B + ((it + j) & 3) * N * 128)) + s * 16, idesc);
        it += C - 1;
      } else if (mode & 16) {
        for (int s = 0; s < 4; s++)  // A from TMEM: columns 256 + 32*stage + 8*s
          mma_ts(tmem + (it & 1) * N, tmem + 256 + st * 32 + s * 8, bd + s * 16, idesc);
      } else {
        for (int s = 0; s < 4; s++)
          mma(tmem + (it & 1) * N, ad + ((mode & 1) ? s * 2 : s * 16), bd + s * 16, idesc);
      }
      if (mode & 2) { commit(&bar); wait(&bar, ph); ph ^= 1; }
      if (mode & 8) commit(&bar2[it & 3]);  // commit only (async arrive), no wait
      if (mode & 4) {  // kernel-shaped sync per k-block (barriers pre-completed by a helper)
        commit(&bar2[it & 3]);
        commit(&bar3[it & 1]);
        wait(&done[0], 0);
        wait(&done[1], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
    }
    commit(&bar); wait(&bar, ph);
    long long t1 = clock64();
    out[0] = (t1 - t0);
  }
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N>
void run(long long* d) {
  const int smem = 4 * 16384 + 4 * N * 128;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* mn[] = {"A none ", "A sw128", "A none +commit/wait each", "A sw128+commit/wait each",
                      "", "A sw128 + kernel-shaped sync", "", "", "", "A sw128 + commit only", "", "", "", "", "", "",
                      "A TMEM", "", "", "", "A TMEM + kernel-shaped sync", "", "", "", "A TMEM + commit only", "", "", "", "", "", "", "", "", "2 chains", "", "", "", "", "", "", "", "", "", "", "", "", "", "", "",
                      "", "", "", "", "", "", "", "", "", "", "", "", "", "", "", "", "4 chains", "", "", "", "4 chains + sync"};
  auto name = [&](int mode) -> const char* {
    if (mode == 129) return "bf16 kind::f16, 8 x K=16";
    if (mode == 133) return "bf16 kind::f16 8x + sync";
    if (mode == 385) return "bf16 kind::f16, 4 x K=16";
    return mn[mode];
  };
  for (int mode : {1, 5, 16, 33, 65, 65 + 4, 129, 129 + 4, 129 + 256}) {
    if (N > 128 && (mode & 16)) continue;
    if (N > 128 && (mode & 64)) continue;
    const int iters = 2000;
    probe<N><<<1, 128, smem>>>(d, iters, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return; }
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    double cyc = (double)h / iters;
    double ops = 2.0 * 128 * N * (mode == 385 ? 64 : 128);
    printf("N=%3d %-30s %7.1f cycles/k-block  %6.0f ops/clk/SM (peak ~15500)\n", N, name(mode), cyc, ops / cyc);
  }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  run<32>(d); run<64>(d); run<128>(d); run<256>(d);
  return 0;
}
