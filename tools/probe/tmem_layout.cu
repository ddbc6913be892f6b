// Which (TMEM lane, column) does register r of thread t land in for tcgen05.st.16x256b.x1?
// One warp stores value (t << 8 | r) and reads lanes 0-31 back with 32x32b.x8.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(unsigned* out) {
  __shared__ uint32_t holder;
  const int lane = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&holder)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = holder;
  uint32_t z = 0xFFFFFFFFu;
  // clear 32 lanes x 8 columns
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(t), "r"(z));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t r0 = (lane << 8) | 0, r1 = (lane << 8) | 1, r2 = (lane << 8) | 2, r3 = (lane << 8) | 3;
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1,%2,%3,%4};" ::"r"(t), "r"(r0), "r"(r1), "r"(r2), "r"(r3));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t v[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < 8; c++) out[lane * 8 + c] = v[c];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  unsigned* d; cudaMalloc(&d, 32 * 8 * 4);
  probe<<<1, 32>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  unsigned h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("lane: column 0..7 = (thread, reg)\n");
  for (int l = 0; l < 16; l++) {
    printf("lane %2d:", l);
    for (int c = 0; c < 8; c++) {
      if (h[l * 8 + c] == 0xFFFFFFFFu) printf("   --  ");
      else printf(" t%02u.r%u", h[l * 8 + c] >> 8, h[l * 8 + c] & 0xff);
    }
    printf("\n");
  }
  return 0;
}
