// BTC-equivalent bit-serial GEMM: AND + popcount over FLXQ-P bit planes.
//
// Restates the reference engine's fused loop (engine.py:251-334) on CUDA
// cores: for every scale group, k-chunk span and plane pair (s, t),
// popcount(w_s & x_t) over the 128-bit chunk row (engine.py:89-95, 196-208),
// weighted by coeff(s)*coeff(t) with the signed MSB (engine.py:114-130,
// bitplane.py:23-29), summed exactly, then the fused dequant
// (engine.py:211-216).  Group spans that do not cover a whole chunk are masked
// (engine.py:165-193); the last group runs through the zero padding.
//
// This is the paper's binary-tensor-core formulation.  sm_100a has no BMMA
// (mma .b1 is emulated with IMMA + MOVM) and POPC issues at 16/clk/SM
// (measured), so this path is compute-bound at p*q/32 POPC per weight per
// token; it is kept for the drop-in group_matmul_fused over FLXQ-P operands
// and as the measured baseline the T6 tensor-core path replaced.
//
// Thread = one weight row; CTA = 128 rows x one K range x one activation chunk.
#include "common.cuh"

namespace flexq {

struct BsParams {
  const uint4* __restrict__ w;   // FLXQ-P weight words, 16 B per (kc, rc, s, r)
  const uint4* __restrict__ x;   // FLXQ-P activation words
  const float* __restrict__ ws;  // [n, G]
  const float* __restrict__ xs;  // [m, G]
  int64_t m, n, k, gs, ng, kc_n, rcw, rcx, m_pad, n_pad;
  int cm, wcm, pb, qb;  // activation / weight chunk_m, plane counts
  int32_t* partials;
  void* y;
  int out_dtype;
  float* ws_part;
  unsigned* counters;
  int ksplit;
};

__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) {
  return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w);
}
__device__ __forceinline__ int popc_and(const uint4& a, const uint4& b) {
  return __popc(a.x & b.x) + __popc(a.y & b.y) + __popc(a.z & b.z) + __popc(a.w & b.w);
}

template <int PB, int QB>
__global__ void __launch_bounds__(128) bitserial_kernel(BsParams p) {
  const int pb = PB ? PB : p.pb, qb = QB ? QB : p.qb;
  const int64_t row = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int64_t split = blockIdx.y, xc = blockIdx.z;
  const int64_t kc0 = split * p.kc_n / p.ksplit, kc1 = (split + 1) * p.kc_n / p.ksplit;
  const int64_t rc = row / p.wcm, rr = row - rc * p.wcm;
  const bool row_ok = row < p.rcw * p.wcm;
  const int cm = p.cm;
  const int64_t k_pad = p.kc_n * kChunkK;

  int P[8];
  float acc[8];
#pragma unroll
  for (int r = 0; r < 8; r++) { P[r] = 0; acc[r] = 0.f; }
  int64_t cur = -1;

  auto drain = [&](int64_t g) {
#pragma unroll
    for (int r = 0; r < 8; r++) {
      if (r >= cm) break;
      const int64_t tok = xc * cm + r;
      if (tok >= p.m || row >= p.n) continue;
      if (p.partials) atomicAdd(&p.partials[(g * p.m + tok) * p.n + row], P[r]);
      if (p.y) acc[r] = fmaf(p.ws[row * p.ng + g] * p.xs[tok * p.ng + g], (float)P[r], acc[r]);
    }
  };

  for (int64_t kc = kc0; kc < kc1; kc++) {
    uint4 wv[8];
    const uint4* wb = p.w + ((kc * p.rcw + rc) * pb) * p.wcm + rr;
#pragma unroll
    for (int s = 0; s < 8; s++) {
      if (s >= pb) break;
      wv[s] = row_ok ? __ldcs(wb + s * p.wcm) : make_uint4(0, 0, 0, 0);
    }
    const uint4* xb = p.x + ((kc * p.rcx + xc) * qb) * cm;
    const int64_t base = kc * kChunkK;
    int64_t g = base / p.gs;
    for (; g < p.ng; g++) {
      const int64_t glo = g * p.gs;
      if (glo >= base + kChunkK) break;
      const int64_t ghi = (g == p.ng - 1) ? k_pad : glo + p.gs;
      const int lo = (int)(glo > base ? glo - base : 0);
      const int hi = (int)(ghi < base + kChunkK ? ghi - base : kChunkK);
      if (g != cur) {
        if (cur >= 0) drain(cur);
        cur = g;
#pragma unroll
        for (int r = 0; r < 8; r++) P[r] = 0;
      }
      uint4 msk = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
      if (lo != 0 || hi != kChunkK) {
        uint32_t mm[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int a = max(lo, 32 * q), b = min(hi, 32 * q + 32);
          mm[q] = a < b ? (((b - a) == 32 ? 0xffffffffu : ((1u << (b - a)) - 1u)) << (a - 32 * q)) : 0u;
        }
        msk = make_uint4(mm[0], mm[1], mm[2], mm[3]);
      }
      uint4 wm[8];
#pragma unroll
      for (int s = 0; s < 8; s++) {
        if (s >= pb) break;
        wm[s] = and4(wv[s], msk);
      }
#pragma unroll
      for (int r = 0; r < 8; r++) {
        if (r >= cm) break;
        int tot = 0;
#pragma unroll
        for (int t = 0; t < 8; t++) {
          if (t >= qb) break;
          const uint4 xv = __ldg(xb + t * cm + r);
          int sum_s = 0;
#pragma unroll
          for (int s = 0; s < 8; s++) {
            if (s >= pb) break;
            const int c = popc_and(wm[s], xv);
            sum_s += (s == pb - 1) ? -(c << s) : (c << s);
          }
          tot += (t == qb - 1) ? -(sum_s << t) : (sum_s << t);
        }
        P[r] += tot;
      }
    }
  }
  if (cur >= 0) drain(cur);
  if (!p.y) return;

  const int64_t tile = (int64_t)blockIdx.z * gridDim.x + blockIdx.x;
  if (p.ksplit > 1) {
    for (int r = 0; r < cm; r++) p.ws_part[(split * p.m_pad + xc * cm + r) * p.n_pad + row] = acc[r];
    __threadfence();
    __syncthreads();
    __shared__ unsigned prev;
    if (threadIdx.x == 0) prev = atomicAdd(&p.counters[tile], 1u);
    __syncthreads();
    if (prev != (unsigned)p.ksplit - 1) return;
    __threadfence();
    for (int r = 0; r < cm; r++) {
      float s = 0.f;
      for (int sp = 0; sp < p.ksplit; sp++) s += __ldcg(&p.ws_part[(sp * p.m_pad + xc * cm + r) * p.n_pad + row]);
      acc[r] = s;
    }
    if (threadIdx.x == 0) p.counters[tile] = 0u;
  }
  if (row >= p.n) return;
  for (int r = 0; r < cm; r++) {
    const int64_t tok = xc * cm + r;
    if (tok >= p.m) break;
    if (p.out_dtype == FLEXQ_OUT_F16)
      reinterpret_cast<__half*>(p.y)[tok * p.n + row] = __float2half_rn(acc[r]);
    else
      reinterpret_cast<float*>(p.y)[tok * p.n + row] = acc[r];
  }
}

static int auto_ksplit_bs(int64_t blocks, int64_t kc_n) {
  int64_t want = cdiv(148 * 8, blocks);
  if (want > kc_n) want = kc_n;
  if (want > 64) want = 64;
  return (int)(want < 1 ? 1 : want);
}

int64_t gemm_bitserial_workspace(int64_t m, int64_t n, int64_t k, int ksplit) {
  // bound over every activation chunk_m in 1..8: token chunks rcx <= m, padded tokens <= m + 7
  const int64_t nb = cdiv(n, 128), kc_n = cdiv(k, kChunkK), m_pad = m + 8;
  if (ksplit <= 0) ksplit = auto_ksplit_bs(nb, kc_n);  // the largest auto split (rcx = 1)
  return cdiv((int64_t)ksplit * m_pad * nb * 128 * 4, 256) * 256 + cdiv(nb * m * 4, 256) * 256;
}

int gemm_bitserial_launch(const uint8_t* wwords, const uint8_t* xwords, const float* wscale,
                          const float* xscale, int64_t m, int64_t n, int64_t k, int wbits,
                          int xbits, int64_t gs, int wcm, int xcm, int32_t* partials, void* y,
                          int out_dtype, void* workspace, int ksplit, cudaStream_t st) {
  if (wcm < 1 || wcm > 8 || xcm < 1 || xcm > 8) {
    set_error("gemm_bitserial: chunk_m must be in 1..8, got weights %d activations %d", wcm, xcm);
    return FLEXQ_ERR_CONFIG;
  }
  if (m < 1 || n < 1 || k < 1 || gs < 1) {
    set_error("gemm_bitserial: dims must be positive, got m=%lld n=%lld k=%lld group=%lld",
              (long long)m, (long long)n, (long long)k, (long long)gs);
    return FLEXQ_ERR_CONFIG;
  }
  if (wbits < 2 || wbits > 8 || xbits < 2 || xbits > 8) {
    set_error("gemm_bitserial: bits must be in 2..8, got (%d, %d)", wbits, xbits);
    return FLEXQ_ERR_CONFIG;
  }
  if (!y && !partials) {
    set_error("gemm_bitserial: nothing to compute (y and partials are both NULL)");
    return FLEXQ_ERR_CONFIG;
  }
  BsParams p;
  p.w = reinterpret_cast<const uint4*>(wwords);
  p.x = reinterpret_cast<const uint4*>(xwords);
  p.ws = wscale;
  p.xs = xscale;
  p.m = m; p.n = n; p.k = k; p.gs = gs;
  p.ng = cdiv(k, gs);
  p.kc_n = cdiv(k, kChunkK);
  p.wcm = wcm;
  p.rcw = cdiv(n, wcm);
  p.cm = xcm;
  p.rcx = cdiv(m, p.cm);
  p.pb = wbits; p.qb = xbits;
  const int64_t nb = cdiv(n, 128);
  if (ksplit <= 0) ksplit = auto_ksplit_bs(nb * p.rcx, p.kc_n);
  if (ksplit > p.kc_n) ksplit = (int)p.kc_n;
  p.ksplit = ksplit;
  p.m_pad = p.rcx * p.cm;
  p.n_pad = nb * 128;
  p.partials = partials;
  p.y = y;
  p.out_dtype = out_dtype;
  p.ws_part = reinterpret_cast<float*>(workspace);
  p.counters = workspace ? reinterpret_cast<unsigned*>(
                               reinterpret_cast<char*>(workspace) +
                               cdiv((int64_t)ksplit * p.m_pad * p.n_pad * 4, 256) * 256)
                         : nullptr;
  if (y && ksplit > 1 && !workspace) {
    set_error("gemm_bitserial: workspace required for ksplit=%d", ksplit);
    return FLEXQ_ERR_CONFIG;
  }
  dim3 grid((unsigned)nb, (unsigned)ksplit, (unsigned)p.rcx);
  if (wbits == 6 && xbits == 6) bitserial_kernel<6, 6><<<grid, 128, 0, st>>>(p);
  else if (wbits == 6 && xbits == 8) bitserial_kernel<6, 8><<<grid, 128, 0, st>>>(p);
  else bitserial_kernel<0, 0><<<grid, 128, 0, st>>>(p);
  FLEXQ_LAUNCH_CHECK("gemm_bitserial");
  return FLEXQ_OK;
}

}  // namespace flexq
