// Offline packers.
//
// 1. FLXQ-P bit planes (the reference layout, byte-identical with
//    pack(decompose(q), cfg): bitplane.py:55-79, packing.py:132-147,
//    docs/format.md:47-84).  One warp owns one (row, 128-k chunk): lane l holds
//    code k = 32*it + l and one __ballot_sync per plane gathers the 32 bits of
//    word `it` -- the intra-warp bit gather of the paper.
// 2. The inverse (packing.py:150-165 + bitplane.py:87-89).
// 3. The T6 layout of the production unpack-to-INT8 path:
//    offset-binary u = code + 32 (6 bits) packed 4 per 3 bytes per lane, so each
//    lane's three 16-byte loads per k-block are its m16n8k32 A fragments for 4
//    k-steps (byte layout: unpack_t6 in common.cuh).
#include "common.cuh"

namespace flexq {

// ---- 1. FLXQ-P pack -----------------------------------------------------------
__global__ void __launch_bounds__(256) pack_planes_kernel(const int8_t* __restrict__ codes,
                                                          int64_t rows, int64_t cols, int bits,
                                                          int cm, int64_t rc_n, int64_t kc_n,
                                                          uint32_t* __restrict__ words) {
  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t rows_pad = rc_n * cm;
  if (item >= rows_pad * kc_n) return;
  const int64_t kc = item / rows_pad, r = item - kc * rows_pad;
  const int64_t rc = r / cm, rr = r - rc * cm;
  const unsigned mask = (1u << bits) - 1u;
  uint32_t mine = 0;
#pragma unroll
  for (int it = 0; it < 4; it++) {
    const int64_t c = kc * kChunkK + it * 32 + lane;
    unsigned enc = 0;
    if (r < rows && c < cols) enc = (unsigned)(int)codes[r * cols + c] & mask;
    for (int s = 0; s < bits; s++) {
      const uint32_t w = __ballot_sync(0xffffffffu, (enc >> s) & 1u);
      if (lane == s * 4 + it) mine = w;
    }
  }
  if (lane < bits * 4) {
    const int s = lane >> 2, it = lane & 3;
    const int64_t base = (((kc * rc_n + rc) * bits + s) * cm + rr) * 4;  // u32 words
    words[base + it] = mine;
  }
}

// ---- 2. FLXQ-P unpack + recompose ----------------------------------------------
__global__ void unpack_planes_kernel(const uint8_t* __restrict__ words, int64_t rows,
                                     int64_t cols, int bits, int cm, int64_t rc_n,
                                     int8_t* __restrict__ codes) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i - r * cols;
  const int64_t rc = r / cm, rr = r - rc * cm, kc = c / kChunkK, j = c - kc * kChunkK;
  int v = 0;
  for (int s = 0; s < bits; s++) {
    const int64_t off = (((kc * rc_n + rc) * bits + s) * cm + rr) * 16 + (j >> 3);
    const int bit = (words[off] >> (j & 7)) & 1;
    v += (s == bits - 1) ? -(bit << s) : (bit << s);  // signed MSB coefficient (bitplane.py:23-29)
  }
  codes[i] = (int8_t)v;
}

// ---- 3. T6 pack --------------------------------------------------------------------
// thread = (row tile, k-block, lane) -> 12 u32: [v = 0, 1, 2] x 4 k-steps, see unpack_t6
__global__ void pack_t6_kernel(const int8_t* __restrict__ codes, T6Geom G,
                               uint32_t* __restrict__ t6) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G.rt * G.kb * 32) return;
  const int lane = (int)(i & 31);
  const int64_t blk = i >> 5;
  const int64_t rt = blk / G.kb, kb = blk - rt * G.kb;
  const int gq = lane >> 2, t = lane & 3;
  const int64_t span = G.spg * kKStep;
  uint32_t out[3][4];
#pragma unroll
  for (int jj = 0; jj < 4; jj++) {
    uint32_t Wv[3] = {0u, 0u, 0u};
    const int64_t ks = kb * 4 + jj;
#pragma unroll
    for (int reg = 0; reg < 4; reg++) {
      const int64_t row = rt * kRowTile + gq + 8 * (reg & 1);
#pragma unroll
      for (int b = 0; b < 4; b++) {
        const int64_t kp = ks * kKStep + 4 * t + b + 16 * (reg >> 1);
        const int64_t g = kp / span, j = kp - g * span;
        const int64_t kk = g * G.gs + j;
        uint32_t u = 0;  // zero padding: contributes nothing whatever the activation
        if (ks < G.ks && g < G.ng && j < G.gs && kk < G.k && row < G.n)
          u = (uint32_t)((int)codes[row * G.k + kk] + 32);
        if (reg < 3) {
          Wv[reg] |= u << (8 * b);
        } else {  // a3: 2 bits into the top of each of the three words
#pragma unroll
          for (int v = 0; v < 3; v++) Wv[v] |= ((u >> (2 * v)) & 3u) << (8 * b + 6);
        }
      }
    }
    out[0][jj] = Wv[0]; out[1][jj] = Wv[1]; out[2][jj] = Wv[2];
  }
#pragma unroll
  for (int v = 0; v < 3; v++) {
    uint4 val = make_uint4(out[v][0], out[v][1], out[v][2], out[v][3]);
    reinterpret_cast<uint4*>(t6)[G.vec_index(rt, kb, v, lane)] = val;
  }
}

// weight scales for the fast epilogue: pairs {s[16rt+gq], s[16rt+gq+8]} at
// T6Geom::scale_index -> [RG, G, 4, 8, 2]
template <typename T>
__global__ void pack_t6_scales_kernel(const double* __restrict__ scales, T6Geom G,
                                      T* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G.rt * G.ng * 16) return;
  const int h = (int)(i & 1), gq = (int)((i >> 1) & 7);
  const int64_t q = i >> 4;
  const int64_t rt = q / G.ng, g = q - rt * G.ng;
  const int64_t row = rt * kRowTile + gq + 8 * h;
  const double s = row < G.n ? scales[row * G.ng + g] : 0.0;
  const int64_t o = G.scale_index(rt, g, gq) * 2 + h;
  if constexpr (sizeof(T) == 2) {
    out[o] = __double2half(s);
  } else {
    out[o] = (float)s;
  }
}

int pack_planes_launch(const int8_t* codes, int64_t rows, int64_t cols, int bits, int cm,
                       uint8_t* words, cudaStream_t st) {
  const int64_t rc_n = cdiv(rows, cm), kc_n = cdiv(cols, kChunkK);
  const int64_t items = rc_n * cm * kc_n;
  pack_planes_kernel<<<(unsigned)cdiv(items, 8), 256, 0, st>>>(
      codes, rows, cols, bits, cm, rc_n, kc_n, reinterpret_cast<uint32_t*>(words));
  FLEXQ_LAUNCH_CHECK("pack_planes");
  return FLEXQ_OK;
}

int unpack_planes_launch(const uint8_t* words, int64_t rows, int64_t cols, int bits, int cm,
                         int8_t* codes, cudaStream_t st) {
  const int64_t rc_n = cdiv(rows, cm);
  unpack_planes_kernel<<<(unsigned)cdiv(rows * cols, 256), 256, 0, st>>>(words, rows, cols, bits,
                                                                         cm, rc_n, codes);
  FLEXQ_LAUNCH_CHECK("unpack_planes");
  return FLEXQ_OK;
}

int pack_t6_launch(const int8_t* codes, const double* scales, int64_t n, int64_t k, int64_t gs,
                   int scale_f16, uint32_t* t6, void* wscale, cudaStream_t st) {
  T6Geom G(n, k, gs);
  const int64_t threads = G.rt * G.kb * 32;
  pack_t6_kernel<<<(unsigned)cdiv(threads, 256), 256, 0, st>>>(codes, G, t6);
  FLEXQ_LAUNCH_CHECK("pack_t6");
  if (wscale) {
    const int64_t cnt = G.rt * G.ng * 16;
    if (scale_f16)
      pack_t6_scales_kernel<__half><<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(
          scales, G, reinterpret_cast<__half*>(wscale));
    else
      pack_t6_scales_kernel<float><<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(
          scales, G, reinterpret_cast<float*>(wscale));
    FLEXQ_LAUNCH_CHECK("pack_t6_scales");
  }
  return FLEXQ_OK;
}

}  // namespace flexq
