// LLaMA-2 decode harness ops around the W6Ax linears (BASELINE config 5, SURVEY.md
// sec. 8(f) f1).  Not part of the reference's path -- the reference has no model code
// -- but the glue an end-to-end decode step needs between the quantized
// linears: rotary embedding + KV-cache append, and single-query attention over the cache.
// Both read the token positions from device memory so a whole decode step can be captured
// once in a CUDA graph and replayed for every position.
#include "common.cuh"
#include "quant_math.cuh"

namespace flexq {

// qkv: [B, 3*H*D] fp16 (q | k | v); pos: [B] int32 (position of this token);
// k_cache / v_cache: [B, H, Lmax, D] fp16; q_out: [B, H, D] fp16.  Rotate-half RoPE with
// inv_freq_i = theta^(-2i/D), angles in fp32.
__global__ void rope_kv_append_kernel(const __half* __restrict__ qkv, const int* __restrict__ pos,
                                      __half* __restrict__ k_cache, __half* __restrict__ v_cache,
                                      __half* __restrict__ q_out, int H, int D, int Lmax,
                                      float theta) {
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.y, hh = blockIdx.x, i = threadIdx.x;  // i < D/2
  const int half = D / 2;
  const int p = pos[b];
  if (p < 0 || p >= Lmax) return;  // no slot: the cache is full (the host raises first)
  const float inv_freq = powf(theta, -2.f * (float)i / (float)D);
  float sn, cs;
  sincosf((float)p * inv_freq, &sn, &cs);
  const __half* q = qkv + (int64_t)b * 3 * H * D + (int64_t)hh * D;
  const __half* k = q + (int64_t)H * D;
  const __half* v = k + (int64_t)H * D;
  const float q0 = __half2float(q[i]), q1 = __half2float(q[i + half]);
  const float k0 = __half2float(k[i]), k1 = __half2float(k[i + half]);
  __half* qo = q_out + ((int64_t)b * H + hh) * D;
  qo[i] = __float2half_rn(q0 * cs - q1 * sn);
  qo[i + half] = __float2half_rn(q1 * cs + q0 * sn);
  const int64_t slot = (((int64_t)b * H + hh) * Lmax + p) * D;
  k_cache[slot + i] = __float2half_rn(k0 * cs - k1 * sn);
  k_cache[slot + i + half] = __float2half_rn(k1 * cs + k0 * sn);
  v_cache[slot + i] = v[i];
  v_cache[slot + i + half] = v[i + half];
}

// out[b, h*D:(h+1)*D] = softmax(q k^T / sqrt(D)) v over keys [0, pos[b]] of the cache.
// One CTA per (head, token), 8 warps; warp w takes keys w, w+8, ... with an online softmax
// (lane owns 4 of the D=128 dims), then the 8 partial states are merged in smem.
constexpr int kAttnWarps = 8;
__global__ void __launch_bounds__(kAttnWarps * 32) attn_decode_kernel(
    const __half* __restrict__ q, const __half* __restrict__ k_cache,
    const __half* __restrict__ v_cache, const int* __restrict__ pos, __half* __restrict__ out,
    int H, int Lmax, float scale) {
  constexpr int D = 128;
  __shared__ float sm_m[kAttnWarps], sm_l[kAttnWarps];
  __shared__ float sm_acc[kAttnWarps][D];
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.y, hh = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int len = min(pos[b] + 1, Lmax);  // never read past the cache
  const __half* qp = q + ((int64_t)b * H + hh) * D + lane * 4;
  const uint2 qraw = *reinterpret_cast<const uint2*>(qp);
  const float2 qa = __half22float2(*reinterpret_cast<const __half2*>(&qraw.x));
  const float2 qb = __half22float2(*reinterpret_cast<const __half2*>(&qraw.y));
  const __half* kb = k_cache + ((int64_t)b * H + hh) * Lmax * D + lane * 4;
  const __half* vb = v_cache + ((int64_t)b * H + hh) * Lmax * D + lane * 4;
  float m = -INFINITY, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int j = warp; j < len; j += kAttnWarps) {
    const uint2 kr = *reinterpret_cast<const uint2*>(kb + (int64_t)j * D);
    const uint2 vr = *reinterpret_cast<const uint2*>(vb + (int64_t)j * D);
    const float2 ka = __half22float2(*reinterpret_cast<const __half2*>(&kr.x));
    const float2 kk = __half22float2(*reinterpret_cast<const __half2*>(&kr.y));
    float s = qa.x * ka.x + qa.y * ka.y + qb.x * kk.x + qb.y * kk.y;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s *= scale;
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn), pj = __expf(s - mn);
    const float2 va = __half22float2(*reinterpret_cast<const __half2*>(&vr.x));
    const float2 vv = __half22float2(*reinterpret_cast<const __half2*>(&vr.y));
    l = l * corr + pj;
    acc[0] = acc[0] * corr + pj * va.x;
    acc[1] = acc[1] * corr + pj * va.y;
    acc[2] = acc[2] * corr + pj * vv.x;
    acc[3] = acc[3] * corr + pj * vv.y;
    m = mn;
  }
  if (lane == 0) { sm_m[warp] = m; sm_l[warp] = l; }
#pragma unroll
  for (int i = 0; i < 4; i++) sm_acc[warp][lane * 4 + i] = acc[i];
  __syncthreads();
  if (warp == 0) {
    float mt = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; w++) mt = fmaxf(mt, sm_m[w]);
    float lt = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int w = 0; w < kAttnWarps; w++) {
      const float f = sm_m[w] == -INFINITY ? 0.f : __expf(sm_m[w] - mt);
      lt += sm_l[w] * f;
#pragma unroll
      for (int i = 0; i < 4; i++) o[i] += sm_acc[w][lane * 4 + i] * f;
    }
    const float inv = 1.f / lt;
    __half* op = out + (int64_t)b * H * D + (int64_t)hh * D + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; i++) op[i] = __float2half_rn(o[i] * inv);
  }
}

// One kernel per (head, token) for the whole attention block of a decode step: RoPE of q
// and k, KV-cache append, single-query attention, and -- since head_dim == group size
// (128) -- the o_proj activation quantizer of group h of token b, written straight into
// o_proj's operand (codes / fp32 scale / correction, bit-identical to quantize() of the
// fp16 attention output).  Replaces rope_kv_append + attn_decode + quantize.
__global__ void __launch_bounds__(kAttnWarps * 32) attn_block_kernel(
    const __half* __restrict__ qkv, const int* __restrict__ pos, __half* __restrict__ k_cache,
    __half* __restrict__ v_cache, __half* __restrict__ out, int H, int Lmax, float theta,
    float scale, int bits, uint8_t* __restrict__ act_frag, float* __restrict__ act_scale,
    int32_t* __restrict__ act_corr, int64_t m_pad, uint32_t* __restrict__ flag) {
  constexpr int D = 128;
  __shared__ float sm_m[kAttnWarps], sm_l[kAttnWarps];
  __shared__ float sm_acc[kAttnWarps][D];
  __shared__ __half sm_q[D];
  pdl_launch_dependents();
  pdl_wait();
  const int b = blockIdx.y, hh = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = pos[b];
  if (p < 0 || p >= Lmax) {  // KV cache full: flag it, touch nothing
    if (tid == 0) atomicOr(flag, FLEXQ_FLAG_KV_OVERFLOW);
    return;
  }
  const int64_t head_base = ((int64_t)b * H + hh) * Lmax * D;
  if (tid < D / 2) {  // RoPE (rotate-half) + append
    const int i = tid;
    const float inv_freq = powf(theta, -2.f * (float)i / (float)D);
    float sn, cs;
    sincosf((float)p * inv_freq, &sn, &cs);
    const __half* q = qkv + (int64_t)b * 3 * H * D + (int64_t)hh * D;
    const __half* k = q + (int64_t)H * D;
    const __half* v = k + (int64_t)H * D;
    const float q0 = __half2float(q[i]), q1 = __half2float(q[i + D / 2]);
    const float k0 = __half2float(k[i]), k1 = __half2float(k[i + D / 2]);
    sm_q[i] = __float2half_rn(q0 * cs - q1 * sn);
    sm_q[i + D / 2] = __float2half_rn(q1 * cs + q0 * sn);
    const int64_t slot = head_base + (int64_t)p * D;
    k_cache[slot + i] = __float2half_rn(k0 * cs - k1 * sn);
    k_cache[slot + i + D / 2] = __float2half_rn(k1 * cs + k0 * sn);
    v_cache[slot + i] = v[i];
    v_cache[slot + i + D / 2] = v[i + D / 2];
  }
  __syncthreads();  // q in smem, this token's k / v visible to the whole CTA
  const float2 qa = __half22float2(*reinterpret_cast<const __half2*>(&sm_q[lane * 4]));
  const float2 qb = __half22float2(*reinterpret_cast<const __half2*>(&sm_q[lane * 4 + 2]));
  const __half* kb = k_cache + head_base + lane * 4;
  const __half* vb = v_cache + head_base + lane * 4;
  float m = -INFINITY, l = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int j = warp; j <= p; j += kAttnWarps) {
    const uint2 kr = *reinterpret_cast<const uint2*>(kb + (int64_t)j * D);
    const uint2 vr = *reinterpret_cast<const uint2*>(vb + (int64_t)j * D);
    const float2 ka = __half22float2(*reinterpret_cast<const __half2*>(&kr.x));
    const float2 kk = __half22float2(*reinterpret_cast<const __half2*>(&kr.y));
    float s = qa.x * ka.x + qa.y * ka.y + qb.x * kk.x + qb.y * kk.y;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    s *= scale;
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn), pj = __expf(s - mn);
    const float2 va = __half22float2(*reinterpret_cast<const __half2*>(&vr.x));
    const float2 vv = __half22float2(*reinterpret_cast<const __half2*>(&vr.y));
    l = l * corr + pj;
    acc[0] = acc[0] * corr + pj * va.x;
    acc[1] = acc[1] * corr + pj * va.y;
    acc[2] = acc[2] * corr + pj * vv.x;
    acc[3] = acc[3] * corr + pj * vv.y;
    m = mn;
  }
  if (lane == 0) { sm_m[warp] = m; sm_l[warp] = l; }
#pragma unroll
  for (int i = 0; i < 4; i++) sm_acc[warp][lane * 4 + i] = acc[i];
  __syncthreads();
  if (warp != 0) return;
  float mt = -INFINITY;
#pragma unroll
  for (int w = 0; w < kAttnWarps; w++) mt = fmaxf(mt, sm_m[w]);
  float lt = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int w = 0; w < kAttnWarps; w++) {
    const float f = sm_m[w] == -INFINITY ? 0.f : __expf(sm_m[w] - mt);
    lt += sm_l[w] * f;
#pragma unroll
    for (int i = 0; i < 4; i++) o[i] += sm_acc[w][lane * 4 + i] * f;
  }
  const float inv = 1.f / lt;
  __half oh[4];
#pragma unroll
  for (int i = 0; i < 4; i++) oh[i] = __float2half_rn(o[i] * inv);
  if (out) {
    __half* op = out + (int64_t)b * H * D + (int64_t)hh * D + lane * 4;
#pragma unroll
    for (int i = 0; i < 4; i++) op[i] = oh[i];
  }
  // o_proj activation quantizer for (token b, group hh): lane holds columns 4*lane..+3
  float v[4];
  bool finite = true;
  float peak = 0.f;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    v[i] = __half2float(oh[i]);
    finite &= isfinite(v[i]);
    peak = fmaxf(peak, fabsf(v[i]));
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) peak = fmaxf(peak, __shfl_xor_sync(0xffffffffu, peak, s));
  if (!__all_sync(0xffffffffu, finite)) {
    if (lane == 0) atomicOr(flag, FLEXQ_FLAG_NONFINITE);
    peak = 0.f;
  }
  int cd[4];
  const double sc = codes4_fp16(v, peak, bits, 1, lane == 0 ? flag : nullptr, cd);
  int csum = 0;
  uint32_t word = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    csum += cd[i];
    word |= (uint32_t)(cd[i] & 0xff) << (8 * i);
  }
  *reinterpret_cast<uint32_t*>(act_frag + operand_word_offset(hh, b, m_pad, lane)) = word;
#pragma unroll
  for (int s = 16; s; s >>= 1) csum += __shfl_xor_sync(0xffffffffu, csum, s);
  if (lane == 0) {
    act_scale[(int64_t)hh * m_pad + b] = (float)sc;
    act_corr[(int64_t)hh * m_pad + b] = kCorrBias + 32 * csum;
  }
}

int attn_block_launch(const void* qkv, const int* pos, void* k_cache, void* v_cache, void* out,
                      int64_t batch, int heads, int head_dim, int64_t lmax, float theta, int bits,
                      int64_t group_size, uint32_t* act_frag, float* act_scale, int32_t* act_corr,
                      int64_t m_pad, uint32_t* flag, cudaStream_t st) {
  if (group_size != head_dim) {
    set_error("attn_block: the fused o_proj quantizer needs group_size == head_dim (%d), got %lld",
              head_dim, (long long)group_size);
    return FLEXQ_ERR_CONFIG;
  }
  if (head_dim != 128 || batch < 1 || heads < 1 || lmax < 1 || bits < 2 || bits > 8 ||
      !act_frag || !act_scale || !act_corr || !flag || m_pad < batch || m_pad % 8) {
    set_error("attn_block: needs head_dim 128 (= the quantizer group) and an operand buffer");
    return FLEXQ_ERR_SHAPE;
  }
  cudaError_t e = launch_pdl(attn_block_kernel, dim3((unsigned)heads, (unsigned)batch),
                             dim3(kAttnWarps * 32), 0, st, reinterpret_cast<const __half*>(qkv),
                             pos, reinterpret_cast<__half*>(k_cache),
                             reinterpret_cast<__half*>(v_cache), reinterpret_cast<__half*>(out),
                             heads, (int)lmax, theta, 1.f / sqrtf((float)head_dim), bits,
                             reinterpret_cast<uint8_t*>(act_frag), act_scale, act_corr, m_pad,
                             flag);
  if (e != cudaSuccess) return cuda_status(e, "attn_block launch");
  return FLEXQ_OK;
}

int rope_kv_append_launch(const void* qkv, const int* pos, void* k_cache, void* v_cache,
                          void* q_out, int64_t batch, int heads, int head_dim, int64_t lmax,
                          float theta, cudaStream_t st) {
  if (batch < 1 || heads < 1 || head_dim < 2 || head_dim % 2 || head_dim > 1024 || lmax < 1) {
    set_error("rope_kv_append: bad geometry");
    return FLEXQ_ERR_SHAPE;
  }
  cudaError_t e = launch_pdl(rope_kv_append_kernel, dim3((unsigned)heads, (unsigned)batch),
                             dim3((unsigned)(head_dim / 2)), 0, st,
                             reinterpret_cast<const __half*>(qkv), pos,
                             reinterpret_cast<__half*>(k_cache), reinterpret_cast<__half*>(v_cache),
                             reinterpret_cast<__half*>(q_out), heads, head_dim, (int)lmax, theta);
  if (e != cudaSuccess) return cuda_status(e, "rope_kv_append launch");
  return FLEXQ_OK;
}

int attn_decode_launch(const void* q, const void* k_cache, const void* v_cache, const int* pos,
                       void* out, int64_t batch, int heads, int head_dim, int64_t lmax,
                       cudaStream_t st) {
  if (head_dim != 128 || batch < 1 || heads < 1 || lmax < 1) {
    set_error("attn_decode: head_dim must be 128 (got %d)", head_dim);
    return FLEXQ_ERR_SHAPE;
  }
  cudaError_t e = launch_pdl(attn_decode_kernel, dim3((unsigned)heads, (unsigned)batch),
                             dim3(kAttnWarps * 32), 0, st, reinterpret_cast<const __half*>(q),
                             reinterpret_cast<const __half*>(k_cache),
                             reinterpret_cast<const __half*>(v_cache), pos,
                             reinterpret_cast<__half*>(out), heads, (int)lmax,
                             1.f / sqrtf((float)head_dim));
  if (e != cudaSuccess) return cuda_status(e, "attn_decode launch");
  return FLEXQ_OK;
}

}  // namespace flexq
