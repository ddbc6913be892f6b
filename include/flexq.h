/*
 * flexq.h -- C ABI of the B200 (sm_100a) W6A6/W6A8 quantized-linear library
 * (libflexq_sm100a.so).  Plain pointers, sizes and a cudaStream_t; no torch
 * types.  All pointers are DEVICE pointers unless stated; nothing here
 * allocates memory on the hot path (workspaces are caller-owned).
 *
 * The reference (FlexQ restatement, package `bitserial`) is pure Python; its
 * FFI for this path would bind one C entry per public Python function.  Each
 * entry below names the reference interface it replaces
 * (paths under /root/reference/pkg/src/bitserial/).  INTEGRATION.md shows the
 * ctypes stub a maintainer would add.
 *
 * Errors: every entry returns an int status (0 = ok, negative = error) and
 * records a message retrievable with flexq_last_error() (thread-local).  The
 * codes map 1:1 to the reference's exception classes (errors.py:8-28).
 * Data-dependent errors (non-finite input, a scale that rounds to zero) are
 * detected on the device and OR-ed into a caller-provided int32 flag word.
 */
#ifndef FLEXQ_H_
#define FLEXQ_H_

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-28) ---------------------------------------- */
#define FLEXQ_OK 0
#define FLEXQ_ERR_INVALID_INPUT (-1) /* InvalidInputError  (errors.py:8)  */
#define FLEXQ_ERR_SHAPE (-2)         /* ShapeError         (errors.py:12) */
#define FLEXQ_ERR_CONFIG (-3)        /* ConfigError        (errors.py:16) */
#define FLEXQ_ERR_FORMAT (-4)        /* FormatError        (errors.py:24) */
#define FLEXQ_ERR_CUDA (-5)          /* CUDA runtime / launch failure      */

/* device flag bits written by the quantizers */
#define FLEXQ_FLAG_NONFINITE 1u      /* quantize.py:135-136 "input contains non-finite values" */
#define FLEXQ_FLAG_NONPOS_SCALE 2u   /* quantize.py:71-72   "all scales must be strictly positive" */
#define FLEXQ_FLAG_KV_OVERFLOW 4u    /* decode harness: a position at or past the KV-cache length */

/* float input dtypes */
#define FLEXQ_DT_F16 0
#define FLEXQ_DT_BF16 1
#define FLEXQ_DT_F32 2
#define FLEXQ_DT_F64 3

/* output dtypes for the fast epilogue */
#define FLEXQ_OUT_F16 0
#define FLEXQ_OUT_F32 1

const char* flexq_last_error(void);
/* The FLEXQ_* debug / A-B environment knobs in effect ("defaults" when none is set); they
 * are read once, at the library's first use, never per launch. */
const char* flexq_tuning(void);
int flexq_version(void);                  /* MAJOR*10000 + MINOR*100 + PATCH */
int flexq_device_check(void);             /* 0 if an sm_100 device is current, else FLEXQ_ERR_CUDA */

/* ---- quantizer ------------------------------------------------------------
 * Replaces quantize(data, bits, group_size, fp16_scales)  (quantize.py:118-148).
 * x: [rows, cols] row-major, dtype `dtype`.  codes: int8 [rows, cols] or NULL.
 * scales: float64 [rows, G] or NULL, G = ceil(cols / group_size).
 * Bit-exact with the reference: float64 divide, half-away rounding, fp16
 * scale rounding directly from float64.  Optional fused outputs for the i8
 * GEMM path (NULL to skip): act_frag (T6 activation fragment layout, see
 * DESIGN.md sec. 3), act_scale_f32 [G, m_pad], act_corr [G, m_pad] (= 32 * sum of
 * codes per group, the offset-binary weight correction).  `m_pad` is the token
 * stride of those arrays (multiple of 8 >= rows). */
int flexq_quantize(const void* x, int dtype, int64_t rows, int64_t cols, int bits,
                   int64_t group_size, int fp16_scales, int8_t* codes, double* scales,
                   uint32_t* act_frag, float* act_scale_f32, int32_t* act_corr, int64_t m_pad,
                   uint32_t* flag, cudaStream_t stream);

/* ---- bit-plane packer (FLXQ-P, byte-identical with the reference) ---------
 * Replaces pack(decompose(q), PackConfig(chunk_m, word_bits))  (bitplane.py:55-84,
 * packing.py:132-147, docs/format.md:47-84).  codes int8 [rows, cols] ->
 * words [KC, RC, bits, chunk_m, 16 bytes] (little-endian, LSB-first). */
int64_t flexq_planes_bytes(int64_t rows, int64_t cols, int bits, int chunk_m);
int flexq_pack_planes(const int8_t* codes, int64_t rows, int64_t cols, int bits, int chunk_m,
                      uint8_t* words, cudaStream_t stream);
/* Replaces recompose(unpack(p, cfg))  (packing.py:150-165, bitplane.py:87-89). */
int flexq_unpack_planes(const uint8_t* words, int64_t rows, int64_t cols, int bits, int chunk_m,
                        int8_t* codes, cudaStream_t stream);

/* ---- T6 weight layout for the unpack-to-INT8 tensor-core path -------------
 * The offline packer of the production path (weight_pack_config analogue,
 * packing.py:74-76): 6-bit codes in offset binary (u = code + 32) split into
 * the low-nibble planes {0..3} and the high planes {4,5}, laid out so every
 * lane's 16-byte loads are its mma A-fragments.  Requires |code| <= 31 (bits<=6).
 * weights: int8 [n, k];  scales float64 [n, G].  t6: u32 [RT, KB, 3, 32, 4];
 * wscale: [RT, G, 8, 2] in fp16 (scale_f16=1, exact only in fp16-scale mode)
 * or fp32. */
int64_t flexq_t6_bytes(int64_t n, int64_t k, int64_t group_size);
int flexq_pack_t6(const int8_t* codes, const double* scales, int64_t n, int64_t k,
                  int64_t group_size, int scale_f16, uint32_t* t6, void* wscale,
                  cudaStream_t stream);
int64_t flexq_act_frag_bytes(int64_t m_pad, int64_t k, int64_t group_size);
/* Token padding of the activation operand for m tokens: a multiple of 8 for the
 * decode GEMV (m <= 16), a whole number of tcgen05 token tiles (32 / 64 / 128)
 * above.  Layout of the operand: [k-block][m_pad/8][8 k-cores]
 * [8 tokens][16 B], the K-major no-swizzle UMMA canonical form, read both as
 * mma.m16n8k32 B fragments and as tcgen05.mma B tiles. */
int64_t flexq_act_m_pad(int64_t m);
/* Already-quantized activations (a QuantTensor: int8 codes [m, k] + float64
 * scales [m, G]) -> the T6 activation operand, for int_matmul_reference-style
 * calls (engine.py:337-365) that skip the float quantizer. */
int flexq_pack_act_t6(const int8_t* codes, const double* scales, int64_t m, int64_t m_pad,
                      int64_t k, int64_t group_size, uint32_t* act_frag, float* act_scale_f32,
                      int32_t* act_corr, cudaStream_t stream);
/* Replaces bmma_chunk (engine.py:89-95): *out = sum popcount(a[i] & b[i]) over
 * nbytes bytes (device int64 result). */
int flexq_popcount_and(const uint8_t* a, const uint8_t* b, int64_t nbytes, int64_t* out,
                       cudaStream_t stream);

/* ---- GEMM cores ------------------------------------------------------------
 * Both produce, per (token m, row n, group g), the exact integer partial
 * P[g,m,n] = sum_{k in g} x[m,k]*w[n,k] and then either
 *   trace:  P written as int32 [G, m, n]   (engine.py:211-216 trace_slot;
 *           caller zeroes it: partial groups are combined with integer atomics)
 *   fast:   y[m,n] = sum_g (xs*ws) * P in fp32, stored fp16/fp32 [m, n].
 * `partials` / `y` may be NULL to skip either.  workspace: see
 * flexq_gemm_workspace_bytes (fp32 split-K partials + per-tile counters; the
 * counters must be zero before the first call and are left zeroed). */
int64_t flexq_gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t group_size,
                                   int ksplit /* 0 = auto */);

/* Production path: unpack-to-INT8 + tensor cores over T6 weights.
 * Replaces int_matmul_reference / group_matmul_fused numerics (engine.py:290-365).
 * act_* are the fused outputs of flexq_quantize (same m_pad).
 * ksplit: 0 = automatic kernel choice (streaming GEMV for M <= 32 with one group per
 * 128-k block, M <= 16 otherwise; tcgen05 above), > 0 = the mma.sync kernel with that
 * k-split, -1 = the mma.sync kernel (automatic split; GEMV for M <= 16), -2 = the tcgen05
 * kernel whenever it supports the shape (M > 16), -3 = the streaming GEMV whenever it
 * supports the shape (M <= 32). */
int flexq_gemm_t6(const uint32_t* t6, const void* wscale, int scale_f16,
                  const uint32_t* act_frag, const float* act_scale, const int32_t* act_corr,
                  int64_t m, int64_t m_pad, int64_t n, int64_t k, int64_t group_size,
                  int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                  cudaStream_t stream);

/* Same, with an optional fused residual (y and residual of out_dtype, [m, n]; residual
 * may alias y): y = acc + residual, one rounding.  Used by the decode step to fold the
 * transformer's residual add into the linear's epilogue. */
int flexq_gemm_t6_ex(const uint32_t* t6, const void* wscale, int scale_f16,
                     const uint32_t* act_frag, const float* act_scale, const int32_t* act_corr,
                     int64_t m, int64_t m_pad, int64_t n, int64_t k, int64_t group_size,
                     int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                     const void* residual, cudaStream_t stream);

/* BTC-equivalent bit-serial path: AND + popcount over FLXQ-P planes.
 * Replaces group_matmul_fused(wp, xp, ...)  (engine.py:290-334): wwords /
 * xwords from flexq_pack_planes with their chunk_m (reference defaults: 8 for
 * weights, min(m, 8) for activations, packing.py:69-76); scales fp32
 * row-major [n, G] / [m, G] (fast epilogue only). */
int flexq_gemm_bitserial(const uint8_t* wwords, const uint8_t* xwords, const float* wscale,
                         const float* xscale, int64_t m, int64_t n, int64_t k, int wbits,
                         int xbits, int64_t group_size, int w_chunk_m, int x_chunk_m,
                         int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                         cudaStream_t stream);

/* Exact float64 epilogue over traced partials: y[m,n] = sum_g (xs*ws)*P in
 * ascending g with separate IEEE multiply/add -- bit-identical with the
 * reference's _scale_accumulate (engine.py:211-216).  y16 (fp16, correctly
 * rounded from the float64 result) may be NULL. */
int flexq_group_epilogue_f64(const int32_t* partials, const double* wscale,
                             const double* xscale, int64_t m, int64_t n, int64_t groups,
                             double* y, uint16_t* y16, cudaStream_t stream);

/* ---- batched fast path with the scales folded into fp16 operands ---------
 * For 32 < M <= 128 at group 128 with fp16 weight scales, flexq_linear_forward(_ex) runs
 * tcgen05.mma.kind::f16 over A = fp16(w * ws) (converted on chip from the T6 stream) and
 * B = fp16(x_code * xs) (written by the activation quantizer), accumulating each tile's whole
 * K range in fp32 TMEM (csrc/gemm_tc16.cu).  Same codes and scales as the
 * reference (quantize.py:118-148); fp16 y within the fast path's tolerance; no INT32 partials
 * (flexq_gemm_t6 with `partials` gives those).  act_f16: the fp16 operand inside an act buffer
 * (flexq_act_f16_operand); workspace: flexq_gemm_workspace_bytes(m, n, k, 128, 0). */
#define FLEXQ_KERNEL_GEMV 0      /* streaming GEMV (mma.sync), decode batches */
#define FLEXQ_KERNEL_TC_I8 1     /* tcgen05 kind::i8, exact INT32 group partials */
#define FLEXQ_KERNEL_TC16 2      /* tcgen05 kind::f16, scales folded into the operands */
#define FLEXQ_KERNEL_MMA_SYNC 3  /* mma.sync (group sizes not aligned to 128 k) */
/* The GEMM kernel flexq_linear_forward uses for this shape (the FLEXQ_KERNEL_* codes). */
int flexq_linear_kernel(int64_t m, int64_t n, int64_t k, int64_t group_size, int scale_f16);
/* Process-wide override of the kind::f16 route for 32 < M <= 256 (A/B runs and tests that cover
 * the kernel on small shapes): -1 = automatic (measured size rule, the default), 0 = never,
 * 1 = whenever gemm_tc16 supports the shape.  Returns the previous mode, or -2 (and sets the
 * error string) for an invalid mode.  No reference counterpart: routing is internal to this
 * library (the reference has one CPU path, engine.py:290). */
int flexq_set_tc16_route(int mode);
int flexq_gemm_tc16(const uint32_t* t6, const void* wscale, const void* act_f16, int64_t m,
                    int64_t n, int64_t k, void* y, int out_dtype, void* workspace,
                    const void* residual, cudaStream_t stream);
/* Address of the fp16 operand inside an act buffer of flexq_act_buf_bytes(m, k, group_size). */
void* flexq_act_f16_operand(void* act_buf, int64_t m, int64_t k, int64_t group_size);

/* ---- one-call online linear (quantized_linear with pre-packed weights) ----
 * Replaces the online half of quantized_linear (engine.py:487-513):
 * quantize activations (fp16 [m, k]) -> T6 GEMM -> fp16 y [m, n].
 * act_buf must hold flexq_act_buf_bytes(); workspace flexq_gemm_workspace_bytes(). */
int64_t flexq_act_buf_bytes(int64_t m, int64_t k, int64_t group_size);  /* m_pad = flexq_act_m_pad(m) */
int flexq_linear_forward(const uint32_t* t6, const void* wscale, int scale_f16, int xbits,
                         const void* x, int64_t m, int64_t n, int64_t k, int64_t group_size,
                         uint16_t* y, void* act_buf, void* workspace, uint32_t* flag,
                         cudaStream_t stream);
/* Same with the output dtype chosen (FLEXQ_OUT_F16 / FLEXQ_OUT_F32 y [m, n]) and an optional
 * fused residual of that dtype [m, n] (may alias y): y = x W^T + residual.  FLEXQ_OUT_F32 is
 * what a row (K) shard emits: its fp32 partial y is summed across ranks before any rounding
 * (the reference's group partials combine in the float epilogue,
 * engine.py:277-286). */
int flexq_linear_forward_ex(const uint32_t* t6, const void* wscale, int scale_f16, int xbits,
                            const void* x, int64_t m, int64_t n, int64_t k, int64_t group_size,
                            void* y, int out_dtype, void* act_buf, void* workspace,
                            uint32_t* flag, const void* residual, cudaStream_t stream);

/* ---- LLaMA-2 decode harness (BASELINE config 5) ---------
 * Producers and glue around the W6Ax linears for an end-to-end decode step.  The
 * reference has no model code; these are NOT part of its drop-in surface.
 * The fused quantizers write the same activation operand as flexq_quantize (same m_pad
 * rules, fp16 scales) from an fp16 intermediate h computed in the kernel:
 *   rmsnorm:  h = weight * fp16(x * rsqrt(mean(x^2) + eps))    (LLaMA RMSNorm)
 *   silu:     h = fp16(fp16(silu(g)) * u),  gate_up row = [g (cols) | u (cols)]
 * and are bit-identical to flexq_quantize applied to that h (h_out may be NULL). */
int flexq_rmsnorm_quantize(const void* x, int64_t x_stride, const void* weight, float eps,
                           int64_t rows, int64_t cols, int bits, int64_t group_size,
                           uint32_t* act_frag, float* act_scale, int32_t* act_corr, int64_t m_pad,
                           uint32_t* flag, void* h_out, cudaStream_t stream);
int flexq_silu_mul_quantize(const void* gate_up, int64_t x_stride, int64_t rows, int64_t cols,
                            int bits, int64_t group_size, uint32_t* act_frag, float* act_scale,
                            int32_t* act_corr, int64_t m_pad, uint32_t* flag, void* h_out,
                            cudaStream_t stream);
/* Rotate-half RoPE of q and k for each token's position pos[b] (device int32), k and v
 * appended to the caches [batch, heads, max_len, head_dim] at pos[b]; q_out [batch, heads,
 * head_dim].  qkv rows are [q | k | v] (heads * head_dim each).  A position outside
 * [0, max_len) writes nothing (attention then reads at most max_len cached positions). */
int flexq_rope_kv_append(const void* qkv, const int32_t* pos, void* k_cache, void* v_cache,
                         void* q_out, int64_t batch, int heads, int head_dim, int64_t max_len,
                         float theta, cudaStream_t stream);
/* The whole attention block of a decode step in one kernel: RoPE + append (as above),
 * attention, and the o_proj activation quantizer (group_size must equal head_dim = 128, so
 * head h of token b is group h; anything else is FLEXQ_ERR_CONFIG): writes o_proj's operand
 * (act_frag / act_scale / act_corr with m_pad = flexq_act_m_pad(batch)), bit-identical to
 * flexq_quantize of the fp16 attention output, which is also stored to
 * out[batch, heads * head_dim] when out is not NULL.  A position outside [0, max_len) sets
 * FLEXQ_FLAG_KV_OVERFLOW in *flag and writes nothing for that token. */
int flexq_attn_block(const void* qkv, const int32_t* pos, void* k_cache, void* v_cache, void* out,
                     int64_t batch, int heads, int head_dim, int64_t max_len, float theta,
                     int bits, int64_t group_size, uint32_t* act_frag, float* act_scale,
                     int32_t* act_corr, int64_t m_pad, uint32_t* flag, cudaStream_t stream);
/* Single-query attention of q over cache positions [0, pos[b]] (head_dim 128). */
int flexq_attn_decode(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos,
                      void* out, int64_t batch, int heads, int head_dim, int64_t max_len,
                      cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FLEXQ_H_ */
