// extern "C" boundary of libflexq_sm100a.so (declared in include/flexq.h).
// Argument validation here mirrors the reference's raising sites so the
// Python wrapper can map status codes to the same exception classes.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace flexq {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
  set_error("%s: CUDA error %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
  return FLEXQ_ERR_CUDA;
}

int quantize_launch(const void*, int, int64_t, int64_t, int, int64_t, int, int8_t*, double*,
                    uint32_t*, float*, int32_t*, int64_t, uint32_t*, cudaStream_t);
int pack_planes_launch(const int8_t*, int64_t, int64_t, int, int, uint8_t*, cudaStream_t);
int unpack_planes_launch(const uint8_t*, int64_t, int64_t, int, int, int8_t*, cudaStream_t);
int pack_t6_launch(const int8_t*, const double*, int64_t, int64_t, int64_t, int, uint32_t*, void*,
                   cudaStream_t);
int64_t gemm_t6_workspace(int64_t, int64_t, int64_t, int64_t, int);
int gemm_t6_launch(const uint32_t*, const void*, int, const uint32_t*, const float*,
                   const int32_t*, int64_t, int64_t, int64_t, int64_t, int64_t, int32_t*, void*,
                   int, void*, int, const void*, cudaStream_t);
int64_t gemm_bitserial_workspace(int64_t, int64_t, int64_t, int);
int gemm_bitserial_launch(const uint8_t*, const uint8_t*, const float*, const float*, int64_t,
                          int64_t, int64_t, int, int, int64_t, int, int, int32_t*, void*, int,
                          void*, int, cudaStream_t);
int codes_to_frag_launch(const int8_t*, const double*, int64_t, int64_t, int64_t, int64_t,
                         uint32_t*, float*, int32_t*, cudaStream_t);
int popcount_and_launch(const uint8_t*, const uint8_t*, int64_t, int64_t*, cudaStream_t);
int64_t tc_act_m_pad(int64_t m);
int fused_quant_launch(int, const void*, int64_t, const void*, float, int64_t, int64_t, int,
                       int64_t, uint32_t*, float*, int32_t*, int64_t, uint32_t*, void*,
                       cudaStream_t);
int rope_kv_append_launch(const void*, const int*, void*, void*, void*, int64_t, int, int, int64_t,
                          float, cudaStream_t);
int attn_decode_launch(const void*, const void*, const void*, const int*, void*, int64_t, int, int,
                       int64_t, cudaStream_t);
int attn_block_launch(const void*, const int*, void*, void*, void*, int64_t, int, int, int64_t,
                      float, int, int64_t, uint32_t*, float*, int32_t*, int64_t, uint32_t*,
                      cudaStream_t);
bool gemm_tc16_supported(int64_t, int64_t, int64_t, int64_t, int);
int gemm_tc16_launch(const uint32_t*, const void*, const void*, int64_t, int64_t, int64_t, void*,
                     int, void*, const void*, cudaStream_t);
int quantize_f16op_launch(const void*, int64_t, int64_t, int, __half*, int64_t, uint32_t*,
                          cudaStream_t);
bool gemv_stream_supported(int64_t m, int64_t spg, int64_t units);
int group_epilogue_launch(const int32_t*, const double*, const double*, int64_t, int64_t, int64_t,
                          double*, uint16_t*, cudaStream_t);

static int check_chunk_m(int cm) {
  if (cm < 1 || cm > 8) {
    set_error("chunk_m (%d) must be in 1..8", cm);
    return FLEXQ_ERR_CONFIG;
  }
  return FLEXQ_OK;
}

// ---- runtime: knobs read once, per-device caches -----------------------------------------
static const char* env(const char* name) { return getenv(name); }

const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning v;
    v.trace = env("FLEXQ_TRACE") != nullptr;
    v.disable_tc = env("FLEXQ_DISABLE_TC") && atoi(env("FLEXQ_DISABLE_TC")) == 1;
    v.gemv_wide = env("FLEXQ_GEMV_WIDE") != nullptr;
    v.gemv_rev = env("FLEXQ_GEMV_REV") != nullptr;
    v.gemv_timeline = env("FLEXQ_GEMV_TIMELINE") != nullptr;
    v.tc_timeline = env("FLEXQ_TC_TIMELINE") != nullptr;
    v.q_early = env("FLEXQ_Q_EARLY") != nullptr;
    v.disable_tc16 = env("FLEXQ_DISABLE_TC16") && atoi(env("FLEXQ_DISABLE_TC16")) == 1;
    if (env("FLEXQ_STREAM_MAX_M") && atoi(env("FLEXQ_STREAM_MAX_M")) >= 1)
      v.stream_max_m = atoi(env("FLEXQ_STREAM_MAX_M"));
    if (env("FLEXQ_STREAM_STAGES")) {
      const int k = atoi(env("FLEXQ_STREAM_STAGES"));
      if (k >= 2 && k <= 4) v.stream_stages = k;
    }
    if (env("FLEXQ_MIN_UNITS") && atoi(env("FLEXQ_MIN_UNITS")) > 0)
      v.min_units = atoi(env("FLEXQ_MIN_UNITS"));
    if (env("FLEXQ_TC_MIN_UNITS") && atoi(env("FLEXQ_TC_MIN_UNITS")) > 0)
      v.tc_min_units = atoi(env("FLEXQ_TC_MIN_UNITS"));
    v.tc_align = !(env("FLEXQ_TC_ALIGN") && atoi(env("FLEXQ_TC_ALIGN")) == 0);
    return v;
  }();
  return t;
}

static std::mutex g_rt_mu;
constexpr int kMaxDevices = 64;

int device_sms() {
  static int sms[kMaxDevices] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

int tc_grid(int64_t units, int64_t kbn, int min_pct) {
  // Measured (tools/ab_tc_grid.sh): with every CTA inside one tile the split tiles have the
  // fewest, equal contributors and the fixups shrink -- 7B q_proj M = 64 / 128 / 256 on
  // kind::i8 21.5 / 30.4 / 32.1 -> 17.9 / 24.3 / 26.9 us, 13B gate_proj M = 128 on kind::f16
  // 43.6 -> 27.9 us -- but a grid that leaves many SMs idle loses (7B down_proj at 64 of 148
  // CTAs: 40.6 -> 48.4 us), hence the per-kernel floor.
  const int64_t sms = device_sms();
  int64_t c = units / tuning().tc_min_units;
  if (c < 1) c = 1;
  if (c > sms) c = sms;
  if (tuning().tc_align && kbn > 0 && units % kbn == 0 && min_pct <= 100) {
    const int64_t need = cdiv(units, c);
    for (int64_t upc = need; upc <= kbn; upc++)
      if (kbn % upc == 0) {
        const int64_t ca = units / upc;
        if (ca * 100 >= sms * min_pct) return (int)ca;
        break;
      }
  }
  return (int)c;
}

cudaError_t ensure_smem(const void* kern, int bytes) {
  struct Entry { int dev; const void* kern; int bytes; };
  static std::vector<Entry> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_rt_mu);
  for (const Entry& e : done)
    if (e.dev == dev && e.kern == kern && e.bytes >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({dev, kern, bytes});
  return e;
}

long long* dbg_trace_buf() {
  static long long* buf = nullptr;
  static const bool on = tuning().trace;
  if (on && !buf) {
    cudaMalloc(&buf, (4 + 4 * kDbgCap) * sizeof(long long));
    cudaMemset(buf, 0, 4 * sizeof(long long));
  }
  return buf;
}

long long dbg_next_launch() {
  static long long n = 0;
  return ++n;
}

}  // namespace flexq

using namespace flexq;

/* Debug: copy out and reset the event trace (FLEXQ_TRACE=1). Returns the record count. */
extern "C" int flexq_debug_trace(long long* host, int max_records) {
  long long* buf = dbg_trace_buf();
  if (!buf) return 0;
  cudaDeviceSynchronize();
  unsigned long long n = 0;
  cudaMemcpy(&n, buf, sizeof(n), cudaMemcpyDeviceToHost);
  if (n > kDbgCap) n = kDbgCap;
  if ((long long)n > max_records) n = max_records;
  cudaMemcpy(host, buf + 4, n * 4 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemset(buf, 0, 4 * sizeof(long long));
  return (int)n;
}

extern "C" {

const char* flexq_last_error(void) { return g_err; }

const char* flexq_tuning(void) {
  static std::string desc;
  static std::once_flag once;
  std::call_once(once, [] {
    const Tuning& t = tuning();
    const Tuning d;
    std::string s;
    auto add = [&](const char* k, const std::string& v) { s += (s.empty() ? "" : ",") + std::string(k) + "=" + v; };
    if (t.trace != d.trace) add("FLEXQ_TRACE", "1");
    if (t.disable_tc != d.disable_tc) add("FLEXQ_DISABLE_TC", "1");
    if (t.gemv_wide != d.gemv_wide) add("FLEXQ_GEMV_WIDE", "1");
    if (t.gemv_rev != d.gemv_rev) add("FLEXQ_GEMV_REV", "1");
    if (t.gemv_timeline != d.gemv_timeline) add("FLEXQ_GEMV_TIMELINE", "1");
    if (t.tc_timeline != d.tc_timeline) add("FLEXQ_TC_TIMELINE", "1");
    if (t.q_early != d.q_early) add("FLEXQ_Q_EARLY", "1");
    if (t.disable_tc16 != d.disable_tc16) add("FLEXQ_DISABLE_TC16", "1");
    if (t.stream_max_m != d.stream_max_m) add("FLEXQ_STREAM_MAX_M", std::to_string(t.stream_max_m));
    if (t.stream_stages != d.stream_stages) add("FLEXQ_STREAM_STAGES", std::to_string(t.stream_stages));
    if (t.min_units != d.min_units) add("FLEXQ_MIN_UNITS", std::to_string(t.min_units));
    if (t.tc_min_units != d.tc_min_units) add("FLEXQ_TC_MIN_UNITS", std::to_string(t.tc_min_units));
    if (t.tc_align != d.tc_align) add("FLEXQ_TC_ALIGN", "0");
    desc = s.empty() ? "defaults" : s;
  });
  return desc.c_str();
}

int flexq_version(void) { return 100; /* 0.1.0 */ }

int flexq_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "flexq_device_check");
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) {
    set_error("libflexq_sm100a needs an sm_100 (B200) device, found sm_%d%d", major, minor);
    return FLEXQ_ERR_CUDA;
  }
  return FLEXQ_OK;
}

int flexq_quantize(const void* x, int dtype, int64_t rows, int64_t cols, int bits,
                   int64_t group_size, int fp16_scales, int8_t* codes, double* scales,
                   uint32_t* act_frag, float* act_scale_f32, int32_t* act_corr, int64_t m_pad,
                   uint32_t* flag, cudaStream_t stream) {
  return quantize_launch(x, dtype, rows, cols, bits, group_size, fp16_scales, codes, scales,
                         act_frag, act_scale_f32, act_corr, m_pad, flag, stream);
}

int64_t flexq_planes_bytes(int64_t rows, int64_t cols, int bits, int chunk_m) {
  if (chunk_m < 1) return 0;
  return cdiv(cols, kChunkK) * cdiv(rows, chunk_m) * bits * chunk_m * 16;
}

int flexq_pack_planes(const int8_t* codes, int64_t rows, int64_t cols, int bits, int chunk_m,
                      uint8_t* words, cudaStream_t stream) {
  int rc = check_chunk_m(chunk_m);
  if (rc) return rc;
  if (bits < 1 || bits > 8) {
    set_error("bits must be in 1..8, got %d", bits);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (rows < 1 || cols < 1) {
    set_error("pack_planes: empty tensor (%lld, %lld)", (long long)rows, (long long)cols);
    return FLEXQ_ERR_SHAPE;
  }
  return pack_planes_launch(codes, rows, cols, bits, chunk_m, words, stream);
}

int flexq_unpack_planes(const uint8_t* words, int64_t rows, int64_t cols, int bits, int chunk_m,
                        int8_t* codes, cudaStream_t stream) {
  int rc = check_chunk_m(chunk_m);
  if (rc) return rc;
  if (bits < 1 || bits > 8 || rows < 1 || cols < 1) {
    set_error("unpack_planes: bad geometry rows=%lld cols=%lld bits=%d", (long long)rows,
              (long long)cols, bits);
    return FLEXQ_ERR_FORMAT;
  }
  return unpack_planes_launch(words, rows, cols, bits, chunk_m, codes, stream);
}

int64_t flexq_t6_bytes(int64_t n, int64_t k, int64_t group_size) {
  T6Geom G(n, k, group_size);
  return G.rt * G.kb * 3 * 32 * 16;
}

int64_t flexq_act_frag_bytes(int64_t m_pad, int64_t k, int64_t group_size) {
  T6Geom G(1, k, group_size);
  return cdiv(m_pad, kTokTile) * G.kb * 32 * 32;
}

int flexq_pack_t6(const int8_t* codes, const double* scales, int64_t n, int64_t k,
                  int64_t group_size, int scale_f16, uint32_t* t6, void* wscale,
                  cudaStream_t stream) {
  if (n < 1 || k < 1 || group_size < 1) {
    set_error("pack_t6: bad geometry n=%lld k=%lld group=%lld", (long long)n, (long long)k,
              (long long)group_size);
    return FLEXQ_ERR_SHAPE;
  }
  if (wscale && !scales) {
    set_error("pack_t6: scales required to pack wscale");
    return FLEXQ_ERR_INVALID_INPUT;
  }
  return pack_t6_launch(codes, scales, n, k, group_size, scale_f16, t6, wscale, stream);
}

int flexq_pack_act_t6(const int8_t* codes, const double* scales, int64_t m, int64_t m_pad,
                      int64_t k, int64_t group_size, uint32_t* act_frag, float* act_scale_f32,
                      int32_t* act_corr, cudaStream_t stream) {
  return codes_to_frag_launch(codes, scales, m, m_pad, k, group_size, act_frag, act_scale_f32,
                              act_corr, stream);
}

int flexq_popcount_and(const uint8_t* a, const uint8_t* b, int64_t nbytes, int64_t* out,
                       cudaStream_t stream) {
  return popcount_and_launch(a, b, nbytes, out, stream);
}

int64_t flexq_gemm_workspace_bytes(int64_t m, int64_t n, int64_t k, int64_t group_size,
                                   int ksplit) {
  int64_t a = gemm_t6_workspace(m, n, k, group_size, ksplit);
  int64_t b = gemm_bitserial_workspace(m, n, k, ksplit);
  return a > b ? a : b;
}

int flexq_gemm_t6(const uint32_t* t6, const void* wscale, int scale_f16,
                  const uint32_t* act_frag, const float* act_scale, const int32_t* act_corr,
                  int64_t m, int64_t m_pad, int64_t n, int64_t k, int64_t group_size,
                  int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                  cudaStream_t stream) {
  return gemm_t6_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k,
                        group_size, partials, y, out_dtype, workspace, ksplit, nullptr, stream);
}

int flexq_gemm_t6_ex(const uint32_t* t6, const void* wscale, int scale_f16,
                     const uint32_t* act_frag, const float* act_scale, const int32_t* act_corr,
                     int64_t m, int64_t m_pad, int64_t n, int64_t k, int64_t group_size,
                     int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                     const void* residual, cudaStream_t stream) {
  return gemm_t6_launch(t6, wscale, scale_f16, act_frag, act_scale, act_corr, m, m_pad, n, k,
                        group_size, partials, y, out_dtype, workspace, ksplit, residual, stream);
}

int flexq_gemm_bitserial(const uint8_t* wwords, const uint8_t* xwords, const float* wscale,
                         const float* xscale, int64_t m, int64_t n, int64_t k, int wbits,
                         int xbits, int64_t group_size, int w_chunk_m, int x_chunk_m,
                         int32_t* partials, void* y, int out_dtype, void* workspace, int ksplit,
                         cudaStream_t stream) {
  return gemm_bitserial_launch(wwords, xwords, wscale, xscale, m, n, k, wbits, xbits, group_size,
                               w_chunk_m, x_chunk_m, partials, y, out_dtype, workspace, ksplit,
                               stream);
}

int flexq_group_epilogue_f64(const int32_t* partials, const double* wscale,
                             const double* xscale, int64_t m, int64_t n, int64_t groups,
                             double* y, uint16_t* y16, cudaStream_t stream) {
  return group_epilogue_launch(partials, wscale, xscale, m, n, groups, y, y16, stream);
}

int64_t flexq_act_m_pad(int64_t m) { return m < 1 ? 0 : tc_act_m_pad(m); }

// The batched forward takes the kind::f16 kernel (gemm_tc16.cu) for 32 < m <= 128 at group 128
// with fp16 weight scales; the fp16 operand then follows the INT8 operand in the act buffer.
static std::atomic<int> g_tc16_mode{-1};  // flexq_set_tc16_route: -1 auto, 0 never, 1 always

static bool tc16_route(int64_t m, int64_t n, int64_t k, int64_t gs, int scale_f16) {
  if (m <= 16 || tuning().disable_tc16 || tuning().disable_tc || !gemm_tc16_supported(m, n, k, gs, scale_f16))
    return false;
  const int mode = g_tc16_mode.load(std::memory_order_relaxed);
  if (mode >= 0) return mode == 1;
  if (m <= 32) return false;  // 16 < M <= 32: the streaming GEMV or kind::i8 (measured faster)
  // Measured A/B against the INT8 kernel (tools/ab_tc16.sh, sweep --tc16-route, LLaMA-2
  // 7B/13B/70B linears, aligned grids): kind::f16 wins on layers of >= 8192 units (70B gate
  // M = 64/128/256: 60/74/120 vs 85/103/187 us) and loses on smaller ones at M <= 128 (7B
  // q_proj M = 128: 40 vs 31 us: too few k-blocks per CTA to fill its deeper pipeline).  For
  // 128 < M <= 256 (one 256-token tile) it also wins on wide layers (7B gate_proj 11008 x 4096
  // M = 256: 36.8 vs 52.3 us; 70B o_proj 54.5 vs 60.0 us) but not on narrow ones (7B down_proj
  // 4096 x 11008: 68.1 vs 49.5 us).
  const int64_t units = cdiv(n, 64) * cdiv(k, 128);
  if (m <= 128) return units >= 8192;
  return units >= 8192 || n >= 8192;
}

int flexq_set_tc16_route(int mode) {
  if (mode < -1 || mode > 1) {
    set_error("set_tc16_route: mode must be -1 (auto), 0 (never) or 1 (always)");
    return -2;
  }
  return g_tc16_mode.exchange(mode);
}

static int64_t act_f16_offset(int64_t m, int64_t k, int64_t group_size) {
  const int64_t m_pad = flexq_act_m_pad(m);
  T6Geom G(1, k, group_size);
  const int64_t frag = cdiv(flexq_act_frag_bytes(m_pad, k, group_size), 256) * 256;
  const int64_t vec = cdiv(G.ng * m_pad * 4, 256) * 256;
  return frag + 2 * vec;
}

int64_t flexq_act_buf_bytes(int64_t m, int64_t k, int64_t group_size) {
  const int64_t base = act_f16_offset(m, k, group_size);
  if (m > 16 && group_size == 128 && k % 128 == 0)  // room for the fp16 operand (gemm_tc16)
    return base + flexq_act_m_pad(m) * k * 2;
  return base;
}

int flexq_linear_kernel(int64_t m, int64_t n, int64_t k, int64_t group_size, int scale_f16) {
  if (m < 1 || n < 1 || k < 1 || group_size < 1) return -1;
  if (tc16_route(m, n, k, group_size, scale_f16)) return FLEXQ_KERNEL_TC16;
  T6Geom G(n, k, group_size);
  if (gemv_stream_supported(m, G.spg, G.rg * G.kb)) return FLEXQ_KERNEL_GEMV;
  if (m > 16 && G.spg % 4 == 0 && !tuning().disable_tc) return FLEXQ_KERNEL_TC_I8;
  return FLEXQ_KERNEL_MMA_SYNC;
}

int flexq_gemm_tc16(const uint32_t* t6, const void* wscale, const void* act_f16, int64_t m,
                    int64_t n, int64_t k, void* y, int out_dtype, void* workspace,
                    const void* residual, cudaStream_t stream) {
  return gemm_tc16_launch(t6, wscale, act_f16, m, n, k, y, out_dtype, workspace, residual, stream);
}

void* flexq_act_f16_operand(void* act_buf, int64_t m, int64_t k, int64_t group_size) {
  if (!act_buf) return nullptr;
  return reinterpret_cast<char*>(act_buf) + act_f16_offset(m, k, group_size);
}

static int linear_forward(const uint32_t* t6, const void* wscale, int scale_f16, int xbits,
                          const void* x, int64_t m, int64_t n, int64_t k, int64_t group_size,
                          void* y, int out_dtype, void* act_buf, void* workspace, uint32_t* flag,
                          const void* residual, cudaStream_t stream) {
  if (!act_buf || !flag || !y) {
    set_error("linear_forward: act_buf, flag and y are required");
    return FLEXQ_ERR_INVALID_INPUT;
  }
  if (out_dtype != FLEXQ_OUT_F16 && out_dtype != FLEXQ_OUT_F32) {
    set_error("linear_forward: unknown out_dtype %d", out_dtype);
    return FLEXQ_ERR_INVALID_INPUT;
  }
  const int64_t m_pad = flexq_act_m_pad(m);
  T6Geom G(1, k, group_size);
  char* base = reinterpret_cast<char*>(act_buf);
  const int64_t frag = cdiv(flexq_act_frag_bytes(m_pad, k, group_size), 256) * 256;
  const int64_t vec = cdiv(G.ng * m_pad * 4, 256) * 256;
  uint32_t* act_frag = reinterpret_cast<uint32_t*>(base);
  float* xs = reinterpret_cast<float*>(base + frag);
  int32_t* corr = reinterpret_cast<int32_t*>(base + frag + vec);
  if (tc16_route(m, n, k, group_size, scale_f16)) {  // batched: scales folded into fp16 operands
    __half* act16 = reinterpret_cast<__half*>(base + frag + 2 * vec);
    int rc = quantize_f16op_launch(x, m, k, xbits, act16, m_pad, flag, stream);
    if (rc) return rc;
    return gemm_tc16_launch(t6, wscale, act16, m, n, k, y, out_dtype, workspace, residual, stream);
  }
  int rc = quantize_launch(x, FLEXQ_DT_F16, m, k, xbits, group_size, 1, nullptr, nullptr,
                           act_frag, xs, corr, m_pad, flag, stream);
  if (rc) return rc;
  return gemm_t6_launch(t6, wscale, scale_f16, act_frag, xs, corr, m, m_pad, n, k, group_size,
                        nullptr, y, out_dtype, workspace, 0, residual, stream);
}

int flexq_linear_forward(const uint32_t* t6, const void* wscale, int scale_f16, int xbits,
                         const void* x, int64_t m, int64_t n, int64_t k, int64_t group_size,
                         uint16_t* y, void* act_buf, void* workspace, uint32_t* flag,
                         cudaStream_t stream) {
  return linear_forward(t6, wscale, scale_f16, xbits, x, m, n, k, group_size, y, FLEXQ_OUT_F16,
                        act_buf, workspace, flag, nullptr, stream);
}

int flexq_linear_forward_ex(const uint32_t* t6, const void* wscale, int scale_f16, int xbits,
                            const void* x, int64_t m, int64_t n, int64_t k, int64_t group_size,
                            void* y, int out_dtype, void* act_buf, void* workspace,
                            uint32_t* flag, const void* residual, cudaStream_t stream) {
  return linear_forward(t6, wscale, scale_f16, xbits, x, m, n, k, group_size, y, out_dtype,
                        act_buf, workspace, flag, residual, stream);
}

/* ---- LLaMA decode harness (BASELINE config 5) ---- */
int flexq_rmsnorm_quantize(const void* x, int64_t x_stride, const void* weight, float eps,
                           int64_t rows, int64_t cols, int bits, int64_t group_size,
                           uint32_t* act_frag, float* act_scale, int32_t* act_corr, int64_t m_pad,
                           uint32_t* flag, void* h_out, cudaStream_t stream) {
  return fused_quant_launch(0, x, x_stride, weight, eps, rows, cols, bits, group_size, act_frag,
                            act_scale, act_corr, m_pad, flag, h_out, stream);
}

int flexq_silu_mul_quantize(const void* gate_up, int64_t x_stride, int64_t rows, int64_t cols,
                            int bits, int64_t group_size, uint32_t* act_frag, float* act_scale,
                            int32_t* act_corr, int64_t m_pad, uint32_t* flag, void* h_out,
                            cudaStream_t stream) {
  return fused_quant_launch(1, gate_up, x_stride, nullptr, 0.f, rows, cols, bits, group_size,
                            act_frag, act_scale, act_corr, m_pad, flag, h_out, stream);
}

int flexq_rope_kv_append(const void* qkv, const int32_t* pos, void* k_cache, void* v_cache,
                         void* q_out, int64_t batch, int heads, int head_dim, int64_t max_len,
                         float theta, cudaStream_t stream) {
  return rope_kv_append_launch(qkv, pos, k_cache, v_cache, q_out, batch, heads, head_dim, max_len,
                               theta, stream);
}

int flexq_attn_decode(const void* q, const void* k_cache, const void* v_cache, const int32_t* pos,
                      void* out, int64_t batch, int heads, int head_dim, int64_t max_len,
                      cudaStream_t stream) {
  return attn_decode_launch(q, k_cache, v_cache, pos, out, batch, heads, head_dim, max_len, stream);
}

int flexq_attn_block(const void* qkv, const int32_t* pos, void* k_cache, void* v_cache, void* out,
                     int64_t batch, int heads, int head_dim, int64_t max_len, float theta,
                     int bits, int64_t group_size, uint32_t* act_frag, float* act_scale,
                     int32_t* act_corr, int64_t m_pad, uint32_t* flag, cudaStream_t stream) {
  return attn_block_launch(qkv, pos, k_cache, v_cache, out, batch, heads, head_dim, max_len, theta,
                           bits, group_size, act_frag, act_scale, act_corr, m_pad, flag, stream);
}

}  // extern "C"
