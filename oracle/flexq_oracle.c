/*
 * CPU oracle (plain C restatement) of the reference's W6Ax quantized-linear path.
 *
 * TEST INFRASTRUCTURE ONLY -- the product package never links or loads this
 * library.  It exists so parity tests can check the CUDA path at LLaMA-2-70B
 * sizes in seconds (the reference's numpy path needs minutes-hours there,
 * SURVEY.md section 7 "Oracle cost at big shapes").  Its own parity is pinned
 * against the golden vectors frozen from the real reference
 * (tests/golden/golden.npz, tests/test_oracle.py).
 *
 * Restated reference functions (paths under /root/reference/pkg/src/bitserial):
 *   oracle_quantize_*    quantize.py:118-148 (group_scales 99-110,
 *                        _round_half_away 29-31, fp16 scale mode 143-144,
 *                        QuantTensor positivity check 71-72)
 *   oracle_int_matmul    engine.py:337-365 (int_matmul_reference) with the
 *                        shared epilogue engine.py:211-216 (_scale_accumulate):
 *                        acc += (xs*ws) * (double)partial, ascending group
 *                        order, no FMA contraction (built -ffp-contract=off).
 *   oracle_pack_planes   bitplane.py:55-79 + packing.py:132-147 (FLXQ-P).
 *
 * Build: oracle/Makefile -> oracle/_build/liboracle.so
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NONFINITE -1
#define ORC_NONPOSITIVE_SCALE -2
#define ORC_BAD_ARG -3

static int qmax_of(int bits) { return (1 << (bits - 1)) - 1; }

static double to_fp16_and_back(double v) {
  _Float16 h = (_Float16)v; /* round-to-nearest-even, direct double->half */
  return (double)h;
}

static double half_bits_to_double(uint16_t b) {
  _Float16 h;
  memcpy(&h, &b, 2);
  return (double)h;
}

/* quantize.py:29-31 */
static double round_half_away(double v) {
  double a = floor(fabs(v) + 0.5);
  return v < 0 ? -a : (v > 0 ? a : 0.0 * v);
}

typedef double (*load_fn)(const void* base, int64_t idx);
static double load_f64(const void* b, int64_t i) { return ((const double*)b)[i]; }
static double load_f32(const void* b, int64_t i) { return (double)((const float*)b)[i]; }
static double load_f16(const void* b, int64_t i) { return half_bits_to_double(((const uint16_t*)b)[i]); }

static int quantize_generic(const void* x, load_fn ld, int64_t rows, int64_t cols, int bits,
                            int64_t gs, int fp16_scales, int8_t* codes, double* scales) {
  if (bits < 2 || bits > 8 || gs < 1 || rows < 0 || cols < 0) return ORC_BAD_ARG;
  const int64_t ng = (cols + gs - 1) / gs;
  const int lim = qmax_of(bits);
  for (int64_t r = 0; r < rows; r++)
    for (int64_t c = 0; c < cols; c++)
      if (!isfinite(ld(x, r * cols + c))) return ORC_NONFINITE;
  for (int64_t r = 0; r < rows; r++) {
    for (int64_t g = 0; g < ng; g++) {
      const int64_t lo = g * gs, hi = (lo + gs < cols) ? lo + gs : cols;
      double peak = 0.0;
      for (int64_t c = lo; c < hi; c++) {
        double a = fabs(ld(x, r * cols + c));
        if (a > peak) peak = a;
      }
      double s = peak > 0.0 ? peak / (double)lim : 1.0; /* quantize.py:110 */
      if (fp16_scales) s = to_fp16_and_back(s);           /* quantize.py:143-144 */
      if (!(s > 0.0)) return ORC_NONPOSITIVE_SCALE;       /* quantize.py:71-72 */
      scales[r * ng + g] = s;
      for (int64_t c = lo; c < hi; c++) {
        double v = round_half_away(ld(x, r * cols + c) / s); /* quantize.py:147 */
        if (v > lim) v = lim;
        if (v < -lim) v = -lim;
        codes[r * cols + c] = (int8_t)v;
      }
    }
  }
  return ORC_OK;
}

int oracle_quantize_f64(const double* x, int64_t rows, int64_t cols, int bits, int64_t gs,
                        int fp16_scales, int8_t* codes, double* scales) {
  return quantize_generic(x, load_f64, rows, cols, bits, gs, fp16_scales, codes, scales);
}
int oracle_quantize_f32(const float* x, int64_t rows, int64_t cols, int bits, int64_t gs,
                        int fp16_scales, int8_t* codes, double* scales) {
  return quantize_generic(x, load_f32, rows, cols, bits, gs, fp16_scales, codes, scales);
}
int oracle_quantize_f16(const uint16_t* x, int64_t rows, int64_t cols, int bits, int64_t gs,
                        int fp16_scales, int8_t* codes, double* scales) {
  return quantize_generic(x, load_f16, rows, cols, bits, gs, fp16_scales, codes, scales);
}

/* ---- engine.py:337-365 int_matmul_reference + engine.py:211-216 ------------ */
typedef struct {
  const int8_t *w, *x;
  const double *ws, *xs;
  int64_t m, n, k, gs, ng, n0, n1;
  double* y;
  int32_t* partials;
} mm_job;

static void* mm_worker(void* arg) {
  mm_job* j = (mm_job*)arg;
  for (int64_t col = j->n0; col < j->n1; col++) {
    const int8_t* wr = j->w + col * j->k;
    for (int64_t row = 0; row < j->m; row++) {
      const int8_t* xr = j->x + row * j->k;
      double acc = 0.0;
      for (int64_t g = 0; g < j->ng; g++) {
        const int64_t lo = g * j->gs, hi = (lo + j->gs < j->k) ? lo + j->gs : j->k;
        int64_t p = 0;
        for (int64_t c = lo; c < hi; c++) p += (int64_t)wr[c] * (int64_t)xr[c];
        if (j->partials) j->partials[(g * j->m + row) * j->n + col] = (int32_t)p;
        double sprod = j->xs[row * j->ng + g] * j->ws[col * j->ng + g];
        acc += sprod * (double)p;
      }
      j->y[row * j->n + col] = acc;
    }
  }
  return NULL;
}

int oracle_int_matmul(const int8_t* w, const int8_t* x, const double* ws, const double* xs,
                      int64_t m, int64_t n, int64_t k, int64_t gs, double* y, int32_t* partials,
                      int nthreads) {
  if (m < 1 || n < 1 || k < 1 || gs < 1) return ORC_BAD_ARG;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  const int64_t ng = (k + gs - 1) / gs;
  pthread_t th[256];
  mm_job jobs[256];
  const int64_t per = (n + nthreads - 1) / nthreads;
  int launched = 0;
  for (int t = 0; t < nthreads; t++) {
    int64_t n0 = t * per, n1 = n0 + per < n ? n0 + per : n;
    if (n0 >= n1) break;
    jobs[t] = (mm_job){w, x, ws, xs, m, n, k, gs, ng, n0, n1, y, partials};
    pthread_create(&th[t], NULL, mm_worker, &jobs[t]);
    launched++;
  }
  for (int t = 0; t < launched; t++) pthread_join(th[t], NULL);
  return ORC_OK;
}

/* ---- bitplane.py:55-79 + packing.py:132-147 (FLXQ-P byte stream) ----------- */
int oracle_pack_planes(const int8_t* codes, int64_t rows, int64_t cols, int bits, int chunk_m,
                       uint8_t* out) {
  if (bits < 1 || bits > 8 || chunk_m < 1 || chunk_m > 8) return ORC_BAD_ARG;
  const int64_t rc_n = (rows + chunk_m - 1) / chunk_m, kc_n = (cols + 127) / 128;
  const int64_t total = kc_n * rc_n * bits * chunk_m * 16;
  memset(out, 0, (size_t)total);
  for (int64_t r = 0; r < rows; r++) {
    const int64_t rc = r / chunk_m, rr = r % chunk_m;
    for (int64_t c = 0; c < cols; c++) {
      const unsigned enc = (unsigned)(int)codes[r * cols + c] & ((1u << bits) - 1u);
      const int64_t kc = c / 128, j = c % 128;
      for (int s = 0; s < bits; s++) {
        if (!((enc >> s) & 1u)) continue;
        const int64_t base = (((kc * rc_n + rc) * bits + s) * chunk_m + rr) * 16;
        out[base + j / 8] |= (uint8_t)(1u << (j % 8));
      }
    }
  }
  return ORC_OK;
}
