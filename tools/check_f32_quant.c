// Exhaustive check behind quant_math.cuh::quant_one_h: for every finite fp16 v and positive fp16 s,
// roundf(fl32(v / s)) (clamped) equals the float64 reference code floor(|v / s| + 0.5); and for
// every positive fp16 peak and bits 2..8, fp16(fl32(peak / lim)) equals fp16(fl64(peak / lim)).
//   gcc -O2 -o /tmp/check_f32_quant tools/check_f32_quant.c -lm && /tmp/check_f32_quant
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
static float h2f(uint16_t h) {
  uint32_t s = (h >> 15) & 1, e = (h >> 10) & 31, m = h & 1023; float v;
  if (e == 0) v = ldexpf((float)m, -24); else if (e == 31) v = m ? NAN : INFINITY; else v = ldexpf((float)(m | 1024), (int)e - 25);
  return s ? -v : v;
}
int main(void) {
  static float vals[65536]; int n = 0;
  for (int h = 0; h < 65536; h++) { float f = h2f((uint16_t)h); if (isfinite(f)) vals[n++] = f; }
  long long bad = 0, tot = 0;
  for (int i = 0; i < n; i++) {
    float s = vals[i]; if (!(s > 0)) continue;
    for (int j = 0; j < n; j++) {
      float v = vals[j];
      double q = (double)v / (double)s;
      double a = floor(fabs(q) + 0.5); if (a > 127) a = 127;
      volatile float q32 = v / s;   /* IEEE correctly rounded fp32 divide */
      float b = roundf(fabsf(q32)); if (b > 127) b = 127;
      int sa = q < 0, sb = q32 < 0;
      tot++;
      if (a != (double)b || (a != 0 && sa != sb)) { if (bad < 5) printf("v=%g s=%g q=%.17g q32=%.9g a=%g b=%g\n", v, s, q, q32, a, b); bad++; }
    }
  }
  printf("codes: pairs %lld mismatches %lld\n", tot, bad);
  /* group scales: fp16(fl32(peak / lim)) vs fp16(fl64(peak / lim)), every positive fp16 peak */
  long sbad = 0, stot = 0;
  for (int hb = 1; hb < 0x7c00; hb++) {
    _Float16 hp; uint16_t hh = (uint16_t)hb; memcpy(&hp, &hh, 2);
    for (int bits = 2; bits <= 8; bits++) {
      int lim = (1 << (bits - 1)) - 1;
      _Float16 a = (_Float16)((double)hp / (double)lim);
      volatile float q32 = (float)hp / (float)lim;
      _Float16 b = (_Float16)q32;
      stot++;
      if (memcmp(&a, &b, 2)) sbad++;
    }
  }
  printf("scales: cases %ld mismatches %ld\n", stot, sbad);
  return (bad || sbad) ? 1 : 0;
}
