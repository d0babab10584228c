/* tests/native/quant_div_check.c -- exhaustive proof that the device
 * quantizer's f32 division gives the reference's codes.
 *
 * Reference (proj/src/quantize.cpp:26-32): q = clamp(llround((double)w /
 * (double)s), -qmax, qmax).  Device (csrc/k_quant.cu): q = clamp(roundf(
 * RN32(w / s)), ...) with roundf = round half away from zero, like llround.
 * For every positive finite fp16 scale s and every finite fp16 weight w with
 * |w| <= (qmax + 1) * s (beyond that both clamp to +-qmax) the two codes must
 * be equal, for qmax = 7 (int4) and 127 (int8).  Argument: a
 * quotient of two fp16 values that is not itself a half-integer lies at
 * least ~2^-13 (relative) away from every half-integer, far beyond the 2^-24
 * error of RN32, and half-integers of magnitude <= 128 are exact in f32.
 * Prints the mismatch count (0 expected). */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static double h2d(uint16_t h) {
  const int e = (h >> 10) & 31, m = h & 1023;
  const double v = e == 0 ? ldexp((double)m, -24) : ldexp((double)(m | 1024), e - 25);
  return (h & 0x8000) ? -v : v;
}

typedef struct {
  int s_lo, s_hi;
  unsigned long long bad, checked;
} job_t;

static int clampi(long long q, int qmax) { return q < -qmax ? -qmax : q > qmax ? qmax : (int)q; }

static void* run(void* p) {
  job_t* j = (job_t*)p;
  for (int su = j->s_lo; su < j->s_hi; ++su) {
    const double sd = h2d((uint16_t)su);
    const float sf = (float)sd;
    for (int wu = 0; wu < 0x7C00; ++wu) {
      const double wd = h2d((uint16_t)wu);
      if (wd > 128.0 * sd) break; /* |q| > 128: both clamp */
      for (int sign = 0; sign < 2; ++sign) {
        const double w = sign ? -wd : wd;
        const long long ref = llround(w / sd);
        volatile float qf = (float)w / sf; /* RN32 division */
        const float r = roundf(qf);
        for (int qmax = 7; qmax <= 127; qmax += 120) {
          if (clampi(ref, qmax) != clampi((long long)r, qmax)) ++j->bad;
        }
        ++j->checked;
      }
    }
  }
  return NULL;
}

int main(void) {
  enum { NT = 16 };
  pthread_t th[NT];
  job_t jobs[NT];
  const int lo = 1, hi = 0x7C00; /* positive finite scales (incl. subnormal) */
  for (int t = 0; t < NT; ++t) {
    jobs[t].s_lo = lo + (hi - lo) * t / NT;
    jobs[t].s_hi = lo + (hi - lo) * (t + 1) / NT;
    jobs[t].bad = jobs[t].checked = 0;
    pthread_create(&th[t], NULL, run, &jobs[t]);
  }
  unsigned long long bad = 0, checked = 0;
  for (int t = 0; t < NT; ++t) {
    pthread_join(th[t], NULL);
    bad += jobs[t].bad;
    checked += jobs[t].checked;
  }
  printf("quant_div_check: %llu (w, s) pairs, %llu mismatches\n", checked, bad);
  return bad != 0;
}
