/* tests/native/expf_check.c -- exhaustive check of the device expf port
 * (paper_2211_10017_b200/csrc/glibc_expf.h) against the host libm expf the
 * reference gate calls (proj/src/routing.cpp:34).  Usage: expf_check [lo hi]
 * over the 32-bit pattern range [lo, hi); prints mismatch count. */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include "glibc_expf.h"

typedef struct { uint64_t lo, hi, bad, first; } job_t;

static void* run(void* p) {
  job_t* j = (job_t*)p;
  for (uint64_t u = j->lo; u < j->hi; ++u) {
    float x = moe_u2f((uint32_t)u);
    float a = expf(x), b = moe_glibc_expf(x);
    uint32_t ua = moe_f2u(a), ub = moe_f2u(b);
    if (ua != ub && !(isnan(a) && isnan(b))) {
      if (!j->bad) j->first = u;
      ++j->bad;
    }
  }
  return NULL;
}

int main(int argc, char** argv) {
  uint64_t lo = 0, hi = 1ull << 32;
  if (argc == 3) { lo = strtoull(argv[1], 0, 0); hi = strtoull(argv[2], 0, 0); }
  int nt = 8;
  pthread_t th[64];
  job_t jobs[64];
  uint64_t step = (hi - lo + nt - 1) / nt;
  for (int i = 0; i < nt; ++i) {
    jobs[i].lo = lo + i * step;
    jobs[i].hi = jobs[i].lo + step > hi ? hi : jobs[i].lo + step;
    jobs[i].bad = 0;
    pthread_create(&th[i], 0, run, &jobs[i]);
  }
  uint64_t bad = 0, first = 0;
  for (int i = 0; i < nt; ++i) {
    pthread_join(th[i], 0);
    if (jobs[i].bad && !bad) first = jobs[i].first;
    bad += jobs[i].bad;
  }
  printf("checked=%llu mismatches=%llu first=0x%08llx\n", (unsigned long long)(hi - lo),
         (unsigned long long)bad, (unsigned long long)first);
  return bad != 0;
}
