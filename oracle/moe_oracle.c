/* oracle/moe_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the
 * product).  Scalar C restatement of the reference MoE-layer hot path; see
 * moe_oracle.h for scope and the top-k extension.  Built with
 * -ffp-contract=off like the reference (proj/CMakeLists.txt:9) so every f32
 * add/mul rounds separately, in the same order as the reference loops.
 */
#include "moe_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return OR_EINVAL;
}

const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------ */
/* binary16 <-> binary32/64.  half.hpp:57-75 widens exactly; half.hpp:81-129
 * narrows f64 with one round-to-nearest-even step (subnormals kept, overflow
 * to inf, NaN -> 0x7E00).  Restated here with integer arithmetic on the
 * binary64 significand. */

float or_half_to_f32(uint16_t h) {
  const int sign = h >> 15, ex = (h >> 10) & 0x1F, man = h & 0x3FF;
  double v;
  if (ex == 0x1F) {
    if (man) return sign ? -NAN : NAN;
    return sign ? -INFINITY : INFINITY;
  }
  if (ex == 0)
    v = ldexp((double)man, -24);
  else
    v = ldexp((double)(man | 0x400), ex - 25);
  return (float)(sign ? -v : v); /* exact: fp16 values are f32-representable */
}

uint16_t or_f64_to_half(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  const uint16_t sign = (uint16_t)((u >> 48) & 0x8000u);
  const int bexp = (int)((u >> 52) & 0x7FF);
  const uint64_t frac = u & 0xFFFFFFFFFFFFFull;
  if (bexp == 0x7FF) return frac ? 0x7E00 : (uint16_t)(sign | 0x7C00);
  if (bexp == 0) return sign; /* f64 subnormals are far below 2^-25 */
  const int e = bexp - 1023;  /* value = 1.frac * 2^e */
  if (e > 15) return (uint16_t)(sign | 0x7C00);
  /* quantum of the target grid: 2^(max(e,-14) - 10) */
  const int q = (e < -14 ? -14 : e) - 10;
  const uint64_t sig = frac | (1ull << 52); /* value = sig * 2^(e-52) */
  const int sh = q - (e - 52);              /* bits to drop, >= 42 */
  if (sh > 63) return sign;
  uint64_t kept = sig >> sh;
  const uint64_t rem = sig & ((1ull << sh) - 1), half = 1ull << (sh - 1);
  if (rem > half || (rem == half && (kept & 1))) ++kept;
  /* kept counts units of 2^q. */
  if (e < -14) return (uint16_t)(sign | kept); /* kept <= 1024: 1024 == min normal */
  int be = e + 15;
  if (kept == 2048) { kept = 1024; ++be; }
  if (be >= 31) return (uint16_t)(sign | 0x7C00);
  return (uint16_t)(sign | (be << 10) | (kept - 1024));
}

uint16_t or_f32_to_half(float x) { return or_f64_to_half((double)x); }

/* half.hpp:136-146: exact f64 op, one RN16. */
uint16_t or_half_add(uint16_t a, uint16_t b) {
  return or_f64_to_half((double)or_half_to_f32(a) + (double)or_half_to_f32(b));
}
uint16_t or_half_sub(uint16_t a, uint16_t b) {
  return or_f64_to_half((double)or_half_to_f32(a) - (double)or_half_to_f32(b));
}
uint16_t or_half_mul(uint16_t a, uint16_t b) {
  return or_f64_to_half((double)or_half_to_f32(a) * (double)or_half_to_f32(b));
}

static int half_finite(uint16_t h) { return (h & 0x7C00) != 0x7C00; }

/* ------------------------------------------------------------------------ */
/* quantizer: src/quantize.cpp */

static int qmax_of(int bits) { return bits == 8 ? 127 : 7; }
static int offset_of(int bits) { return bits == 8 ? 128 : 8; }

/* quantize.cpp:14-24 */
uint16_t or_quant_scale(float maxabs, int qmax) {
  if (maxabs == 0.0f) return 0x3C00;
  const float s32 = maxabs / (float)qmax;
  const uint16_t s16 = or_f32_to_half(s32);
  if ((s16 & 0x7FFF) == 0) return 0x0001;
  return s16;
}

/* quantize.cpp:26-32: llround(f64(w)/f64(s)) (half away from zero), clamp. */
uint8_t or_quant_encode(uint16_t w, uint16_t scale, int bits) {
  const int qmax = qmax_of(bits);
  long q = llround((double)or_half_to_f32(w) / (double)or_half_to_f32(scale));
  if (q < -qmax) q = -qmax;
  if (q > qmax) q = qmax;
  return (uint8_t)(q + offset_of(bits));
}

/* quantize.cpp:34-50: [v0..v7] -> {v0|v2<<4, v4|v6<<4, v1|v3<<4, v5|v7<<4} */
int or_pack_int4(const uint8_t* v, size_t count, uint8_t* out) {
  if (count % 8) return fail("pack_int4_interleaved: length must be a multiple of 8");
  for (size_t i = 0; i < count; ++i)
    if (v[i] >= 16) return fail("pack_int4_interleaved: value does not fit a nibble");
  for (size_t g = 0; g < count / 8; ++g) {
    const uint8_t* s = v + 8 * g;
    uint8_t* d = out + 4 * g;
    d[0] = (uint8_t)(s[0] | (s[2] << 4));
    d[1] = (uint8_t)(s[4] | (s[6] << 4));
    d[2] = (uint8_t)(s[1] | (s[3] << 4));
    d[3] = (uint8_t)(s[5] | (s[7] << 4));
  }
  return OR_OK;
}

/* quantize.cpp:52-72 */
int or_unpack_int4(const uint8_t* p, size_t count, uint8_t* out) {
  if (count % 8) return fail("unpack_int4_interleaved: count must be a multiple of 8");
  for (size_t g = 0; g < count / 8; ++g) {
    const uint8_t* b = p + 4 * g;
    uint8_t* v = out + 8 * g;
    v[0] = b[0] & 15; v[2] = b[0] >> 4;
    v[4] = b[1] & 15; v[6] = b[1] >> 4;
    v[1] = b[2] & 15; v[3] = b[2] >> 4;
    v[5] = b[3] & 15; v[7] = b[3] >> 4;
  }
  return OR_OK;
}

/* quantize.cpp:74-122 */
int or_quantize(const uint16_t* w, size_t e, size_t m, size_t n, int bits,
                uint8_t* packed, uint16_t* scales) {
  if (bits != 4 && bits != 8) return fail("bits must be 4 or 8");
  if (!(e > 0 && m > 0 && n > 0)) return fail("quantize: empty weight tensor");
  if (bits == 4 && n % 8)
    return fail("quantize: 4-bit packing needs the column count divisible by 8");
  const size_t total = e * m * n;
  for (size_t i = 0; i < total; ++i)
    if (!half_finite(w[i])) {
      snprintf(g_err, sizeof g_err, "quantize: non-finite weight at flat index %zu", i);
      return OR_EINVAL;
    }
  const int qmax = qmax_of(bits);
  uint8_t* codes = bits == 8 ? packed : (uint8_t*)malloc(total);
  for (size_t ei = 0; ei < e; ++ei)
    for (size_t ni = 0; ni < n; ++ni) {
      float mx = 0.0f;
      for (size_t mi = 0; mi < m; ++mi) {
        const float a = fabsf(or_half_to_f32(w[(ei * m + mi) * n + ni]));
        if (a > mx) mx = a; /* std::max(maxabs, a) keeps maxabs on ties */
      }
      const uint16_t s = or_quant_scale(mx, qmax);
      scales[ei * n + ni] = s;
      for (size_t mi = 0; mi < m; ++mi)
        codes[(ei * m + mi) * n + ni] = or_quant_encode(w[(ei * m + mi) * n + ni], s, bits);
    }
  if (bits == 4) {
    or_pack_int4(codes, total, packed);
    free(codes);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* dequantizer: dequant.hpp / dequant.cpp.  MOE_FAULT_INJECT (dequant.cpp:12-30)
 * is honoured so the fault drill can be reproduced against the oracle. */

static int fault_mode(void) { /* 0 none, 8 corrupt u8, 4 corrupt u4 */
  const char* v = getenv("MOE_FAULT_INJECT");
  if (!v || !*v) return 0;
  return strcmp(v, "i2f4") == 0 ? 4 : 8;
}
uint16_t or_debias_u8(void) { return fault_mode() == 8 ? 0x6481 : 0x6480; }
uint16_t or_debias_u4(void) { return fault_mode() == 4 ? 0x6409 : 0x6408; }

/* one logical code -> fp16 value (code - offset), either path */
static uint16_t code_value(uint8_t code, int bits, int fast) {
  if (!fast) /* dequant.cpp:61-63: RN16(q) (exact) */
    return or_f64_to_half((double)((int)code - offset_of(bits)));
  /* dequant.hpp:40-63: (0x6400 | code) - debias, one fp16 subtraction */
  return or_half_sub((uint16_t)(0x6400 | code), bits == 8 ? or_debias_u8() : or_debias_u4());
}

/* logical code (ei, mi, ni) from the reference packing */
static uint8_t code_at(const uint8_t* packed, size_t m, size_t n, int bits,
                       size_t ei, size_t mi, size_t ni) {
  const size_t flat = (ei * m + mi) * n + ni;
  if (bits == 8) return packed[flat];
  const uint8_t* b = packed + (flat / 8) * 4;
  const int j = (int)(flat % 8);
  /* j even -> bytes 0,1 ; odd -> bytes 2,3 (quantize.cpp:44-47) */
  const int byte = (j & 1) * 2 + (j >> 2);
  const int hi = (j >> 1) & 1;
  return hi ? (uint8_t)(b[byte] >> 4) : (uint8_t)(b[byte] & 15);
}

/* dequant.cpp:55-112 */
int or_dequantize(const uint8_t* packed, const uint16_t* scales, size_t e,
                  size_t m, size_t n, int bits, int fast, uint16_t* out) {
  if (!(e > 0 && m > 0 && n > 0)) return fail("dequantize: empty tensor");
  if (bits == 4 && n % 8) return fail("dequantize: 4-bit column count not a multiple of 8");
  for (size_t ei = 0; ei < e; ++ei)
    for (size_t mi = 0; mi < m; ++mi)
      for (size_t ni = 0; ni < n; ++ni) {
        const uint16_t v = code_value(code_at(packed, m, n, bits, ei, mi, ni), bits, fast);
        out[(ei * m + mi) * n + ni] = or_half_mul(v, scales[ei * n + ni]);
      }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* LayerNorm: model.cpp:175-195.  Every f32 op rounds separately. */

static void ln_row(const uint16_t* x, size_t d, const uint16_t* g,
                   const uint16_t* b, uint16_t* out) {
  float mean = 0.0f;
  for (size_t i = 0; i < d; ++i) mean += or_half_to_f32(x[i]);
  mean /= (float)d;
  float var = 0.0f;
  for (size_t i = 0; i < d; ++i) {
    const float dx = or_half_to_f32(x[i]) - mean;
    var += dx * dx;
  }
  var /= (float)d;
  const float inv = 1.0f / sqrtf(var + 1e-5f);
  for (size_t i = 0; i < d; ++i) {
    const float y = (or_half_to_f32(x[i]) - mean) * inv * or_half_to_f32(g[i]) +
                    or_half_to_f32(b[i]);
    out[i] = or_f32_to_half(y);
  }
}

int or_layer_norm(const uint16_t* x, size_t T, size_t d, const uint16_t* g,
                  const uint16_t* b, uint16_t* out) {
  for (size_t r = 0; r < T; ++r) ln_row(x + r * d, d, g, b, out + r * d);
  return OR_OK;
}

/* model.cpp:273-297: acc += f32(x)*f32(w) for k ascending, then + bias */
int or_gate_logits(const uint16_t* xn, size_t T, size_t d, const uint16_t* gw,
                   const uint16_t* gb, size_t E, float* logits) {
  for (size_t r = 0; r < T; ++r)
    for (size_t j = 0; j < E; ++j) {
      float acc = 0.0f;
      for (size_t k = 0; k < d; ++k)
        acc += or_half_to_f32(xn[r * d + k]) * or_half_to_f32(gw[k * E + j]);
      logits[r * E + j] = acc + or_half_to_f32(gb[j]);
    }
  return OR_OK;
}

float or_expf(float x) { return expf(x); }

/* routing.cpp:11-41 (top-1), generalised to top-k (see header). */
int or_gate_topk(const float* logits, size_t T, size_t E, int k,
                 uint32_t* expert, uint16_t* scale) {
  if (!(T > 0 && E > 0)) return fail("gate_top1: empty input");
  if (k < 1 || (size_t)k > E) return fail("gate_topk: k must be in [1, n_experts]");
  for (size_t i = 0; i < T * E; ++i)
    if (!isfinite(logits[i])) {
      snprintf(g_err, sizeof g_err, "gate_top1: non-finite logit at row %zu", i / E);
      return OR_EINVAL;
    }
  unsigned char* taken = (unsigned char*)calloc(E, 1);
  for (size_t r = 0; r < T; ++r) {
    const float* l = logits + r * E;
    memset(taken, 0, E);
    for (int s = 0; s < k; ++s) {
      size_t best = E;
      for (size_t j = 0; j < E; ++j) {
        if (taken[j]) continue;
        if (best == E || l[j] > l[best]) best = j; /* strict: ties keep lowest */
      }
      taken[best] = 1;
      expert[r * k + s] = (uint32_t)best;
    }
    const float mx = l[expert[r * k]];
    float sum = 0.0f;
    for (size_t j = 0; j < E; ++j) sum += expf(l[j] - mx);
    for (int s = 0; s < k; ++s) {
      /* s == 0: expf(0) == 1 -> RN16(1/sum), routing.cpp:37-38 */
      const float num = s == 0 ? 1.0f : expf(l[expert[r * k + s]] - mx);
      scale[r * k + s] = or_f32_to_half(num / sum);
    }
  }
  free(taken);
  return OR_OK;
}

/* routing.cpp:43-87: stable counting sort, finished -> key E (tail). */
int or_routing_plan(const uint32_t* expert, const uint8_t* finished, size_t T,
                    int k, size_t E, uint32_t* perm, uint32_t* inv,
                    uint32_t* offsets, uint32_t* active) {
  if (T == 0) return fail("build_routing_plan: no rows");
  const size_t S = T * (size_t)k;
  for (size_t i = 0; i < S; ++i)
    if (expert[i] >= E) return fail("build_routing_plan: expert out of range");
  uint32_t* cnt = (uint32_t*)calloc(E + 1, 4);
  uint32_t* cur = (uint32_t*)calloc(E + 1, 4);
  for (size_t i = 0; i < S; ++i) ++cnt[finished[i / k] ? E : expert[i]];
  uint32_t run = 0;
  for (size_t e = 0; e <= E; ++e) {
    cur[e] = run;
    if (e < E) offsets[e] = run;
    run += cnt[e];
  }
  const uint32_t act = (uint32_t)S - cnt[E];
  offsets[E] = act;
  *active = act;
  for (size_t i = 0; i < S; ++i) {
    const uint32_t pos = cur[finished[i / k] ? E : expert[i]]++;
    perm[pos] = (uint32_t)i;
    inv[i] = pos;
  }
  free(cnt);
  free(cur);
  return OR_OK;
}

size_t or_make_problems(const uint32_t* offsets, size_t E, uint32_t* problems) {
  size_t np = 0;
  for (size_t e = 0; e < E; ++e)
    if (offsets[e] < offsets[e + 1]) {
      problems[3 * np] = (uint32_t)e;
      problems[3 * np + 1] = offsets[e];
      problems[3 * np + 2] = offsets[e + 1];
      ++np;
    }
  return np;
}

void or_permute(const uint16_t* x, size_t cols, const uint32_t* perm, size_t S,
                int k, uint16_t* xp) {
  for (size_t p = 0; p < S; ++p)
    memcpy(xp + p * cols, x + (size_t)(perm[p] / k) * cols, cols * 2);
}

void or_unpermute_scale(const uint16_t* y, size_t T, size_t cols,
                        const uint32_t* perm, uint32_t active,
                        const uint16_t* scale, uint16_t* out) {
  memset(out, 0, T * cols * 2);
  for (size_t i = 0; i < active; ++i) {
    const uint32_t r = perm[i];
    for (size_t c = 0; c < cols; ++c)
      out[r * cols + c] = or_half_mul(y[i * cols + c], scale[r]);
  }
}

/* ------------------------------------------------------------------------ */
/* grouped GEMM: grouped_gemm.cpp:19-214.  Weight staged as f32 of the fp16
 * (dequantized) value; acc k-sequential; + bias; ReLU via !(h > 0); RN16. */

static float weight_f32(int bits, const uint16_t* w16, const uint8_t* packed,
                        const uint16_t* scales, size_t m, size_t n, size_t e,
                        size_t k, size_t j) {
  if (bits == 16) return or_half_to_f32(w16[(e * m + k) * n + j]);
  const uint16_t v = code_value(code_at(packed, m, n, bits, e, k, j), bits, 1);
  return or_half_to_f32(or_half_mul(v, scales[e * n + j]));
}

int or_grouped_gemm(const uint16_t* x, size_t rows, size_t m,
                    const uint32_t* problems, size_t np, int bits,
                    const uint16_t* w16, const uint8_t* packed,
                    const uint16_t* scales, size_t E, size_t n,
                    const uint16_t* bias, int relu, int separate, uint16_t* out,
                    uint64_t* traffic) {
  for (size_t p = 0; p < np; ++p) {
    if (problems[3 * p] >= E) return fail("grouped_gemm: expert out of range");
    if (!(problems[3 * p + 1] <= problems[3 * p + 2] && problems[3 * p + 2] <= rows))
      return fail("grouped_gemm: problem rows out of range");
  }
  memset(out, 0, rows * n * 2);
  float* wcol = (float*)malloc(m * n * sizeof(float));
  uint64_t wb = 0, ab = 0, ob = 0;
  for (size_t p = 0; p < np; ++p) {
    const size_t e = problems[3 * p], r0 = problems[3 * p + 1], r1 = problems[3 * p + 2];
    for (size_t k = 0; k < m; ++k)
      for (size_t j = 0; j < n; ++j)
        wcol[k * n + j] = weight_f32(bits, w16, packed, scales, m, n, e, k, j);
    for (size_t r = r0; r < r1; ++r)
      for (size_t j = 0; j < n; ++j) {
        float acc = 0.0f;
        for (size_t k = 0; k < m; ++k) acc += or_half_to_f32(x[r * m + k]) * wcol[k * n + j];
        float h = acc + or_half_to_f32(bias[e * n + j]);
        if (relu && !(h > 0.0f)) h = 0.0f;
        out[r * n + j] = or_f32_to_half(h);
      }
    const uint64_t nr = r1 - r0;
    if (bits == 16)
      wb += (uint64_t)m * n * 2;
    else
      wb += (uint64_t)(bits == 8 ? m * n : m * n / 2) + (uint64_t)n * 2;
    ab += (nr * m + n) * 2;
    ob += nr * n * 2;
    if (separate && bits != 16) {
      wb += (uint64_t)m * n * 2;
      ob += (uint64_t)m * n * 2;
    }
  }
  free(wcol);
  if (traffic) {
    traffic[0] = wb;
    traffic[1] = ab;
    traffic[2] = ob;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* whole layer: model.cpp:299-349 (batched, top-k extension) */

int or_moe_forward(const or_layer* L, const uint16_t* x, size_t T,
                   const uint8_t* finished, int k, uint16_t* out,
                   uint32_t* expert_o, uint16_t* scale_o, uint32_t* perm_o,
                   uint32_t* inv_o, uint32_t* offsets_o, uint32_t* active_o) {
  const size_t d = L->d, f = L->f, E = L->E, S = T * (size_t)k;
  int st = OR_OK;
  uint16_t* xn = (uint16_t*)malloc(T * d * 2);
  float* logits = (float*)malloc(T * E * 4);
  uint32_t* ex = (uint32_t*)malloc(S * 4);
  uint16_t* sc = (uint16_t*)malloc(S * 2);
  uint32_t* perm = (uint32_t*)malloc(S * 4);
  uint32_t* inv = (uint32_t*)malloc(S * 4);
  uint32_t* offs = (uint32_t*)malloc((E + 1) * 4);
  uint32_t* probs = (uint32_t*)malloc(3 * E * 4);
  uint16_t* xp = (uint16_t*)malloc(S * d * 2);
  uint16_t* h = (uint16_t*)malloc(S * f * 2);
  uint16_t* y = (uint16_t*)malloc(S * d * 2);
  uint32_t active = 0;
  or_layer_norm(x, T, d, L->ln_g, L->ln_b, xn);
  or_gate_logits(xn, T, d, L->gw, L->gb, E, logits);
  st = or_gate_topk(logits, T, E, k, ex, sc);
  if (st == OR_OK) st = or_routing_plan(ex, finished, T, k, E, perm, inv, offs, &active);
  if (st == OR_OK) {
    const size_t np = or_make_problems(offs, E, probs);
    or_permute(xn, d, perm, S, k, xp);
    st = or_grouped_gemm(xp, S, d, probs, np, L->bits, L->w1, L->q1, L->s1, E, f, L->b1,
                         1, 0, h, NULL);
    if (st == OR_OK)
      st = or_grouped_gemm(h, S, f, probs, np, L->bits, L->w2, L->q2, L->s2, E, d, L->b2,
                           0, 0, y, NULL);
  }
  if (st == OR_OK) {
    for (size_t r = 0; r < T; ++r) {
      uint16_t* o = out + r * d;
      memcpy(o, x + r * d, d * 2);
      if (finished[r]) continue;
      for (int s = 0; s < k; ++s) {
        const uint16_t* yr = y + (size_t)inv[r * k + s] * d;
        for (size_t c = 0; c < d; ++c) o[c] = or_half_add(o[c], or_half_mul(yr[c], sc[r * k + s]));
      }
    }
    if (expert_o) memcpy(expert_o, ex, S * 4);
    if (scale_o) memcpy(scale_o, sc, S * 2);
    if (perm_o) memcpy(perm_o, perm, S * 4);
    if (inv_o) memcpy(inv_o, inv, S * 4);
    if (offsets_o) memcpy(offsets_o, offs, (E + 1) * 4);
    if (active_o) *active_o = active;
  }
  free(xn); free(logits); free(ex); free(sc); free(perm); free(inv);
  free(offs); free(probs); free(xp); free(h); free(y);
  return st;
}

/* reference.cpp:167-239: one token at a time, no routing machinery. */
int or_moe_per_token(const or_layer* L, const uint16_t* x, size_t T,
                     const uint8_t* finished, int k, uint16_t* out) {
  const size_t d = L->d, f = L->f, E = L->E;
  uint16_t* xn = (uint16_t*)malloc(d * 2);
  float* lg = (float*)malloc(E * 4);
  uint32_t* ex = (uint32_t*)malloc((size_t)k * 4);
  uint16_t* sc = (uint16_t*)malloc((size_t)k * 2);
  uint16_t* h = (uint16_t*)malloc(f * 2);
  uint16_t* y = (uint16_t*)malloc(d * 2);
  int st = OR_OK;
  for (size_t r = 0; r < T && st == OR_OK; ++r) {
    uint16_t* o = out + r * d;
    memcpy(o, x + r * d, d * 2);
    if (finished[r]) continue;
    ln_row(x + r * d, d, L->ln_g, L->ln_b, xn);
    or_gate_logits(xn, 1, d, L->gw, L->gb, E, lg);
    st = or_gate_topk(lg, 1, E, k, ex, sc);
    for (int s = 0; s < k && st == OR_OK; ++s) {
      const uint32_t e = ex[s];
      uint32_t prob[3] = {e, 0, 1};
      st = or_grouped_gemm(xn, 1, d, prob, 1, L->bits, L->w1, L->q1, L->s1, E, f, L->b1, 1,
                           0, h, NULL);
      if (st == OR_OK)
        st = or_grouped_gemm(h, 1, f, prob, 1, L->bits, L->w2, L->q2, L->s2, E, d, L->b2,
                             0, 0, y, NULL);
      for (size_t c = 0; c < d; ++c) o[c] = or_half_add(o[c], or_half_mul(y[c], sc[s]));
    }
  }
  free(xn); free(lg); free(ex); free(sc); free(h); free(y);
  return st;
}
