/* oracle/moe_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C11, scalar, single-threaded) of the reference's
 * MoE-layer hot path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER.  The product path never links or calls
 * it.  Each function cites the reference file:line it restates (paths are
 * relative to /root/reference/proj).
 *
 * Parity pinning: checked against the reference's own known-answer tests
 * (tests/test_oracle_golden.py) and against the compiled reference
 * (oracle/_ref/libmoeref.so, tests/test_oracle_vs_ref.py, plus committed
 * fixtures under tests/golden/ produced by tests/golden/make_golden.py).
 *
 * The top-k (k > 1) gating and slot-ordered combine are an EXTENSION: the
 * reference is top-1 only.  Conventions: slots
 * chosen by repeated argmax (strict '>', ties -> lowest index); softmax over
 * all E experts with the top-1 logit subtracted; slot scale
 * RN16(RN32(expf(l_s - mx) / sum)); plan = stable counting sort over slot
 * index r*k+s; combine folds slots in order with fp16 rounding per step.
 * For k == 1 every one of these reduces to the reference exactly.
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes, same meaning as include/moe_cuda.h */
#define OR_OK 0
#define OR_EINVAL 1

const char* or_last_error(void);

/* ---- binary16 helpers (include/moeinfer/half.hpp:57-146) ---- */
float or_half_to_f32(uint16_t h);
uint16_t or_f64_to_half(double x);
uint16_t or_f32_to_half(float x);
uint16_t or_half_add(uint16_t a, uint16_t b);
uint16_t or_half_sub(uint16_t a, uint16_t b);
uint16_t or_half_mul(uint16_t a, uint16_t b);

/* ---- quantizer (src/quantize.cpp:14-122) ---- */
uint16_t or_quant_scale(float maxabs, int qmax);
uint8_t or_quant_encode(uint16_t w, uint16_t scale, int bits);
int or_pack_int4(const uint8_t* values, size_t count, uint8_t* out);
int or_unpack_int4(const uint8_t* packed, size_t count, uint8_t* out);
int or_quantize(const uint16_t* w, size_t e, size_t m, size_t n, int bits,
                uint8_t* packed, uint16_t* scales);

/* ---- dequantizer (include/moeinfer/dequant.hpp:39-70, src/dequant.cpp:45-112) */
uint16_t or_debias_u8(void);
uint16_t or_debias_u4(void);
int or_dequantize(const uint8_t* packed, const uint16_t* scales, size_t e,
                  size_t m, size_t n, int bits, int fast, uint16_t* out);

/* ---- LayerNorm + gate (src/model.cpp:175-205, 273-297) ---- */
int or_layer_norm(const uint16_t* x, size_t T, size_t d, const uint16_t* gamma,
                  const uint16_t* beta, uint16_t* out);
int or_gate_logits(const uint16_t* xn, size_t T, size_t d, const uint16_t* gw,
                   const uint16_t* gb, size_t E, float* logits);

/* ---- gating (src/routing.cpp:11-41, top-k extension) ---- */
int or_gate_topk(const float* logits, size_t T, size_t E, int k,
                 uint32_t* expert, uint16_t* scale);

/* ---- routing plan (src/routing.cpp:43-87) over S = T*k slots ---- */
int or_routing_plan(const uint32_t* expert, const uint8_t* finished, size_t T,
                    int k, size_t E, uint32_t* perm, uint32_t* inv,
                    uint32_t* offsets, uint32_t* active);
/* make_grouped_problems (src/grouped_gemm.cpp:109-121); returns count */
size_t or_make_problems(const uint32_t* offsets, size_t E, uint32_t* problems);
/* permute_rows (src/routing.cpp:89-97): xp[p] = x[perm[p] / k] */
void or_permute(const uint16_t* x, size_t cols, const uint32_t* perm, size_t S,
                int k, uint16_t* xp);
/* unpermute_and_scale (src/routing.cpp:99-116), k == 1 form */
void or_unpermute_scale(const uint16_t* y, size_t T, size_t cols,
                        const uint32_t* perm, uint32_t active,
                        const uint16_t* scale, uint16_t* out);

/* ---- grouped GEMM (src/grouped_gemm.cpp:19-214) ----
 * problems: np triples (expert, row_begin, row_end).  weights: bits == 16
 * -> fp16 (E,m,n) in w16; bits 8/4 -> reference-packed codes + scales.
 * traffic (may be NULL): weight, activation, written bytes (analytic,
 * src/grouped_gemm.cpp:155-160, 201-211); separate != 0 adds the
 * separate-pass bytes. */
int or_grouped_gemm(const uint16_t* x, size_t rows, size_t m,
                    const uint32_t* problems, size_t np, int bits,
                    const uint16_t* w16, const uint8_t* packed,
                    const uint16_t* scales, size_t E, size_t n,
                    const uint16_t* bias, int relu, int separate,
                    uint16_t* out, uint64_t* traffic);

/* ---- whole MoE layer (src/model.cpp:299-349 + top-k extension) ---- */
typedef struct {
  size_t d, f, E;
  int bits; /* 16, 8 or 4 */
  const uint16_t *ln_g, *ln_b, *gw, *gb, *b1, *b2;
  const uint16_t *w1, *w2;          /* bits == 16 */
  const uint8_t *q1, *q2;           /* bits 8/4: reference layout */
  const uint16_t *s1, *s2;
} or_layer;

/* out: T x d fp16.  Optional diagnostics (may be NULL): expert/scale T*k,
 * perm/inv T*k, offsets E+1, active. */
int or_moe_forward(const or_layer* L, const uint16_t* x, size_t T,
                   const uint8_t* finished, int k, uint16_t* out,
                   uint32_t* expert, uint16_t* scale, uint32_t* perm,
                   uint32_t* inv, uint32_t* offsets, uint32_t* active);

/* ref::moe_per_token (src/reference.cpp:167-239), generalised to top-k. */
int or_moe_per_token(const or_layer* L, const uint16_t* x, size_t T,
                     const uint8_t* finished, int k, uint16_t* out);

/* glibc expf as the reference calls it (routing.cpp:34); exported so tests
 * can compare the device port against it. */
float or_expf(float x);

#ifdef __cplusplus
}
#endif
#endif
