// k_ln_gate.cu -- K2 gating as ONE kernel per block of token rows:
//   LayerNorm (proj/src/model.cpp:175-205) -> f32 gate logits (:273-297) ->
//   top-k softmax gate (proj/src/routing.cpp:11-41, top-k extension) ->
//   per-block routing-key histogram (routing.cpp:55-62, first counting-sort
//   pass, consumed by plan_scan in k_route.cu).  Bit-exact with the oracle.
//
// Everything on this path is a serial f32 chain: per row the LN mean and
// variance chains (2*d dependent FADDs), per (row, expert) the k-ordered
// logit chain (d dependent FMAs -- fp16 x fp16 products are exact in f32, so
// fmaf == the reference's multiply-then-add).  The floor is therefore chain
// LATENCY (~4 cycles per step), not bandwidth or FLOPs, unless the chains
// outnumber the FMA lanes.  The kernel is sized for that:
//
// * rb rows per CTA, rb = ceil(T / (148 * waves)) -- every SM gets rows, one
//   CTA per SM; waves > 1 only when the rows' fp16 copies exceed the
//   shared-memory budget (d = 1024: 79 rows).
// * The rows arrive by bulk copies issued by one elected lane; the f32 gate
//   weights stream through a ring of bulk-copied k-chunks (the whole matrix
//   when it fits, E = 8 / d = 512: 16 KB).
// * LN: one thread per row runs both chains over the fp16 row (conversion
//   inline, loads prefetched); then all threads normalise in place (fp16 xn
//   stays in shared memory for the logits) and write xn for the FFN gather.
// * Logits: a thread owns RPT rows x EPG experts of chains (EPG >= 2 as
//   FFMA2 pairs).  (EPG, RPT) is the smallest that fits 256 threads, so small
//   T runs many short-latency threads and large T few FMA-dense ones.
// * Tail: logits + bias -> shared memory; selection (strict '>', first
//   maximum) one thread per row; every expf (glibc port) in parallel; the
//   softmax denominator summed serially per row in expert order; scales,
//   expert ids and the key histogram.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace moecu {

namespace g3 {
constexpr int kMaxRows = 256;
constexpr size_t kXBudget = 160 * 1024;   // fp16 rows in shared memory
constexpr size_t kXfBudget = 64 * 1024;   // f32 row copies for the LN chains
constexpr size_t kWBudget = 128 * 1024;   // f32 gate weights resident whole
constexpr size_t kSmemMax = 220 * 1024;

struct Cfg {
  int nt, rb, epg, rpt, ng, nrg, ntask, kc, nch, ns, xp, wide;
  size_t off_xf, off_w, wslot, off_st, off_sel, off_hist, off_gb, off_bias, off_tab, off_fin,
      off_bar, total;
};

// nt threads; wide: the LN chains read an f32 copy of the rows (and of the
// squared deviations) made by all threads, so the chain thread issues only
// its dependent FADDs
__host__ __device__ inline Cfg cfg1(int64_t d, int64_t E, int64_t gwp, int rb, int epg, int rpt,
                                    int nt, bool whole, int maxns = 3) {
  Cfg c;
  c.nt = nt;
  c.rb = rb;
  c.epg = epg;
  c.rpt = rpt;
  c.ng = (int)((E + epg - 1) / epg);
  c.nrg = (rb + rpt - 1) / rpt;
  c.ntask = c.ng * c.nrg;
  // the whole weight matrix when it fits (no per-chunk barriers), else
  // 16 KB chunks through a ring of up to maxns slots
  int kc = whole && (size_t)d * gwp * 4 <= kWBudget ? (int)d : (int)(16384 / (gwp * 4)) / 8 * 8;
  if (kc < 8) kc = 8;
  if (kc > d) kc = (int)d;  // d % 8 == 0
  c.kc = kc;
  c.nch = (int)((d + kc - 1) / kc);
  c.ns = c.nch < maxns ? c.nch : maxns;
  c.xp = (int)d + 8;  // 16-byte row pitch, rows on distinct 16-byte bank groups
  // (rb + rpt) rows + slack: a thread's last row group and the operand
  // prefetch may read past the rows (never used)
  const size_t xbytes = ((size_t)(rb + rpt) * c.xp * 2 + 256 + 127) & ~size_t(127);
  const size_t xf = (size_t)rb * (d + 4) * 4;  // pitch d + 4: chain rows on distinct banks
  c.wide = xf <= kXfBudget ? 1 : 0;
  c.off_xf = xbytes;
  c.off_w = c.off_xf + (c.wide ? (xf + 127) & ~size_t(127) : 0);
  c.wslot = (size_t)kc * gwp * 4;
  const size_t wring = (size_t)c.ns * c.wslot + (size_t)48 * gwp * 4;  // + prefetch slack
  const size_t lg = (size_t)2 * rb * (E + 1) * 4;  // logits | expf values (reuse the ring)
  const size_t body = (wring > lg ? wring : lg) + 64;
  c.off_st = (c.off_w + body + 15) & ~size_t(15);
  c.off_sel = c.off_st + (size_t)2 * rb * 4;
  c.off_hist = c.off_sel + (size_t)rb * 8 * 4;
  c.off_gb = (c.off_hist + (size_t)(E + 1) * 4 + 15) & ~size_t(15);  // LN gamma | beta, f32
  c.off_bias = c.off_gb + (size_t)2 * d * 4;
  c.off_tab = (c.off_bias + (size_t)E * 4 + 15) & ~size_t(15);
  c.off_fin = c.off_tab + 32 * 8;
  c.off_bar = (c.off_fin + rb + 15) & ~size_t(15);
  c.total = c.off_bar + (size_t)(1 + c.ns) * 8 + 16;  // rows barrier + one per slot
  return c;
}
__host__ __device__ inline Cfg cfg(int64_t d, int64_t E, int64_t gwp, int rb, int epg, int rpt,
                                   int nt) {
  const Cfg c = cfg1(d, E, gwp, rb, epg, rpt, nt, true);
  if (c.total <= kSmemMax) return c;
  // chunked weights: the deepest ring that fits (each 16 KB chunk is an L2
  // round trip; C4's 256 KB of f32 gate weights stream 16 chunks per CTA)
  for (int ns = 8; ns > 3; --ns) {
    const Cfg r = cfg1(d, E, gwp, rb, epg, rpt, nt, false, ns);
    if (r.total <= kSmemMax) return r;
  }
  return cfg1(d, E, gwp, rb, epg, rpt, nt, false, 3);
}

// c += a * b on two lanes (FFMA2), each RN: exact products, k order per chain
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  uint64_t r;
  const uint64_t bb = (uint64_t)__float_as_uint(b.x) | ((uint64_t)__float_as_uint(b.y) << 32);
  const uint64_t cc = (uint64_t)__float_as_uint(c.x) | ((uint64_t)__float_as_uint(c.y) << 32);
  const uint64_t aa = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
  return make_float2(__uint_as_float((uint32_t)r), __uint_as_float((uint32_t)(r >> 32)));
}

__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
}  // namespace g3

// dev-only trace (MOE_GATE_TRACE): [0..7] CTA 0 phase clocks, [16 + 2b] per-CTA
// global-time span
#define G3_TRACE(i)                                                                \
  do {                                                                             \
    if (trace != nullptr && tid == 0) {                                            \
      if ((i) == 0) trace[16 + 2 * blockIdx.x] = g3::gtime();                      \
      if ((i) == 5) trace[16 + 2 * blockIdx.x + 1] = g3::gtime();                  \
      if (blockIdx.x == 0) trace[i] = clock64();                                   \
    }                                                                              \
  } while (0)

// One weight chunk of the logit chains: inputs [0, kn) of the rows
// xr + i*rstride (i < RPT; f32 when XF, else fp16) against the pair-blocked
// weights wg.  Operands of KS inputs per step stream through a DEPTH-step
// register ring with no branches in the loop body (a guarded load lets
// ptxas sink it under the previous step's FMAs); loads past kn read padding
// and are never used.  x arrives converted (f32 copy) when XF.
template <int EPG, int RPT, int KS, int DEPTH, bool XF>
__device__ __forceinline__ void logit_chunk(float2 (&acc)[RPT][EPG >= 2 ? EPG / 2 : 1],
                                            const void* xr, int rstride, const float* wg,
                                            int wstride, int kn) {
  constexpr int NP = EPG >= 2 ? EPG / 2 : 1;
  struct Step {
    float x[RPT][KS];
    uint32_t xh[RPT][KS / 2];
    float w[KS][EPG];
  };
  auto load = [&](Step& o, int kk) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if constexpr (XF) {
        const float* p = reinterpret_cast<const float*>(xr) + (size_t)i * rstride + kk;
#pragma unroll
        for (int q = 0; q < KS; q += 4) {
          const float4 v = *reinterpret_cast<const float4*>(p + q);
          o.x[i][q] = v.x;
          o.x[i][q + 1] = v.y;
          o.x[i][q + 2] = v.z;
          o.x[i][q + 3] = v.w;
        }
      } else {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(xr) + (size_t)i * rstride + kk;
        if constexpr (KS == 8) {
          const uint4 v = *reinterpret_cast<const uint4*>(p);
          o.xh[i][0] = v.x;
          o.xh[i][1] = v.y;
          o.xh[i][2] = v.z;
          o.xh[i][3] = v.w;
        } else {
          const uint2 v = *reinterpret_cast<const uint2*>(p);
          o.xh[i][0] = v.x;
          o.xh[i][1] = v.y;
        }
      }
    }
    const float* w0 = wg + (size_t)(kk >> 1) * wstride;
#pragma unroll
    for (int q = 0; q < KS; q += 2) {  // one input pair: 2 * EPG floats
      const float* wq = w0 + (q >> 1) * wstride;
      if constexpr (EPG == 1) {
        // expert e0 inside its expert pair: inputs q, q+1 are 2 floats apart
        // (wg was shifted back by e0 & 1 by the caller)
        o.w[q][0] = wq[0];
        o.w[q + 1][0] = wq[2];
      } else {
#pragma unroll
        for (int j = 0; j < EPG; j += 2) {  // experts e0+j, e0+j+1 x inputs q, q+1
          const float4 w4 = *reinterpret_cast<const float4*>(wq + 2 * j);
          o.w[q][j] = w4.x;
          o.w[q][j + 1] = w4.y;
          o.w[q + 1][j] = w4.z;
          o.w[q + 1][j + 1] = w4.w;
        }
      }
    }
  };
  auto fma_step = [&](const Step& o) {
#pragma unroll
    for (int q = 0; q < KS; ++q) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        float xq;
        if constexpr (XF) {
          xq = o.x[i][q];
        } else {
          const uint32_t hw = o.xh[i][q / 2];
          xq = h2f((uint16_t)((q & 1) ? (hw >> 16) : (hw & 0xFFFFu)));
        }
        if constexpr (EPG == 1) {
          // one chain per thread: plain FFMA (half the dependent latency of
          // FFMA2 -- the latency-bound small-T configs)
          acc[i][0].x = fmaf(xq, o.w[q][0], acc[i][0].x);
        } else {
#pragma unroll
          for (int j = 0; j < NP; ++j)
            acc[i][j] = g3::ffma2(xq, make_float2(o.w[q][2 * j], o.w[q][2 * j + 1]), acc[i][j]);
        }
      }
    }
  };
  Step r[DEPTH];
#pragma unroll
  for (int d = 0; d < DEPTH; ++d) load(r[d], d * KS);
  int kk = 0;
  for (; kk + DEPTH * KS <= kn; kk += DEPTH * KS) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      fma_step(r[d]);
      load(r[d], kk + (DEPTH + d) * KS);
    }
  }
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)  // remaining kn % (DEPTH * KS) inputs (multiple of 8)
    if (kk + d * KS < kn) fma_step(r[d]);
}

// LNONLY: the LayerNorm half alone (xn to global, finished-row passthrough)
// for the wide-gate path (k_gate_tile.cu): no gate weights, E = gwp = 0;
// a lean instantiation that fits three CTAs per SM
template <int EPG, int RPT, int NT, bool LNONLY = false>
__global__ void __launch_bounds__(NT, LNONLY ? 3 : 1) ln_gate_kernel(
    const uint16_t* __restrict__ x, int64_t T, int d, const uint16_t* __restrict__ lng,
    const uint16_t* __restrict__ lnb, const float* __restrict__ gw32, int gwp,
    const uint16_t* __restrict__ gb, int E, int k, const uint8_t* __restrict__ finished,
    uint16_t* __restrict__ xn, uint32_t* __restrict__ expert, uint16_t* __restrict__ scale,
    uint32_t* __restrict__ blockcnt, uint32_t* bad_row, int rb, uint16_t* __restrict__ out_fin,
    long long* trace, int pdl, int ln_wide) {
  extern __shared__ __align__(128) uint8_t sm[];
  const g3::Cfg C = g3::cfg(d, E, gwp, rb, EPG, RPT, NT);
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm);
  float* xf = reinterpret_cast<float*>(sm + C.off_xf);  // [rb][d + 4] (wide form only)
  const int fp = d + 4;
  float* st = reinterpret_cast<float*>(sm + C.off_st);  // mean[rb] | inv[rb]
  uint32_t* sel = reinterpret_cast<uint32_t*>(sm + C.off_sel);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + C.off_hist);
  float* gsm = reinterpret_cast<float*>(sm + C.off_gb);  // gamma[d] | beta[d]
  float* bsm = reinterpret_cast<float*>(sm + C.off_bias);
  uint64_t* tab = reinterpret_cast<uint64_t*>(sm + C.off_tab);
  uint8_t* fsm = sm + C.off_fin;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C.off_bar);  // [0] rows, [1 + s] weight slots
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * rb;
  const int nrow = (int)::min((int64_t)rb, T - r0);
  const int d8 = d / 8, xp = C.xp;
  G3_TRACE(0);

  griddep_launch();
  if (tid < 32) {  // warp 0 converged, one elected lane issues every copy
    if (elect_one()) {
      mbar_init(&bars[0], 1);
      for (int s = 0; s < C.ns; ++s) mbar_init(&bars[1 + s], 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(&bars[0], (uint32_t)nrow * d * 2);
    }
    __syncwarp();
    auto weights = [&] {
      for (int c = 0; c < C.ns; ++c) {
        const uint32_t bytes = (uint32_t)::min(C.kc, d - c * C.kc) * gwp * 4;
        if (elect_one()) {
          mbar_arrive_expect_tx(&bars[1 + c], bytes);
          bulk_load(sm + C.off_w + c * C.wslot, gw32 + (size_t)c * C.kc * gwp, bytes, &bars[1 + c]);
        }
      }
    };
    // launched early (PDL): the gate weights never change, fetch them while
    // the previous kernel retires; otherwise the rows first (the LN chains
    // wait on them; the weights are needed only by the logit phase)
    if (!LNONLY && pdl) weights();
    griddep_wait();  // x and finished may be the previous kernel's output
    for (int r = tid; r < nrow; r += 32)
      bulk_load(xs + (size_t)r * xp, x + (r0 + r) * d, (uint32_t)d * 2, &bars[0]);
    __syncwarp();
    if (!LNONLY && !pdl) weights();
  } else {
    // the small operands every later phase reads, fetched while the rows
    // land (each would otherwise cost an L2 round trip on the critical path)
    for (int i = tid - 32; i < 2 * d8; i += NT - 32) {  // 16-byte loads, all in flight
      const int c = i < d8 ? i : i - d8;
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(i < d8 ? lng : lnb) + c);
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
      float4* o = reinterpret_cast<float4*>(gsm + (i < d8 ? 0 : d) + c * 8);
      o[0] = make_float4(h2f(h[0]), h2f(h[1]), h2f(h[2]), h2f(h[3]));
      o[1] = make_float4(h2f(h[4]), h2f(h[5]), h2f(h[6]), h2f(h[7]));
    }
    for (int i = tid - 32; i < E; i += NT - 32) bsm[i] = h2f(gb[i]);
    for (int i = tid - 32; i < 32; i += NT - 32) tab[i] = moe_expf_tab_dev[i];
    griddep_wait();
    for (int i = tid - 32; i < nrow; i += NT - 32) fsm[i] = finished != nullptr ? finished[r0 + i] : 0;
  }
  for (int i = tid; i <= E; i += NT) hist[i] = 0;
  __syncthreads();
  mbar_wait_warp(&bars[0], 0);
  G3_TRACE(1);
  if (out_fin != nullptr) {  // fused k = 1 combine: finished tokens pass through (out = x)
    for (int i = tid; i < nrow * d8; i += NT) {
      const int r = i / d8, c = i - r * d8;
      if (fsm[r] != 0)
        *reinterpret_cast<uint4*>(out_fin + (r0 + r) * d + c * 8) =
            *reinterpret_cast<const uint4*>(xs + (size_t)r * xp + c * 8);
    }
  }

  // ---- LayerNorm chains (model.cpp:178-192): one thread per row, serial RN.
  // ln_wide (few rows per CTA): all threads first widen the rows to f32 and
  // later write the squared deviations, so the chain threads issue only
  // FADDs; otherwise the chain threads convert the fp16 row inline (the
  // conversion, dx and dx*dx sit off the dependent FADD chain) -- with 28
  // rows per CTA (C2) the two extra passes cost 1790 + 1975 cycles.
  if (C.wide && ln_wide) {
    for (int i = tid; i < nrow * d8; i += NT) {  // widen (exact)
      const int r = i / d8, c = i - r * d8;
      const uint4 v = *reinterpret_cast<const uint4*>(xs + (size_t)r * xp + c * 8);
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
      float4* dst = reinterpret_cast<float4*>(xf + (size_t)r * fp + c * 8);
      dst[0] = make_float4(h2f(h[0]), h2f(h[1]), h2f(h[2]), h2f(h[3]));
      dst[1] = make_float4(h2f(h[4]), h2f(h[5]), h2f(h[6]), h2f(h[7]));
    }
    __syncthreads();
    G3_TRACE(8);
    const int d4 = d / 4;
    if (tid < nrow) {  // sum chain: loads run three pieces ahead of the FADDs
      const float4* row = reinterpret_cast<const float4*>(xf + (size_t)tid * fp);
      float s = 0.f;
      float4 c0 = row[0], c1 = row[::min(1, d4 - 1)], c2 = row[::min(2, d4 - 1)];
      for (int c = 0; c < d4; ++c) {
        const float4 v = c0;
        c0 = c1;
        c1 = c2;
        c2 = row[::min(c + 3, d4 - 1)];
        s = __fadd_rn(s, v.x);
        s = __fadd_rn(s, v.y);
        s = __fadd_rn(s, v.z);
        s = __fadd_rn(s, v.w);
      }
      st[tid] = __fdiv_rn(s, (float)d);
    }
    if (tid == 0) G3_TRACE(9);
    __syncthreads();
    G3_TRACE(10);
    for (int i = tid; i < nrow * d4; i += NT) {  // squared deviations, in place
      const int r = i / d4;
      float4* p = reinterpret_cast<float4*>(xf + (size_t)r * fp + (size_t)(i - r * d4) * 4);
      const float mean = st[r];
      float4 v = *p;
      const float a = __fsub_rn(v.x, mean), b = __fsub_rn(v.y, mean);
      const float c = __fsub_rn(v.z, mean), e = __fsub_rn(v.w, mean);
      v = make_float4(__fmul_rn(a, a), __fmul_rn(b, b), __fmul_rn(c, c), __fmul_rn(e, e));
      *p = v;
    }
    __syncthreads();
    G3_TRACE(11);
    if (tid < nrow) {
      const float4* row = reinterpret_cast<const float4*>(xf + (size_t)tid * fp);
      float v2 = 0.f;
      float4 c0 = row[0], c1 = row[::min(1, d4 - 1)], c2 = row[::min(2, d4 - 1)];
      for (int c = 0; c < d4; ++c) {
        const float4 v = c0;
        c0 = c1;
        c1 = c2;
        c2 = row[::min(c + 3, d4 - 1)];
        v2 = __fadd_rn(v2, v.x);
        v2 = __fadd_rn(v2, v.y);
        v2 = __fadd_rn(v2, v.z);
        v2 = __fadd_rn(v2, v.w);
      }
      st[rb + tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v2, (float)d), 1e-5f)));
    }
  } else if (tid < nrow) {
    // 8 inputs per 16-byte load, two loads ahead of the FADDs
    const uint4* row = reinterpret_cast<const uint4*>(xs + (size_t)tid * xp);
    float s = 0.f;
    uint4 c0 = row[0], c1 = row[d8 > 1 ? 1 : 0];
    for (int c = 0; c < d8; ++c) {
      const uint4 cur = c0;
      c0 = c1;
      c1 = row[c + 2 < d8 ? c + 2 : d8 - 1];
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&cur);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __fadd_rn(s, h2f(h[i]));
    }
    const float mean = __fdiv_rn(s, (float)d);
    G3_TRACE(9);
    float v2 = 0.f;
    c0 = row[0];
    c1 = row[d8 > 1 ? 1 : 0];
    for (int c = 0; c < d8; ++c) {
      const uint4 cur = c0;
      c0 = c1;
      c1 = row[c + 2 < d8 ? c + 2 : d8 - 1];
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&cur);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float dx = __fsub_rn(h2f(h[i]), mean);
        v2 = __fadd_rn(v2, __fmul_rn(dx, dx));
      }
    }
    st[tid] = mean;
    st[rb + tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v2, (float)d), 1e-5f)));
  }
  __syncthreads();
  G3_TRACE(2);

  // ---- normalise in place (model.cpp:193-194); xn also to global for the
  // gather.  A thread owns one 8-column chunk (gamma / beta in registers)
  // over every rsplit-th row: no per-element index division, and a row's
  // chunks are one coalesced store per warp
  {
    const int rsplit = d8 >= NT ? 1 : NT / d8;
    for (int q = tid; q < d8 * rsplit; q += NT) {
      const int c = q % d8, rs = q / d8;
      const float4 g0 = reinterpret_cast<const float4*>(gsm)[2 * c];
      const float4 g1 = reinterpret_cast<const float4*>(gsm)[2 * c + 1];
      const float4 b0 = reinterpret_cast<const float4*>(gsm + d)[2 * c];
      const float4 b1 = reinterpret_cast<const float4*>(gsm + d)[2 * c + 1];
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
      const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      for (int r = rs; r < nrow; r += rsplit) {
        uint4 v = *reinterpret_cast<const uint4*>(xs + (size_t)r * xp + c * 8);
        uint16_t* h = reinterpret_cast<uint16_t*>(&v);
        const float mean = st[r], inv = st[rb + r];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          h[j] = f2h(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(h2f(h[j]), mean), inv), gg[j]), bb[j]));
        *reinterpret_cast<uint4*>(xn + (r0 + r) * d + c * 8) = v;
        if constexpr (!LNONLY) {
          *reinterpret_cast<uint4*>(xs + (size_t)r * xp + c * 8) = v;
          if (C.wide) {  // f32 copy for the logit chains (no conversion on their path)
            float4* dst = reinterpret_cast<float4*>(xf + (size_t)r * fp + c * 8);
            dst[0] = make_float4(h2f(h[0]), h2f(h[1]), h2f(h[2]), h2f(h[3]));
            dst[1] = make_float4(h2f(h[4]), h2f(h[5]), h2f(h[6]), h2f(h[7]));
          }
        }
      }
    }
  }
  __syncthreads();
  G3_TRACE(3);
  if constexpr (LNONLY) {
    G3_TRACE(5);
    return;
  }

  // ---- logit chains (model.cpp:273-297): RPT rows x EPG experts per thread.
  // Operands of KS inputs per step; with few chains per thread the chain
  // latency leaves room for a three-step-deep prefetch ring.
  constexpr int NP = EPG >= 2 ? EPG / 2 : 1;
  constexpr int KS = EPG * RPT <= 4 ? 8 : 4;
  const int rg = tid % C.nrg, eg = tid / C.nrg, e0 = eg * EPG;
  const bool active = tid < C.ntask;
  float2 acc[RPT][NP];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[i][j] = make_float2(0.f, 0.f);

  for (int c = 0; c < C.nch; ++c) {
    const int s = c % C.ns;
    mbar_wait_warp(&bars[1 + s], (uint32_t)((c / C.ns) & 1));
    if (active) {
      // weights blocked by (input pair, expert pair) (k_gate_fused.cu):
      // inputs 2j, 2j+1 of experts e0.. are the contiguous floats
      // [j * 2 * gwp + 2 * e0, ... + 2 * EPG)
      // EPG = 1: an odd expert's floats start one before 2 * e0 in its pair
      const float* wg = reinterpret_cast<const float*>(sm + C.off_w + s * C.wslot) + 2 * e0 -
                        (EPG == 1 ? (e0 & 1) : 0);
      const int kn = ::min(C.kc, d - c * C.kc);  // multiple of 8
      if (C.wide)  // f32 copy of xn (written by the normalise pass)
        logit_chunk<EPG, RPT, KS, (EPG * RPT <= 2 ? 4 : 2), true>(
            acc, xf + (size_t)rg * fp + c * C.kc, C.nrg * fp, wg, 2 * gwp, kn);
      else
        logit_chunk<EPG, RPT, KS, 2, false>(acc, xs + (size_t)rg * xp + c * C.kc, C.nrg * xp,
                                            wg, 2 * gwp, kn);
    }
    __syncthreads();  // slot s fully read
    if (c + C.ns < C.nch && tid < 32) {
      const int cn = c + C.ns;
      const uint32_t bytes = (uint32_t)::min(C.kc, d - cn * C.kc) * gwp * 4;
      if (elect_one()) {
        mbar_arrive_expect_tx(&bars[1 + s], bytes);
        bulk_load(sm + C.off_w + s * C.wslot, gw32 + (size_t)cn * C.kc * gwp, bytes, &bars[1 + s]);
      }
      __syncwarp();
    }
  }
  G3_TRACE(4);

  // ---- logits + bias into shared memory (the weight ring is drained)
  float* lg = reinterpret_cast<float*>(sm + C.off_w);
  const int lp = E + 1;
  float* ex = lg + (size_t)rb * lp;
  if (active) {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = rg + i * C.nrg;
#pragma unroll
      for (int j = 0; j < EPG; ++j) {
        const float a = (j & 1) ? acc[i][j / 2].y : acc[i][j / 2].x;
        if (e0 + j < E && r < nrow) lg[r * lp + e0 + j] = __fadd_rn(a, bsm[e0 + j]);
      }
    }
  }
  __syncthreads();

  // ---- top-k selection (routing.cpp:15-31): strict '>', lowest index first
  if (E <= 16) {
    if (tid < nrow) {
      const float* l = lg + tid * lp;
      float lv[16];
      bool ok = true;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        lv[j] = j < E ? l[j] : 0.f;
        ok &= j >= E || isfinite(lv[j]);
      }
      if (!ok) {
        atomicMin(bad_row, (uint32_t)(r0 + tid));
        sel[tid * 8] = 0xFFFFFFFFu;
      } else {
        uint32_t taken = 0;
        for (int s2 = 0; s2 < k; ++s2) {
          int bj = -1;
          float bv = 0.f;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (j < E && !((taken >> j) & 1u) && (bj < 0 || lv[j] > bv)) {
              bj = j;
              bv = lv[j];
            }
          taken |= 1u << bj;
          sel[tid * 8 + s2] = (uint32_t)bj;
        }
      }
    }
  } else {
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = warp; r < nrow; r += NT / 32) {
      const float* l = lg + r * lp;
      bool ok = true;
      for (int j = lane; j < E; j += 32) ok &= isfinite(l[j]);
      ok = __all_sync(0xffffffffu, ok);
      if (!ok) {
        if (lane == 0) {
          atomicMin(bad_row, (uint32_t)(r0 + r));
          sel[r * 8] = 0xFFFFFFFFu;
        }
        continue;
      }
      for (int s2 = 0; s2 < k; ++s2) {
        float bv = -INFINITY;
        int bj = 0x7FFFFFFF;
        for (int j = lane; j < E; j += 32) {
          bool tk = false;
          for (int q = 0; q < s2; ++q) tk |= sel[r * 8 + q] == (uint32_t)j;
          const float v = l[j];
          if (!tk && (v > bv || bj == 0x7FFFFFFF)) {  // lane-local first maximum
            bv = v;
            bj = j;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
          if (oj != 0x7FFFFFFF && (bj == 0x7FFFFFFF || ov > bv || (ov == bv && oj < bj))) {
            bv = ov;
            bj = oj;
          }
        }
        if (lane == 0) sel[r * 8 + s2] = (uint32_t)bj;
        __syncwarp();
      }
    }
  }
  __syncthreads();
  G3_TRACE(6);
  // ---- expf(l_j - max) for every (row, expert) in parallel (routing.cpp:34)
  for (int i = tid; i < nrow * E; i += NT) {
    const int r = i / E, j = i - r * E;
    const uint32_t s0 = sel[r * 8];
    if (s0 == 0xFFFFFFFFu) continue;
    const float* l = lg + r * lp;
    ex[r * lp + j] = moe_glibc_expf_t(__fsub_rn(l[j], l[s0]), tab);
  }
  __syncthreads();
  G3_TRACE(7);
  // ---- serial sum in expert order, scales, routing keys (routing.cpp:33-38, 55-62)
  if (tid < nrow) {
    const int r = tid;
    const int64_t row = r0 + r;
    const bool fin = fsm[r] != 0;
    if (sel[r * 8] == 0xFFFFFFFFu) {
      for (int s2 = 0; s2 < k; ++s2) {
        expert[row * k + s2] = 0;
        scale[row * k + s2] = 0;
        atomicAdd(&hist[fin ? E : 0], 1u);
      }
    } else {
      const float* exr = ex + r * lp;
      float sum = 0.f;
      int j = 0;
      for (; j + 8 <= E; j += 8) {  // loads ahead of the dependent adds
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = exr[j + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) sum = __fadd_rn(sum, v[q]);
      }
      for (; j < E; ++j) sum = __fadd_rn(sum, exr[j]);
      for (int s2 = 0; s2 < k; ++s2) {
        const uint32_t e = sel[r * 8 + s2];
        const float num = s2 == 0 ? 1.0f : exr[e];
        expert[row * k + s2] = e;
        scale[row * k + s2] = f2h(__fdiv_rn(num, sum));
        atomicAdd(&hist[fin ? (uint32_t)E : e], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i <= E; i += NT) blockcnt[(int64_t)i * gridDim.x + blockIdx.x] = hist[i];
  G3_TRACE(5);
}

// ============================================================ host side
// rows per CTA and (EPG, RPT, threads): every SM gets rows (waves only when
// the fp16 rows overflow the shared-memory budget), then the fewest chains
// per thread that fit 256 threads.
struct G3Pick {
  int rb, epg, rpt, nt;
};

static bool g3_fits(int64_t d, int64_t E, int64_t gwp, int rb, int epg, int rpt, int nt, int k) {
  const g3::Cfg c = g3::cfg(d, E, gwp, rb, epg, rpt, nt);
  // scalar chains only while they are few (latency-bound: C3 decode); with
  // more chains FFMA2 pairs issue half the instructions (measured, C2)
  if (epg == 1 && c.ntask > 128) return false;
  return c.ntask <= nt && c.total <= g3::kSmemMax && (int64_t)rb * k <= 1024;
}

static bool g3_pick(int64_t T, int64_t d, int64_t E, int k, G3Pick* p) {
  const int64_t gwp = gate_fused_pitch(E);
  const int64_t sms = sm_count();
  int64_t rbmax = (int64_t)(g3::kXBudget / ((size_t)(d + 8) * 2)) - 2;
  rbmax = std::min<int64_t>(rbmax, g3::kMaxRows);
  rbmax = std::min<int64_t>(rbmax, 1024 / k);
  if (rbmax < 1) return false;
  const int64_t per_sm = (T + sms - 1) / sms;
  const int64_t waves = (per_sm + rbmax - 1) / rbmax;
  int rb = (int)std::max<int64_t>(1, (T + sms * waves - 1) / (sms * waves));
  // EPG = 1 (one scalar-FFMA chain per thread) is kept for A/B only
  // (MOE_GATE_EPG1=1): measured slower than FFMA2 pairs at C2 (7114 vs 5880
  // cycles in the logit phase) and at C3 T = 1 (9399 vs 8006)
  static const int kE[] = {1, 2, 4, 8, 8};
  static const int kR[] = {1, 1, 1, 1, 2};
  static const int kT[] = {256, 256, 256, 256, 256};
  static const int first = std::getenv("MOE_GATE_EPG1") ? 0 : 1;
  // dev A/B: MOE_GATE_CFG="EPG,RPT[,threads]" forces a chain layout when it fits
  if (const char* f = std::getenv("MOE_GATE_CFG")) {
    int fe = 0, fr = 0, fnt = 256;
    if (std::sscanf(f, "%d,%d,%d", &fe, &fr, &fnt) >= 2 && (fnt == 256 || fnt == 512) &&
        g3_fits(d, E, gwp, rb, fe, fr, fnt, k)) {
      *p = G3Pick{rb, fe, fr, fnt};
      return true;
    }
  }
  for (;;) {
    for (int i = first; i < 5; ++i)
      if (g3_fits(d, E, gwp, rb, kE[i], kR[i], kT[i], k)) {
        *p = G3Pick{rb, kE[i], kR[i], kT[i]};
        return true;
      }
    if (rb == 1) return false;
    rb = (rb + 1) / 2;  // too many chains for one CTA: halve the rows
  }
}

bool ln_gate_supported(int64_t T, int64_t d, int64_t E, int k) {
  if (d % 8 != 0 || k < 1 || k > 8 || E < 1 || E > 256 || T < 1) return false;
  G3Pick p;
  return g3_pick(T, d, E, k, &p);
}

int ln_gate_rows(int64_t T, int64_t d, int64_t E, int k) {
  G3Pick p;
  return g3_pick(T, d, E, k, &p) ? p.rb : 0;
}

template <int EPG, int RPT, int NT>
static int launch_g3(const GateFusedArgs& a, int rb, cudaStream_t st) {
  const g3::Cfg C = g3::cfg(a.d, a.E, a.gwp, rb, EPG, RPT, NT);
  static size_t attr = 0;
  if (C.total > 48 * 1024 && C.total > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(ln_gate_kernel<EPG, RPT, NT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.total));
    attr = C.total;
  }
  const unsigned grid = (unsigned)((a.T + rb - 1) / rb);
  static long long* dtrace = nullptr;
  const bool tr = std::getenv("MOE_GATE_TRACE") != nullptr;
  if (tr && !dtrace) MOE_CUDA_TRY(cudaMalloc(&dtrace, 8 * (16 + 2 * 65536)));
  const int pdl = pdl_enabled(5) ? 1 : 0;
  // widened LN chains only for a few rows per CTA (decode: the passes are
  // short and the FADD-only chain is faster -- C3 T=1 10710 vs 12869 cycles);
  // many rows (C2: 28): inline conversion (6980 vs 9196 cycles)
  static const int force_wide = std::getenv("MOE_GATE_LN_WIDE") ? std::atoi(std::getenv("MOE_GATE_LN_WIDE")) : -1;
  const int ln_wide = force_wide >= 0 ? force_wide : (rb <= 8 ? 1 : 0);
  MOE_CUDA_TRY(launch_k(5, ln_gate_kernel<EPG, RPT, NT>, dim3(grid), dim3(NT), C.total, st, a.x,
                        a.T, (int)a.d, a.g, a.b, a.gw32, (int)a.gwp, a.gb, (int)a.E, a.k,
                        a.finished, a.xn, a.expert, a.scale, a.blockcnt, a.bad_row, rb,
                        a.out_fin, tr ? dtrace : nullptr, pdl, ln_wide));
  note_launch();
  if (tr && grid <= 65536) {
    std::vector<long long> h(16 + 2 * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost);
    long long lo = h[16], hi = h[17], sum = 0;
    for (unsigned i = 0; i < grid; ++i) {
      lo = std::min(lo, h[16 + 2 * i]);
      hi = std::max(hi, h[17 + 2 * i]);
      sum += h[17 + 2 * i] - h[16 + 2 * i];
    }
    std::fprintf(stderr,
                 "ln_gate EPG=%d RPT=%d NT=%d grid=%u rb=%d kc=%d nch=%d tasks=%d wide=%d: "
                 "span=%lld ns cta mean=%lld ns; cta0 clocks rows=%lld chains=%lld norm=%lld "
                 "logits=%lld tail=%lld (select %lld, expf %lld, sums %lld) [widen %lld, mean chain %lld, sync %lld, sqdev %lld, var chain+ %lld]\n",
                 EPG, RPT, NT, grid, rb, C.kc, C.nch, C.ntask, C.wide, hi - lo, sum / grid,
                 h[1] - h[0], h[2] - h[1], h[3] - h[2], h[4] - h[3], h[5] - h[4],
                 h[6] - h[4], h[7] - h[6], h[5] - h[7], h[8] - h[1], h[9] - h[8], h[10] - h[9], h[11] - h[10], h[2] - h[11]);
  }
  return check_launch("ln_gate");
}

// LN only: rows per CTA sized for ~60 KB of shared memory (three CTAs per SM)
int launch_ln_rows(const GateFusedArgs& a, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  if (a.d % 8 != 0) return set_error(MOE_EINVAL, "ln_rows: d must be a multiple of 8");
  const int rb = (int)std::max<int64_t>(1, std::min<int64_t>(64, 60 * 1024 / ((a.d + 8) * 2) - 1));
  const g3::Cfg C = g3::cfg(a.d, 0, 0, rb, 2, 1, 256);
  static size_t attr = 0;
  if (C.total > 48 * 1024 && C.total > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(ln_gate_kernel<2, 1, 256, true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.total));
    attr = C.total;
  }
  const unsigned grid = (unsigned)((a.T + rb - 1) / rb);
  static long long* dtrace = nullptr;
  const bool tr = std::getenv("MOE_GATE_TRACE") != nullptr && grid <= 65536;
  if (tr && !dtrace) MOE_CUDA_TRY(cudaMalloc(&dtrace, 8 * (16 + 2 * 65536)));
  MOE_CUDA_TRY(launch_k(0, ln_gate_kernel<2, 1, 256, true>, dim3(grid), dim3(256), C.total, st, a.x,
                        a.T, (int)a.d, a.g, a.b, (const float*)nullptr, 0, (const uint16_t*)nullptr,
                        0, 1, a.finished, a.xn, (uint32_t*)nullptr, (uint16_t*)nullptr,
                        (uint32_t*)nullptr, a.bad_row, rb, a.out_fin, tr ? dtrace : nullptr, 0,
                        rb <= 8 ? 1 : 0));
  note_launch();
  if (tr) {  // dev: per-CTA spans and CTA 0 phase clocks
    std::vector<long long> h(16 + 2 * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost);
    long long lo = h[16], hi = h[17], sum = 0;
    for (unsigned i = 0; i < grid; ++i) {
      lo = std::min(lo, h[16 + 2 * i]);
      hi = std::max(hi, h[17 + 2 * i]);
      sum += h[17 + 2 * i] - h[16 + 2 * i];
    }
    std::fprintf(stderr,
                 "ln_rows grid=%u rb=%d: span=%lld ns cta mean=%lld ns; cta0 clocks rows=%lld chains=%lld "
                 "norm=%lld [mean chain %lld]\n",
                 grid, rb, hi - lo, sum / grid, h[1] - h[0], h[2] - h[1], h[3] - h[2], h[9] - h[1]);
  }
  return check_launch("ln_rows");
}

int launch_ln_gate(const GateFusedArgs& a, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  G3Pick p;
  if (!g3_pick(a.T, a.d, a.E, a.k, &p)) return set_error(MOE_EINVAL, "ln_gate: unsupported shape");
  if (p.rb != a.rows) return set_error(MOE_EINVAL, "ln_gate: row block mismatch");
  if (p.nt == 512) {  // dev A/B layouts with 16 warps
    if (p.epg == 8) return p.rpt == 1 ? launch_g3<8, 1, 512>(a, p.rb, st) : launch_g3<8, 2, 512>(a, p.rb, st);
    if (p.epg == 4) return launch_g3<4, 1, 512>(a, p.rb, st);
    return launch_g3<2, 1, 512>(a, p.rb, st);
  }
  if (p.epg == 1) return launch_g3<1, 1, 256>(a, p.rb, st);
  if (p.epg == 2) return p.rpt == 1 ? launch_g3<2, 1, 256>(a, p.rb, st) : launch_g3<2, 2, 256>(a, p.rb, st);
  if (p.epg == 4) return p.rpt == 1 ? launch_g3<4, 1, 256>(a, p.rb, st) : launch_g3<4, 2, 256>(a, p.rb, st);
  if (p.rpt == 1) return launch_g3<8, 1, 256>(a, p.rb, st);
  return launch_g3<8, 2, 256>(a, p.rb, st);
}

}  // namespace moecu
