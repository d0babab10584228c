// k_gate_fused.cu -- K2 gating for the layer hot path, bit-exact with
//   LayerNorm (proj/src/model.cpp:175-205) -> f32 gate logits (:273-297) ->
//   top-k softmax gate (proj/src/routing.cpp:11-41, top-k extension) ->
//   per-block routing-key histogram (routing.cpp:55-62, first counting-sort
//   pass), as two kernels:
//
// ln_rows_kernel -- 32 token rows per CTA arrive by bulk copy (TMA engine);
//   one lane per row runs the reference's two serial f32 chains (sum, then
//   centred sum of squares, every op RN32, no contraction); all threads then
//   normalise and write xn.  The chains are the latency floor of the whole
//   layer at decode sizes (2*d dependent FADDs per row).
//
// gate_topk_kernel -- every (row, expert) logit is its own serial k-chain;
//   products of two fp16 values are exact in f32, so fmaf == the reference's
//   mul-then-add and only the k order matters.  A thread owns RPT rows x EPG
//   experts of chains in registers (FMA-bound, ~1.25 issue slots per FMA);
//   xn and the pre-widened f32 gate weights stream through a 3-stage cp.async
//   ring of KC-input chunks (weights read as warp broadcasts, rows
//   conflict-free).  Then: warp-shuffle argmax (value desc, index asc == the
//   reference's first maximum under strict '>'), expf of every logit in
//   parallel (device port of glibc expf), one thread per row sums them in
//   expert order, gate scales, and a shared-memory histogram of routing keys
//   (finished ? E : expert) written key-major as blockcnt[key][block] for
//   plan_scan (k_route.cu), whose blocks are this kernel's RB*k slots.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace moecu {

// =================================================================== LN rows
// The two serial chains run one lane per row over an f32 copy of the rows
// that all 128 threads widen first (the chain lane then issues one FADD per
// element in pass 1 and FADD2/FMUL2 pairs + one chained FADD per element in
// pass 2 -- latency-bound, not issue-bound); every op is the reference's
// RN32 step in the same order.
namespace lnr {
constexpr int ROWS = 16;
constexpr int kThreads = 128;
__host__ __device__ inline size_t smem(int d) {
  return (size_t)ROWS * (d + 8) * 2 + (size_t)ROWS * (d + 4) * 4 + 2 * ROWS * 4 + 16;
}
}  // namespace lnr

// dev-only timing (MOE_GATE_TRACE): per-CTA [start, end] global time (ns)
// and CTA 0's phase clocks
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define LN_TRACE(i)                                                            \
  do {                                                                         \
    if (trace != nullptr && tid == 0) {                                        \
      if ((i) == 0) trace[16 + 2 * blockIdx.x] = gtime();                      \
      if ((i) == 3) trace[16 + 2 * blockIdx.x + 1] = gtime();                  \
      if (blockIdx.x == 0) trace[i] = clock64();                               \
    }                                                                          \
  } while (0)

__global__ void __launch_bounds__(lnr::kThreads) ln_rows_kernel(
    const uint16_t* __restrict__ x, int64_t T, int d, const uint16_t* __restrict__ g,
    const uint16_t* __restrict__ b, uint16_t* __restrict__ xn, long long* trace) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int xp = d + 8, fp = d + 4;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm);
  float* xf = reinterpret_cast<float*>(sm + (size_t)lnr::ROWS * xp * 2);
  float* st = xf + (size_t)lnr::ROWS * fp;  // mean, inv
  uint64_t* bar = reinterpret_cast<uint64_t*>(st + 2 * lnr::ROWS);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * lnr::ROWS;
  const int nrow = (int)::min((int64_t)lnr::ROWS, T - r0);
  const int d8 = d / 8, d4 = d / 4;
  if (tid < 32) {  // warp 0 converged, one elected lane issues (uniform copy operands)
    if (elect_one()) {
      mbar_init(bar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(bar, (uint32_t)nrow * d * 2);
    }
    __syncwarp();
    for (int r = 0; r < nrow; ++r)
      if (elect_one()) bulk_load(xs + r * xp, x + (r0 + r) * d, (uint32_t)d * 2, bar);
  }
  LN_TRACE(0);
  __syncthreads();
  mbar_wait(bar, 0);
  LN_TRACE(1);
  for (int i = tid; i < nrow * d8; i += lnr::kThreads) {  // widen (exact)
    const int r = i / d8, c = i % d8;
    const uint4 v = *reinterpret_cast<const uint4*>(xs + r * xp + c * 8);
    const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
    float4* dst = reinterpret_cast<float4*>(xf + r * fp + c * 8);
    dst[0] = make_float4(h2f(h[0]), h2f(h[1]), h2f(h[2]), h2f(h[3]));
    dst[1] = make_float4(h2f(h[4]), h2f(h[5]), h2f(h[6]), h2f(h[7]));
  }
  __syncthreads();
  if (tid < nrow) {  // model.cpp:178-192, serial
    // shared loads run two pieces ahead of the dependent adds (LDS latency
    // would otherwise sit on the chain)
    const float4* row = reinterpret_cast<const float4*>(xf + tid * fp);
    float s = 0.f;
    float4 c0 = row[0], c1 = row[d4 > 1 ? 1 : 0];
    for (int c = 0; c < d4; ++c) {
      const float4 v = c0;
      c0 = c1;
      c1 = row[c + 2 < d4 ? c + 2 : c];
      s = __fadd_rn(s, v.x);
      s = __fadd_rn(s, v.y);
      s = __fadd_rn(s, v.z);
      s = __fadd_rn(s, v.w);
    }
    const float mean = __fdiv_rn(s, (float)d);
    const float2 m2 = make_float2(mean, mean);
    float v2 = 0.f;
    c0 = row[0];
    c1 = row[d4 > 1 ? 1 : 0];
    for (int c = 0; c < d4; ++c) {
      const float4 v = c0;
      c0 = c1;
      c1 = row[c + 2 < d4 ? c + 2 : c];
      const float2 d01 = f2_sub(make_float2(v.x, v.y), m2);
      const float2 d23 = f2_sub(make_float2(v.z, v.w), m2);
      const float2 q01 = f2_mul(d01, d01), q23 = f2_mul(d23, d23);
      v2 = __fadd_rn(v2, q01.x);
      v2 = __fadd_rn(v2, q01.y);
      v2 = __fadd_rn(v2, q23.x);
      v2 = __fadd_rn(v2, q23.y);
    }
    st[tid] = mean;
    st[lnr::ROWS + tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v2, (float)d), 1e-5f)));
  }
  __syncthreads();
  LN_TRACE(2);
  for (int i = tid; i < nrow * d8; i += lnr::kThreads) {  // model.cpp:193-194
    const int r = i / d8, c = i % d8;
    const float4* src = reinterpret_cast<const float4*>(xf + r * fp + c * 8);
    const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g) + c);
    const uint4 bv = __ldg(reinterpret_cast<const uint4*>(b) + c);
    const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gv);
    const uint16_t* bh = reinterpret_cast<const uint16_t*>(&bv);
    const float mean = st[r], inv = st[lnr::ROWS + r];
    uint4 o;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
    // scalar RN ops: ptxas contracts a packed f32x2 mul followed by a packed
    // add into FFMA2 even under --fmad=false, which would change the bits
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float4 v = src[h];
      const float xv[4] = {v.x, v.y, v.z, v.w};
      float y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        y[q] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[q], mean), inv), h2f(gh[h * 4 + q])),
                         h2f(bh[h * 4 + q]));
      ow[2 * h] = (uint32_t)f2h(y[0]) | ((uint32_t)f2h(y[1]) << 16);
      ow[2 * h + 1] = (uint32_t)f2h(y[2]) | ((uint32_t)f2h(y[3]) << 16);
    }
    *reinterpret_cast<uint4*>(xn + (r0 + r) * d + c * 8) = o;
  }
  LN_TRACE(3);
}

// Large-T form: 32 rows per CTA, conversions inline (higher occupancy; the
// kernel is issue-bound there, not latency-bound).
__global__ void __launch_bounds__(128) ln_rows_wide_kernel(
    const uint16_t* __restrict__ x, int64_t T, int d, const uint16_t* __restrict__ g,
    const uint16_t* __restrict__ b, uint16_t* __restrict__ xn, long long* trace) {
  constexpr int ROWS = 32;
  extern __shared__ __align__(16) uint8_t sm[];
  const int xp = d + 8;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm);
  float* st = reinterpret_cast<float*>(sm + (size_t)ROWS * xp * 2);  // mean, inv
  uint64_t* bar = reinterpret_cast<uint64_t*>(st + 2 * ROWS);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int nrow = (int)::min((int64_t)ROWS, T - r0);
  const int d8 = d / 8;
  if (tid < 32) {  // warp 0 converged, one elected lane issues (uniform copy operands)
    if (elect_one()) {
      mbar_init(bar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(bar, (uint32_t)nrow * d * 2);
    }
    __syncwarp();
    for (int r = 0; r < nrow; ++r)
      if (elect_one()) bulk_load(xs + r * xp, x + (r0 + r) * d, (uint32_t)d * 2, bar);
  }
  LN_TRACE(0);
  __syncthreads();
  mbar_wait(bar, 0);
  LN_TRACE(1);
  if (tid < nrow) {  // model.cpp:178-192, serial
    const uint4* row = reinterpret_cast<const uint4*>(xs + tid * xp);
    float s = 0.f;
    uint4 cur = row[0];
    for (int c = 0; c < d8; ++c) {
      const uint4 nxt = row[c + 1 < d8 ? c + 1 : c];
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&cur);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __fadd_rn(s, h2f(h[i]));
      cur = nxt;
    }
    const float mean = __fdiv_rn(s, (float)d);
    float v2 = 0.f;
    cur = row[0];
    for (int c = 0; c < d8; ++c) {
      const uint4 nxt = row[c + 1 < d8 ? c + 1 : c];
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&cur);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float dx = __fsub_rn(h2f(h[i]), mean);
        v2 = __fadd_rn(v2, __fmul_rn(dx, dx));
      }
      cur = nxt;
    }
    st[tid] = mean;
    st[ROWS + tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v2, (float)d), 1e-5f)));
  }
  __syncthreads();
  LN_TRACE(2);
  for (int i = tid; i < nrow * d8; i += 128) {  // model.cpp:193-194
    const int r = i / d8, c = i % d8;
    uint4 v = *reinterpret_cast<const uint4*>(xs + r * xp + c * 8);
    const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g) + c);
    const uint4 bv = __ldg(reinterpret_cast<const uint4*>(b) + c);
    uint16_t* h = reinterpret_cast<uint16_t*>(&v);
    const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gv);
    const uint16_t* bh = reinterpret_cast<const uint16_t*>(&bv);
    const float mean = st[r], inv = st[ROWS + r];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      h[j] = f2h(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(h2f(h[j]), mean), inv), h2f(gh[j])),
                           h2f(bh[j])));
    *reinterpret_cast<uint4*>(xn + (r0 + r) * d + c * 8) = v;
  }
  LN_TRACE(3);
}

// ========================================================== logits + top-k
namespace gk {
constexpr int kThreads = 256;
constexpr int NS = 3;
constexpr int kMaxCopies = 8;  // cp.async per thread per chunk, for x and for w each

struct Cfg {
  int ng;       // expert groups (power of two)
  int rt;       // row-threads = kThreads / ng
  int rb;       // rows per CTA = rt * rpt
  int kc;       // inputs per pipeline chunk
  int xpitch;   // fp16 xn chunk row pitch (halves)
  int fpitch;   // f32 xn chunk row pitch (floats)
  size_t xbytes, wbytes, stage, off_xf, body, total;
};

__host__ __device__ inline int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

__host__ __device__ inline Cfg cfg(int E, int gwp, int epg, int rpt) {
  Cfg c;
  c.ng = pow2_at_least((E + epg - 1) / epg);
  if (c.ng > kThreads) c.ng = kThreads;
  c.rt = kThreads / c.ng;
  c.rb = c.rt * rpt;
  int kc = (int)(16384 / ((size_t)gwp * 4)) / 8 * 8;
  c.kc = kc < 16 ? 16 : (kc > 64 ? 64 : kc);
  c.xpitch = c.kc + 8;
  c.fpitch = c.kc + 4;  // 16-byte rows, consecutive row-threads on distinct banks
  c.xbytes = (size_t)c.rb * c.xpitch * 2;
  // gate weights staged transposed, [group][k][EPG]: a thread's EPG weights
  // for consecutive k are contiguous (compile-time offsets, 16-byte loads)
  c.wbytes = (size_t)c.ng * epg * c.kc * 4;
  c.stage = (c.xbytes + c.wbytes + 15) & ~size_t(15);
  c.off_xf = NS * c.stage;
  const size_t pipe = c.off_xf;
  const size_t lg = (size_t)2 * c.rb * (E + 1) * 4;  // logits + expf values (reuse the ring)
  c.body = ((pipe > lg ? pipe : lg) + 15) & ~size_t(15);
  c.total = c.body + (size_t)c.rb * 8 * 4 + (size_t)(E + 1) * 4 + 16;  // + sel[8], hist
  return c;
}

// two independent f32 FMAs in one instruction (FFMA2, sm_100): c += a * b, each lane RN
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  uint64_t r;
  const uint64_t bb = (uint64_t)__float_as_uint(b.x) | ((uint64_t)__float_as_uint(b.y) << 32);
  const uint64_t cc = (uint64_t)__float_as_uint(c.x) | ((uint64_t)__float_as_uint(c.y) << 32);
  const uint64_t aa = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
  return make_float2(__uint_as_float((uint32_t)r), __uint_as_float((uint32_t)(r >> 32)));
}
}  // namespace gk

template <int EPG, int RPT>
__global__ void __launch_bounds__(gk::kThreads, 2) gate_topk_kernel(
    const uint16_t* __restrict__ xn, int64_t T, int d, const float* __restrict__ gw32, int gwp,
    const uint16_t* __restrict__ gb, int E, int k, const uint8_t* __restrict__ finished,
    uint32_t* __restrict__ expert, uint16_t* __restrict__ scale, uint32_t* __restrict__ blockcnt,
    uint32_t* bad_row, long long* trace) {
  extern __shared__ __align__(16) uint8_t sm[];
  const gk::Cfg C = gk::cfg(E, gwp, EPG, RPT);
  long long tw = 0, tc = 0, t_0 = clock64();  // dev-only phase trace (MOE_GATE_TRACE)
  if (trace != nullptr && threadIdx.x == 0) trace[16 + 2 * blockIdx.x] = gtime();
  uint32_t* sel = reinterpret_cast<uint32_t*>(sm + C.body);  // [rb][8]
  uint32_t* hist = sel + C.rb * 8;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rt = tid % C.rt, eg = tid / C.rt;  // row-thread fastest: a warp shares eg
  const int e0 = eg * EPG;
  const int64_t r0 = (int64_t)blockIdx.x * C.rb;
  const int nrow = (int)::min((int64_t)C.rb, T - r0);
  const int KC = C.kc, nch = (d + KC - 1) / KC;

  for (int i = tid; i <= E; i += gk::kThreads) hist[i] = 0;

  // Every chunk copies the same (row, piece) / (k, expert-chunk) pattern, only
  // shifted by k0: each thread's copy descriptors are computed once.
  constexpr int CW = EPG >= 4 ? 4 : EPG;  // experts per weight copy (16 / 8 / 4 bytes)
  constexpr int MAXC = gk::kMaxCopies;     // copies per thread per chunk (host-checked)
  const int wc = (E + CW - 1) / CW;
  const int nx = C.rb * (KC / 8), nw = KC * wc;
  int xsrc[MAXC], xdst[MAXC], wsrc[MAXC], wdst[MAXC];
#pragma unroll
  for (int j = 0; j < MAXC; ++j) {  // fully unrolled: descriptors stay in registers
    const int i = tid + j * gk::kThreads;
    const int r = i / (KC / 8), q = i % (KC / 8);
    xsrc[j] = (i < nx && r < nrow) ? (int)(r * d + q * 8) : -1;  // elements from row r0
    xdst[j] = r * C.xpitch + q * 8;
    const int kk = i / wc, e = (i % wc) * CW;
    wsrc[j] = i < nw ? kk * gwp + e : -1;
    wdst[j] = ((e / EPG) * KC + kk) * EPG + (e % EPG);
  }
  const uint16_t* xbase = xn + r0 * d;
  auto issue = [&](int c) {
    if (c < nch) {
      uint8_t* stg = sm + (size_t)(c % gk::NS) * C.stage;
      uint16_t* xs = reinterpret_cast<uint16_t*>(stg);
      float* ws = reinterpret_cast<float*>(stg + C.xbytes);
      const int k0 = c * KC;
      const bool full = k0 + KC <= d;
#pragma unroll
      for (int j = 0; j < MAXC; ++j) {
        if (tid + j * gk::kThreads >= nx) break;
        const bool ok = xsrc[j] >= 0 && (full || (xsrc[j] % d) + k0 < d);
        cp_async16(xs + xdst[j], ok ? xbase + xsrc[j] + k0 : xn, ok);
      }
      const float* wk = gw32 + (size_t)k0 * gwp;
#pragma unroll
      for (int j = 0; j < MAXC; ++j) {
        if (wsrc[j] < 0) break;
        if (!full && wsrc[j] / gwp + k0 >= d) continue;
        if constexpr (CW == 4) cp_async16(ws + wdst[j], wk + wsrc[j], true);
        else if constexpr (CW == 2) cp_async8(ws + wdst[j], wk + wsrc[j]);
        else cp_async4(ws + wdst[j], wk + wsrc[j]);
      }
    }
    cp_async_commit();
  };
  for (int c = 0; c < gk::NS - 1; ++c) issue(c);

  // chains: RPT rows x EPG experts; EPG >= 2 as float2 pairs (FFMA2)
  constexpr int NP = EPG >= 2 ? EPG / 2 : 1;
  float2 acc[RPT][NP];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[i][j] = make_float2(0.f, 0.f);

  const long long t_1 = clock64();
  for (int c = 0; c < nch; ++c) {
    const long long ta = clock64();
    cp_async_wait<gk::NS - 2>();
    __syncthreads();  // chunk c landed for every thread; chunk c-1 fully consumed
    tw += clock64() - ta;
    issue(c + gk::NS - 1);
    const long long tb = clock64();
    const uint8_t* stg = sm + (size_t)(c % gk::NS) * C.stage;
    const uint16_t* xr = reinterpret_cast<const uint16_t*>(stg) + rt * C.xpitch;
    const float* wg = reinterpret_cast<const float*>(stg + C.xbytes) + (size_t)eg * KC * EPG;
    const int kc = ::min(KC, d - c * KC);
    if (e0 < E) {
      // 4-input steps, operands of step i+1 loaded while step i's FMAs run
      struct Ops {
        uint2 xh[RPT];
        float w[4][EPG];
      };
      auto load = [&](Ops& o, int kk) {
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          o.xh[i] = *reinterpret_cast<const uint2*>(xr + i * C.rt * C.xpitch + kk);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if constexpr (EPG >= 4) {
#pragma unroll
            for (int j = 0; j < EPG; j += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(wg + (kk + q) * EPG + j);
              o.w[q][j] = w4.x;
              o.w[q][j + 1] = w4.y;
              o.w[q][j + 2] = w4.z;
              o.w[q][j + 3] = w4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < EPG; ++j) o.w[q][j] = wg[(kk + q) * EPG + j];
          }
        }
      };
      auto fma_step = [&](const Ops& o) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            const float xq = h2f(reinterpret_cast<const uint16_t*>(&o.xh[i])[q]);
            if constexpr (EPG >= 2) {
#pragma unroll
              for (int j = 0; j < NP; ++j)  // exact products, k order kept per chain
                acc[i][j] = gk::ffma2(xq, make_float2(o.w[q][2 * j], o.w[q][2 * j + 1]), acc[i][j]);
            } else {
              acc[i][0].x = fmaf(xq, o.w[q][0], acc[i][0].x);
            }
          }
        }
      };
      Ops a, b;
      load(a, 0);
      for (int kk = 0; kk < kc; kk += 8) {
        load(b, kk + 4);  // kc is a multiple of 8
        fma_step(a);
        if (kk + 8 < kc) load(a, kk + 8);
        fma_step(b);
      }
    }
  }
  const long long t_2 = clock64();
  (void)tc;
  cp_async_wait<0>();
  __syncthreads();  // ring free: reuse as logits / expf buffers

  float* lg = reinterpret_cast<float*>(sm);
  const int lp = E + 1;
  float* ex = lg + (size_t)C.rb * lp;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = rt + i * C.rt;
#pragma unroll
    for (int j = 0; j < EPG; ++j) {
      const float a = (j & 1) ? acc[i][j / 2].y : acc[i][j / 2].x;
      if (e0 + j < E && r < nrow) lg[r * lp + e0 + j] = __fadd_rn(a, h2f(gb[e0 + j]));
    }
  }
  __syncthreads();

  if (E <= 16) {
    // few experts: one thread per row does the reference's serial selection
    // (strict '>', index order) and its expf values directly -- no shuffles
    if (tid < nrow) {
      const float* l = lg + tid * lp;
      float* exr = ex + tid * lp;
      bool ok = true;
      for (int j = 0; j < E; ++j) ok &= isfinite(l[j]);
      if (!ok) {
        atomicMin(bad_row, (uint32_t)(r0 + tid));
        sel[tid * 8] = 0xFFFFFFFFu;
      } else {
        uint32_t taken = 0;  // E <= 16: bitmask
        for (int s2 = 0; s2 < k; ++s2) {
          int bj = -1;
          float bv = 0.f;
          for (int j = 0; j < E; ++j)
            if (!((taken >> j) & 1u) && (bj < 0 || l[j] > bv)) {
              bj = j;
              bv = l[j];
            }
          taken |= 1u << bj;
          sel[tid * 8 + s2] = (uint32_t)bj;
        }
        const float mx = l[sel[tid * 8]];
        for (int j = 0; j < E; ++j) exr[j] = moe_glibc_expf(__fsub_rn(l[j], mx));
      }
    }
    __syncthreads();
  } else {
    // ---- top-k selection (routing.cpp:15-31): one warp per row, shuffles
    for (int r = warp; r < nrow; r += gk::kThreads / 32) {
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
      for (int s = 0; s < k; ++s) {
        float bv = -INFINITY;
        int bj = 0x7FFFFFFF;
        for (int j = lane; j < E; j += 32) {
          bool taken = false;
          for (int q = 0; q < s; ++q) taken |= sel[r * 8 + q] == (uint32_t)j;
          const float v = l[j];
          if (!taken && (v > bv || bj == 0x7FFFFFFF)) {  // lane-local first maximum
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
        if (lane == 0) sel[r * 8 + s] = (uint32_t)bj;
        __syncwarp();
      }
    }
    __syncthreads();
    // expf(l_j - mx) for every (row, expert) in parallel (routing.cpp:34)
    for (int i = tid; i < nrow * E; i += gk::kThreads) {
      const int r = i / E, j = i % E;
      const uint32_t s0 = sel[r * 8];
      if (s0 == 0xFFFFFFFFu) continue;
      const float* l = lg + r * lp;
      ex[r * lp + j] = moe_glibc_expf(__fsub_rn(l[j], l[s0]));
    }
    __syncthreads();
  }
  // serial sum in expert order, scales, routing keys (routing.cpp:33-38, 55-62)
  if (tid < nrow) {
    const int r = tid;
    const int64_t row = r0 + r;
    const bool fin = finished != nullptr && finished[row] != 0;
    if (sel[r * 8] == 0xFFFFFFFFu) {
      for (int s = 0; s < k; ++s) {
        expert[row * k + s] = 0;
        scale[row * k + s] = 0;
        atomicAdd(&hist[fin ? E : 0], 1u);
      }
    } else {
      const float* exr = ex + r * lp;
      float sum = 0.f;
      for (int j = 0; j < E; ++j) sum = __fadd_rn(sum, exr[j]);
      for (int s = 0; s < k; ++s) {
        const uint32_t e = sel[r * 8 + s];
        const float num = s == 0 ? 1.0f : exr[e];
        expert[row * k + s] = e;
        scale[row * k + s] = f2h(__fdiv_rn(num, sum));
        atomicAdd(&hist[fin ? (uint32_t)E : e], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = tid; i <= E; i += gk::kThreads) blockcnt[(int64_t)i * gridDim.x + blockIdx.x] = hist[i];
  if (trace != nullptr && tid == 0) trace[16 + 2 * blockIdx.x + 1] = gtime();
  if (trace != nullptr && blockIdx.x == 0 && tid == 0) {
    trace[0] = t_1 - t_0;  // prologue (first issues)
    trace[1] = tw;         // chunk waits + barriers
    trace[2] = tc;         // chunk compute
    trace[3] = t_2 - t_1;  // whole chunk loop
    trace[4] = clock64() - t_2;  // top-k, expf, scales, histogram
    trace[5] = nch;
  }
}

// ================================================================= launchers
__global__ void widen_gate_kernel(const uint16_t* __restrict__ gw, int64_t d, int64_t E,
                                  int64_t gwp, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * gwp) return;
  const int64_t r = i / gwp, c = i % gwp;
  out[i] = c < E ? h2f(gw[r * E + c]) : 0.f;
}

int launch_widen_gate(const uint16_t* gw, int64_t d, int64_t E, int64_t gwp, float* out,
                      cudaStream_t st) {
  const int64_t n = d * gwp;
  widen_gate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gw, d, E, gwp, out);
  note_launch();
  return check_launch("widen_gate");
}

int64_t gate_fused_pitch(int64_t E) { return (E + 7) / 8 * 8; }  // EPG <= 8 groups stay in-row

// copy descriptors of a config fit the per-thread register arrays
static bool copies_fit(int64_t E, int epg, const gk::Cfg& c) {
  const int cw = epg >= 4 ? 4 : epg;
  const int64_t nx = (int64_t)c.rb * (c.kc / 8), nw = (int64_t)c.kc * ((E + cw - 1) / cw);
  return nx <= (int64_t)gk::kThreads * gk::kMaxCopies && nw <= (int64_t)gk::kThreads * gk::kMaxCopies;
}

// (EPG, RPT): the most chains per thread (FFMA2 pairs, shared weight loads)
// that still fills the machine; below that the gate is latency-bound and
// 8 expert chains per thread beat many one-chain CTAs.
static void pick(int64_t T, int64_t E, int k, int* epg, int* rpt) {
  const int64_t gwp = gate_fused_pitch(E);
  if (const char* ov = std::getenv("MOE_GATE_CFG")) {  // dev experiments: "EPG,RPT"
    int a = 0, b = 0;
    if (std::sscanf(ov, "%d,%d", &a, &b) == 2 && (a == 1 || a == 2 || a == 4 || a == 8) &&
        (b == 1 || (b == 2 && a == 8))) {
      *epg = a;
      *rpt = b;
      return;
    }
  }
  // Measured on B200 (scripts/route_probe.py): the machine must be filled
  // first (C2: 1 chain/thread over 128 CTAs beats 8 chains/thread over 16),
  // then more chains per thread win (C4: 8x2 over 256 CTAs); below one CTA
  // per SM, 4 chains per thread balance latency and parallelism (C3 decode).
  static const int kE[] = {8, 8, 4, 2, 1};
  static const int kR[] = {2, 1, 1, 1, 1};
  for (int i = 0; i < 5; ++i) {
    const gk::Cfg c = gk::cfg((int)E, (int)gwp, kE[i], kR[i]);
    if ((int64_t)c.rb * k <= 1024 && copies_fit(E, kE[i], c) && (T + c.rb - 1) / c.rb >= 148) {
      *epg = kE[i];
      *rpt = kR[i];
      return;
    }
  }
  // otherwise: the most CTAs if that still covers half the SMs, else 4 chains
  const gk::Cfg c1 = gk::cfg((int)E, (int)gwp, 1, 1);
  const gk::Cfg c4 = gk::cfg((int)E, (int)gwp, 4, 1);
  const bool ok1 = copies_fit(E, 1, c1), ok4 = copies_fit(E, 4, c4) && (int64_t)c4.rb * k <= 1024;
  *epg = (ok1 && ((T + c1.rb - 1) / c1.rb >= 74 || !ok4)) ? 1 : 4;
  *rpt = 1;
}

int gate_fused_rows(int64_t T, int64_t E, int k) {
  int epg, rpt;
  pick(T, E, k, &epg, &rpt);
  return gk::cfg((int)E, (int)gate_fused_pitch(E), epg, rpt).rb;
}

bool gate_fused_supported(int64_t d, int64_t E, int k) {
  if (d % 8 != 0 || k < 1 || k > 8 || E < 1 || E > 256) return false;
  if (lnr::smem((int)d) > 200 * 1024) return false;
  // slots of one gate block must fit a plan_place block (<= 1024 threads),
  // and the EPG=4 fallback must fit the copy descriptors
  const gk::Cfg c = gk::cfg((int)E, (int)gate_fused_pitch(E), 4, 1);
  return (int64_t)c.rb * k <= 1024 && copies_fit(E, 4, c) && c.total <= 200 * 1024;
}

template <int EPG, int RPT>
static int launch_gk(const GateFusedArgs& a, cudaStream_t st) {
  const gk::Cfg C = gk::cfg((int)a.E, (int)a.gwp, EPG, RPT);
  static size_t attr = 0;
  if (C.total > 48 * 1024 && C.total > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gate_topk_kernel<EPG, RPT>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.total));
    attr = C.total;
  }
  const unsigned grid = (unsigned)((a.T + C.rb - 1) / C.rb);
  static long long* dtrace = nullptr;
  const bool tr = std::getenv("MOE_GATE_TRACE") != nullptr;
  if (tr && !dtrace) MOE_CUDA_TRY(cudaMalloc(&dtrace, 8 * (16 + 2 * 65536)));
  gate_topk_kernel<EPG, RPT><<<grid, gk::kThreads, C.total, st>>>(
      a.xn, a.T, (int)a.d, a.gw32, (int)a.gwp, a.gb, (int)a.E, a.k, a.finished, a.expert,
      a.scale, a.blockcnt, a.bad_row, tr ? dtrace : nullptr);
  note_launch();
  if (tr) {
    static std::vector<long long> hv;
    hv.assign(16 + 2 * grid, 0);
    cudaStreamSynchronize(st);
    cudaMemcpy(hv.data(), dtrace, hv.size() * 8, cudaMemcpyDeviceToHost);
    const long long* trace = hv.data();
    long long lo = trace[16], hi = trace[17], sum = 0, mx = 0;
    for (unsigned i = 0; i < grid; ++i) {
      lo = std::min(lo, trace[16 + 2 * i]);
      hi = std::max(hi, trace[16 + 2 * i + 1]);
      sum += trace[16 + 2 * i + 1] - trace[16 + 2 * i];
      mx = std::max(mx, trace[16 + 2 * i + 1] - trace[16 + 2 * i]);
    }
    std::fprintf(stderr, "gate_trace EPG=%d RPT=%d grid=%u rb=%d kc=%d: span=%lld ns cta mean=%lld max=%lld ns; cta0 clocks pro=%lld wait=%lld loop=%lld tail=%lld nch=%lld\n",
                 EPG, RPT, grid, C.rb, C.kc, hi - lo, sum / grid, mx, trace[0], trace[1], trace[3], trace[4], trace[5]);
  }
  return check_launch("gate_topk");
}

// dev-only: summarise an LN trace (per-CTA global-time spans, CTA 0 phases)
static void ln_trace_report(long long* dtr, unsigned grid, const char* name) {
  static std::vector<long long> h;
  h.assign(16 + 2 * grid, 0);
  cudaDeviceSynchronize();
  cudaMemcpy(h.data(), dtr, h.size() * 8, cudaMemcpyDeviceToHost);
  const long long* tr = h.data();
  long long lo = tr[16], hi = tr[17], sum = 0, mx = 0;
  for (unsigned i = 0; i < grid; ++i) {
    lo = std::min(lo, tr[16 + 2 * i]);
    hi = std::max(hi, tr[16 + 2 * i + 1]);
    sum += tr[16 + 2 * i + 1] - tr[16 + 2 * i];
    mx = std::max(mx, tr[16 + 2 * i + 1] - tr[16 + 2 * i]);
  }
  std::fprintf(stderr, "ln_trace %s grid=%u: span=%lld ns cta mean=%lld max=%lld ns; cta0 clocks load=%lld chains=%lld norm=%lld\n",
               name, grid, hi - lo, sum / grid, mx, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2]);
}

int launch_gate_fused(const GateFusedArgs& a, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  static long long* ltr = nullptr;
  const bool ltrace = std::getenv("MOE_GATE_TRACE") != nullptr;
  if (ltrace && !ltr) MOE_CUDA_TRY(cudaMalloc(&ltr, 8 * (16 + 2 * 65536)));
  // 1. LayerNorm rows: latency-bound below ~1 row per SM thread group (f32
  //    widening + packed ops), issue-bound above (inline conversions, more CTAs)
  if (a.T <= 2048) {
    const size_t smem = lnr::smem((int)a.d);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      MOE_CUDA_TRY(cudaFuncSetAttribute(ln_rows_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    const unsigned grid = (unsigned)((a.T + lnr::ROWS - 1) / lnr::ROWS);
    ln_rows_kernel<<<grid, lnr::kThreads, smem, st>>>(a.x, a.T, (int)a.d, a.g, a.b, a.xn,
                                                      ltrace ? ltr : nullptr);
    if (ltrace) ln_trace_report(ltr, grid, "ln_rows");
  } else {
    const size_t smem = (size_t)32 * (a.d + 8) * 2 + 64 * 4 + 16;
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
      MOE_CUDA_TRY(cudaFuncSetAttribute(ln_rows_wide_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = smem;
    }
    const unsigned grid = (unsigned)((a.T + 31) / 32);
    ln_rows_wide_kernel<<<grid, 128, smem, st>>>(a.x, a.T, (int)a.d, a.g, a.b, a.xn,
                                                 ltrace ? ltr : nullptr);
    if (ltrace) ln_trace_report(ltr, grid, "ln_rows_wide");
  }
  note_launch();
  const int s1 = check_launch("ln_rows");
  if (s1 != MOE_OK) return s1;
  // 2. logits + top-k + key histogram
  int epg, rpt;
  pick(a.T, a.E, a.k, &epg, &rpt);
  if (epg == 8 && rpt == 2) return launch_gk<8, 2>(a, st);
  if (epg == 8) return launch_gk<8, 1>(a, st);
  if (epg == 4) return launch_gk<4, 1>(a, st);
  if (epg == 2) return launch_gk<2, 1>(a, st);
  return launch_gk<1, 1>(a, st);
}

}  // namespace moecu
