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
#include "kernels.cuh"

namespace moecu {

// =================================================================== LN rows
namespace lnr {
constexpr int ROWS = 32;  // one full warp of row chains
constexpr int kThreads = 128;
}  // namespace lnr

__global__ void __launch_bounds__(lnr::kThreads) ln_rows_kernel(
    const uint16_t* __restrict__ x, int64_t T, int d, const uint16_t* __restrict__ g,
    const uint16_t* __restrict__ b, uint16_t* __restrict__ xn) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int xp = d + 8;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm);
  float* st = reinterpret_cast<float*>(sm + (size_t)lnr::ROWS * xp * 2);  // mean, inv
  uint64_t* bar = reinterpret_cast<uint64_t*>(st + 2 * lnr::ROWS);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * lnr::ROWS;
  const int nrow = (int)::min((int64_t)lnr::ROWS, T - r0);
  const int d8 = d / 8;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(bar, (uint32_t)nrow * d * 2);
    for (int r = 0; r < nrow; ++r) bulk_load(xs + r * xp, x + (r0 + r) * d, (uint32_t)d * 2, bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  if (tid < nrow) {  // model.cpp:178-192, serial
    // the next 16 bytes are loaded while the current 8 adds run (the shared
    // load latency would otherwise sit on the dependent chain)
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
    st[lnr::ROWS + tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v2, (float)d), 1e-5f)));
  }
  __syncthreads();
  for (int i = tid; i < nrow * d8; i += lnr::kThreads) {  // model.cpp:193-194
    const int r = i / d8, c = i % d8;
    uint4 v = *reinterpret_cast<const uint4*>(xs + r * xp + c * 8);
    const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g) + c);
    const uint4 bv = __ldg(reinterpret_cast<const uint4*>(b) + c);
    uint16_t* h = reinterpret_cast<uint16_t*>(&v);
    const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gv);
    const uint16_t* bh = reinterpret_cast<const uint16_t*>(&bv);
    const float mean = st[r], inv = st[lnr::ROWS + r];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      h[j] = f2h(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(h2f(h[j]), mean), inv), h2f(gh[j])),
                           h2f(bh[j])));
    *reinterpret_cast<uint4*>(xn + (r0 + r) * d + c * 8) = v;
  }
}

// ========================================================== logits + top-k
namespace gk {
constexpr int kThreads = 256;
constexpr int NS = 3;

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
  c.wbytes = (size_t)c.kc * gwp * 4 + 64;  // + over-read slack of the last expert group
  c.stage = (c.xbytes + c.wbytes + 15) & ~size_t(15);
  c.off_xf = NS * c.stage;  // f32 copy of the current xn chunk
  const size_t pipe = c.off_xf + (size_t)c.rb * c.fpitch * 4;
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
__global__ void __launch_bounds__(gk::kThreads) gate_topk_kernel(
    const uint16_t* __restrict__ xn, int64_t T, int d, const float* __restrict__ gw32, int gwp,
    const uint16_t* __restrict__ gb, int E, int k, const uint8_t* __restrict__ finished,
    uint32_t* __restrict__ expert, uint16_t* __restrict__ scale, uint32_t* __restrict__ blockcnt,
    uint32_t* bad_row) {
  extern __shared__ __align__(16) uint8_t sm[];
  const gk::Cfg C = gk::cfg(E, gwp, EPG, RPT);
  uint32_t* sel = reinterpret_cast<uint32_t*>(sm + C.body);  // [rb][8]
  uint32_t* hist = sel + C.rb * 8;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rt = tid % C.rt, eg = tid / C.rt;  // row-thread fastest: a warp shares eg
  const int e0 = eg * EPG;
  const int64_t r0 = (int64_t)blockIdx.x * C.rb;
  const int nrow = (int)::min((int64_t)C.rb, T - r0);
  const int KC = C.kc, nch = (d + KC - 1) / KC;
  const int wq = (E + 3) / 4;  // 16-byte pieces per gate-weight row

  for (int i = tid; i <= E; i += gk::kThreads) hist[i] = 0;

  auto issue = [&](int c) {
    if (c < nch) {
      uint8_t* stg = sm + (size_t)(c % gk::NS) * C.stage;
      uint16_t* xs = reinterpret_cast<uint16_t*>(stg);
      float* ws = reinterpret_cast<float*>(stg + C.xbytes);
      const int k0 = c * KC, kc = ::min(KC, d - k0), kq = kc / 8;
      for (int i = tid; i < C.rb * kq; i += gk::kThreads) {
        const int r = i / kq, q = i % kq;
        const bool ok = r < nrow;
        cp_async16(xs + r * C.xpitch + q * 8, ok ? xn + (r0 + r) * d + k0 + q * 8 : xn, ok);
      }
      for (int i = tid; i < kc * wq; i += gk::kThreads) {
        const int kk = i / wq, q = i % wq;
        cp_async16(ws + kk * gwp + q * 4, gw32 + (size_t)(k0 + kk) * gwp + q * 4, true);
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
  float* xf = reinterpret_cast<float*>(sm + C.off_xf);

  for (int c = 0; c < nch; ++c) {
    cp_async_wait<gk::NS - 2>();
    __syncthreads();  // chunk c landed; previous chunk's f32 copy fully consumed
    const uint8_t* stg = sm + (size_t)(c % gk::NS) * C.stage;
    const uint16_t* xs = reinterpret_cast<const uint16_t*>(stg);
    const int kc = ::min(KC, d - c * KC), kq = kc / 8;
    // widen the chunk once (fp16 -> f32 exactly), instead of per expert group
    for (int i = tid; i < C.rb * kq; i += gk::kThreads) {
      const int r = i / kq, q = i % kq;
      const uint4 v = *reinterpret_cast<const uint4*>(xs + r * C.xpitch + q * 8);
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
      float4* dst = reinterpret_cast<float4*>(xf + r * C.fpitch + q * 8);
      dst[0] = make_float4(h2f(h[0]), h2f(h[1]), h2f(h[2]), h2f(h[3]));
      dst[1] = make_float4(h2f(h[4]), h2f(h[5]), h2f(h[6]), h2f(h[7]));
    }
    issue(c + gk::NS - 1);
    __syncthreads();
    const float* wp = reinterpret_cast<const float*>(stg + C.xbytes) + e0;
    if (e0 < E) {
      const float* xr = xf + rt * C.fpitch;
      for (int kk = 0; kk < kc; kk += 4) {
        float4 xv[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i)
          xv[i] = *reinterpret_cast<const float4*>(xr + i * C.rt * C.fpitch + kk);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* wr = wp + (kk + q) * gwp;
          if constexpr (EPG >= 2) {
            float2 w[NP];
            if constexpr (EPG >= 4) {
#pragma unroll
              for (int j = 0; j < NP; j += 2) {
                const float4 w4 = *reinterpret_cast<const float4*>(wr + 2 * j);
                w[j] = make_float2(w4.x, w4.y);
                w[j + 1] = make_float2(w4.z, w4.w);
              }
            } else {
              w[0] = *reinterpret_cast<const float2*>(wr);
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const float xq = q == 0 ? xv[i].x : q == 1 ? xv[i].y : q == 2 ? xv[i].z : xv[i].w;
#pragma unroll
              for (int j = 0; j < NP; ++j) acc[i][j] = gk::ffma2(xq, w[j], acc[i][j]);  // exact products
            }
          } else {
            const float w0 = wr[0];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
              const float xq = q == 0 ? xv[i].x : q == 1 ? xv[i].y : q == 2 ? xv[i].z : xv[i].w;
              acc[i][0].x = fmaf(xq, w0, acc[i][0].x);
            }
          }
        }
      }
    }
  }
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

int64_t gate_fused_pitch(int64_t E) { return (E + 3) / 4 * 4; }

// (EPG, RPT): the most chains per thread (FFMA2 pairs, shared weight loads)
// that still fills the machine; below that the gate is latency-bound and
// 8 expert chains per thread beat many one-chain CTAs.
static void pick(int64_t T, int64_t E, int k, int* epg, int* rpt) {
  const int64_t gwp = gate_fused_pitch(E);
  const gk::Cfg c82 = gk::cfg((int)E, (int)gwp, 8, 2);
  if ((int64_t)c82.rb * k <= 1024 && (T + c82.rb - 1) / c82.rb >= 148) {
    *epg = 8;
    *rpt = 2;
    return;
  }
  static const int kEpg[] = {8, 4, 2, 1};
  for (int i = 0; i < 4; ++i) {
    const gk::Cfg c = gk::cfg((int)E, (int)gwp, kEpg[i], 1);
    if ((int64_t)c.rb * k <= 1024) {
      *epg = kEpg[i];
      *rpt = 1;
      return;
    }
  }
  *epg = 1;
  *rpt = 1;
}

int gate_fused_rows(int64_t T, int64_t E, int k) {
  int epg, rpt;
  pick(T, E, k, &epg, &rpt);
  return gk::cfg((int)E, (int)gate_fused_pitch(E), epg, rpt).rb;
}

bool gate_fused_supported(int64_t d, int64_t E, int k) {
  if (d % 8 != 0 || k < 1 || k > 8 || E < 1 || E > 256) return false;
  if ((size_t)lnr::ROWS * (d + 8) * 2 + 256 > 200 * 1024) return false;
  // slots of one gate block must fit a plan_place block (<= 1024 threads)
  const gk::Cfg c = gk::cfg((int)E, (int)gate_fused_pitch(E), 1, 1);
  return (int64_t)c.rb * k <= 1024 && c.total <= 200 * 1024;
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
  gate_topk_kernel<EPG, RPT><<<grid, gk::kThreads, C.total, st>>>(
      a.xn, a.T, (int)a.d, a.gw32, (int)a.gwp, a.gb, (int)a.E, a.k, a.finished, a.expert,
      a.scale, a.blockcnt, a.bad_row);
  note_launch();
  return check_launch("gate_topk");
}

int launch_gate_fused(const GateFusedArgs& a, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  // 1. LayerNorm rows
  const size_t smem = (size_t)lnr::ROWS * (a.d + 8) * 2 + 2 * lnr::ROWS * 4 + 16;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(ln_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    attr = smem;
  }
  ln_rows_kernel<<<(unsigned)((a.T + lnr::ROWS - 1) / lnr::ROWS), lnr::kThreads, smem, st>>>(
      a.x, a.T, (int)a.d, a.g, a.b, a.xn);
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
