// k_gate_fused.cu -- K2 fused gating for the layer hot path:
//   LayerNorm (proj/src/model.cpp:175-205) -> f32 gate logits (:273-297) ->
//   top-k softmax gate (proj/src/routing.cpp:11-41, top-k extension) ->
//   per-block routing-key histogram (routing.cpp:55-62, first pass of the
//   counting sort) in ONE kernel, bit-exact with the reference.
//
// A CTA owns ROWS token rows (staged once in shared memory by cp.async) and
// runs every serial chain the reference defines on them:
//   * LN: one thread per row does the left-to-right f32 sum and the centred
//     sum of squares (the only true serial chains); all 256 threads then
//     normalise and write xn (shared + global, 16-byte stores).
//   * logits: every (row, expert) pair is an independent serial chain over
//     k; lane -> row, (warp, lane / ROWS) -> a group of EPG experts held in
//     registers.  fp16 x fp16 products are exact in f32, so fmaf == the
//     reference's mul-then-add; only the k order matters and is kept.  Gate
//     weights are pre-widened to f32 once per layer and streamed through a
//     3-stage cp.async ring of KC-row chunks (warp-broadcast reads).
//   * top-k: argmax by warp shuffle (value desc, index asc == the
//     reference's first maximum with strict '>'), expf of every logit in
//     parallel (device port of glibc expf), then one thread per row sums
//     them in expert order.
//   * histogram: key = finished ? E : expert per slot r*k+s, counted in
//     shared memory; blockcnt[block][E+1] feeds plan_scan (k_route.cu),
//     whose blocks are exactly this kernel's ROWS*k slots.
#include "kernels.cuh"

namespace moecu {

namespace gf {
constexpr int kThreads = 256;
constexpr int kMaxRing = 16;            // mbarriers in the gate-weight ring
constexpr size_t kBudget = 100 * 1024;  // target smem per CTA (2 CTAs / SM)

struct Smem {
  int xp;      // row pitch (halves)
  int lp;      // logits row pitch (floats)
  int kc;      // gate-weight rows per chunk
  int ring;    // chunks resident at once
  size_t off_w, off_l, off_st, off_h, off_bar, total;
};

// gwp = pitch (floats) of the widened gate weights in global and shared memory
__host__ __device__ inline Smem layout(int rows, int d, int E, int gwp) {
  Smem s;
  s.xp = d + 8;
  s.lp = E + 1;
  size_t off = (size_t)rows * s.xp * 2;
  off = (off + 15) & ~size_t(15);
  s.off_w = off;
  const size_t fixed = off + (size_t)2 * rows * s.lp * 4 + (size_t)rows * 10 * 4 +
                       (size_t)(E + 1) * 4 + kMaxRing * 8 + 256;
  // chunk: a multiple of 8 rows, ~8-16 KB; ring: as deep as the budget allows
  int kc = (int)(16384 / ((size_t)gwp * 4)) / 8 * 8;
  kc = kc < 8 ? 8 : (kc > 128 ? 128 : kc);
  if (kc > d) kc = (d + 7) / 8 * 8;
  const int nch = (d + kc - 1) / kc;
  const size_t cb = (size_t)kc * gwp * 4;
  int ring = fixed + cb * 2 < kBudget ? (int)((kBudget - fixed) / cb) : 2;
  ring = ring < 2 ? 2 : (ring > kMaxRing ? kMaxRing : ring);
  if (ring > nch) ring = nch;
  s.kc = kc;
  s.ring = ring;
  off += cb * ring + 64;  // + over-read slack of the last expert group
  off = (off + 15) & ~size_t(15);
  s.off_l = off;
  off += (size_t)2 * rows * s.lp * 4;  // logits, then expf values
  s.off_st = off;
  off += (size_t)rows * 2 * 4 + (size_t)rows * 8 * 4;  // mean, inv, sel[8]
  s.off_h = off;
  off += (size_t)(E + 1) * 4;
  off = (off + 7) & ~size_t(7);
  s.off_bar = off;
  off += (kMaxRing + 1) * 8;
  s.total = (off + 15) & ~size_t(15);
  return s;
}
}  // namespace gf

template <int ROWS, int EPG>
__global__ void __launch_bounds__(gf::kThreads) gate_fused_kernel(
    const uint16_t* __restrict__ x, int64_t T, int d, const uint16_t* __restrict__ g,
    const uint16_t* __restrict__ b, const float* __restrict__ gw32, int gwp,
    const uint16_t* __restrict__ gb, int E, int k, const uint8_t* __restrict__ finished,
    uint16_t* __restrict__ xn_out, uint32_t* __restrict__ expert, uint16_t* __restrict__ scale,
    uint32_t* __restrict__ blockcnt, uint32_t* bad_row) {
  constexpr int RPW = 32 / ROWS;       // row groups per warp
  extern __shared__ __align__(16) uint8_t sm[];
  const gf::Smem L = gf::layout(ROWS, d, E, gwp);
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm);
  float* ws = reinterpret_cast<float*>(sm + L.off_w);
  float* lg = reinterpret_cast<float*>(sm + L.off_l);
  float* st_mean = reinterpret_cast<float*>(sm + L.off_st);
  float* st_inv = st_mean + ROWS;
  uint32_t* sel = reinterpret_cast<uint32_t*>(st_inv + ROWS);  // [ROWS][8]
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + L.off_h);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.off_bar);  // [ring] chunks, [kMaxRing] rows

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = (int64_t)blockIdx.x * ROWS;
  const int nrow = (int)::min((int64_t)ROWS, T - r0);
  const int d8 = d / 8;
  const int KC = L.kc, NSL = L.ring;
  const int nch = (d + KC - 1) / KC;

  for (int i = tid; i <= E; i += gf::kThreads) hist[i] = 0;

  // ---- bulk-copy the rows and the first NSL gate-weight chunks (TMA engine)
  auto issue = [&](int c) {  // thread 0 only
    const int stg = c % NSL;
    const int kc = ::min(KC, d - c * KC);
    const uint32_t bytes = (uint32_t)kc * gwp * 4;
    mbar_arrive_expect_tx(&bars[stg], bytes);
    bulk_load(ws + (size_t)stg * KC * gwp, gw32 + (size_t)c * KC * gwp, bytes, &bars[stg]);
  };
  if (tid == 0) {
    for (int i = 0; i <= gf::kMaxRing; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
    uint64_t* bx = &bars[gf::kMaxRing];
    mbar_arrive_expect_tx(bx, (uint32_t)nrow * d * 2);
    for (int r = 0; r < nrow; ++r) bulk_load(xs + r * L.xp, x + (r0 + r) * d, (uint32_t)d * 2, bx);
    for (int c = 0; c < ::min(NSL, nch); ++c) issue(c);
  }
  __syncthreads();
  mbar_wait(&bars[gf::kMaxRing], 0);  // rows landed

  // ---- LN statistics: one serial chain per row (model.cpp:178-192)
  if (tid < nrow) {
    const uint16_t* row = xs + tid * L.xp;
    float s = 0.f;
    for (int c = 0; c < d8; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + c * 8);
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = __fadd_rn(s, h2f(h[i]));
    }
    const float mean = __fdiv_rn(s, (float)d);
    float v2 = 0.f;
    for (int c = 0; c < d8; ++c) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + c * 8);
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float dx = __fsub_rn(h2f(h[i]), mean);
        v2 = __fadd_rn(v2, __fmul_rn(dx, dx));
      }
    }
    const float var = __fdiv_rn(v2, (float)d);
    st_mean[tid] = mean;
    st_inv[tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  }
  __syncthreads();

  // ---- normalise (model.cpp:193-194): xs <- xn, and xn -> global
  for (int i = tid; i < nrow * d8; i += gf::kThreads) {
    const int r = i / d8, c = i % d8;
    uint4 v = *reinterpret_cast<const uint4*>(xs + r * L.xp + c * 8);
    const uint4 gv = __ldg(reinterpret_cast<const uint4*>(g) + c);
    const uint4 bv = __ldg(reinterpret_cast<const uint4*>(b) + c);
    uint16_t* h = reinterpret_cast<uint16_t*>(&v);
    const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gv);
    const uint16_t* bh = reinterpret_cast<const uint16_t*>(&bv);
    const float mean = st_mean[r], inv = st_inv[r];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      h[j] = f2h(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(h2f(h[j]), mean), inv), h2f(gh[j])),
                           h2f(bh[j])));
    *reinterpret_cast<uint4*>(xs + r * L.xp + c * 8) = v;
    *reinterpret_cast<uint4*>(xn_out + (r0 + r) * d + c * 8) = v;
  }

  // ---- logits: serial k chains (model.cpp:284-288)
  const int rr = lane % ROWS;
  const int grp = warp * RPW + lane / ROWS;
  const int e0 = grp * EPG;
  float acc[EPG];
#pragma unroll
  for (int j = 0; j < EPG; ++j) acc[j] = 0.f;
  const uint16_t* xrow = xs + rr * L.xp;
  __syncthreads();  // xn complete in shared memory
  for (int c = 0; c < nch; ++c) {
    const int stg = c % NSL;
    mbar_wait(&bars[stg], (uint32_t)(c / NSL) & 1u);
    const float* wc = ws + (size_t)stg * KC * gwp + e0;
    const int k0 = c * KC, kc = ::min(KC, d - k0);
    if (e0 < E) {
      for (int kk = 0; kk < kc; kk += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(xrow + k0 + kk);
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xv = h2f(h[i]);
          const float* wr = wc + (kk + i) * gwp;
          if constexpr (EPG >= 4) {
#pragma unroll
            for (int j = 0; j < EPG; j += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(wr + j);
              acc[j] = fmaf(xv, w4.x, acc[j]);
              acc[j + 1] = fmaf(xv, w4.y, acc[j + 1]);
              acc[j + 2] = fmaf(xv, w4.z, acc[j + 2]);
              acc[j + 3] = fmaf(xv, w4.w, acc[j + 3]);
            }
          } else {
#pragma unroll
            for (int j = 0; j < EPG; ++j) acc[j] = fmaf(xv, wr[j], acc[j]);
          }
        }
      }
    }
    __syncthreads();  // stage consumed by every thread
    if (tid == 0 && c + NSL < nch) issue(c + NSL);
  }
#pragma unroll
  for (int j = 0; j < EPG; ++j)
    if (e0 + j < E && rr < nrow) lg[rr * L.lp + e0 + j] = __fadd_rn(acc[j], h2f(gb[e0 + j]));
  __syncthreads();

  // ---- top-k selection (routing.cpp:15-31): one warp per row, shuffles
  for (int r = warp; r < nrow; r += 8) {
    const float* l = lg + r * L.lp;
    bool fin_ok = true;
    for (int j = lane; j < E; j += 32) fin_ok &= isfinite(l[j]);
    fin_ok = __all_sync(0xffffffffu, fin_ok);
    if (!fin_ok) {
      if (lane == 0) {
        atomicMin(bad_row, (uint32_t)(r0 + r));
        for (int s = 0; s < k; ++s) sel[r * 8 + s] = 0xFFFFFFFFu;
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
        if (!taken && (v > bv || bj == 0x7FFFFFFF)) {  // lane-local: first max (j ascends)
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
  float* ex = lg + ROWS * L.lp;
  for (int i = tid; i < nrow * E; i += gf::kThreads) {
    const int r = i / E, j = i % E;
    const uint32_t s0 = sel[r * 8];
    if (s0 == 0xFFFFFFFFu) continue;
    const float* l = lg + r * L.lp;
    ex[r * L.lp + j] = moe_glibc_expf(__fsub_rn(l[j], l[s0]));
  }
  __syncthreads();
  // serial Σ and scales, one thread per row (routing.cpp:33-38)
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
      const float* exr = ex + r * L.lp;
      float sum = 0.f;
      for (int j = 0; j < E; ++j) sum = __fadd_rn(sum, exr[j]);  // expert order
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
  for (int i = tid; i <= E; i += gf::kThreads) blockcnt[(int64_t)i * gridDim.x + blockIdx.x] = hist[i];
}

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

int gate_fused_rows(int64_t T) {
  if (T >= 32 * 148) return 32;
  if (T >= 16 * 148) return 16;
  return 8;
}

template <int ROWS, int EPG>
static int launch_gf(const GateFusedArgs& a, cudaStream_t st) {
  const gf::Smem L = gf::layout(ROWS, (int)a.d, (int)a.E, (int)a.gwp);
  static size_t attr = 0;
  if (L.total > 48 * 1024 && L.total > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gate_fused_kernel<ROWS, EPG>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total));
    attr = L.total;
  }
  const unsigned grid = (unsigned)((a.T + ROWS - 1) / ROWS);
  gate_fused_kernel<ROWS, EPG><<<grid, gf::kThreads, L.total, st>>>(
      a.x, a.T, (int)a.d, a.g, a.b, a.gw32, (int)a.gwp, a.gb, (int)a.E, a.k, a.finished, a.xn,
      a.expert, a.scale, a.blockcnt, a.bad_row);
  note_launch();
  return check_launch("gate_fused");
}

template <int ROWS>
static int launch_gf_rows(const GateFusedArgs& a, cudaStream_t st) {
  constexpr int NG = 8 * (32 / ROWS);
  const int64_t need = (a.E + NG - 1) / NG;
  if (need <= 1) return launch_gf<ROWS, 1>(a, st);
  if (need <= 2) return launch_gf<ROWS, 2>(a, st);
  if (need <= 4) return launch_gf<ROWS, 4>(a, st);
  if (need <= 8) return launch_gf<ROWS, 8>(a, st);
  return launch_gf<ROWS, 16>(a, st);
}

int64_t gate_fused_pitch(int64_t E) {
  // covers every expert group's float4 reads at every ROWS (see layout)
  return (E + 3) / 4 * 4;
}

bool gate_fused_supported(int64_t d, int64_t E, int k) {
  if (d % 8 != 0 || k < 1 || k > 8 || E < 1) return false;
  if (E > 128) return false;  // EPG <= 16 at ROWS = 32 (8 expert groups)
  const gf::Smem L = gf::layout(32, (int)d, (int)E, (int)gate_fused_pitch(E));
  return L.total <= 220 * 1024;
}

int launch_gate_fused(const GateFusedArgs& a, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  switch (a.rows) {
    case 32: return launch_gf_rows<32>(a, st);
    case 16: return launch_gf_rows<16>(a, st);
    default: return launch_gf_rows<8>(a, st);
  }
}

}  // namespace moecu
