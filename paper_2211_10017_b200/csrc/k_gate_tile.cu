// k_gate_tile.cu -- K2 for wide gates (C4: E = 64, 16384 tokens; C5: E = 128):
// the f32 gate logits (proj/src/model.cpp:273-297) as a register-tiled
// CUDA-core GEMM, fused with top-k softmax (routing.cpp:11-41, top-k
// extension) and the routing-key histogram; the LayerNorm runs before it
// (ln_gate_kernel in LN-only mode writes xn).
//
// Why a separate kernel: in the one-kernel gate every CTA holds its rows for
// the serial LN chains, so at C4 it runs one CTA of 8 warps per SM (12.5 %
// warps active) over two waves and re-streams the 256 KB of f32 gate weights
// per CTA; its logit phase ran at ~35 % of the FMA pipe.  Here a CTA owns a
// tile of TR rows x all experts, 256 threads as 16 x 16, each thread RPT
// rows x EPT experts of chains (k ascending per chain -- exact: fp16 x fp16
// products are exact in f32, so FFMA2 == the reference's mul-then-add).
// Per input a thread reads RPT x values (two addresses per warp: broadcasts)
// and EPT weights from shared memory and issues RPT*EPT/2 FFMA2.  Inputs
// arrive in chunks of KC: x transposed to f32 [KC][TR], weights f32
// [KC][EP], double-buffered, the next chunk's global loads in flight during
// the current chunk's FMAs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace moecu {

namespace gt {
constexpr int KC = 32;  // inputs per staged chunk

__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  uint64_t r;
  const uint64_t bb = (uint64_t)__float_as_uint(b.x) | ((uint64_t)__float_as_uint(b.y) << 32);
  const uint64_t cc = (uint64_t)__float_as_uint(c.x) | ((uint64_t)__float_as_uint(c.y) << 32);
  const uint64_t aa = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
  return make_float2(__uint_as_float((uint32_t)r), __uint_as_float((uint32_t)(r >> 32)));
}

// RG x EG threads (RG % 8 == 0, EG % 4 == 0), each RPT rows x EPT experts
template <int RPT, int EPT, int RG, int EG>
struct Cfg {
  static constexpr int TR = RG * RPT, EP = EG * EPT, NT = RG * EG;
  static constexpr int XS = KC * TR, WS = KC * EP;     // floats per buffer
  static constexpr int STAGE = 2 * (XS + WS);          // two buffers
  static constexpr int LG = TR * (EP + 1);             // logits | expf
  static constexpr int BODY = STAGE > 2 * LG ? STAGE : 2 * LG;
  // [body floats] [bias EP] [sel TR*8 u32] [hist EP+1] [fin TR] [tab 32 u64]
  static constexpr int OFF_BIAS = BODY * 4;
  static constexpr int OFF_SEL = OFF_BIAS + EP * 4;
  static constexpr int OFF_HIST = OFF_SEL + TR * 8 * 4;
  static constexpr int OFF_FIN = OFF_HIST + (EP + 1) * 4;
  static constexpr int OFF_TAB = (OFF_FIN + TR + 15) / 16 * 16;
  static constexpr int SMEM = OFF_TAB + 32 * 8;
};
}  // namespace gt

template <int RPT, int EPT, int RG, int EG>
__global__ void __launch_bounds__(RG * EG, 1) gate_tile_kernel(
    const uint16_t* __restrict__ xn, int64_t T, int d, const float* __restrict__ gw32, int gwp,
    const uint16_t* __restrict__ gb, int E, int k, const uint8_t* __restrict__ finished,
    uint32_t* __restrict__ expert, uint16_t* __restrict__ scale, uint32_t* __restrict__ blockcnt,
    uint32_t* bad_row) {
  using C = gt::Cfg<RPT, EPT, RG, EG>;
  constexpr int TR = C::TR, EP = C::EP, KC = gt::KC, NT = C::NT;
  extern __shared__ __align__(16) uint8_t sm[];
  float* body = reinterpret_cast<float*>(sm);
  float* bsm = reinterpret_cast<float*>(sm + C::OFF_BIAS);
  uint32_t* sel = reinterpret_cast<uint32_t*>(sm + C::OFF_SEL);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sm + C::OFF_HIST);
  uint8_t* fsm = sm + C::OFF_FIN;
  uint64_t* tab = reinterpret_cast<uint64_t*>(sm + C::OFF_TAB);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * TR;
  const int nrow = (int)::min((int64_t)TR, T - r0);
  griddep_launch();
  griddep_wait();
  for (int i = tid; i < EP; i += NT) bsm[i] = i < E ? h2f(gb[i]) : 0.f;
  for (int i = tid; i <= E; i += NT) hist[i] = 0;
  for (int i = tid; i < 32; i += NT) tab[i] = moe_expf_tab_dev[i];
  for (int i = tid; i < TR; i += NT) fsm[i] = i < nrow && finished != nullptr ? finished[r0 + i] : 0;

  // ---- staging: chunk c of x (transposed, f32) and of the gate weights
  constexpr int XQ = TR * (KC / 8);        // 16-byte x pieces per chunk
  constexpr int XPT = (XQ + NT - 1) / NT;  // per thread
  constexpr int WQ = (KC / 2) * (EP / 2);  // float4 weight pieces (2 inputs x 2 experts)
  constexpr int WPT = (WQ + NT - 1) / NT;
  const int nch = (d + KC - 1) / KC;
  uint4 xr[XPT];
  float4 wr[WPT];
  auto load = [&](int c) {
    const int k0 = c * KC;
#pragma unroll
    for (int j = 0; j < XPT; ++j) {
      const int i = tid + j * NT;
      const int r = i % TR, q = i / TR;  // consecutive threads: consecutive rows
      const int kk = k0 + q * 8;
      const bool ok = i < XQ && r < nrow && kk < d;
      xr[j] = ok ? __ldg(reinterpret_cast<const uint4*>(xn + (r0 + r) * d + kk)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const int i = tid + j * NT;
      const int ep = i % (EP / 2), kp = i / (EP / 2);  // expert pair, input pair
      const int kk = k0 + 2 * kp;
      const bool ok = i < WQ && kk < d && 2 * ep < gwp;
      // gw32 [k/2][e/2][k%2][e%2]: inputs kk, kk+1 x experts 2ep, 2ep+1
      wr[j] = ok ? __ldg(reinterpret_cast<const float4*>(gw32 + (int64_t)(kk >> 1) * 2 * gwp + ep * 4))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
    float* xT = body + buf * (C::XS + C::WS);
    float* wS = xT + C::XS;
#pragma unroll
    for (int j = 0; j < XPT; ++j) {
      const int i = tid + j * NT;
      if (i >= XQ) break;
      const int r = i % TR, q = i / TR;
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&xr[j]);
#pragma unroll
      for (int u = 0; u < 8; ++u) xT[(q * 8 + u) * TR + r] = h2f(h[u]);
    }
#pragma unroll
    for (int j = 0; j < WPT; ++j) {
      const int i = tid + j * NT;
      if (i >= WQ) break;
      const int ep = i % (EP / 2), kp = i / (EP / 2);
      *reinterpret_cast<float2*>(wS + (2 * kp) * EP + 2 * ep) = make_float2(wr[j].x, wr[j].y);
      *reinterpret_cast<float2*>(wS + (2 * kp + 1) * EP + 2 * ep) = make_float2(wr[j].z, wr[j].w);
    }
  };

  // ---- the logit chains: thread (rg, eg) owns rows rg*RPT.. and experts
  // eg*EPT..; a warp covers 8 row groups x 4 expert groups, so each half-warp
  // reads 4 distinct x vectors and 4 distinct weight vectors per input (one
  // shared-memory wavefront each)
  constexpr int WE = EG / 4;  // warps along the experts
  const int eg = ((tid >> 5) % WE) * 4 + (tid & 3), rg = ((tid >> 5) / WE) * 8 + ((tid & 31) >> 2);
  float2 acc[RPT][EPT / 2];
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < EPT / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  load(0);
  store(0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) load(c + 1);  // in flight during this chunk's FMAs
    const float* xT = body + buf * (C::XS + C::WS);
    const float* wS = xT + C::XS;
    const int kn = ::min(KC, d - c * KC);
#pragma unroll 4
    for (int kk = 0; kk < kn; ++kk) {
      float xv[RPT];
      float wv[EPT];
      if constexpr (RPT % 4 == 0) {
#pragma unroll
        for (int i = 0; i < RPT; i += 4) {
          const float4 v = *reinterpret_cast<const float4*>(xT + kk * TR + rg * RPT + i);
          xv[i] = v.x;
          xv[i + 1] = v.y;
          xv[i + 2] = v.z;
          xv[i + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < RPT; i += 2) {
          const float2 v = *reinterpret_cast<const float2*>(xT + kk * TR + rg * RPT + i);
          xv[i] = v.x;
          xv[i + 1] = v.y;
        }
      }
#pragma unroll
      for (int j = 0; j < EPT; j += 4)  // one LDS.128 per 4 experts
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(wv[j]), "=f"(wv[j + 1]), "=f"(wv[j + 2]), "=f"(wv[j + 3])
                     : "r"(smem_u32(wS + kk * EP + eg * EPT + j)));
#pragma unroll
      for (int i = 0; i < RPT; ++i)
#pragma unroll
        for (int j = 0; j < EPT / 2; ++j)
          acc[i][j] = gt::ffma2(xv[i], make_float2(wv[2 * j], wv[2 * j + 1]), acc[i][j]);
    }
    if (c + 1 < nch) store(buf ^ 1);
    __syncthreads();
  }

  // ---- logits + bias (model.cpp:288-289) -> shared memory (staging drained)
  constexpr int LP = EP + 1;
  float* lg = body;
  float* ex = body + TR * LP;
#pragma unroll
  for (int i = 0; i < RPT; ++i)
#pragma unroll
    for (int j = 0; j < EPT; ++j) {
      const int r = rg * RPT + i, e = eg * EPT + j;
      const float a = (j & 1) ? acc[i][j / 2].y : acc[i][j / 2].x;
      lg[r * LP + e] = __fadd_rn(a, bsm[e]);
    }
  __syncthreads();

  // ---- top-k (routing.cpp:15-31): warp per row, strict '>', lowest index first
  const int warp = tid >> 5, lane = tid & 31;
  for (int r = warp; r < nrow; r += NT / 32) {
    const float* l = lg + r * LP;
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
        if (!tk && (v > bv || bj == 0x7FFFFFFF)) {
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
  __syncthreads();
  // ---- expf(l_j - max) for every (row, expert) in parallel (routing.cpp:34)
  for (int i = tid; i < nrow * E; i += NT) {
    const int r = i / E, j = i - r * E;
    const uint32_t s0 = sel[r * 8];
    if (s0 == 0xFFFFFFFFu) continue;
    const float* l = lg + r * LP;
    ex[r * LP + j] = moe_glibc_expf_t(__fsub_rn(l[j], l[s0]), tab);
  }
  __syncthreads();
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
      const float* exr = ex + r * LP;
      float sum = 0.f;
      int j = 0;
      for (; j + 8 <= E; j += 8) {
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
}

// ============================================================ host side
// Wide gates only: E a multiple of 16 in [48, 128] and enough (row x expert)
// work to fill the GPU; RPT picked so the tiles cover the SMs once.
// E = 64 only: at E = 128 (C5 widths, 4096 tokens) the tiles cannot fill
// the SMs with enough warps and the one-kernel gate is faster (measured
// 156 vs 142 us); MOE_GATE_TILE=128 admits it for A/B runs
bool gate_tile_supported(int64_t T, int64_t d, int64_t E, int k) {
  static const bool off = std::getenv("MOE_GATE_NO_TILE") != nullptr;  // dev A/B
  static const bool e128 = std::getenv("MOE_GATE_TILE") && std::atoi(std::getenv("MOE_GATE_TILE")) == 128;
  return !off && d % 8 == 0 && (E == 64 || (e128 && E == 128)) && k >= 1 && k <= 8 &&
         T * E >= (int64_t)1 << 18;
}

int gate_tile_rows(int64_t T, int64_t E) {
  static const int force = std::getenv("MOE_GATE_TILE_RPT") ? std::atoi(std::getenv("MOE_GATE_TILE_RPT")) : 0;
  if (force == 2 || force == 4 || force == 8) return 16 * force;
  // rows per tile: 16 * RPT, RPT in {2, 4, 8}: the largest whose tiles still
  // give every SM one
  const int64_t sms = sm_count();
  for (int rpt : {8, 4})
    if ((T + 16 * rpt - 1) / (16 * rpt) >= sms) return 16 * rpt;
  return 32;
}

template <int RPT, int EPT, int RG, int EG>
static int launch_tile(const GateFusedArgs& a, cudaStream_t st) {
  using C = gt::Cfg<RPT, EPT, RG, EG>;
  static bool attr = false;
  if (!attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gate_tile_kernel<RPT, EPT, RG, EG>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const unsigned grid = (unsigned)((a.T + C::TR - 1) / C::TR);
  MOE_CUDA_TRY(launch_k(0, gate_tile_kernel<RPT, EPT, RG, EG>, dim3(grid), dim3(C::NT), C::SMEM, st,
                        (const uint16_t*)a.xn, a.T, (int)a.d, a.gw32, (int)a.gwp, a.gb, (int)a.E,
                        a.k, a.finished, a.expert, a.scale, a.blockcnt, a.bad_row));
  note_launch();
  return check_launch("gate_tile");
}

// tile shapes (rows per tile tr): 256 threads (16 row groups x 16 expert
// groups) x {8,4,2} rows x E/16 experts.  Measured at C4: 4 x 4 (tr 64) 90 us,
// 8 x 4 (tr 128) 90 us, 128 threads x 8 x 8 (tr 128) 106 us
int launch_gate_tile(const GateFusedArgs& a, int tr, cudaStream_t st) {
  if (a.T == 0) return MOE_OK;
  if (!gate_tile_supported(a.T, a.d, a.E, a.k)) return set_error(MOE_EINVAL, "gate_tile: unsupported shape");
  if (a.E == 64) {
    static const int shape = std::getenv("MOE_GATE_TILE_SHAPE") ? std::atoi(std::getenv("MOE_GATE_TILE_SHAPE")) : 0;
    if (tr == 64 && shape == 1) return launch_tile<8, 2, 8, 32>(a, st);  // dev A/B thread tiles
    if (tr == 64 && shape == 2) return launch_tile<2, 8, 32, 8>(a, st);
    if (tr == 128) return launch_tile<8, 4, 16, 16>(a, st);
    if (tr == 64) return launch_tile<4, 4, 16, 16>(a, st);
    if (tr == 32) return launch_tile<2, 4, 16, 16>(a, st);
  } else {
    if (tr == 128) return launch_tile<8, 8, 16, 16>(a, st);
    if (tr == 64) return launch_tile<4, 8, 16, 16>(a, st);
    if (tr == 32) return launch_tile<2, 8, 16, 16>(a, st);
  }
  return set_error(MOE_EINVAL, "gate_tile: no tile for E=%lld rows=%d", (long long)a.E, tr);
}

}  // namespace moecu
