// k_gate.cu -- K2 gating: LayerNorm, f32 gate logits, top-k softmax gate.
//
// Bit-exactness with the reference (proj/src/model.cpp:175-205, 273-297;
// proj/src/routing.cpp:11-41) requires the reference's SERIAL f32 orders:
//   * LN mean/var are left-to-right sums over d, every op RN32 separately
//     (no contraction: __fadd_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn);
//   * a logit is acc = acc + x_k*w_kj for k ascending, then + b_j; the
//     fp16 x fp16 product is exact in f32, so fmaf() == mul-then-add here;
//   * the softmax sum runs over experts in index order using the host libm
//     expf (glibc_expf.h, bit-exact port).
// Parallelism therefore comes from independent chains: rows (LN), and
// (row, expert) pairs register-blocked 4x4 per thread (logits).
#include "kernels.cuh"

namespace moecu {

// ------------------------------------------------------------------- LayerNorm
// One warp per row: the row is staged in shared memory with 16-byte loads,
// lane 0 runs the two serial reductions, all lanes normalise.
__global__ void __launch_bounds__(128) layer_norm_kernel(const uint16_t* __restrict__ x,
                                                         int64_t T, int64_t d,
                                                         const uint16_t* __restrict__ g,
                                                         const uint16_t* __restrict__ b,
                                                         uint16_t* __restrict__ out) {
  extern __shared__ float ln_sm[];  // 4 warps x d floats
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 4 + warp;
  if (r >= T) return;
  const int64_t stride = (d + 3) & ~int64_t(3);
  float* row = ln_sm + (size_t)warp * stride;
  const uint16_t* xr = x + r * d;
  for (int64_t i = lane; i < d; i += 32) row[i] = h2f(xr[i]);
  __syncwarp();
  float mean = 0.f, inv = 0.f;
  if (lane == 0) {
    float s0 = 0.f;
    int64_t i = 0;
    for (; i + 4 <= d; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(row + i);
      s0 = __fadd_rn(s0, v.x);
      s0 = __fadd_rn(s0, v.y);
      s0 = __fadd_rn(s0, v.z);
      s0 = __fadd_rn(s0, v.w);
    }
    for (; i < d; ++i) s0 = __fadd_rn(s0, row[i]);
    mean = __fdiv_rn(s0, (float)d);
    float v0 = 0.f;
    for (i = 0; i < d; ++i) {
      const float dx = __fsub_rn(row[i], mean);
      v0 = __fadd_rn(v0, __fmul_rn(dx, dx));
    }
    const float var = __fdiv_rn(v0, (float)d);
    inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  }
  mean = __shfl_sync(0xffffffffu, mean, 0);
  inv = __shfl_sync(0xffffffffu, inv, 0);
  uint16_t* orow = out + r * d;
  for (int64_t i = lane; i < d; i += 32) {
    const float y = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(row[i], mean), inv), h2f(g[i])),
                              h2f(b[i]));
    orow[i] = f2h(y);
  }
}

int launch_layer_norm(const uint16_t* x, int64_t T, int64_t d, const uint16_t* g,
                      const uint16_t* b, uint16_t* out, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  const size_t smem = (size_t)4 * ((d + 3) & ~int64_t(3)) * sizeof(float);
  if (smem > 48 * 1024) {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(layer_norm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      set = true;
    }
  }
  layer_norm_kernel<<<(unsigned)((T + 3) / 4), 128, smem, st>>>(x, T, d, g, b, out);
  note_launch();
  return check_launch("layer_norm");
}

// ----------------------------------------------------------------- gate logits
// Each thread owns a 4-row x 4-expert block of serial chains (16 independent
// accumulators, so the FMA latency of one chain is hidden by the others).
// A 64-thread block covers (64/EB)*4 rows x EB*4 experts, EB = expert groups
// chosen so small E does not waste lanes; x rows and gate-weight columns are
// staged in shared memory 32 k at a time (padded rows: conflict-free).
constexpr int GL_THREADS = 64;
constexpr int GL_KC = 32;

__global__ void __launch_bounds__(GL_THREADS) gate_logits_kernel(
    const uint16_t* __restrict__ xn, int64_t T, int64_t d, const uint16_t* __restrict__ gw,
    const uint16_t* __restrict__ gb, int64_t E, int EB, float* __restrict__ logits) {
  extern __shared__ float gl_sm[];
  const int RB = GL_THREADS / EB;
  float* xs = gl_sm;                          // [RB*4][GL_KC+1]
  float* ws = gl_sm + RB * 4 * (GL_KC + 1);   // [EB*4][GL_KC+1]
  const int tid = threadIdx.x;
  const int rg = tid / EB, eg = tid % EB;
  const int64_t r0 = (int64_t)blockIdx.x * RB * 4;
  const int64_t e0 = (int64_t)blockIdx.y * EB * 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int64_t k0 = 0; k0 < d; k0 += GL_KC) {
    const int kc = (int)::min((int64_t)GL_KC, d - k0);
    __syncthreads();
    for (int i = tid; i < RB * 4 * GL_KC; i += GL_THREADS) {
      const int rr = i / GL_KC, kk = i % GL_KC;
      const int64_t r = r0 + rr;
      xs[rr * (GL_KC + 1) + kk] = (r < T && kk < kc) ? h2f(xn[r * d + k0 + kk]) : 0.f;
    }
    for (int i = tid; i < EB * 4 * GL_KC; i += GL_THREADS) {
      const int kk = i / (EB * 4), ee = i % (EB * 4);
      const int64_t e = e0 + ee;
      ws[ee * (GL_KC + 1) + kk] = (e < E && kk < kc) ? h2f(gw[(k0 + kk) * E + e]) : 0.f;
    }
    __syncthreads();
    const float* xr = xs + rg * 4 * (GL_KC + 1);
    const float* wr = ws + eg * 4 * (GL_KC + 1);
    for (int kk = 0; kk < kc; ++kk) {
      float xv[4], wv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xr[i * (GL_KC + 1) + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) wv[j] = wr[j * (GL_KC + 1) + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);  // exact product
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + rg * 4 + i;
    if (r >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t e = e0 + eg * 4 + j;
      if (e < E) logits[r * E + e] = __fadd_rn(acc[i][j], h2f(gb[e]));
    }
  }
}

int launch_gate_logits(const uint16_t* xn, int64_t T, int64_t d, const uint16_t* gw,
                       const uint16_t* gb, int64_t E, float* logits, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  int EB = 1;
  while (EB < 8 && EB * 4 < E) EB *= 2;
  const int RB = GL_THREADS / EB;
  const size_t smem = (size_t)(RB * 4 + EB * 4) * (GL_KC + 1) * sizeof(float);
  dim3 grid((unsigned)((T + RB * 4 - 1) / (RB * 4)), (unsigned)((E + EB * 4 - 1) / (EB * 4)));
  gate_logits_kernel<<<grid, GL_THREADS, smem, st>>>(xn, T, d, gw, gb, E, EB, logits);
  note_launch();
  return check_launch("gate_logits");
}

// ---------------------------------------------------------------- top-k gate
// One thread per row, serial over experts in index order (routing.cpp:24-38).
constexpr int kMaxTopK = 8;

__global__ void gate_topk_kernel(const float* __restrict__ logits, int64_t T, int64_t E, int k,
                                 uint32_t* __restrict__ expert, uint16_t* __restrict__ scale,
                                 uint32_t* bad_row) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= T) return;
  const float* l = logits + r * E;
  for (int64_t j = 0; j < E; ++j) {
    if (!isfinite(l[j])) {
      atomicMin(bad_row, (uint32_t)r);
      return;
    }
  }
  uint32_t sel[kMaxTopK];
  for (int s = 0; s < k; ++s) {
    int64_t best = -1;
    float bv = 0.f;
    for (int64_t j = 0; j < E; ++j) {
      bool taken = false;
      for (int q = 0; q < s; ++q) taken |= sel[q] == (uint32_t)j;
      if (taken) continue;
      const float v = l[j];
      if (best < 0 || v > bv) {  // strict: ties keep the lowest index
        best = j;
        bv = v;
      }
    }
    sel[s] = (uint32_t)best;
  }
  const float mx = l[sel[0]];
  float sum = 0.f;
  for (int64_t j = 0; j < E; ++j) sum = __fadd_rn(sum, moe_glibc_expf(__fsub_rn(l[j], mx)));
  for (int s = 0; s < k; ++s) {
    const float num = s == 0 ? 1.0f : moe_glibc_expf(__fsub_rn(l[sel[s]], mx));
    expert[r * k + s] = sel[s];
    scale[r * k + s] = f2h(__fdiv_rn(num, sum));
  }
}

int launch_gate_topk(const float* logits, int64_t T, int64_t E, int k, uint32_t* expert,
                     uint16_t* scale, uint32_t* bad_row, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  if (k < 1 || k > kMaxTopK || k > E)
    return set_error(MOE_EINVAL, "gate_topk: k must be in [1, min(n_experts, %d)]", kMaxTopK);
  gate_topk_kernel<<<(unsigned)((T + 127) / 128), 128, 0, st>>>(logits, T, E, k, expert, scale,
                                                                bad_row);
  note_launch();
  return check_launch("gate_topk");
}

}  // namespace moecu
