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

// Row-per-thread form for d % 8 == 0 (the hot path).  The serial chains are
// the latency floor, so each thread owns one row's chain and the block
// streams 64 rows x 64 columns at a time through a 4-deep cp.async ring;
// three passes (sum, centred sum of squares, normalise) re-stream the rows
// (the second and third hit L2).  Reading 8 fp16 per LDS.128 from 144-byte
// row pitches is bank-conflict free per quarter warp.
constexpr int LN_R = 64, LN_KC = 64, LN_NS = 4, LN_PITCH = LN_KC + 8;

__global__ void __launch_bounds__(LN_R) layer_norm_rows_kernel(const uint16_t* __restrict__ x,
                                                               int64_t T, int64_t d,
                                                               const uint16_t* __restrict__ g,
                                                               const uint16_t* __restrict__ b,
                                                               uint16_t* __restrict__ out) {
  __shared__ __align__(16) uint16_t buf[LN_NS][LN_R][LN_PITCH];
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * LN_R, row = r0 + tid;
  const int nch = (int)((d + LN_KC - 1) / LN_KC);
  auto issue = [&](int c) {
    if (c < nch) {
      uint16_t(*dst)[LN_PITCH] = buf[c % LN_NS];
      for (int i = tid; i < LN_R * (LN_KC / 8); i += LN_R) {
        const int rr = i / (LN_KC / 8), ch = i % (LN_KC / 8);
        const int64_t gr = r0 + rr, col = (int64_t)c * LN_KC + ch * 8;
        const bool ok = gr < T && col < d;
        cp_async16(&dst[rr][ch * 8], ok ? x + gr * d + col : x, ok);
      }
    }
    cp_async_commit();
  };
  float mean = 0.f, inv = 0.f;
  for (int pass = 0; pass < 3; ++pass) {
    float acc = 0.f;
    for (int c = 0; c < LN_NS - 1; ++c) issue(c);
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<LN_NS - 2>();
      __syncthreads();
      issue(c + LN_NS - 1);
      const uint16_t* rp = buf[c % LN_NS][tid];
      const int kc = (int)::min((int64_t)LN_KC, d - (int64_t)c * LN_KC);
      for (int j = 0; j < kc; j += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(rp + j);
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
        if (pass == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc = __fadd_rn(acc, h2f(h[i]));
        } else if (pass == 1) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float dx = __fsub_rn(h2f(h[i]), mean);
            acc = __fadd_rn(acc, __fmul_rn(dx, dx));
          }
        } else if (row < T) {
          const int64_t col = (int64_t)c * LN_KC + j;
          const uint4 gv = *reinterpret_cast<const uint4*>(g + col);
          const uint4 bv = *reinterpret_cast<const uint4*>(b + col);
          const uint16_t* gh = reinterpret_cast<const uint16_t*>(&gv);
          const uint16_t* bh = reinterpret_cast<const uint16_t*>(&bv);
          uint4 o;
          uint16_t* oh = reinterpret_cast<uint16_t*>(&o);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            oh[i] = f2h(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(h2f(h[i]), mean), inv), h2f(gh[i])),
                                  h2f(bh[i])));
          *reinterpret_cast<uint4*>(out + row * d + col) = o;
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    if (pass == 0) {
      mean = __fdiv_rn(acc, (float)d);
    } else if (pass == 1) {
      const float var = __fdiv_rn(acc, (float)d);
      inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
    }
  }
}

int launch_layer_norm(const uint16_t* x, int64_t T, int64_t d, const uint16_t* g,
                      const uint16_t* b, uint16_t* out, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  if (d % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (reinterpret_cast<uintptr_t>(g) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(b) & 15) == 0) {
    layer_norm_rows_kernel<<<(unsigned)((T + LN_R - 1) / LN_R), LN_R, 0, st>>>(x, T, d, g, b, out);
    note_launch();
    return check_launch("layer_norm");
  }
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
// One thread per row holding EC expert chains (EC in {1,2,4,8}, picked so
// T*E/EC threads fill the GPU: the serial k-chain latency is the floor).  The
// thread streams its own xn row with 16-byte loads; the block's EC gate
// columns are staged as f32 in shared memory and read as warp broadcasts.
constexpr int GL_ROWS = 128, GL_KCH = 256;

template <int EC>
__global__ void __launch_bounds__(GL_ROWS) gate_logits_kernel(
    const uint16_t* __restrict__ xn, int64_t T, int64_t d, const uint16_t* __restrict__ gw,
    const uint16_t* __restrict__ gb, int64_t E, int vec, float* __restrict__ logits) {
  __shared__ __align__(16) float ws[GL_KCH][EC];
  const int tid = threadIdx.x;
  const int64_t row = (int64_t)blockIdx.x * GL_ROWS + tid;
  const int64_t e0 = (int64_t)blockIdx.y * EC;
  const bool live = row < T;
  const uint16_t* xr = xn + (live ? row : 0) * d;
  float acc[EC];
#pragma unroll
  for (int j = 0; j < EC; ++j) acc[j] = 0.f;
  for (int64_t k0 = 0; k0 < d; k0 += GL_KCH) {
    const int kc = (int)::min((int64_t)GL_KCH, d - k0);
    __syncthreads();
    for (int i = tid; i < GL_KCH * EC; i += GL_ROWS) {
      const int kk = i / EC, j = i % EC;
      ws[kk][j] = (kk < kc && e0 + j < E) ? h2f(gw[(k0 + kk) * E + e0 + j]) : 0.f;
    }
    __syncthreads();
    if (!live) continue;
    if (vec) {
      for (int kk = 0; kk < kc; kk += 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(xr + k0 + kk);
        const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float xv = h2f(h[i]);
#pragma unroll
          for (int j = 0; j < EC; ++j) acc[j] = fmaf(xv, ws[kk + i][j], acc[j]);  // exact product
        }
      }
    } else {
      for (int kk = 0; kk < kc; ++kk) {
        const float xv = h2f(xr[k0 + kk]);
#pragma unroll
        for (int j = 0; j < EC; ++j) acc[j] = fmaf(xv, ws[kk][j], acc[j]);
      }
    }
  }
  if (!live) return;
#pragma unroll
  for (int j = 0; j < EC; ++j)
    if (e0 + j < E) logits[row * E + e0 + j] = __fadd_rn(acc[j], h2f(gb[e0 + j]));
}

int launch_gate_logits(const uint16_t* xn, int64_t T, int64_t d, const uint16_t* gw,
                       const uint16_t* gb, int64_t E, float* logits, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  int EC = 8;
  while (EC > 1 && (EC > E || T * ((E + EC - 1) / EC) < 16384)) EC >>= 1;
  const int vec = (d % 8 == 0) && (reinterpret_cast<uintptr_t>(xn) & 15) == 0;
  dim3 grid((unsigned)((T + GL_ROWS - 1) / GL_ROWS), (unsigned)((E + EC - 1) / EC));
  switch (EC) {
    case 8: gate_logits_kernel<8><<<grid, GL_ROWS, 0, st>>>(xn, T, d, gw, gb, E, vec, logits); break;
    case 4: gate_logits_kernel<4><<<grid, GL_ROWS, 0, st>>>(xn, T, d, gw, gb, E, vec, logits); break;
    case 2: gate_logits_kernel<2><<<grid, GL_ROWS, 0, st>>>(xn, T, d, gw, gb, E, vec, logits); break;
    default: gate_logits_kernel<1><<<grid, GL_ROWS, 0, st>>>(xn, T, d, gw, gb, E, vec, logits); break;
  }
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
