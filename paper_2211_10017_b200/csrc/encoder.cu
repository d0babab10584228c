// encoder.cu -- encoder_forward (proj/src/model.cpp:351-398) of a .moec
// checkpoint on the GPU.  Per encoder layer:
//   attention_forward (model.cpp:207-256): LN -> Q, K, V = gemm_f16 ->
//     per (sentence, head) attend_one (attn_inner.hpp:20-50) -> O = gemm_f16
//     -> x + O (half_add);
//   then the layer's FFN: the MoE block (layer_forward, top-1, no finished
//   rows: model.cpp:387) or dense_ffn_forward (model.cpp:258-271: LN ->
//   gemm_f16 ReLU -> gemm_f16 -> half_add);
// then the final LayerNorm.  EXACT mode is bit-identical to the reference:
// LayerNorm and the gemm_f16 panels run the reference's serial f32 chains
// (k_gate.cu, k_gemm_exact.cu), attend_one's chains are restated below in
// the same order (f32 products and sums RN, glibc expf port, p = s_j / sum
// per element), half_add is fp16 RN.  FAST mode runs the projections and the
// MoE experts on the tcgen05 path (within the layer tolerance).
#include <cmath>
#include <cstring>

#include "encoder.cuh"
#include "glibc_expf.h"

namespace moecu {

EncoderDev::~EncoderDev() {
  for (void* p : allocs) cudaFree(p);
  for (void* p : {(void*)x, (void*)x2, (void*)xn, (void*)q, (void*)k, (void*)v, (void*)ctx,
                  (void*)o, (void*)h, (void*)tokens, (void*)problem, (void*)bad, (void*)ident,
                  (void*)ones})
    if (p) cudaFree(p);
}

int enc_upload(EncoderDev* E, const uint16_t* host, int64_t count, uint16_t** out) {
  MOE_CUDA_TRY(cudaMalloc(out, count * 2));
  E->allocs.push_back(*out);
  MOE_CUDA_TRY(cudaMemcpy(*out, host, count * 2, cudaMemcpyHostToDevice));
  return MOE_OK;
}

int enc_linear(EncoderDev* E, const uint16_t* w, const uint16_t* b, int64_t m, int64_t n,
               DevLinear* out) {
  out->m = m;
  out->n = n;
  uint16_t* tmp = nullptr;
  MOE_CUDA_TRY(cudaMalloc(&tmp, m * n * 2));
  MOE_CUDA_TRY(cudaMemcpy(tmp, w, m * n * 2, cudaMemcpyHostToDevice));
  MOE_CUDA_TRY(cudaMalloc(&out->tiled, tiled_bytes(1, m, n, 16)));
  E->allocs.push_back(out->tiled);
  const int st = launch_tile_weights(tmp, 1, m, n, 16, out->tiled, nullptr);
  MOE_CUDA_TRY(cudaDeviceSynchronize());
  cudaFree(tmp);
  TRY(st);
  return enc_upload(E, b, n, &out->bias);
}

namespace {

__device__ __forceinline__ uint16_t hadd(uint16_t a, uint16_t b) {
  return __half_as_ushort(__hadd_rn(__ushort_as_half(a), __ushort_as_half(b)));
}

// x[s * len + p] = tok_embed[src[s][p]] (+) pos_embed[p]   (model.cpp:373-382)
__global__ void embed_kernel(const int32_t* __restrict__ tok, int64_t t, int64_t len, int64_t d,
                             const uint16_t* __restrict__ te, const uint16_t* __restrict__ pe,
                             int64_t vocab, uint16_t* __restrict__ x, uint32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d, c = i - r * d;
    const int32_t id = tok[r];
    if (id < 0 || id >= vocab) {
      atomicMin(bad, (uint32_t)r);
      x[i] = 0;
      continue;
    }
    x[i] = hadd(te[(int64_t)id * d + c], pe[(r % len) * d + c]);
  }
}

// out = a (+) b, fp16 RN (the residuals: model.cpp:252-254, 267-269)
__global__ void add_kernel(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b,
                           int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hadd(a[i], b[i]);
}

// attend_one (attn_inner.hpp:20-50) for every query row of one sentence and
// one head: CTA (sentence, head).  Every chain keeps the reference's order;
// the chains themselves are independent, so they are spread over the
// threads, four per thread in flight:
//   1. s[r][j] = (sum_c q[r][c] k[j][c]) * inv_sqrt_dk   (c ascending)
//   2. per row: max, e_j = expf(s_j - max), sum_j e_j (j ascending),
//      p[r][j] = e_j / sum (the reference's per-element division)
//   3. ctx[r][c] = sum_j p[r][j] v[j][c]                   (j ascending)
// q rows, the head's K and V slices and the score matrix live in shared
// memory; the expf table too.
__global__ void attention_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ k,
                                 const uint16_t* __restrict__ v, int len, int64_t d, int64_t ld,
                                 int dk, float inv_sqrt_dk, uint16_t* __restrict__ ctx) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(sm);
  float* sc = reinterpret_cast<float*>(sm + 32 * 8);  // [len][len + 1]
  const int lp = len + 1;
  // K rows at a pitch of dk + 2 halves: lanes reading one column of
  // consecutive keys hit consecutive banks (at dk they all hit one bank)
  const int kp = dk + 4;  // 8-byte aligned rows for the 4-column vector loads
  uint16_t* qs = reinterpret_cast<uint16_t*>(sc + (int64_t)len * lp);  // [len][kp]
  uint16_t* ks = qs + len * kp;                                        // [len][kp]
  uint16_t* vs = ks;  // V replaces K after the scores (two CTAs per SM at len 128)
  float* rsum = reinterpret_cast<float*>(ks + len * kp);              // [len]
  const int64_t s0 = (int64_t)blockIdx.x * len;  // first row of the sentence
  const int h0 = blockIdx.y * dk;
  const int nt = blockDim.x;
  for (int i = threadIdx.x; i < 32; i += nt) tab[i] = moe_expf_tab_dev[i];
  for (int i = threadIdx.x; i < len * dk; i += nt) {
    const int j = i / dk, c = i - j * dk;
    const int64_t g = (s0 + j) * ld + h0 + c;
    qs[j * kp + c] = q[g];
    ks[j * kp + c] = k[g];
  }
  __syncthreads();
  // 1. scores: a thread owns a 4 x 4 tile of (query row, key) chains; per
  // input column c it reads 4 q and 4 k values (4-column vectors) and runs
  // 16 independent chains (c ascending in each)
  const int nr4 = (len + 3) / 4, ntile = nr4 * nr4;
  for (int tix = threadIdx.x; tix < ntile; tix += nt) {
    const int r0 = (tix / nr4) * 4, j0 = (tix % nr4) * 4;
    float a[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) a[u][w] = 0.f;
    const uint16_t* qr[4];
    const uint16_t* kr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      qr[u] = qs + ::min(r0 + u, len - 1) * kp;
      kr[u] = ks + ::min(j0 + u, len - 1) * kp;
    }
    for (int c0 = 0; c0 < dk; c0 += 4) {
      uint2 qv[4], kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        qv[u] = *reinterpret_cast<const uint2*>(qr[u] + c0);
        kv[u] = *reinterpret_cast<const uint2*>(kr[u] + c0);
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float qf[4], kf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t qw = cc < 2 ? qv[u].x : qv[u].y, kw = cc < 2 ? kv[u].x : kv[u].y;
          qf[u] = h2f((uint16_t)((cc & 1) ? qw >> 16 : qw & 0xFFFFu));
          kf[u] = h2f((uint16_t)((cc & 1) ? kw >> 16 : kw & 0xFFFFu));
        }
        // fp16 x fp16 products are exact in f32, so one FMA equals the
        // reference's separately rounded multiply-then-add
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int w = 0; w < 4; ++w) a[u][w] = __fmaf_rn(qf[u], kf[w], a[u][w]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (r0 + u < len && j0 + w < len) sc[(r0 + u) * lp + j0 + w] = __fmul_rn(a[u][w], inv_sqrt_dk);
  }
  __syncthreads();
  // V into the K slots (K is no longer read)
  for (int i = threadIdx.x; i < len * dk; i += nt) {
    const int j = i / dk, c = i - j * dk;
    vs[j * kp + c] = v[(s0 + j) * ld + h0 + c];
  }
  // 2. softmax (attend_one's order where it matters): the row max is exact
  // in any order (a warp per row); every expf in parallel; the row sums
  // serially in key order (a thread per row); every p = e / sum in parallel
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < len; r += nt / 32) {
    float m = -INFINITY;
    for (int j = lane; j < len; j += 32) m = fmaxf(m, sc[r * lp + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) rsum[r] = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < len * len; i += nt) {
    const int r = i / len, j = i - r * len;
    sc[r * lp + j] = moe_glibc_expf_t(__fsub_rn(sc[r * lp + j], rsum[r]), tab);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < len; r += nt) {
    const float* e = sc + r * lp;
    float sum = 0.0f;
    for (int j = 0; j < len; ++j) sum = __fadd_rn(sum, e[j]);
    rsum[r] = sum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < len * len; i += nt) {
    const int r = i / len, j = i - r * len;
    sc[r * lp + j] = __fdiv_rn(sc[r * lp + j], rsum[r]);
  }
  __syncthreads();
  // 3. context: a thread owns 4 rows x 4 columns of outputs; per key j it
  // reads 4 probabilities and one 4-column vector of v (j ascending)
  const int nc4 = dk / 4, nout = nr4 * nc4;
  for (int tix = threadIdx.x; tix < nout; tix += nt) {
    const int r0 = (tix / nc4) * 4, c0 = (tix % nc4) * 4;
    float a[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int w = 0; w < 4; ++w) a[u][w] = 0.f;
    const float* pr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) pr[u] = sc + ::min(r0 + u, len - 1) * lp;
    for (int j = 0; j < len; ++j) {
      const uint2 vv = *reinterpret_cast<const uint2*>(vs + j * kp + c0);
      const float vf[4] = {h2f((uint16_t)(vv.x & 0xFFFFu)), h2f((uint16_t)(vv.x >> 16)),
                           h2f((uint16_t)(vv.y & 0xFFFFu)), h2f((uint16_t)(vv.y >> 16))};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float pu = pr[u][j];
#pragma unroll
        for (int w = 0; w < 4; ++w) a[u][w] = __fadd_rn(a[u][w], __fmul_rn(pu, vf[w]));
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (r0 + u < len)
#pragma unroll
        for (int w = 0; w < 4; ++w) ctx[(s0 + r0 + u) * d + h0 + c0 + w] = f2h(a[u][w]);
  }
}

// FAST mode (sentences of <= 128 tokens, head width a multiple of 16): the
// same attention on the tensor cores, flash-style in registers -- a warp owns
// 16 query rows: S = Q K^T by mma.m16n8k16 (f16 in, f32 accumulate), scale,
// row max / exp / row sum by quad shuffles, P = e / sum rounded to fp16 and
// reused in registers as the A operand of O = P V (V transposed in shared
// memory).  Not bit-exact (tensor-core sums, fp16 P, fast exp); within the
// layer tolerance.
constexpr int kAttMaxLen = 128;

__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  return (uint32_t)f2h(lo) | ((uint32_t)f2h(hi) << 16);
}

template <int DK>
__global__ void __launch_bounds__(256) attention_tc_kernel(const uint16_t* __restrict__ q,
                                                           const uint16_t* __restrict__ k,
                                                           const uint16_t* __restrict__ v, int len,
                                                           int64_t d, int64_t ld,
                                                           float inv_sqrt_dk,
                                                           uint16_t* __restrict__ ctx) {
  constexpr int P = DK + 8;                  // Q / K / V row pitch (halves): conflict-free
  constexpr int NT = kAttMaxLen / 8;         // key tiles of 8
  extern __shared__ __align__(16) uint16_t att_sm[];
  uint16_t* Qs = att_sm;                    // [kAttMaxLen][P]
  uint16_t* Ks = Qs + kAttMaxLen * P;       // [kAttMaxLen][P]
  uint16_t* Vs = Ks + kAttMaxLen * P;       // [kAttMaxLen][P] (row-major; ldmatrix.trans)
  const int Lp = (len + 15) & ~15;
  const int64_t s0 = (int64_t)blockIdx.x * len;
  const int h0 = blockIdx.y * DK;
  constexpr int C8 = DK / 8;  // 16-byte pieces per head row
  for (int i = threadIdx.x; i < Lp * C8; i += blockDim.x) {
    const int j = i / C8, c = (i - j * C8) * 8;
    uint4 qv = make_uint4(0, 0, 0, 0), kv = qv, vv = qv;
    if (j < len) {
      const int64_t g = (s0 + j) * ld + h0 + c;
      qv = *reinterpret_cast<const uint4*>(q + g);
      kv = *reinterpret_cast<const uint4*>(k + g);
      vv = *reinterpret_cast<const uint4*>(v + g);
    }
    *reinterpret_cast<uint4*>(Qs + j * P + c) = qv;
    *reinterpret_cast<uint4*>(Ks + j * P + c) = kv;
    *reinterpret_cast<uint4*>(Vs + j * P + c) = vv;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (warp * 16 >= Lp) return;
  const int r0 = warp * 16;
  const int ntile = Lp / 8;
  float acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  // S = Q K^T
#pragma unroll
  for (int kk = 0; kk < DK / 16; ++kk) {
    const uint16_t* qa = Qs + (r0 + g) * P + kk * 16 + 2 * t;
    const uint32_t a0 = *reinterpret_cast<const uint32_t*>(qa);
    const uint32_t a1 = *reinterpret_cast<const uint32_t*>(qa + 8 * P);
    const uint32_t a2 = *reinterpret_cast<const uint32_t*>(qa + 8);
    const uint32_t a3 = *reinterpret_cast<const uint32_t*>(qa + 8 * P + 8);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      if (j < ntile) {
        const uint16_t* kb = Ks + (j * 8 + g) * P + kk * 16 + 2 * t;
        mma16816(acc[j], a0, a1, a2, a3, *reinterpret_cast<const uint32_t*>(kb),
                 *reinterpret_cast<const uint32_t*>(kb + 8));
      }
    }
  }
  // softmax over keys (rows g and g + 8 of the strip; columns 8j + 2t, +1)
  float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < ntile) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = j * 8 + 2 * t + (e & 1);
        acc[j][e] = key < len ? acc[j][e] * inv_sqrt_dk : -INFINITY;
      }
      mx0 = fmaxf(mx0, fmaxf(acc[j][0], acc[j][1]));
      mx1 = fmaxf(mx1, fmaxf(acc[j][2], acc[j][3]));
    }
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    if (j < ntile) {
      acc[j][0] = __expf(acc[j][0] - mx0);
      acc[j][1] = __expf(acc[j][1] - mx0);
      acc[j][2] = __expf(acc[j][2] - mx1);
      acc[j][3] = __expf(acc[j][3] - mx1);
      sum0 += acc[j][0] + acc[j][1];
      sum1 += acc[j][2] + acc[j][3];
    }
  }
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    sum0 += __shfl_xor_sync(0xffffffffu, sum0, o);
    sum1 += __shfl_xor_sync(0xffffffffu, sum1, o);
  }
  const float is0 = 1.f / sum0, is1 = 1.f / sum1;
  // O = P V: the S accumulators of key tiles 2u, 2u + 1 are the A fragment
  // of k-step u
  float o[DK / 8][4];
#pragma unroll
  for (int c8 = 0; c8 < DK / 8; ++c8) o[c8][0] = o[c8][1] = o[c8][2] = o[c8][3] = 0.f;
#pragma unroll
  for (int u = 0; u < NT / 2; ++u) {
    if (2 * u < ntile) {
      const uint32_t a0 = pack_h2(acc[2 * u][0] * is0, acc[2 * u][1] * is0);
      const uint32_t a1 = pack_h2(acc[2 * u][2] * is1, acc[2 * u][3] * is1);
      const uint32_t a2 = pack_h2(acc[2 * u + 1][0] * is0, acc[2 * u + 1][1] * is0);
      const uint32_t a3 = pack_h2(acc[2 * u + 1][2] * is1, acc[2 * u + 1][3] * is1);
#pragma unroll
      for (int c8 = 0; c8 < DK / 8; ++c8) {
        // B (keys x columns) fragment of V[16u.., 8c8..] by a transposing
        // matrix load: lanes 0-15 address the 16 key rows
        uint32_t b0, b1;
        const uint16_t* vrow = Vs + (u * 16 + (lane & 15)) * P + c8 * 8;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                     : "=r"(b0), "=r"(b1) : "r"(smem_u32(vrow)));
        mma16816(o[c8], a0, a1, a2, a3, b0, b1);
      }
    }
  }
#pragma unroll
  for (int c8 = 0; c8 < DK / 8; ++c8) {
    const int col = h0 + c8 * 8 + 2 * t;
    const int ra = r0 + g, rb2 = r0 + g + 8;
    if (ra < len)
      *reinterpret_cast<uint32_t*>(ctx + (s0 + ra) * d + col) = pack_h2(o[c8][0], o[c8][1]);
    if (rb2 < len)
      *reinterpret_cast<uint32_t*>(ctx + (s0 + rb2) * d + col) = pack_h2(o[c8][2], o[c8][3]);
  }
}

int blocks_for(int64_t n);

// y = x W + b (ReLU); residual non-null: out = residual (+) y.  FAST mode
// folds the residual into the tcgen05 epilogue (its k = 1 combine form with
// an identity row map and unit scales -- the same fp16 RN add); EXACT keeps
// the separate add so every op stays the reference's.
int gemm(EncoderDev* E, const uint16_t* x, int64_t t, const DevLinear& w, int relu, int mode,
         uint16_t* out, cudaStream_t st, const uint16_t* residual = nullptr,
         uint16_t* res_out = nullptr) {
  GemmArgs g{x, t, w.m, E->problem, 1, w.tiled, nullptr, 16, 1, w.n, w.bias, relu, out,
             0, t};
  if (mode == MOE_MODE_EXACT) {
    TRY(launch_gemm_exact(g, st));
  } else {
    if (residual) {
      g.cx = residual;
      g.cperm = E->ident;
      g.cscale = E->ones;
      g.cout = res_out;
    }
    TRY(launch_gemm_tc(g, st));
    if (residual) return MOE_OK;
  }
  if (residual) {
    add_kernel<<<blocks_for(t * w.n), 256, 0, st>>>(residual, out, t * w.n, res_out);
    note_launch();
  }
  return MOE_OK;
}

__global__ void fill_ident_kernel(uint32_t* ident, uint16_t* ones, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ident[i] = (uint32_t)i;
    ones[i] = 0x3C00;  // 1.0
  }
}

int blocks_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 8); }

// LayerNorm rows (model.cpp:175-195): the LN-only instantiation of the fused
// gate kernel (same serial chains; rows staged by bulk copies) when the rows
// are 16-byte aligned, else the standalone row kernel
int layer_norm(EncoderDev* E, const uint16_t* x, int64_t t, const uint16_t* g, const uint16_t* b,
               uint16_t* out, cudaStream_t st) {
  const int64_t d = E->d;
  if (d % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    GateFusedArgs a{x, t, d, g, b, nullptr, 0, nullptr, 0, 1, nullptr, out, nullptr, nullptr,
                    nullptr, E->bad, 0, nullptr};
    return launch_ln_rows(a, st);
  }
  return launch_layer_norm(x, t, d, g, b, out, st);
}

}  // namespace
}  // namespace moecu

using namespace moecu;

struct moe_moec;
namespace moecu {
EncoderDev* moec_encoder(moe_moec* M);
moe_layer* moec_layer(moe_moec* M, int i);
}  // namespace moecu

extern "C" int moe_encoder_forward(moe_moec* M, const int32_t* tokens, int64_t batch, int64_t len,
                                   int mode, uint16_t* out, moe_stream_t stream) {
  if (!M) return set_error(MOE_EINVAL, "encoder: null argument");
  // encoder_forward's checks first (model.cpp:354-366)
  if (batch <= 0 || !tokens) return set_error(MOE_EINVAL, "encoder: empty batch");
  if (!out) return set_error(MOE_EINVAL, "encoder: null argument");
  EncoderDev* E = moec_encoder(M);
  if (!E) return set_error(MOE_EINVAL, "encoder: checkpoint was loaded without device layers");
  if (mode != MOE_MODE_EXACT && mode != MOE_MODE_FAST) return set_error(MOE_EINVAL, "encoder: bad mode");
  if (len < 1 || len > E->maxlen) return set_error(MOE_EINVAL, "encoder: source length out of range");
  const int64_t t = batch * len, d = E->d;
  if (len > 256) return set_error(MOE_EINVAL, "encoder: sentences longer than 256 tokens");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (t > E->cap_t) {
    for (void* p : {(void*)E->x, (void*)E->x2, (void*)E->xn, (void*)E->q, (void*)E->k, (void*)E->v,
                    (void*)E->ctx, (void*)E->o, (void*)E->h, (void*)E->tokens})
      if (p) cudaFree(p);
    if (E->ident) cudaFree(E->ident);
    if (E->ones) cudaFree(E->ones);
    for (uint16_t** p : {&E->x, &E->x2, &E->xn, &E->ctx, &E->o})
      MOE_CUDA_TRY(cudaMalloc(p, t * d * 2));
    MOE_CUDA_TRY(cudaMalloc(&E->q, t * 3 * d * 2));  // Q | K | V rows
    MOE_CUDA_TRY(cudaMalloc(&E->h, t * E->f * 2));
    MOE_CUDA_TRY(cudaMalloc(&E->tokens, t * 4));
    MOE_CUDA_TRY(cudaMalloc(&E->ident, t * 4));
    MOE_CUDA_TRY(cudaMalloc(&E->ones, t * 2));
    fill_ident_kernel<<<blocks_for(t), 256, 0, st>>>(E->ident, E->ones, t);
    note_launch();
    E->cap_t = t;
  }
  if (!E->problem) {
    MOE_CUDA_TRY(cudaMalloc(&E->problem, 3 * 4));
    MOE_CUDA_TRY(cudaMalloc(&E->bad, 4));
  }
  const uint32_t prob[3] = {0u, 0u, (uint32_t)t};
  MOE_CUDA_TRY(cudaMemcpyAsync(E->problem, prob, 12, cudaMemcpyHostToDevice, st));
  MOE_CUDA_TRY(cudaMemcpyAsync(E->tokens, tokens, t * 4, cudaMemcpyHostToDevice, st));
  MOE_CUDA_TRY(cudaMemsetAsync(E->bad, 0xFF, 4, st));
  embed_kernel<<<blocks_for(t * d), 256, 0, st>>>(E->tokens, t, len, d, E->tok, E->pos, E->vocab,
                                                  E->x, E->bad);
  note_launch();
  uint32_t bad = 0;
  MOE_CUDA_TRY(cudaMemcpyAsync(&bad, E->bad, 4, cudaMemcpyDeviceToHost, st));
  MOE_CUDA_TRY(cudaStreamSynchronize(st));
  if (bad != 0xFFFFFFFFu) return set_error(MOE_EINVAL, "encoder: token id out of range");
  const int dk = (int)(d / E->heads);
  if (dk % 4 != 0) return set_error(MOE_EINVAL, "encoder: head width (d_model / n_heads) must be a multiple of 4");
  const float inv_sqrt_dk = 1.0f / std::sqrt((float)dk);
  const size_t att_smem = 32 * 8 + (size_t)len * (len + 1) * 4 + (size_t)2 * len * (dk + 4) * 2 + (size_t)len * 4 + 16;
  if (att_smem > 220 * 1024)
    return set_error(MOE_EINVAL, "encoder: sentence too long for the attention kernel's shared memory");
  if (att_smem > 48 * 1024)
    MOE_CUDA_TRY(cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)att_smem));
  uint16_t* x = E->x;
  uint16_t* y = E->x2;
  for (const EncLayerDev& l : E->layers) {
    // attention_forward (model.cpp:207-256)
    TRY(layer_norm(E, x, t, l.ln_g, l.ln_b, E->xn, st));
    // Q | K | V as one projection (W_q | W_k | W_v column-concatenated at load:
    // every output column's chain is unchanged, xn is read once)
    TRY(gemm(E, E->xn, t, l.qkv, 0, mode, E->q, st));
    const uint16_t* qp = E->q;
    const uint16_t* kp = E->q + d;
    const uint16_t* vp = E->q + 2 * d;
    const int64_t ld = 3 * d;
    if (mode == MOE_MODE_FAST && len <= kAttMaxLen && (dk == 64 || dk == 16 || dk == 32 || dk == 128)) {
      const dim3 grid((unsigned)batch, (unsigned)E->heads);
      const size_t tsm = (size_t)3 * kAttMaxLen * (dk + 8) * 2;
      auto go = [&](auto kern) -> int {
        if (tsm > 48 * 1024)
          MOE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
        kern<<<grid, 256, tsm, st>>>(qp, kp, vp, (int)len, d, ld, inv_sqrt_dk, E->ctx);
        return MOE_OK;
      };
      TRY(dk == 64 ? go(attention_tc_kernel<64>) : dk == 16 ? go(attention_tc_kernel<16>)
                   : dk == 32 ? go(attention_tc_kernel<32>) : go(attention_tc_kernel<128>));
    } else {
      attention_kernel<<<dim3((unsigned)batch, (unsigned)E->heads), 256, att_smem, st>>>(
          qp, kp, vp, (int)len, d, ld, dk, inv_sqrt_dk, E->ctx);
    }
    note_launch();
    TRY(check_launch("encoder attention"));
    TRY(gemm(E, E->ctx, t, l.o, 0, mode, E->o, st, x, y));  // y = x (+) O
    std::swap(x, y);
    // the FFN: MoE block (moe_ffn_forward, no finished rows) or dense
    if (l.moe_block >= 0) {
      TRY(layer_forward(moec_layer(M, l.moe_block), x, nullptr, t, 1, mode, y, st));
    } else {
      TRY(layer_norm(E, x, t, l.fln_g, l.fln_b, E->xn, st));
      TRY(gemm(E, E->xn, t, l.w1, 1, mode, E->h, st));
      TRY(gemm(E, E->h, t, l.w2, 0, mode, E->o, st, x, y));  // y = x (+) FFN
    }
    std::swap(x, y);
  }
  TRY(layer_norm(E, x, t, E->ln_g, E->ln_b, out, st));
  return check_launch("encoder");
}
