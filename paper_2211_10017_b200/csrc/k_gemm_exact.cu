// k_gemm_exact.cu -- EXACT-mode grouped expert GEMM (CUDA cores).
//
// Reproduces proj/src/grouped_gemm.cpp:19-95 bit for bit: weight value
// w = RN16(((0x6400|code) - debias) * s) (fused magic dequant, dequant.hpp),
// acc = acc + x_k * w_k for k ascending in f32 (the fp16 x fp16 product is
// exact, so fmaf is the same single rounding), h = acc + bias,
// ReLU as !(h > 0) -> +0, one RN16.  This is the parity path (and the path
// the reference's own k-sequential test needs: 65504^2 + 1 - 65504^2 == 0);
// the throughput path is k_gemm_tc.cu.
//
// Work unit: (problem, 8 rows, 128 output columns); one thread per output
// column holding 8 row accumulators, walking the tiled weights
// (moe_tile_weights layout) one 64-wide k-block at a time with the
// activations staged in shared memory.
#include "kernels.cuh"

namespace moecu {

constexpr int kExRows = 8;

__device__ __forceinline__ int find_problem(const uint32_t* pre, int np, uint32_t t) {
  int lo = 0, hi = np - 1;  // largest p with pre[p] <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(128) gemm_exact_kernel(GemmArgs a) {
  extern __shared__ uint32_t ex_sm[];
  uint32_t* pre = ex_sm;                                        // np+1 tile prefix
  float* xs = reinterpret_cast<float*>(ex_sm + a.np + 1 + 3);  // [kExRows][64]
  const int tid = threadIdx.x;
  const int np = (int)a.np;
  const int64_t nft = (a.n + 127) / 128, nkb = (a.m + 63) / 64;
  if (tid == 0) {
    uint32_t run = 0;
    for (int p = 0; p < np; ++p) {
      pre[p] = run;
      const uint32_t len = a.problems[3 * p + 2] - a.problems[3 * p + 1];
      run += (len + kExRows - 1) / kExRows * (uint32_t)nft;
    }
    pre[np] = run;
  }
  __syncthreads();
  const uint32_t total = pre[np];
  const int wb = wblock_bytes(a.bits);
  const uint32_t db = a.debias;
  for (uint32_t t = blockIdx.x; t < total; t += gridDim.x) {
    const int p = find_problem(pre, np, t);
    const uint32_t local = t - pre[p];
    const int64_t ft = local % nft, rt = local / nft;
    const int64_t e = a.problems[3 * p];
    const int64_t r0 = a.problems[3 * p + 1] + rt * kExRows;
    const int64_t r1 = a.problems[3 * p + 2];
    const int64_t col = ft * 128 + tid;
    const bool live_col = col < a.n;
    const uint16_t s = (a.bits != 16 && live_col) ? a.scales[e * a.n + col] : 0x3C00;
    float acc[kExRows];
#pragma unroll
    for (int r = 0; r < kExRows; ++r) acc[r] = 0.f;
    const uint8_t* wbase = static_cast<const uint8_t*>(a.tiled) + ((e * nft + ft) * nkb) * wb;
    for (int64_t kb = 0; kb < nkb; ++kb) {
      __syncthreads();
      for (int i = tid; i < kExRows * 64; i += 128) {
        const int rr = i / 64, kk = i % 64;
        const int64_t row = r0 + rr, k = kb * 64 + kk;
        xs[i] = (row < r1 && k < a.m) ? h2f(a.x[row * a.m + k]) : 0.f;
      }
      __syncthreads();
      const uint8_t* blk = wbase + kb * wb;
      const int kmax = (int)::min((int64_t)64, a.m - kb * 64);
      // 64 weights of this column in k order, as f32 of the fp16 value
      float w[64];
      if (a.bits == 4) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint4 c = reinterpret_cast<const uint4*>(blk)[h * 128 + tid];
          const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t pr[4];
            i2f_u4(wd[q], db | (db << 16), pr);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint32_t v = hmul2_u32(pr[j], s | ((uint32_t)s << 16));
              w[h * 32 + q * 8 + 2 * j] = h2f((uint16_t)(v & 0xFFFF));
              w[h * 32 + q * 8 + 2 * j + 1] = h2f((uint16_t)(v >> 16));
            }
          }
        }
      } else if (a.bits == 8) {
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const uint4 c = reinterpret_cast<const uint4*>(blk)[c4 * 128 + tid];
          const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t pr[2];
            i2f_u8(wd[q], db | (db << 16), pr);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint32_t v = hmul2_u32(pr[j], s | ((uint32_t)s << 16));
              w[c4 * 16 + q * 4 + 2 * j] = h2f((uint16_t)(v & 0xFFFF));
              w[c4 * 16 + q * 4 + 2 * j + 1] = h2f((uint16_t)(v >> 16));
            }
          }
        }
      } else {
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint4 c = reinterpret_cast<const uint4*>(blk)[c8 * 128 + tid];
          const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            w[c8 * 8 + 2 * q] = h2f((uint16_t)(wd[q] & 0xFFFF));
            w[c8 * 8 + 2 * q + 1] = h2f((uint16_t)(wd[q] >> 16));
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < 64; ++kk) {
        if (kk < kmax) {
#pragma unroll
          for (int r = 0; r < kExRows; ++r) acc[r] = fmaf(xs[r * 64 + kk], w[kk], acc[r]);
        }
      }
    }
    if (live_col) {
      const float b = h2f(a.bias[e * a.n + col]);
#pragma unroll
      for (int r = 0; r < kExRows; ++r) {
        const int64_t row = r0 + r;
        if (row >= r1) break;
        float h = __fadd_rn(acc[r], b);
        if (a.relu && !(h > 0.0f)) h = 0.0f;
        a.out[row * a.n + col] = f2h(h);
      }
    }
  }
}

int launch_gemm_exact(const GemmArgs& a, cudaStream_t st) {
  if (a.np == 0) return MOE_OK;
  if (a.np > 4096) return set_error(MOE_EINVAL, "grouped_gemm: at most 4096 problems");
  const size_t smem = (a.np + 4) * 4 + kExRows * 64 * sizeof(float);
  const unsigned grid = (unsigned)(sm_count() * 8);
  gemm_exact_kernel<<<grid, 128, smem, st>>>(a);
  note_launch();
  return check_launch("gemm_exact");
}

}  // namespace moecu
