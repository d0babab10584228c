// k_gemv.cu -- K5: decode-sized grouped expert GEMM ("dequant-GEMV").
//
// Same math as the FAST tcgen05 path (proj/src/grouped_gemm.cpp:165-214
// semantics, per-channel scale applied to the f32 accumulator), for the
// decode regime where each active expert sees only a few token rows and the
// layer is bound by streaming the packed expert weights from HBM.
//
// Work item = (problem, 128-feature tile, k-split).  One CTA = 8 warps; warp
// w owns features 16w..16w+15 of the tile.  Per 64-input k-block a lane
// reads its fragment words straight from the weight-tile layout the tcgen05
// path uses (k_quant.cu tile_weights: [e][ft][kb][chunk][feat][16B]) -- no
// second copy of the weights -- turns them into fp16 pairs with the magic
// I2F trick (proj/include/moeinfer/dequant.hpp:39-63) and feeds
// mma.sync.m16n8k16 (row = feature, col = token).  The k order inside an
// MMA is permuted consistently for A and B (lane t covers k = 16t..16t+15 of
// the block), which the f32 tensor accumulation does not care about.
// Loads run U k-blocks ahead (double-buffered registers) so every warp keeps
// 2-4 KB in flight.  Split-K partials (f32) are reduced in a fixed order by
// the last CTA of each (problem, feature tile) -- deterministic.
#include "kernels.cuh"

namespace moecu {

namespace gv {
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int NT = 16;  // token rows per pass (2 MMA n-tiles)

template <int BITS>
struct Frag {
  static constexpr int NW = BITS == 4 ? 4 : BITS == 8 ? 8 : 16;  // words per lane per k-block
  static constexpr int U = BITS == 4 ? 8 : BITS == 8 ? 4 : 2;    // k-blocks in flight
};

__device__ __forceinline__ void mma_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Lane (g = lane/4, t = lane%4) words of one k-block for features g and g+8
// of its warp's 16-feature group: k = 16t .. 16t+15 of the block.
template <int BITS>
__device__ __forceinline__ void load_frag(const uint8_t* blk, int fg, int t,
                                          uint32_t (&w)[Frag<BITS>::NW]) {
  if constexpr (BITS == 4) {
    // chunk h = t>>1 holds k 32h..32h+31; half (t&1) = words 2(t&1), 2(t&1)+1
    const uint8_t* p = blk + (t >> 1) * 2048 + (t & 1) * 8;
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(p + fg * 16));
    const uint2 b = __ldg(reinterpret_cast<const uint2*>(p + (fg + 8) * 16));
    w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y;
  } else if constexpr (BITS == 8) {
    const uint8_t* p = blk + t * 2048;  // chunk t: k 16t..16t+15
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p + fg * 16));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(p + (fg + 8) * 16));
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  } else {
    const uint8_t* p = blk + 2 * t * 2048;  // chunks 2t, 2t+1: k 16t..16t+15
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(p + c * 2048 + fg * 16));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(p + c * 2048 + (fg + 8) * 16));
      w[4 * c + 0] = a.x; w[4 * c + 1] = a.y; w[4 * c + 2] = a.z; w[4 * c + 3] = a.w;
      w[8 + 4 * c + 0] = b.x; w[8 + 4 * c + 1] = b.y; w[8 + 4 * c + 2] = b.z; w[8 + 4 * c + 3] = b.w;
    }
  }
}

// fp16 pairs (k 16t+2p, +1), p = 0..7, for feature g (lo) and g+8 (hi)
template <int BITS>
__device__ __forceinline__ void dequant_frag(const uint32_t (&w)[Frag<BITS>::NW], uint32_t db2,
                                             uint32_t (&lo)[8], uint32_t (&hi)[8]) {
  if constexpr (BITS == 4) {
    i2f_u4(w[0], db2, &lo[0]);
    i2f_u4(w[1], db2, &lo[4]);
    i2f_u4(w[2], db2, &hi[0]);
    i2f_u4(w[3], db2, &hi[4]);
  } else if constexpr (BITS == 8) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      i2f_u8(w[q], db2, &lo[2 * q]);
      i2f_u8(w[4 + q], db2, &hi[2 * q]);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      lo[q] = w[q];
      hi[q] = w[8 + q];
    }
  }
}

struct Params {
  const uint16_t* x;      // (rows, m) expert-sorted activations
  const uint8_t* tiled;   // tile_weights layout
  const uint16_t* scales; // (E, n) or null (W16)
  const uint16_t* bias;   // (E, n)
  const uint32_t* problems;
  uint16_t* out;          // (rows, n)
  float* part;            // split-K partials [nsplit][rows][n]
  uint32_t* ticket;       // [E][nft] arrival counters (self-resetting)
  int64_t m, n, rows, nft, nkb;
  int np, nsplit, kbs_per_split, relu;
  uint32_t db2;           // debias constant in both halves
};

template <int BITS>
__global__ void __launch_bounds__(kThreads, 2) gemv_kernel(const Params P) {
  using F = Frag<BITS>;
  constexpr int WBYTES = wblock_bytes(BITS);
  extern __shared__ __align__(16) uint16_t xs[];  // [NT][kp]
  __shared__ uint32_t s_last;
  const int split = blockIdx.x % P.nsplit;
  const int ft = (blockIdx.x / P.nsplit) % P.nft;
  const int p = blockIdx.x / (P.nsplit * (int)P.nft);
  if (p >= P.np) return;
  const int64_t e = P.problems[3 * p];
  const int64_t r0 = P.problems[3 * p + 1], r1 = P.problems[3 * p + 2];
  if (r1 <= r0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int kb0 = split * P.kbs_per_split;
  const int kb1 = (int)(P.nkb < (int64_t)(kb0 + P.kbs_per_split) ? P.nkb : (int64_t)(kb0 + P.kbs_per_split));
  if (kb0 >= kb1) return;
  const int kspan = (kb1 - kb0) * 64;
  const int kp = kspan + 8;  // conflict-free fragment reads (see header)
  const int fg = warp * 16 + g;
  const uint8_t* wbase = P.tiled + ((e * P.nft + ft) * P.nkb) * (int64_t)WBYTES;
  const int64_t feat0 = (int64_t)ft * 128 + warp * 16;
  float sc[2] = {1.f, 1.f}, bi[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t f = feat0 + g + 8 * h;
    if (f < P.n) {
      if (P.scales) sc[h] = h2f(P.scales[e * P.n + f]);
      bi[h] = h2f(P.bias[e * P.n + f]);
    }
  }

  using W = uint32_t[F::U][F::NW];
  auto load_group = [&](int kb, W& w) {
#pragma unroll
    for (int u = 0; u < F::U; ++u)
      if (kb + u < kb1) load_frag<BITS>(wbase + (int64_t)(kb + u) * WBYTES, fg, t, w[u]);
  };
  for (int64_t rb = r0; rb < r1; rb += NT) {
    const int nrow = (int)(r1 - rb < (int64_t)NT ? r1 - rb : (int64_t)NT);
    uint32_t wa[F::U][F::NW], wb[F::U][F::NW];
    __syncthreads();  // previous pass done with xs
    // first weight group in flight before waiting for the activations
    load_group(kb0, wa);
    // stage x[rb .. rb+nrow)[k range] (zero-filled past m / past nrow)
    const int kq = kspan / 8;
    for (int i = threadIdx.x; i < NT * kq; i += kThreads) {
      const int r = i / kq, c = i % kq;
      const int64_t k = (int64_t)kb0 * 64 + c * 8;
      const bool ok = r < nrow && k < P.m;
      cp_async16(xs + r * kp + c * 8, ok ? P.x + (rb + r) * P.m + k : P.x, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();

    // two independent accumulator chains per n-tile (even / odd MMA of a
    // k-block) halve the dependent mma.sync latency chain
    float acc[2][2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[j][c][q] = 0.f;

    auto compute_group = [&](int kb, const W& w) {
#pragma unroll
      for (int u = 0; u < F::U; ++u) {
        if (kb + u >= kb1) break;
        uint32_t lo[8], hi[8];
        dequant_frag<BITS>(w[u], P.db2, lo, hi);
        const uint16_t* xk = xs + (kb + u - kb0) * 64 + 16 * t;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j * 8 >= nrow) break;
          const uint4 xa = *reinterpret_cast<const uint4*>(xk + (j * 8 + g) * kp);
          const uint4 xb = *reinterpret_cast<const uint4*>(xk + (j * 8 + g) * kp + 8);
          const uint32_t xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t a[4] = {lo[2 * i], hi[2 * i], lo[2 * i + 1], hi[2 * i + 1]};
            mma_16816(acc[j][i & 1], a, xv[2 * i], xv[2 * i + 1]);
          }
        }
      }
    };
    for (int kb = kb0; kb < kb1; kb += 2 * F::U) {
      load_group(kb + F::U, wb);
      compute_group(kb, wa);
      if (kb + F::U >= kb1) break;
      load_group(kb + 2 * F::U, wa);
      compute_group(kb + F::U, wb);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[j][0][q] += acc[j][1][q];

    // D fragment: acc[j][0..1] -> feature g, tokens 8j+2t, +1; [2..3] -> feature g+8
    if (P.nsplit == 1) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tok = j * 8 + 2 * t + (q & 1), h = q >> 1;
          const int64_t f = feat0 + g + 8 * h;
          if (tok < nrow && f < P.n) {
            float v = fmaf(acc[j][0][q], sc[h], bi[h]);
            if (P.relu) v = v > 0.f ? v : 0.f;
            P.out[(rb + tok) * P.n + f] = f2h(v);
          }
        }
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int tok = j * 8 + 2 * t + (q & 1), h = q >> 1;
          const int64_t f = feat0 + g + 8 * h;
          if (tok < nrow && f < P.n) P.part[((int64_t)split * P.rows + rb + tok) * P.n + f] = acc[j][0][q];
        }
    }
  }
  if (P.nsplit == 1) return;
  // last CTA of this (problem, feature tile) reduces the splits in order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&P.ticket[e * P.nft + ft], 1u);
    s_last = prev == (uint32_t)P.nsplit - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t nrows = r1 - r0;
  const int64_t fbase = (int64_t)ft * 128;
  for (int64_t i = threadIdx.x; i < nrows * 128; i += kThreads) {
    const int64_t r = r0 + i / 128, f = fbase + i % 128;
    if (f >= P.n) continue;
    float a = 0.f;
    for (int s = 0; s < P.nsplit; ++s) a += __ldcg(&P.part[((int64_t)s * P.rows + r) * P.n + f]);
    float v = fmaf(a, P.scales ? h2f(P.scales[e * P.n + f]) : 1.f, h2f(P.bias[e * P.n + f]));
    if (P.relu) v = v > 0.f ? v : 0.f;
    P.out[r * P.n + f] = f2h(v);
  }
  if (threadIdx.x == 0) P.ticket[e * P.nft + ft] = 0;
}
}  // namespace gv

int gemv_splits(int64_t m, int64_t n, double active_experts) {
  const int64_t nft = (n + 127) / 128, nkb = (m + 63) / 64;
  int s = 1;
  while (s < 16 && nkb / (2 * s) >= 4 && active_experts * nft * s < 2.0 * 148) s *= 2;
  return s;
}

size_t gemv_smem(int64_t m, int nsplit) {
  const int64_t nkb = (m + 63) / 64;
  const int64_t kbs = (nkb + nsplit - 1) / nsplit;
  return (size_t)gv::NT * (kbs * 64 + 8) * 2;
}

template <int BITS>
static int run_gemv(const GemmArgs& a, const GemvWork& w, cudaStream_t st) {
  gv::Params P;
  P.x = a.x;
  P.tiled = static_cast<const uint8_t*>(a.tiled);
  P.scales = BITS == 16 ? nullptr : a.scales;
  P.bias = a.bias;
  P.problems = a.problems;
  P.out = a.out;
  P.part = w.part;
  P.ticket = w.ticket;
  P.m = a.m;
  P.n = a.n;
  P.rows = a.rows;
  P.nft = (a.n + 127) / 128;
  P.nkb = (a.m + 63) / 64;
  P.np = (int)a.np;
  P.kbs_per_split = (int)((P.nkb + w.nsplit - 1) / w.nsplit);
  P.nsplit = (int)((P.nkb + P.kbs_per_split - 1) / P.kbs_per_split);  // no empty splits
  P.relu = a.relu;
  P.db2 = (uint32_t)a.debias | ((uint32_t)a.debias << 16);
  const size_t smem = gemv_smem(a.m, w.nsplit);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gv::gemv_kernel<BITS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  const int64_t grid = a.np * P.nft * P.nsplit;
  gv::gemv_kernel<BITS><<<(unsigned)grid, gv::kThreads, smem, st>>>(P);
  note_launch();
  return check_launch("gemv");
}

int launch_gemv(const GemmArgs& a, const GemvWork& w, cudaStream_t st) {
  if (a.np == 0 || a.rows == 0) return MOE_OK;
  if (a.m % 8 != 0) return set_error(MOE_EINVAL, "gemv: m must be a multiple of 8");
  if (w.nsplit > 1 && (w.part == nullptr || w.ticket == nullptr))
    return set_error(MOE_EINVAL, "gemv: split-K workspace missing");
  if (gemv_smem(a.m, w.nsplit) > 200 * 1024)
    return set_error(MOE_EINVAL, "gemv: k range too long for one CTA (raise nsplit)");
  switch (a.bits) {
    case 4: return run_gemv<4>(a, w, st);
    case 8: return run_gemv<8>(a, w, st);
    default: return run_gemv<16>(a, w, st);
  }
}

}  // namespace moecu
