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
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "kernels.cuh"

namespace moecu {

namespace gv {
constexpr int kMaxGemvProblems = 1024;
constexpr int kWarps = 8;                 // compute warps, 16 features each
constexpr int kThreads = 32 * (kWarps + 1);  // + one producer warp
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
  uint32_t hb2;           // -(64 + debias - 1024) in both halves (i2f_u4_fast)
  int nitems;             // np * nft * nsplit work items, strided over persistent CTAs
  int early;              // second GEMM of an FFN pair: problems and weights are read before
                          // the programmatic-dependent-launch wait (only x is the previous
                          // kernel's output)
  long long* trace;       // dev-only (MOE_GEMV_TRACE): per CTA [start, prologue, items, k-loop ns, x-stage ns, epi ns, end]
};

__device__ __forceinline__ long long gv_time() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Weight blocks stream through a ring of NST stages (TMA bulk copies issued
// by a producer warp, mbarrier full/empty handshake); the 8 compute warps read
// their fragment words from shared memory.  Registers stay free for
// occupancy, and every CTA keeps NST x WBYTES of weights in flight.
template <int BITS>
struct Ring {
  static constexpr int WB = wblock_bytes(BITS);
  static constexpr int NST = BITS == 4 ? 8 : BITS == 8 ? 6 : 4;
};

template <int BITS>
__device__ __forceinline__ void frag_from_smem(const uint8_t* blk, int fg, int t,
                                               uint32_t (&w)[Frag<BITS>::NW]) {
  if constexpr (BITS == 4) {
    const uint8_t* p = blk + (t >> 1) * 2048 + (t & 1) * 8;
    const uint2 a = *reinterpret_cast<const uint2*>(p + fg * 16);
    const uint2 b = *reinterpret_cast<const uint2*>(p + (fg + 8) * 16);
    w[0] = a.x; w[1] = a.y; w[2] = b.x; w[3] = b.y;
  } else if constexpr (BITS == 8) {
    const uint8_t* p = blk + t * 2048;
    const uint4 a = *reinterpret_cast<const uint4*>(p + fg * 16);
    const uint4 b = *reinterpret_cast<const uint4*>(p + (fg + 8) * 16);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
  } else {
    const uint8_t* p = blk + 2 * t * 2048;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint4 a = *reinterpret_cast<const uint4*>(p + c * 2048 + fg * 16);
      const uint4 b = *reinterpret_cast<const uint4*>(p + c * 2048 + (fg + 8) * 16);
      w[4 * c + 0] = a.x; w[4 * c + 1] = a.y; w[4 * c + 2] = a.z; w[4 * c + 3] = a.w;
      w[8 + 4 * c + 0] = b.x; w[8 + 4 * c + 1] = b.y; w[8 + 4 * c + 2] = b.z; w[8 + 4 * c + 3] = b.w;
    }
  }
}

constexpr int kCompute = 32 * kWarps;  // compute threads; warp kWarps is the producer

template <int BITS>
__device__ __forceinline__ void dequant_fast(const uint32_t (&w)[Frag<BITS>::NW], uint32_t db2,
                                             uint32_t hb2, uint32_t (&lo)[8], uint32_t (&hi)[8]) {
  if constexpr (BITS == 4) {
    i2f_u4_fast(w[0], db2, hb2, &lo[0]);
    i2f_u4_fast(w[1], db2, hb2, &lo[4]);
    i2f_u4_fast(w[2], db2, hb2, &hi[0]);
    i2f_u4_fast(w[3], db2, hb2, &hi[4]);
  } else {
    dequant_frag<BITS>(w, db2, lo, hi);
  }
}

struct Item {
  int64_t e, r0, r1;
  int ft, split, kb0, kb1;
};

// item order: feature tile fastest, then k-split, then problem -- a CTA's
// consecutive items share the expert rows it has staged
__device__ __forceinline__ Item item_at(const Params& P, const int* live, int i) {
  Item it;
  it.ft = i % (int)P.nft;
  it.split = (i / (int)P.nft) % P.nsplit;
  const int p = live[i / (P.nsplit * (int)P.nft)];
  it.e = P.problems[3 * p];
  it.r0 = P.problems[3 * p + 1];
  it.r1 = P.problems[3 * p + 2];
  it.kb0 = it.split * P.kbs_per_split;
  const int64_t hi = (int64_t)it.kb0 + P.kbs_per_split;
  it.kb1 = (int)(P.nkb < hi ? P.nkb : hi);
  return it;
}

// Persistent: CTA b handles work items b, b + grid, ...  The producer warp
// streams the weight blocks of all of them back to back through the ring
// (it never drains between items); the compute warps stage only the live
// rows of each item (the MMA's unused B rows only feed discarded columns).
template <int BITS>
__global__ void __launch_bounds__(kThreads, 3) gemv_kernel(const Params P) {
  using F = Frag<BITS>;
  using RG = Ring<BITS>;
  extern __shared__ __align__(1024) uint8_t gsm[];
  uint8_t* ring = gsm;                                            // [NST][WB]
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + RG::NST * RG::WB);
  uint64_t* empty = full + RG::NST;
  uint16_t* xs = reinterpret_cast<uint16_t*>(empty + RG::NST);  // [NT][kp]
  __shared__ uint32_t s_last;
  __shared__ int s_live[kMaxGemvProblems];  // non-empty problems, in order
  __shared__ int s_nlive;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int kp = P.kbs_per_split * 64 + 8;  // row pitch of xs (conflict-free fragments)
  const long long t_start = P.trace ? gv_time() : 0;
  long long t_k = 0, t_x = 0, t_e = 0;
  int n_it = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < RG::NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kWarps);
    }
    fence_barrier_init();
  }
  griddep_launch();
  // FFN1: problems and activations come from the previous kernel.  FFN2
  // (early): the problems were written two kernels back (complete before
  // FFN1 started), the weights never change -- the prologue and the weight
  // stream start while FFN1 retires; the compute warps wait before reading x
  if (!P.early) griddep_wait();
  if (warp == 0) {  // compact the live problems: work items cover only those
    int base = 0;
    for (int p0 = 0; p0 < P.np; p0 += 32) {
      const int p = p0 + lane;
      const bool live = p < P.np && P.problems[3 * p + 2] > P.problems[3 * p + 1];
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (live) s_live[base + __popc(m & ((1u << lane) - 1u))] = p;
      base += __popc(m);
    }
    if (lane == 0) s_nlive = base;
  }
  __syncthreads();
  const int nitems = s_nlive * P.nsplit * (int)P.nft;
  const long long t_pro = P.trace ? gv_time() : 0;

  if (warp == kWarps) {
    // ------------------------------------------------------------- producer
    // converged warp, one elected lane issues: a lane-0-only loop makes
    // ptxas re-uniformise the copy operands per instruction (R2UR waterfall)
    {
      int s = 0;
      uint32_t ph = 0;
      int n = 0;
      const int i0 = (int)((int64_t)blockIdx.x * nitems / gridDim.x);  // balanced blocks
      const int i1 = (int)((int64_t)(blockIdx.x + 1) * nitems / gridDim.x);
      for (int i = i0; i < i1; ++i) {
        const Item it = item_at(P, s_live, i);
        if (it.r1 <= it.r0) continue;
        const uint8_t* wb = P.tiled + ((it.e * P.nft + it.ft) * P.nkb) * (int64_t)RG::WB;
        const int npass = (int)((it.r1 - it.r0 + NT - 1) / NT);
        for (int pass = 0; pass < npass; ++pass)
          for (int kb = it.kb0; kb < it.kb1; ++kb, ++n) {
            if (n >= RG::NST) mbar_wait_warp(&empty[s], ph ^ 1u);
            if (elect_one()) {
              mbar_arrive_expect_tx(&full[s], RG::WB);
              bulk_load(ring + s * RG::WB, wb + (int64_t)kb * RG::WB, RG::WB, &full[s]);
            }
            __syncwarp();
            if (++s == RG::NST) {
              s = 0;
              ph ^= 1u;
            }
          }
      }
    }
  } else {
    // -------------------------------------------------------------- compute
    if (P.early) griddep_wait();  // x = the previous kernel's output
    int s = 0;
    uint32_t ph = 0;
    const int fg = warp * 16 + g;
    const int i0 = (int)((int64_t)blockIdx.x * nitems / gridDim.x);
    const int i1 = (int)((int64_t)(blockIdx.x + 1) * nitems / gridDim.x);
    int64_t staged_r = -1;  // first row staged in xs (-1: none)
    int staged_kb = -1;
    for (int i = i0; i < i1; ++i) {
      const Item it = item_at(P, s_live, i);
      if (it.r1 <= it.r0) continue;
      const int64_t feat0 = (int64_t)it.ft * 128 + warp * 16;
      float sc[2] = {1.f, 1.f}, bi[2] = {0.f, 0.f};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t f = feat0 + g + 8 * h;
        if (f < P.n) {
          if (P.scales) sc[h] = h2f(P.scales[it.e * P.n + f]);
          bi[h] = h2f(P.bias[it.e * P.n + f]);
        }
      }
      const int nkbl = it.kb1 - it.kb0;
      const int kq = nkbl * 8;  // 16-byte pieces per staged row
      for (int64_t rb = it.r0; rb < it.r1; rb += NT) {
        const int nrow = (int)(it.r1 - rb < (int64_t)NT ? it.r1 - rb : (int64_t)NT);
        long long tt0 = P.trace ? gv_time() : 0;
        if (rb != staged_r || it.kb0 != staged_kb) {  // same rows as the last item: reuse
          named_bar_sync(1, kCompute);  // everyone done with xs
          for (int q = threadIdx.x; q < nrow * kq; q += kCompute) {
            const int r = q / kq, c = q % kq;
            const int64_t k = (int64_t)it.kb0 * 64 + c * 8;
            const bool ok = k < P.m;
            cp_async16(xs + r * kp + c * 8, ok ? P.x + (rb + r) * P.m + k : P.x, ok);
          }
          cp_async_commit();
          cp_async_wait<0>();
          named_bar_sync(1, kCompute);
          staged_r = rb;
          staged_kb = it.kb0;
        }

        long long tt1 = P.trace ? gv_time() : 0;
        t_x += tt1 - tt0;
        ++n_it;
        float acc[2][2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][c][q] = 0.f;
        const uint16_t* xk0 = xs + 16 * t + g * kp;
        auto kloop = [&](auto ntile_c) {
          constexpr int NTL = decltype(ntile_c)::value;
          const uint16_t* xk = xk0;
          for (int kbl = 0; kbl < nkbl; ++kbl, xk += 64) {
            mbar_wait_warp(&full[s], ph);
            uint32_t w[F::NW];
            frag_from_smem<BITS>(ring + s * RG::WB, fg, t, w);
            uint32_t lo[8], hi[8];
            dequant_fast<BITS>(w, P.db2, P.hb2, lo, hi);
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
              const uint4 xa = *reinterpret_cast<const uint4*>(xk + j * 8 * kp);
              const uint4 xb = *reinterpret_cast<const uint4*>(xk + j * 8 * kp + 8);
              const uint32_t xv[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t a[4] = {lo[2 * q], hi[2 * q], lo[2 * q + 1], hi[2 * q + 1]};
                mma_16816(acc[j][q & 1], a, xv[2 * q], xv[2 * q + 1]);
              }
            }
            // the MMAs consumed every word loaded from the stage (in every
            // lane): only now may the producer refill it
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (++s == RG::NST) {
              s = 0;
              ph ^= 1u;
            }
          }
        };
        if (nrow > 8)
          kloop(std::integral_constant<int, 2>{});
        else
          kloop(std::integral_constant<int, 1>{});
        long long tt2 = P.trace ? gv_time() : 0;
        t_k += tt2 - tt1;
        tt0 = tt2;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[j][0][q] += acc[j][1][q];
        // D fragment: acc[j][0][0..1] -> feature g, tokens 8j+2t, +1; [2..3] -> g+8
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int tok = j * 8 + 2 * t + (q & 1), h = q >> 1;
            const int64_t f = feat0 + g + 8 * h;
            if (tok < nrow && f < P.n) {
              if (P.nsplit == 1) {
                float v = fmaf(acc[j][0][q], sc[h], bi[h]);
                if (P.relu) v = v > 0.f ? v : 0.f;
                P.out[(rb + tok) * P.n + f] = f2h(v);
              } else {
                P.part[((int64_t)it.split * P.rows + rb + tok) * P.n + f] = acc[j][0][q];
              }
            }
          }
      }
      const long long te0 = P.trace ? gv_time() : 0;
      if (P.nsplit > 1) {
        // last CTA of this (expert, feature tile) reduces the splits in order
        __threadfence();
        named_bar_sync(1, kCompute);
        if (threadIdx.x == 0) {
          const uint32_t prev = atomicAdd(&P.ticket[it.e * P.nft + it.ft], 1u);
          s_last = prev == (uint32_t)P.nsplit - 1;
        }
        named_bar_sync(1, kCompute);
        if (s_last) {
          __threadfence();
          const int64_t nrows = it.r1 - it.r0;
          const int64_t fbase = (int64_t)it.ft * 128;
          for (int64_t q = threadIdx.x; q < nrows * 128; q += kCompute) {
            const int64_t r = it.r0 + q / 128, f = fbase + q % 128;
            if (f >= P.n) continue;
            float a = 0.f;
            for (int s2 = 0; s2 < P.nsplit; ++s2)
              a += __ldcg(&P.part[((int64_t)s2 * P.rows + r) * P.n + f]);
            float v = fmaf(a, P.scales ? h2f(P.scales[it.e * P.n + f]) : 1.f,
                           h2f(P.bias[it.e * P.n + f]));
            if (P.relu) v = v > 0.f ? v : 0.f;
            P.out[r * P.n + f] = f2h(v);
          }
          if (threadIdx.x == 0) P.ticket[it.e * P.nft + it.ft] = 0;
        }
      }
      if (P.trace) t_e += gv_time() - te0;
    }
    if (P.trace && threadIdx.x == 0) {
      long long* tr = P.trace + 8 * blockIdx.x;
      tr[0] = t_start;
      tr[1] = t_pro - t_start;
      tr[2] = n_it;
      tr[3] = t_k;
      tr[4] = t_x;
      tr[5] = t_e;
      tr[6] = gv_time();
    }
  }
}
}  // namespace gv

int gemv_splits(int64_t m, int64_t n, double active_experts) {
  const int64_t nft = (n + 127) / 128, nkb = (m + 63) / 64;
  int s = 1;
  while (s < 16 && nkb / (2 * s) >= 4 && active_experts * nft * s < 2.0 * 148) s *= 2;
  while (s < 64 && (nkb + s - 1) / s > 16) s *= 2;  // <= 1024 inputs staged per CTA
  return s;
}

static size_t ring_bytes(int bits) {
  const int nst = bits == 4 ? gv::Ring<4>::NST : bits == 8 ? gv::Ring<8>::NST : gv::Ring<16>::NST;
  return (size_t)nst * wblock_bytes(bits) + 2 * nst * 8;
}

size_t gemv_smem(int64_t m, int nsplit, int bits) {
  const int64_t nkb = (m + 63) / 64;
  const int64_t kbs = (nkb + nsplit - 1) / nsplit;
  return ring_bytes(bits) + (size_t)gv::NT * (kbs * 64 + 8) * 2;
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
  {
    const int off = (int)(a.debias & 0x3FF);  // debias - 1024 (8; 9 under MOE_FAULT_INJECT)
    const uint16_t hb = (uint16_t)(0x8000 | (21 << 10) | (off << 4));  // -(64 + off)
    P.hb2 = (uint32_t)hb | ((uint32_t)hb << 16);
  }
  P.nitems = (int)(a.np * P.nft * P.nsplit);
  // no programmatic dependent launch by default: an early-started second
  // GEMV competes with the first one's tail for SM slots and HBM (C3 T=64:
  // 86.7 us per layer with it, 82.3 without); MOE_PDL=5 opts in (early
  // prologue: weights stream before the wait, only x waits)
  P.early = a.second && pdl_enabled(4) ? 1 : 0;
  const size_t smem = gemv_smem(a.m, w.nsplit, BITS);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gv::gemv_kernel<BITS>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  // persistent: enough CTAs for the live items (empty problems are skipped
  // inside), at most 3 per SM
  // at most min(np, rows) problems are live (each holds >= 1 row): size the
  // grid for those -- at T = 1 a grid for all E problems launched ~3x more
  // CTAs than there were items, each paying the prologue
  const int64_t live = std::max<int64_t>(1, std::min<int64_t>(a.np, a.rows));
  static const int per_sm = std::getenv("MOE_GEMV_CTAS") ? std::atoi(std::getenv("MOE_GEMV_CTAS")) : 3;
  const int64_t grid =
      std::max<int64_t>(1, std::min<int64_t>(live * P.nft * P.nsplit, per_sm * (int64_t)sm_count()));
  static long long* dtrace = nullptr;
  const bool tr = std::getenv("MOE_GEMV_TRACE") != nullptr;
  if (tr && !dtrace) MOE_CUDA_TRY(cudaMalloc(&dtrace, 8 * 8 * 4096));
  P.trace = tr ? dtrace : nullptr;
  if (tr) MOE_CUDA_TRY(cudaMemsetAsync(dtrace, 0, 8 * 8 * grid, st));
  MOE_CUDA_TRY(launch_k(4, gv::gemv_kernel<BITS>, dim3((unsigned)grid), dim3(gv::kThreads), smem,
                        st, P));
  note_launch();
  if (tr) {  // dev instrumentation: per-CTA phase times (ns)
    std::vector<long long> h(8 * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost);
    long long lo = h[0], hi = h[6];
    double pro = 0, items = 0, tk = 0, tx = 0, te = 0, span = 0;
    for (int64_t b = 0; b < grid; ++b) {
      lo = std::min(lo, h[8 * b]);
      hi = std::max(hi, h[8 * b + 6]);
      pro += h[8 * b + 1];
      items += h[8 * b + 2];
      tk += h[8 * b + 3];
      tx += h[8 * b + 4];
      te += h[8 * b + 5];
      span += h[8 * b + 6] - h[8 * b];
    }
    std::fprintf(stderr,
                 "gemv m=%lld n=%lld rows=%lld nsplit=%d grid=%lld: kernel span %lld ns; per CTA mean: "
                 "life %.0f ns, prologue %.0f, items %.2f, x-stage %.0f, k-loop %.0f, epilogue %.0f\n",
                 (long long)a.m, (long long)a.n, (long long)a.rows, P.nsplit, (long long)grid,
                 hi - lo, span / grid, pro / grid, items / grid, tx / grid, tk / grid, te / grid);
  }
  return check_launch("gemv");
}

int launch_gemv(const GemmArgs& a, const GemvWork& w, cudaStream_t st) {
  if (a.np == 0 || a.rows == 0) return MOE_OK;
  if (a.np > gv::kMaxGemvProblems) return set_error(MOE_EINVAL, "gemv: at most 1024 problems");
  if (a.m % 8 != 0) return set_error(MOE_EINVAL, "gemv: m must be a multiple of 8");
  if (w.nsplit > 1 && (w.part == nullptr || w.ticket == nullptr))
    return set_error(MOE_EINVAL, "gemv: split-K workspace missing");
  if (gemv_smem(a.m, w.nsplit, a.bits) > 200 * 1024)
    return set_error(MOE_EINVAL, "gemv: k range too long for one CTA (raise nsplit)");
  switch (a.bits) {
    case 4: return run_gemv<4>(a, w, st);
    case 8: return run_gemv<8>(a, w, st);
    default: return run_gemv<16>(a, w, st);
  }
}

}  // namespace moecu
