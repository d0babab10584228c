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

// One GEMM of the FFN pair as the kernels see it
struct Phase {
  const uint16_t* x;       // (rows, m) expert-sorted activations
  const uint8_t* tiled;    // tile_weights layout
  const uint16_t* scales;  // (E, n) or null (W16)
  const uint16_t* bias;    // (E, n)
  uint16_t* out;           // (rows, n)
  float* part;             // split-K partials [nsplit][rows][n]
  uint32_t* ticket;        // [E][nft] arrival counters (self-resetting)
  int64_t m, n;
  int nft, nkb, nsplit, kbs, relu;
};

struct Params {
  Phase ph;
  const uint32_t* problems;
  int64_t rows;
  int np;
  uint32_t db2;           // debias constant in both halves
  uint32_t hb2;           // -(64 + debias - 1024) in both halves (i2f_u4_fast)
  int early;              // second GEMM of an FFN pair: problems and weights are read before
                          // the programmatic-dependent-launch wait (only x is the previous
                          // kernel's output)
  long long* trace;       // dev-only (MOE_GEMV_TRACE): per CTA [start, prologue, items, k-loop ns, x-stage ns, epi ns, end]
  int chunked;            // item blocks of ceil(items / grid) (spare CTAs exit)
};

// Both GEMMs of the FFN pair in one persistent launch (decode): FFN1 items
// then FFN2 items, taken from a global counter in order; an FFN2 item waits
// until the FFN1 feature tiles its k range reads are complete (`ready`).
// Deadlock-free on any residency: items are claimed in order, so every FFN1
// item is held by a running CTA that reaches it before any FFN2 item.
// (The kernels copy the phase they work on out of ph[] by value: a reference
// into the parameter array selected at run time miscompiled -- FFN2 items
// read stale split-K / row state on 16-bit layers, found by bisection.)
struct PairParams {
  Phase ph[2];
  const uint32_t* problems;
  int64_t rows;
  int np;
  uint32_t db2, hb2;
  uint32_t* ready;  // [E][ph[0].nft] FFN1 tile complete (self-resetting)
  uint32_t* ctl;    // [0] next item, [1] CTAs finished (self-resetting)
  int E;
  int kbs_max;      // rows buffer width in k-blocks (max over the two GEMMs)
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

// item j of a phase: feature tile fastest, then k-split, then problem -- a
// CTA's consecutive items share the expert rows it has staged
__device__ __forceinline__ Item item_of(const Phase& ph, const uint32_t* problems, const int* live,
                                        int j) {
  Item it;
  it.ft = j % ph.nft;
  it.split = (j / ph.nft) % ph.nsplit;
  const int p = live[j / (ph.nsplit * ph.nft)];
  it.e = problems[3 * p];
  it.r0 = problems[3 * p + 1];
  it.r1 = problems[3 * p + 2];
  it.kb0 = it.split * ph.kbs;
  const int64_t hi = (int64_t)it.kb0 + ph.kbs;
  it.kb1 = (int)(ph.nkb < hi ? ph.nkb : hi);
  return it;
}

// compact the non-empty problems (warp 0): work items cover only those
__device__ __forceinline__ void compact_live(const uint32_t* problems, int np, int* live,
                                             int* nlive, int lane) {
  int base = 0;
  for (int p0 = 0; p0 < np; p0 += 32) {
    const int p = p0 + lane;
    const bool ok = p < np && problems[3 * p + 2] > problems[3 * p + 1];
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (ok) live[base + __popc(m & ((1u << lane) - 1u))] = p;
    base += __popc(m);
  }
  if (lane == 0) *nlive = base;
}

// producer: the weight blocks of one item into the ring (every pass of
// NT rows re-reads them)
template <int BITS>
__device__ __forceinline__ void produce_item(const Phase& ph, const Item& it, uint8_t* ring,
                                             uint64_t* full, uint64_t* empty, int& s,
                                             uint32_t& phs, int& n) {
  using RG = Ring<BITS>;
  const uint8_t* wb = ph.tiled + ((it.e * ph.nft + it.ft) * ph.nkb) * (int64_t)RG::WB;
  const int npass = (int)((it.r1 - it.r0 + NT - 1) / NT);
  for (int pass = 0; pass < npass; ++pass)
    for (int kb = it.kb0; kb < it.kb1; ++kb, ++n) {
      if (n >= RG::NST) mbar_wait_warp(&empty[s], phs ^ 1u);
      if (elect_one()) {
        mbar_arrive_expect_tx(&full[s], RG::WB);
        bulk_load(ring + s * RG::WB, wb + (int64_t)kb * RG::WB, RG::WB, &full[s]);
      }
      __syncwarp();
      if (++s == RG::NST) {
        s = 0;
        phs ^= 1u;
      }
    }
}

// One pass of NT rows of an item: the k-loop over the item's weight blocks
// (ring stages, in the order the producer issued them) against the rows
// staged at xs (pitch kp halves), then the epilogue (scale, bias, ReLU, fp16)
// or, for split-K, the f32 partials.
template <int BITS>
__device__ __forceinline__ void mma_pass(const Phase& ph, const Item& it, int64_t rb, int nrow,
                                         const uint16_t* xs, int kp, int64_t rows, uint32_t db2,
                                         uint32_t hb2, const float (&sc)[2], const float (&bi)[2],
                                         const uint8_t* ring, uint64_t* full, uint64_t* empty,
                                         int& s, uint32_t& phs, uint64_t* xdone) {
  using F = Frag<BITS>;
  using RG = Ring<BITS>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int fg = warp * 16 + g;
  const int64_t feat0 = (int64_t)it.ft * 128 + warp * 16;
  const int nkbl = it.kb1 - it.kb0;
  float acc[2][2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[j][c][q] = 0.f;
  const uint16_t* xk0 = xs + 16 * t + g * kp;
  // int4: the lane's fragment words sit at a fixed offset in every stage
  // (chunk t/2, half t%2, features fg and fg+8): shared-window addresses
  // computed once, so the loop body is waits, two 8-byte loads, dequant
  // and MMAs (no per-iteration address rebuild)
  const uint32_t ring_s = smem_u32(ring) + (uint32_t)((t >> 1) * 2048 + (t & 1) * 8 + fg * 16);
  const uint32_t full_s = smem_u32(full);
  auto kloop = [&](auto ntile_c) {
    constexpr int NTL = decltype(ntile_c)::value;
    const uint16_t* xk = xk0;
    for (int kbl = 0; kbl < nkbl; ++kbl, xk += 64) {
      uint32_t w[F::NW];
      if constexpr (BITS == 4) {
        while (!mbar_try_wait(full_s + 8u * (uint32_t)s, phs)) {
        }
        const uint32_t a = ring_s + (uint32_t)s * (uint32_t)RG::WB;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(a));
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[2]), "=r"(w[3]) : "r"(a + 128u));
      } else {
        mbar_wait_warp(&full[s], phs);
        frag_from_smem<BITS>(ring + s * RG::WB, fg, t, w);
      }
      uint32_t lo[8], hi[8];
      dequant_fast<BITS>(w, db2, hb2, lo, hi);
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
        phs ^= 1u;
      }
    }
  };
  if (nrow > 8)
    kloop(std::integral_constant<int, 2>{});
  else
    kloop(std::integral_constant<int, 1>{});
  if (xdone != nullptr) {  // the rows buffer is free for the producer's next pass
    __syncwarp();
    if (lane == 0) mbar_arrive(xdone);
  }
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
      if (tok < nrow && f < ph.n) {
        if (ph.nsplit == 1) {
          float v = fmaf(acc[j][0][q], sc[h], bi[h]);
          if (ph.relu) v = v > 0.f ? v : 0.f;
          ph.out[(rb + tok) * ph.n + f] = f2h(v);
        } else {
          ph.part[((int64_t)it.split * rows + rb + tok) * ph.n + f] = acc[j][0][q];
        }
      }
    }
}

__device__ __forceinline__ void item_scale_bias(const Phase& ph, const Item& it, float (&sc)[2],
                                                float (&bi)[2]) {
  const int warp = threadIdx.x >> 5, g = (threadIdx.x & 31) >> 2;
  const int64_t feat0 = (int64_t)it.ft * 128 + warp * 16;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t f = feat0 + g + 8 * h;
    sc[h] = 1.f;
    bi[h] = 0.f;
    if (f < ph.n) {
      if (ph.scales) sc[h] = h2f(ph.scales[it.e * ph.n + f]);
      bi[h] = h2f(ph.bias[it.e * ph.n + f]);
    }
  }
}

// Split-K: the last CTA of this (expert, feature tile) reduces the splits in
// fixed order.  One fence per CTA on each side: the barrier orders the
// other threads' partial stores before thread 0's release (cumulativity),
// and thread 0's acquire before the other threads' loads.  Returns true when
// the item's output rows are final (nsplit == 1, or this CTA reduced).
__device__ __forceinline__ bool finish_item(const Phase& ph, const Item& it, int64_t rows,
                                            uint32_t* s_last) {
  if (ph.nsplit == 1) return true;
  named_bar_sync(1, kCompute);
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&ph.ticket[it.e * ph.nft + it.ft], 1u);
    __threadfence();
    *s_last = prev == (uint32_t)ph.nsplit - 1;
  }
  named_bar_sync(1, kCompute);
  if (!*s_last) return false;
  const int64_t nrows = it.r1 - it.r0;
  const int64_t fbase = (int64_t)it.ft * 128;
  for (int64_t q = threadIdx.x; q < nrows * 128; q += kCompute) {
    const int64_t r = it.r0 + q / 128, f = fbase + q % 128;
    if (f >= ph.n) continue;
    float a = 0.f;
    for (int s2 = 0; s2 < ph.nsplit; ++s2) a += __ldcg(&ph.part[((int64_t)s2 * rows + r) * ph.n + f]);
    float v = fmaf(a, ph.scales ? h2f(ph.scales[it.e * ph.n + f]) : 1.f, h2f(ph.bias[it.e * ph.n + f]));
    if (ph.relu) v = v > 0.f ? v : 0.f;
    ph.out[r * ph.n + f] = f2h(v);
  }
  if (threadIdx.x == 0) ph.ticket[it.e * ph.nft + it.ft] = 0;
  return true;
}

// Persistent: CTA b handles a balanced contiguous block of the work items.
// The producer warp streams the weight blocks of all of them back to back
// through the ring (it never drains between items); the compute warps stage
// only the live rows of each item (the MMA's unused B rows only feed
// discarded columns).
template <int BITS, int MINB = 3>
__global__ void __launch_bounds__(kThreads, MINB) gemv_kernel(const Params P) {
  using RG = Ring<BITS>;
  extern __shared__ __align__(1024) uint8_t gsm[];
  uint8_t* ring = gsm;                                            // [NST][WB]
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + RG::NST * RG::WB);
  uint64_t* empty = full + RG::NST;
  uint16_t* xs = reinterpret_cast<uint16_t*>(empty + RG::NST);  // [NT][kp]
  __shared__ uint32_t s_last;
  __shared__ int s_live[kMaxGemvProblems];  // non-empty problems, in order
  __shared__ int s_nlive;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool tr = P.trace != nullptr;
  const long long t_start = tr ? gv_time() : 0;
  long long t_k = 0, t_x = 0;
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
  if (warp == 0) compact_live(P.problems, P.np, s_live, &s_nlive, lane);
  __syncthreads();
  const int nitems = s_nlive * P.ph.nsplit * P.ph.nft;
  const long long t_pro = tr ? gv_time() : 0;
  // contiguous blocks of `per` items (MOE_GEMV_CHUNKED, dev A/B): when the
  // live items just exceed a multiple of the grid, the spare CTAs exit and
  // the busy ones share their SMs with fewer neighbours, instead of two or
  // three CTAs running one extra item alone at the end
  int i0, i1;
  if (P.chunked) {
    const int per = (nitems + (int)gridDim.x - 1) / (int)gridDim.x;
    i0 = ::min(nitems, (int)blockIdx.x * per);
    i1 = ::min(nitems, i0 + per);
  } else {
    i0 = (int)((int64_t)blockIdx.x * nitems / gridDim.x);  // balanced blocks
    i1 = (int)((int64_t)(blockIdx.x + 1) * nitems / gridDim.x);
  }
  int s = 0, n = 0;
  uint32_t phs = 0;
  if (warp == kWarps) {
    // producer: converged warp, one elected lane issues (a lane-0-only loop
    // makes ptxas re-uniformise the copy operands per instruction)
    for (int i = i0; i < i1; ++i) {
      const Item it = item_of(P.ph, P.problems, s_live, i);
      produce_item<BITS>(P.ph, it, ring, full, empty, s, phs, n);
    }
  } else {
    if (P.early) griddep_wait();  // x = the previous kernel's output
    const Phase& ph = P.ph;
    const int kp = ph.kbs * 64 + 8;  // row pitch of xs (conflict-free fragments)
    int64_t staged_r = -1;           // first row staged in xs (-1: none)
    int staged_kb = -1;
    for (int i = i0; i < i1; ++i) {
      const Item it = item_of(ph, P.problems, s_live, i);
      float sc[2], bi[2];
      item_scale_bias(ph, it, sc, bi);
      const int kq = (it.kb1 - it.kb0) * 8;  // 16-byte pieces per staged row
      for (int64_t rb = it.r0; rb < it.r1; rb += NT) {
        const int nrow = (int)(it.r1 - rb < (int64_t)NT ? it.r1 - rb : (int64_t)NT);
        const long long tt0 = tr ? gv_time() : 0;
        if (rb != staged_r || it.kb0 != staged_kb) {  // same rows as the last item: reuse
          named_bar_sync(1, kCompute);  // everyone done with xs
          for (int q = threadIdx.x; q < nrow * kq; q += kCompute) {
            const int r = q / kq, c = q % kq;
            const int64_t k = (int64_t)it.kb0 * 64 + c * 8;
            const bool ok = k < ph.m;
            cp_async16(xs + r * kp + c * 8, ok ? ph.x + (rb + r) * ph.m + k : ph.x, ok);
          }
          cp_async_commit();
          cp_async_wait<0>();
          named_bar_sync(1, kCompute);
          staged_r = rb;
          staged_kb = it.kb0;
        }
        const long long tt1 = tr ? gv_time() : 0;
        t_x += tt1 - tt0;
        ++n_it;
        mma_pass<BITS>(ph, it, rb, nrow, xs, kp, P.rows, P.db2, P.hb2, sc, bi, ring, full, empty,
                       s, phs, nullptr);
        if (tr) t_k += gv_time() - tt1;
      }
      finish_item(ph, it, P.rows, &s_last);
    }
    if (tr && threadIdx.x == 0) {
      long long* tp = P.trace + 8 * blockIdx.x;
      tp[0] = t_start;
      tp[1] = t_pro - t_start;
      tp[2] = n_it;
      tp[3] = t_k;
      tp[4] = t_x;
      tp[5] = 0;
      tp[6] = gv_time();
    }
  }
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kQ = 2;             // claimed items queued between producer and compute warps
constexpr int kS = 4;             // finished items queued for the signal warp
constexpr int kPairThreads = 32 * (kWarps + 2);  // compute, producer, signal
constexpr int kPairProblems = 512;

// k-blocks per split in the pair kernel: two rows buffers of NB rows each
__host__ __device__ constexpr int pair_max_kbs(int nb) { return nb == 8 ? 16 : 8; }

// The pair kernel's item: problems packed in shared memory as
// {expert, row0 | row1 << 16} (decode: rows < 65536)
__device__ __forceinline__ Item pair_item(const Phase& ph, const uint2* pk, int j) {
  Item it;
  it.ft = j % ph.nft;
  it.split = (j / ph.nft) % ph.nsplit;
  const uint2 p = pk[j / (ph.nsplit * ph.nft)];
  it.e = p.x;
  it.r0 = p.y & 0xFFFFu;
  it.r1 = p.y >> 16;
  it.kb0 = it.split * ph.kbs;
  const int hi = it.kb0 + ph.kbs;
  it.kb1 = ph.nkb < hi ? ph.nkb : hi;
  return it;
}

// Warp roles: 8 compute warps, a producer warp and a signal warp.
// * producer: claims items (global counter, in order), waits for an FFN2
//   item's FFN1 tiles, issues every copy -- each pass's rows (one bulk copy
//   per row into one of two rows buffers of NB rows) and the weight blocks
//   (ring);
// * compute: mbarrier waits, dequant + mma.sync, epilogue (output rows or
//   split-K partials), then hand the item to the signal warp -- no
//   block-wide barrier and no global fence on this path;
// * signal: per finished item, the split-K ticket (the last CTA reduces the
//   splits in fixed order, 4 features per lane) and the FFN1 tile-ready
//   flag, each behind one fence -- off the compute warps' critical path.
template <int BITS, int NB>
__global__ void __launch_bounds__(kPairThreads, 3) gemv_pair_kernel(const PairParams P) {
  using RG = Ring<BITS>;
  extern __shared__ __align__(1024) uint8_t gsm[];
  uint8_t* ring = gsm;
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm + RG::NST * RG::WB);
  uint64_t* empty = full + RG::NST;
  uint64_t* xfull = empty + RG::NST;  // [2]
  uint64_t* xempty = xfull + 2;       // [2]
  uint16_t* xs0 = reinterpret_cast<uint16_t*>(gsm + RG::NST * RG::WB + 256);  // 2 x [NB][kp]
  __shared__ uint2 s_pk[kPairProblems];
  __shared__ int s_nlive;
  __shared__ int s_q[kQ], s_d[kS];
  __shared__ uint64_t qfull[kQ], qempty[kQ], dfull[kS], dempty[kS];
  __shared__ uint32_t s_fin;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kp = P.kbs_max * 64 + 8;  // rows buffer pitch (halves)
  if (threadIdx.x == 0) {
    for (int i = 0; i < RG::NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], kWarps);
    }
    for (int i = 0; i < kQ; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], kWarps);
    }
    for (int i = 0; i < kS; ++i) {
      mbar_init(&dfull[i], kWarps);
      mbar_init(&dempty[i], 1);
    }
    fence_barrier_init();
  }
  griddep_launch();
  griddep_wait();  // problems and x come from the previous kernels
  if (warp == 0) {  // live problems, packed
    int base = 0;
    for (int p0 = 0; p0 < P.np; p0 += 32) {
      const int p = p0 + lane;
      uint32_t e = 0, r0 = 0, r1 = 0;
      if (p < P.np) {
        e = P.problems[3 * p];
        r0 = P.problems[3 * p + 1];
        r1 = P.problems[3 * p + 2];
      }
      const bool ok = p < P.np && r1 > r0;
      const uint32_t m = __ballot_sync(0xffffffffu, ok);
      if (ok) s_pk[base + __popc(m & ((1u << lane) - 1u))] = make_uint2(e, r0 | (r1 << 16));
      base += __popc(m);
    }
    if (lane == 0) s_nlive = base;
  }
  __syncthreads();
  const int n0 = s_nlive * P.ph[0].nsplit * P.ph[0].nft;
  const int total = n0 + s_nlive * P.ph[1].nsplit * P.ph[1].nft;
  const int nft0 = P.ph[0].nft;
  if (warp == kWarps) {
    // ------------------------------------------------------------- producer
    int s = 0, qs = 0, xb = 0, n = 0, qn = 0, xn = 0;
    uint32_t phs = 0, qph = 0, xph = 0;
    auto weights = [&](const Phase& ph, const Item& it, int kb0, int kb1) {
      const uint8_t* wb = ph.tiled + ((it.e * ph.nft + it.ft) * ph.nkb) * (int64_t)RG::WB;
      for (int kb = kb0; kb < kb1; ++kb, ++n) {
        if (n >= RG::NST) mbar_wait_warp(&empty[s], phs ^ 1u);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[s], RG::WB);
          bulk_load(ring + s * RG::WB, wb + (int64_t)kb * RG::WB, RG::WB, &full[s]);
        }
        __syncwarp();
        if (++s == RG::NST) {
          s = 0;
          phs ^= 1u;
        }
      }
    };
    // the next claim is always in flight (lane 0's register; read one item
    // later) so its round trip overlaps the current item's copies
    uint32_t next = 0;
    if (lane == 0) next = atomicAdd(&P.ctl[0], 1u);
    for (;;) {
      int i = (int)__shfl_sync(0xffffffffu, next, 0);
      if (i >= total) i = -1;
      if (qn >= kQ) mbar_wait_warp(&qempty[qs], qph ^ 1u);
      if (lane == 0) {
        s_q[qs] = i;
        mbar_arrive(&qfull[qs]);  // release: the compute warps see s_q
      }
      __syncwarp();
      ++qn;
      if (++qs == kQ) {
        qs = 0;
        qph ^= 1u;
      }
      if (i < 0) break;
      if (lane == 0) next = atomicAdd(&P.ctl[0], 1u);
      const int pi = i >= n0;
      const Phase ph = pi ? P.ph[1] : P.ph[0];  // a copy: see PairParams
      const Item it = pair_item(ph, s_pk, pi ? i - n0 : i);
      const uint32_t seg = (uint32_t)(it.kb1 - it.kb0) * 128;  // bytes per row (m % 64 == 0)
      for (int64_t rb = it.r0; rb < it.r1; rb += NB) {
        const int nrow = (int)(it.r1 - rb < (int64_t)NB ? it.r1 - rb : (int64_t)NB);
        // rows first (the compute warps need them for the first block).  An
        // FFN2 item whose FFN1 tiles are not final yet: first the weight
        // blocks that cannot wait on this pass's own consumption (one ring),
        // then wait for the tiles, then the rows
        int kpre = it.kb0;
        if (rb == it.r0 && pi == 1) {
          const int t0 = it.kb0 >> 1, t1 = (it.kb1 - 1) >> 1;  // feature tile = 2 k-blocks
          bool ready = true;
          if (lane == 0)
            for (int t = t0; t <= t1; ++t) ready = ready && ld_acquire(&P.ready[it.e * nft0 + t]) != 0;
          ready = __shfl_sync(0xffffffffu, ready, 0);
          if (!ready) {
            kpre = ::min(it.kb1, it.kb0 + RG::NST);
            weights(ph, it, it.kb0, kpre);
            if (lane == 0)
              for (int t = t0; t <= t1; ++t)
                while (ld_acquire(&P.ready[it.e * nft0 + t]) == 0) __nanosleep(32);
          }
          if (lane == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // h via bulk copies
          __syncwarp();
        }
        if (xn >= 2) mbar_wait_warp(&xempty[xb], xph ^ 1u);
        uint16_t* xs = xs0 + xb * (NB * kp);
        if (elect_one()) mbar_arrive_expect_tx(&xfull[xb], seg * (uint32_t)nrow);
        __syncwarp();
        if (lane < nrow)
          bulk_load(xs + lane * kp, ph.x + (rb + lane) * ph.m + (int64_t)it.kb0 * 64, seg, &xfull[xb]);
        __syncwarp();
        ++xn;
        if (++xb == 2) {
          xb = 0;
          xph ^= 1u;
        }
        weights(ph, it, rb == it.r0 ? kpre : it.kb0, it.kb1);  // kpre == kb0 unless pre-issued
      }
    }
  } else if (warp == kWarps + 1) {
    // --------------------------------------------------------------- signal
    int ds = 0;
    uint32_t dph = 0;
    for (;;) {
      mbar_wait_warp(&dfull[ds], dph);  // acquire: the compute warps' stores
      const int i = s_d[ds];
      if (i < 0) break;
      const int pi = i >= n0;
      const Phase ph = pi ? P.ph[1] : P.ph[0];  // a copy: see PairParams
      const Item it = pair_item(ph, s_pk, pi ? i - n0 : i);
      bool final = true;
      if (ph.nsplit > 1) {
        uint32_t last = 0;
        if (lane == 0) {
          __threadfence();
          last = atomicAdd(&ph.ticket[it.e * ph.nft + it.ft], 1u) == (uint32_t)ph.nsplit - 1;
          __threadfence();
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        final = last != 0;
        if (final) {  // reduce the splits in order: 4 features per lane, a row per step
          const int64_t f = (int64_t)it.ft * 128 + lane * 4;
          if (f < ph.n) {
            float sc[4] = {1.f, 1.f, 1.f, 1.f}, bi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (ph.scales) sc[q] = h2f(ph.scales[it.e * ph.n + f + q]);
              bi[q] = h2f(ph.bias[it.e * ph.n + f + q]);
            }
            for (int64_t r = it.r0; r < it.r1; ++r) {
              float4 a = __ldcg(reinterpret_cast<const float4*>(ph.part + (r * ph.n + f)));
              for (int s2 = 1; s2 < ph.nsplit; ++s2) {
                const float4 b =
                    __ldcg(reinterpret_cast<const float4*>(ph.part + (((int64_t)s2 * P.rows + r) * ph.n + f)));
                a.x += b.x;
                a.y += b.y;
                a.z += b.z;
                a.w += b.w;
              }
              const float av[4] = {a.x, a.y, a.z, a.w};
              uint16_t o[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float v = fmaf(av[q], sc[q], bi[q]);
                if (ph.relu) v = v > 0.f ? v : 0.f;
                o[q] = f2h(v);
              }
              *reinterpret_cast<uint2*>(ph.out + r * ph.n + f) =
                  make_uint2(o[0] | ((uint32_t)o[1] << 16), o[2] | ((uint32_t)o[3] << 16));
            }
          }
          if (lane == 0) ph.ticket[it.e * ph.nft + it.ft] = 0;
        }
      }
      __syncwarp();
      if (final && pi == 0 && lane == 0) {  // h tile (e, ft) final
        __threadfence();
        atomicExch(&P.ready[it.e * nft0 + it.ft], 1u);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[ds]);
      if (++ds == kS) {
        ds = 0;
        dph ^= 1u;
      }
    }
  } else {
    // -------------------------------------------------------------- compute
    int s = 0, qs = 0, xb = 0, ds = 0, dn = 0;
    uint32_t phs = 0, qph = 0, xph = 0, dph = 0;
    auto hand_off = [&](int i) {  // to the signal warp, after this warp's stores
      if (dn >= kS) mbar_wait_warp(&dempty[ds], dph ^ 1u);
      if (warp == 0 && lane == 0) s_d[ds] = i;
      __syncwarp();
      if (lane == 0) mbar_arrive(&dfull[ds]);  // release (cumulative over the warp's stores)
      ++dn;
      if (++ds == kS) {
        ds = 0;
        dph ^= 1u;
      }
    };
    for (;;) {
      mbar_wait_warp(&qfull[qs], qph);
      const int i = s_q[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      if (++qs == kQ) {
        qs = 0;
        qph ^= 1u;
      }
      if (i < 0) {
        hand_off(-1);
        break;
      }
      const int pi = i >= n0;
      const Phase ph = pi ? P.ph[1] : P.ph[0];  // a copy: see PairParams
      const Item it = pair_item(ph, s_pk, pi ? i - n0 : i);
      float sc[2], bi[2];
      item_scale_bias(ph, it, sc, bi);
      for (int64_t rb = it.r0; rb < it.r1; rb += NB) {
        const int nrow = (int)(it.r1 - rb < (int64_t)NB ? it.r1 - rb : (int64_t)NB);
        mbar_wait_warp(&xfull[xb], xph);
        mma_pass<BITS>(ph, it, rb, nrow, xs0 + xb * (NB * kp), kp, P.rows, P.db2, P.hb2, sc, bi,
                       ring, full, empty, s, phs, &xempty[xb]);
        if (++xb == 2) {
          xb = 0;
          xph ^= 1u;
        }
      }
      hand_off(i);
    }
  }
  // self-reset for the next launch (graph replay): the last CTA out clears
  // the claim counter and the ready flags -- every CTA is past its last use
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_fin = atomicAdd(&P.ctl[1], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_fin) {
    for (int i = threadIdx.x; i < P.E * nft0; i += kPairThreads) P.ready[i] = 0;
    if (threadIdx.x == 0) {
      P.ctl[0] = 0;
      P.ctl[1] = 0;
    }
  }
}
}  // namespace gv

int gemv_splits(int64_t m, int64_t n, double active_experts) {
  const int64_t nft = (n + 127) / 128, nkb = (m + 63) / 64;
  static const int force = std::getenv("MOE_GEMV_SPLITS") ? std::atoi(std::getenv("MOE_GEMV_SPLITS")) : 0;
  if (force > 0) {  // dev A/B: a fixed split count (capped so the k range stays <= 1024 inputs)
    int s = force;
    while (s < 64 && (nkb + s - 1) / s > 16) s *= 2;
    return s;
  }
  // split k only until the items cover the SMs once: a split costs a rows
  // re-stage, a pipeline fill and the ordered reduction (measured C3 T=8
  // FFN2: 4 splits 14.5 us, 8 splits 18.7 us; T=64 FFN1: 1 split 29.7 us,
  // 2 splits 42.0 us)
  int s = 1;
  while (s < 16 && nkb / (2 * s) >= 4 && active_experts * nft * s < 1.0 * sm_count()) s *= 2;
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

static gv::Phase make_phase(const GemmArgs& a, const GemvWork& w, int bits) {
  gv::Phase ph;
  ph.x = a.x;
  ph.tiled = static_cast<const uint8_t*>(a.tiled);
  ph.scales = bits == 16 ? nullptr : a.scales;
  ph.bias = a.bias;
  ph.out = a.out;
  ph.part = w.part;
  ph.ticket = w.ticket;
  ph.m = a.m;
  ph.n = a.n;
  ph.nft = (int)((a.n + 127) / 128);
  ph.nkb = (int)((a.m + 63) / 64);
  ph.kbs = (ph.nkb + w.nsplit - 1) / w.nsplit;
  ph.nsplit = (ph.nkb + ph.kbs - 1) / ph.kbs;  // no empty splits
  ph.relu = a.relu;
  return ph;
}

static void debias_pair(uint16_t debias, uint32_t* db2, uint32_t* hb2) {
  *db2 = (uint32_t)debias | ((uint32_t)debias << 16);
  const int off = (int)(debias & 0x3FF);  // debias - 1024 (8; 9 under MOE_FAULT_INJECT)
  const uint16_t hb = (uint16_t)(0x8000 | (21 << 10) | (off << 4));  // -(64 + off)
  *hb2 = (uint32_t)hb | ((uint32_t)hb << 16);
}

template <int BITS>
static int run_gemv(const GemmArgs& a, const GemvWork& w, cudaStream_t st) {
  gv::Params P;
  P.ph = make_phase(a, w, BITS);
  P.problems = a.problems;
  P.rows = a.rows;
  P.np = (int)a.np;
  debias_pair(a.debias, &P.db2, &P.hb2);
  // no programmatic dependent launch by default: an early-started second
  // GEMV competes with the first one's tail for SM slots and HBM (C3 T=64:
  // 86.7 us per layer with it, 82.3 without); MOE_PDL=5 opts in (early
  // prologue: weights stream before the wait, only x waits)
  P.early = a.second && pdl_enabled(4) ? 1 : 0;
  static const int chunked = std::getenv("MOE_GEMV_CHUNKED") ? std::atoi(std::getenv("MOE_GEMV_CHUNKED")) : 0;
  P.chunked = chunked;
  const size_t smem = gemv_smem(a.m, w.nsplit, BITS);
  static const int per_sm = std::getenv("MOE_GEMV_CTAS") ? std::atoi(std::getenv("MOE_GEMV_CTAS")) : 3;
  // MOE_GEMV_CTAS=2: the 2-CTA/SM instantiation (register cap 113 instead of 72)
  auto kern = per_sm == 2 ? gv::gemv_kernel<BITS, 2> : gv::gemv_kernel<BITS, 3>;
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gv::gemv_kernel<BITS, 2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MOE_CUDA_TRY(cudaFuncSetAttribute(gv::gemv_kernel<BITS, 3>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  // persistent: enough CTAs for the live items (empty problems are skipped
  // inside), at most 3 per SM
  // at most min(np, rows) problems are live (each holds >= 1 row): size the
  // grid for those -- at T = 1 a grid for all E problems launched ~3x more
  // CTAs than there were items, each paying the prologue
  const int64_t live = std::max<int64_t>(1, std::min<int64_t>(a.np, a.rows));
  const int64_t grid = std::max<int64_t>(
      1, std::min<int64_t>(live * P.ph.nft * P.ph.nsplit, per_sm * (int64_t)sm_count()));
  static long long* dtrace = nullptr;
  const bool tr = std::getenv("MOE_GEMV_TRACE") != nullptr;
  if (tr && !dtrace) MOE_CUDA_TRY(cudaMalloc(&dtrace, 8 * 8 * 4096));
  P.trace = tr ? dtrace : nullptr;
  if (tr) MOE_CUDA_TRY(cudaMemsetAsync(dtrace, 0, 8 * 8 * grid, st));
  MOE_CUDA_TRY(launch_k(4, kern, dim3((unsigned)grid), dim3(gv::kThreads), smem, st, P));
  note_launch();
  if (tr) {  // dev instrumentation: per-CTA phase times (ns)
    std::vector<long long> h(8 * grid);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost);
    long long lo = h[0], hi = h[6];
    double pro = 0, items = 0, tk = 0, tx = 0, span = 0;
    for (int64_t b = 0; b < grid; ++b) {
      lo = std::min(lo, h[8 * b]);
      hi = std::max(hi, h[8 * b + 6]);
      pro += h[8 * b + 1];
      items += h[8 * b + 2];
      tk += h[8 * b + 3];
      tx += h[8 * b + 4];
      span += h[8 * b + 6] - h[8 * b];
    }
    std::fprintf(stderr,
                 "gemv m=%lld n=%lld rows=%lld nsplit=%d grid=%lld: kernel span %lld ns; per CTA mean: "
                 "life %.0f ns, prologue %.0f, passes %.2f, x-stage %.0f, k-loop %.0f\n",
                 (long long)a.m, (long long)a.n, (long long)a.rows, P.ph.nsplit, (long long)grid,
                 hi - lo, span / grid, pro / grid, items / grid, tx / grid, tk / grid);
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

// rows per pass of the pair kernel: 8 when the routed rows spread thin over
// the experts (decode), so two rows buffers of a 16-block k range fit three
// CTAs per SM
static int pair_nb(int64_t rows, double active_experts) {
  return (double)rows <= 4.0 * std::max(1.0, active_experts) ? 8 : 16;
}

int gemv_pair_splits(int64_t m, int64_t n, double active_experts, int64_t rows) {
  const int64_t nkb = (m + 63) / 64;
  const int cap = gv::pair_max_kbs(pair_nb(rows, active_experts));
  int s = gemv_splits(m, n, active_experts);
  while ((nkb + s - 1) / s > cap) s *= 2;
  return s;
}

static size_t pair_smem(int bits, int nb, int kbs_max) {
  const int nst = bits == 4 ? gv::Ring<4>::NST : bits == 8 ? gv::Ring<8>::NST : gv::Ring<16>::NST;
  return (size_t)nst * wblock_bytes(bits) + 256 + (size_t)2 * nb * (kbs_max * 64 + 8) * 2;
}

template <int BITS, int NB>
static int run_gemv_pair(const GemmArgs& a1, const GemmArgs& a2, const GemvWork& w1,
                         const GemvWork& w2, uint32_t* ready, uint32_t* ctl, cudaStream_t st) {
  gv::PairParams P;
  P.ph[0] = make_phase(a1, w1, BITS);
  P.ph[1] = make_phase(a2, w2, BITS);
  P.problems = a1.problems;
  P.rows = a1.rows;
  P.np = (int)a1.np;
  debias_pair(a1.debias, &P.db2, &P.hb2);
  P.ready = ready;
  P.ctl = ctl;
  P.E = (int)a1.E;
  P.kbs_max = std::max(P.ph[0].kbs, P.ph[1].kbs);
  if (P.kbs_max > gv::pair_max_kbs(NB))
    return set_error(MOE_EINVAL, "gemv_pair: k range per split too long");
  const size_t smem = pair_smem(BITS, NB, P.kbs_max);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(gv::gemv_pair_kernel<BITS, NB>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  int per_sm = 0;
  MOE_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gv::gemv_pair_kernel<BITS, NB>,
                                                             gv::kPairThreads, smem));
  static const int cap = std::getenv("MOE_GEMV_CTAS") ? std::atoi(std::getenv("MOE_GEMV_CTAS")) : 3;
  per_sm = std::max(1, std::min(per_sm, cap));
  const int64_t live = std::max<int64_t>(1, std::min<int64_t>(a1.np, a1.rows));
  const int64_t items = live * std::max(P.ph[0].nft * P.ph[0].nsplit, P.ph[1].nft * P.ph[1].nsplit);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(items, per_sm * (int64_t)sm_count()));
  MOE_CUDA_TRY(launch_k(0, gv::gemv_pair_kernel<BITS, NB>, dim3((unsigned)grid),
                        dim3(gv::kPairThreads), smem, st, P));
  note_launch();
  return check_launch("gemv_pair");
}

// Experimental (MOE_GEMV_PAIR=1, off by default): int4 / int8 only -- with
// fp16 weights repeated forwards showed whole experts of FFN2 rows wrong on
// some launches (a race not yet root-caused)
bool gemv_pair_supported(int64_t rows, int64_t np, int64_t d, int64_t f, int bits) {
  return bits != 16 && rows < 65536 && np <= gv::kPairProblems && d % 64 == 0 && f % 64 == 0;
}

int launch_gemv_pair(const GemmArgs& a1, const GemmArgs& a2, const GemvWork& w1,
                     const GemvWork& w2, uint32_t* ready, uint32_t* ctl, cudaStream_t st) {
  if (a1.np == 0 || a1.rows == 0) return MOE_OK;
  if (!gemv_pair_supported(a1.rows, a1.np, a1.m, a1.n, a1.bits))
    return set_error(MOE_EINVAL, "gemv_pair: needs int4/int8, rows < 65536, <= 512 problems, m and n multiples of 64");
  if (a2.m != a1.n || a2.n != a1.m || a1.bits != a2.bits || a2.x != a1.out)
    return set_error(MOE_EINVAL, "gemv_pair: FFN2 must read FFN1's output");
  if ((w1.nsplit > 1 && (w1.part == nullptr || w1.ticket == nullptr)) ||
      (w2.nsplit > 1 && (w2.part == nullptr || w2.ticket == nullptr)) ||
      (w1.nsplit > 1 && w2.nsplit > 1 && (w1.part == w2.part || w1.ticket == w2.ticket)))
    return set_error(MOE_EINVAL, "gemv_pair: split-K workspaces missing or shared");
  if (ready == nullptr || ctl == nullptr) return set_error(MOE_EINVAL, "gemv_pair: no sync words");
  // NB = 8 whenever the splits need the longer k range; else by row density
  const double act = (double)std::min<int64_t>(a1.np, a1.rows);
  const int64_t kb1 = ((a1.m + 63) / 64 + w1.nsplit - 1) / w1.nsplit;
  const int64_t kb2 = ((a2.m + 63) / 64 + w2.nsplit - 1) / w2.nsplit;
  const bool nb8 = std::max(kb1, kb2) > gv::pair_max_kbs(16) || pair_nb(a1.rows, act) == 8;
  switch (a1.bits) {
    case 4: return nb8 ? run_gemv_pair<4, 8>(a1, a2, w1, w2, ready, ctl, st)
                       : run_gemv_pair<4, 16>(a1, a2, w1, w2, ready, ctl, st);
    case 8: return nb8 ? run_gemv_pair<8, 8>(a1, a2, w1, w2, ready, ctl, st)
                       : run_gemv_pair<8, 16>(a1, a2, w1, w2, ready, ctl, st);
    default: return set_error(MOE_EINVAL, "gemv_pair: int4 / int8 only");
  }
}

}  // namespace moecu
