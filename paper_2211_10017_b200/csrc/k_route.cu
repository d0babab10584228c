// k_route.cu -- K3 routing plan + gather, unpermute, K6 combine.
//
// build_routing_plan (proj/src/routing.cpp:43-87) is a STABLE counting sort
// of S = T*k slots by key = finished ? E : expert.  GPU form, three passes:
//   1. count : per 256-slot block, a shared-memory histogram of keys;
//   2. scan  : one CTA turns the (block x key) histogram into global key
//              offsets (= expert_offsets, active_rows) and per-block bases,
//              and emits the per-expert problem list for the grouped GEMMs;
//   3. place : per block, each slot's rank among equal keys in slot order is
//              (rank inside its warp via __match_any_sync + popc) + (equal
//              keys in earlier warps) -> pos = base + rank; writes perm/inv
//              and gathers the activation row into expert-sorted order with
//              16-byte vector copies (permute_rows, routing.cpp:89-97).
// Everything is integer and order-deterministic: bit-identical to the
// reference counting sort.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace moecu {

constexpr int kPlanBlock = 256;

int64_t plan_blocks(int64_t S) { return (S + kPlanBlock - 1) / kPlanBlock; }

__device__ __forceinline__ uint32_t slot_key(const uint32_t* expert, const uint8_t* finished,
                                             int64_t slot, int k, int64_t E, uint32_t* bad) {
  const uint32_t e = expert[slot];
  if (e >= (uint32_t)E) atomicMin(bad, (uint32_t)slot);
  if (finished != nullptr && finished[slot / k] != 0) return (uint32_t)E;
  return e >= (uint32_t)E ? (uint32_t)E : e;
}

__global__ void __launch_bounds__(kPlanBlock) plan_count_kernel(
    const uint32_t* __restrict__ expert, const uint8_t* __restrict__ finished, int64_t S, int k,
    int64_t E, uint32_t* __restrict__ blockcnt, uint32_t* bad) {
  extern __shared__ uint32_t hist[];
  for (int64_t i = threadIdx.x; i <= E; i += kPlanBlock) hist[i] = 0;
  __syncthreads();
  const int64_t slot = (int64_t)blockIdx.x * kPlanBlock + threadIdx.x;
  if (slot < S) atomicAdd(&hist[slot_key(expert, finished, slot, k, E, bad)], 1u);
  __syncthreads();
  for (int64_t i = threadIdx.x; i <= E; i += kPlanBlock)
    blockcnt[i * gridDim.x + blockIdx.x] = hist[i];  // key-major [E+1][nblk]
}

// One CTA of 1024 threads over the key-major histogram cnt[key][block]:
//   pass 1: warp w sums keys w, w+32, ... over all blocks (coalesced rows);
//   scan  : exclusive scan of the key totals -> expert_offsets, active_rows;
//   pass 2: per key, a warp-wide running scan over blocks writes
//           base[key][block] = offsets[key] + (count of key in earlier blocks).
__global__ void __launch_bounds__(1024) plan_scan_kernel(
    const uint32_t* __restrict__ blockcnt, int64_t nblk, int64_t E,
    uint32_t* __restrict__ blockbase, uint32_t* __restrict__ offsets,
    uint32_t* __restrict__ problems, uint32_t* __restrict__ active) {
  __shared__ uint32_t tot[1024 + 1];
  __shared__ uint32_t warp_sum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t keys = E + 1;
  // loads are issued 8 per lane before any use (latency, not bandwidth, bound)
  for (int64_t key = warp; key < keys; key += 32) {
    const uint32_t* row = blockcnt + key * nblk;
    uint32_t s = 0;
    for (int64_t b0 = 0; b0 < nblk; b0 += 256) {
      uint32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t b = b0 + j * 32 + lane;
        v[j] = b < nblk ? row[b] : 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) s += v[j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) tot[key] = s;
  }
  __syncthreads();
  const uint32_t t = tid < keys ? tot[tid] : 0u;
  uint32_t incl = t;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t ws = warp_sum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += v;
    }
    warp_sum[lane] = ws;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t excl = incl - t + (warp > 0 ? warp_sum[warp - 1] : 0);
  __syncthreads();  // every thread has read tot[] / warp_sum[]
  if (tid < keys) {
    tot[tid] = excl;
    offsets[tid] = excl;  // offsets[E] = start of the finished tail = active_rows
  }
  __syncthreads();
  for (int64_t key = warp; key < keys; key += 32) {
    const uint32_t* row = blockcnt + key * nblk;
    uint32_t* brow = blockbase + key * nblk;
    uint32_t carry = tot[key];
    for (int64_t b0 = 0; b0 < nblk; b0 += 256) {  // lane owns 8 consecutive blocks
      uint32_t v[8], pre[8], run = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t b = b0 + lane * 8 + j;
        v[j] = b < nblk ? row[b] : 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        pre[j] = run;
        run += v[j];
      }
      uint32_t in = run;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, in, o);
        if (lane >= o) in += u;
      }
      const uint32_t base = carry + in - run;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t b = b0 + lane * 8 + j;
        if (b < nblk) brow[b] = base + pre[j];
      }
      carry += __shfl_sync(0xffffffffu, in, 31);
    }
  }
  if (tid < E && problems != nullptr) {
    problems[3 * tid] = (uint32_t)tid;
    problems[3 * tid + 1] = tot[tid];
    problems[3 * tid + 2] = tot[tid + 1];
  }
  if (tid == 0 && active != nullptr) *active = tot[E];
}

// One CTA per routing key: the key's exclusive prefix over the blocks,
// blockbase[key][b] = sum of cnt[key][b' < b] (WITHOUT the key's offset), and
// its total keytot[key].  (E+1) CTAs in parallel instead of one CTA walking
// the whole (key x block) table: the key offsets are a 1-2 warp scan over
// keytot that every place CTA redoes (plan_place_kernel with keytot).
__global__ void __launch_bounds__(256) plan_keyscan_kernel(const uint32_t* __restrict__ blockcnt,
                                                           int64_t nblk,
                                                           uint32_t* __restrict__ blockbase,
                                                           uint32_t* __restrict__ keytot) {
  __shared__ uint32_t wsum[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* row = blockcnt + (int64_t)blockIdx.x * nblk;
  uint32_t* brow = blockbase + (int64_t)blockIdx.x * nblk;
  uint32_t carry = 0;
  for (int64_t b0 = 0; b0 < nblk; b0 += 256 * 8) {  // thread owns 8 consecutive blocks
    uint32_t v[8], pre[8], run = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t b = b0 + tid * 8 + j;
      v[j] = b < nblk ? row[b] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      pre[j] = run;
      run += v[j];
    }
    uint32_t in = run;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, in, o);
      if (lane >= o) in += u;
    }
    if (lane == 31) wsum[warp] = in;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t x = wsum[w];
      wpre += w < warp ? x : 0u;
      tot += x;
    }
    const uint32_t base = carry + wpre + in - run;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t b = b0 + tid * 8 + j;
      if (b < nblk) brow[b] = base + pre[j];
    }
    carry += tot;
    __syncthreads();  // wsum reused
  }
  if (tid == 0) keytot[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(1024) plan_place_kernel(int spb,
    const uint32_t* __restrict__ expert, const uint8_t* __restrict__ finished, int64_t S, int k,
    int64_t E, const uint32_t* __restrict__ blockbase, uint32_t* __restrict__ perm,
    uint32_t* __restrict__ inv, const uint16_t* __restrict__ src, int64_t cols,
    uint16_t* __restrict__ dst, uint32_t* bad, const uint32_t* __restrict__ keytot = nullptr,
    uint32_t* __restrict__ offsets = nullptr, uint32_t* __restrict__ problems = nullptr,
    uint32_t* __restrict__ active = nullptr) {
  // spb = slots per plan block (blockDim.x >= spb, a multiple of 32).
  // keytot non-null: blockbase holds per-key prefixes only (plan_keyscan);
  // the key offsets are scanned here and block 0 publishes them.
  extern __shared__ uint32_t wcnt[];  // [warps][E+1], pos list, [keytot: key offsets]
  const int64_t keys = E + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int64_t i = threadIdx.x; i < nwarp * keys; i += blockDim.x) wcnt[i] = 0;
  uint32_t* koff = wcnt + nwarp * keys + blockDim.x;
  if (keytot != nullptr && warp == 0) {
    uint32_t carry = 0;
    for (int64_t k0 = 0; k0 < keys; k0 += 32) {
      const int64_t kk = k0 + lane;
      const uint32_t v = kk < keys ? keytot[kk] : 0u;
      uint32_t in = v;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, in, o);
        if (lane >= o) in += u;
      }
      if (kk < keys) koff[kk] = carry + in - v;
      carry += __shfl_sync(0xffffffffu, in, 31);
    }
  }
  __syncthreads();
  if (keytot != nullptr && blockIdx.x == 0) {
    for (int64_t kk = threadIdx.x; kk < keys; kk += blockDim.x) offsets[kk] = koff[kk];
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
      problems[3 * e] = (uint32_t)e;
      problems[3 * e + 1] = koff[e];
      problems[3 * e + 2] = koff[e + 1];
    }
    if (threadIdx.x == 0 && active != nullptr) *active = koff[E];
  }
  const int64_t slot = (int64_t)blockIdx.x * spb + threadIdx.x;
  const bool live = (int)threadIdx.x < spb && slot < S;
  const uint32_t key = live ? slot_key(expert, finished, slot, k, E, bad) : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t rank_w = __popc(peers & lt);
  if (live && (peers >> lane) == 1u) wcnt[warp * keys + key] = __popc(peers);  // highest peer
  __syncthreads();
  uint32_t* pos_l = wcnt + nwarp * keys;
  if (live) {
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wcnt[w * keys + key];
    const uint32_t pos = blockbase[(int64_t)key * gridDim.x + blockIdx.x] + before + rank_w +
                         (keytot != nullptr ? koff[key] : 0u);
    perm[pos] = (uint32_t)slot;
    inv[slot] = pos;
    pos_l[threadIdx.x] = pos;
  }
  if (dst == nullptr) return;
  __syncthreads();
  // gather: dst[pos] = src[slot / k], one warp per row, 16-byte vectors
  const int64_t nslots = ::min((int64_t)spb, S - (int64_t)blockIdx.x * spb);
  const bool vec = (cols % 8) == 0;
  for (int64_t i = warp; i < nslots; i += nwarp) {
    const int64_t s = (int64_t)blockIdx.x * spb + i;
    const uint16_t* a = src + (s / k) * cols;
    uint16_t* b = dst + (int64_t)pos_l[i] * cols;
    if (vec) {
      const uint4* a4 = reinterpret_cast<const uint4*>(a);
      uint4* b4 = reinterpret_cast<uint4*>(b);
      for (int64_t c = lane; c < cols / 8; c += 32) b4[c] = a4[c];
    } else {
      for (int64_t c = lane; c < cols; c += 32) b[c] = a[c];
    }
  }
}

// Scan + place + gather in ONE kernel for plans whose (block x key)
// histogram is small (every CTA re-derives the key offsets and its own
// bases from the whole histogram -- (E+1) x nblk words from L2 -- instead of
// waiting on a single-CTA scan kernel), then ranks its slots exactly as
// plan_place_kernel and gathers the rows it placed with all its threads
// (loads batched ahead of the stores).
constexpr int kPlaceThreads = 256;
constexpr int64_t kFusedScanMax = 8192;  // (E+1) * nblk words, staged in shared memory

__global__ void __launch_bounds__(1024) plan_place_fused_kernel(int spb,
    const uint32_t* __restrict__ expert, const uint8_t* __restrict__ finished, int64_t S, int k,
    int64_t E, const uint32_t* __restrict__ blockcnt, uint32_t* __restrict__ perm,
    uint32_t* __restrict__ inv, uint32_t* __restrict__ offsets, uint32_t* __restrict__ problems,
    uint32_t* __restrict__ active, const uint16_t* __restrict__ src, int64_t cols,
    uint16_t* __restrict__ dst, uint32_t* bad, long long* trace, int stage_rows) {
  extern __shared__ __align__(16) uint32_t sh[];
  const int64_t keys = E + 1, nblk = gridDim.x;
#define PL_TRACE(i)                                                               \
  do {                                                                            \
    if (trace != nullptr && threadIdx.x == 0) {                                   \
      long long g_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                      \
      if ((i) == 0) trace[16 + 2 * blockIdx.x] = g_;                              \
      if ((i) == 5) trace[16 + 2 * blockIdx.x + 1] = g_;                          \
      if (blockIdx.x == 0) trace[i] = clock64();                                  \
    }                                                                             \
  } while (0)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  uint32_t* tot = sh;                 // [keys]  totals, then exclusive offsets
  uint32_t* base = tot + keys + 1;    // [keys]  this block's first position per key
  uint32_t* wcnt = base + keys;       // [nwarp][keys]
  uint32_t* pos_l = wcnt + nwarp * keys;  // [blockDim]
  uint32_t* cnt = pos_l + blockDim.x;     // [keys][nblk + 1] staged histogram (then srow)
  const int64_t b = blockIdx.x;
  griddep_launch();
  griddep_wait();
  PL_TRACE(0);
  // stage_rows: this block's source rows are bulk-copied into shared memory
  // now (they do not depend on the placement), overlapping the histogram
  // and scan phases; the gather at the end is then bulk stores only
  const int nslots_b = (int)::min((int64_t)spb, S - b * spb);
  const int64_t ncnt_w = std::max<int64_t>(keys * (nblk + 1), (int64_t)blockDim.x);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(cnt + ncnt_w) + 15) & ~uintptr_t(15));
  uint16_t* rows_sm = reinterpret_cast<uint16_t*>(rbar + 2);
  if (stage_rows && dst != nullptr && warp == 0) {
    // one lane issues every copy (measured: one copy per lane was ~600
    // cycles slower to stage the histogram, C2)
    if (elect_one()) {
      mbar_init(rbar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(rbar, (uint32_t)(nslots_b * cols * 2));
      int64_t q = (b * spb) / k;
      int r = (int)((b * spb) % k);
      for (int i = 0; i < nslots_b; ++i) {
        bulk_load(rows_sm + (int64_t)i * cols, src + q * cols, (uint32_t)(cols * 2), rbar);
        if (++r == k) {
          r = 0;
          ++q;
        }
      }
    }
    __syncwarp();
  }
  // this thread's slot key, loaded up front (overlaps the histogram loads)
  const int64_t slot = b * spb + threadIdx.x;
  const bool live = (int)threadIdx.x < spb && slot < S;
  const uint32_t key = live ? slot_key(expert, finished, slot, k, E, bad) : 0xFFFFFFFFu;
  // 1. stage the whole (key x block) histogram (all loads in flight at once),
  //    then per key: total over all blocks and the count in blocks before b
  // (pitch nblk + 1: one thread per key walks its row without bank conflicts)
  // (loads batched 8 per thread ahead of the stores: one L2 round trip,
  // not one per element)
  const int ncnt = (int)(keys * nblk), cp = (int)nblk + 1;
  for (int i0 = threadIdx.x; i0 < ncnt; i0 += 8 * (int)blockDim.x) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      v[u] = i < ncnt ? blockcnt[i] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < ncnt) {
        const int kk = i / (int)nblk;
        cnt[kk * cp + (i - kk * (int)nblk)] = v[u];
      }
    }
  }
  for (int64_t i = threadIdx.x; i < nwarp * keys; i += blockDim.x) wcnt[i] = 0;
  __syncthreads();
  // a warp per key: lanes take strided blocks, then a shuffle reduction
  // (integer sums: order-free)
  for (int64_t kk = warp; kk < keys; kk += nwarp) {
    const uint32_t* row = cnt + kk * cp;
    uint32_t t = 0, pre = 0;
    for (int bb = lane; bb < (int)nblk; bb += 32) {
      const uint32_t v = row[bb];
      t += v;
      pre += bb < b ? v : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
    }
    if (lane == 0) {
      tot[kk] = t;
      base[kk] = pre;
    }
  }
  __syncthreads();
  PL_TRACE(1);
  // 2. exclusive scan of the key totals: warp 0, 32 keys per round
  //    (lane-interleaved, conflict-free), carry across rounds
  if (warp == 0) {
    uint32_t carry = 0;
    for (int64_t k0 = 0; k0 < keys; k0 += 32) {
      const int64_t key = k0 + lane;
      const uint32_t v = key < keys ? tot[key] : 0u;
      uint32_t in = v;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, in, o);
        if (lane >= o) in += u;
      }
      if (key < keys) {
        tot[key] = carry + in - v;
        base[key] += carry + in - v;
      }
      carry += __shfl_sync(0xffffffffu, in, 31);
    }
  }
  __syncthreads();
  if (b == 0) {
    for (int64_t key = threadIdx.x; key < keys; key += blockDim.x) offsets[key] = tot[key];
    for (int64_t e = threadIdx.x; e < E; e += blockDim.x)
      if (problems != nullptr) {
        problems[3 * e] = (uint32_t)e;
        problems[3 * e + 1] = tot[e];
        problems[3 * e + 2] = tot[e + 1];
      }
    if (threadIdx.x == 0 && active != nullptr) *active = tot[E];
  }
  PL_TRACE(2);
  // 3. place (as plan_place_kernel): rank among equal keys in slot order
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const uint32_t rank_w = __popc(peers & ((1u << lane) - 1u));
  if (live && (peers >> lane) == 1u) wcnt[warp * keys + key] = __popc(peers);
  __syncthreads();
  if (live) {
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wcnt[w * keys + key];
    const uint32_t pos = base[key] + before + rank_w;
    perm[pos] = (uint32_t)slot;
    inv[slot] = pos;
    pos_l[threadIdx.x] = pos;
  }
  if (dst == nullptr) return;
  // source row of each slot (one 64-bit division per slot, not per piece)
  uint32_t* srow = cnt;  // the staged histogram is no longer needed
  if (live) srow[threadIdx.x] = (uint32_t)(slot / k);
  __syncthreads();
  PL_TRACE(3);
  if (stage_rows) {  // rows already in shared memory: bulk stores to their positions
    if (warp == 0) {
      mbar_wait_warp(rbar, 0);
      if (elect_one()) {
        for (int i = 0; i < nslots_b; ++i)
          bulk_store(dst + (int64_t)pos_l[i] * cols, rows_sm + (int64_t)i * cols,
                     (uint32_t)(cols * 2));
        bulk_commit();
        bulk_wait_read<0>();  // shared memory stays valid until the stores have read it
      }
      __syncwarp();
    }
    PL_TRACE(5);
    return;
  }
  // 4. gather dst[pos] = src[slot / k]: 16-byte pieces, 8 loads in flight per
  //    thread (32-bit index math: a 64-bit division per piece costs more
  //    than the copy)
  const int nslots = (int)::min((int64_t)spb, S - b * spb);
  const int c8 = (int)(cols / 8), total = nslots * c8;
  const bool pow2 = (c8 & (c8 - 1)) == 0;
  const int sh_c8 = __ffs(c8) - 1;
  constexpr int U = 8;
  for (int i0 = threadIdx.x; i0 < total; i0 += U * (int)blockDim.x) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < total) {
        const int sl = pow2 ? i >> sh_c8 : i / c8, c = i - sl * c8;
        v[u] = reinterpret_cast<const uint4*>(src + (int64_t)srow[sl] * cols)[c];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * (int)blockDim.x;
      if (i < total) {
        const int sl = pow2 ? i >> sh_c8 : i / c8, c = i - sl * c8;
        reinterpret_cast<uint4*>(dst + (int64_t)pos_l[sl] * cols)[c] = v[u];
      }
    }
  }
  PL_TRACE(5);
#undef PL_TRACE
}

int launch_routing_plan(const uint32_t* expert, const uint8_t* finished, int64_t T, int k,
                        int64_t E, uint32_t* perm, uint32_t* inv, uint32_t* offsets,
                        uint32_t* problems, uint32_t* active, const PlanWork& w,
                        const uint16_t* gather_src, int64_t cols, uint16_t* gather_dst,
                        cudaStream_t st) {
  const int64_t S = T * k;
  if (S == 0) return MOE_OK;
  if (E + 1 > 1024) return set_error(MOE_EINVAL, "routing plan: at most 1023 experts");
  const int64_t nblk = plan_blocks(S);
  plan_count_kernel<<<(unsigned)nblk, kPlanBlock, (E + 1) * 4, st>>>(expert, finished, S, k, E,
                                                                      w.blockcnt, w.bad);
  note_launch();
  plan_scan_kernel<<<1, 1024, 0, st>>>(w.blockcnt, nblk, E, w.blockbase, offsets, problems,
                                       active);
  note_launch();
  const size_t smem = (8 * (E + 1) + kPlanBlock) * 4;
  // The row gather runs as its own wide launch (one warp per row): folding
  // it into plan_place left only S/256 CTAs to move S*cols*2 bytes.
  plan_place_kernel<<<(unsigned)nblk, kPlanBlock, smem, st>>>(
      kPlanBlock, expert, finished, S, k, E, w.blockbase, perm, inv, nullptr, 0, nullptr, w.bad);
  note_launch();
  const int s1 = check_launch("routing_plan");
  if (s1 != MOE_OK || gather_dst == nullptr) return s1;
  return launch_permute(gather_src, cols, perm, S, k, gather_dst, st);
}

// Plan from per-block counts already produced by the fused gate kernel
// (k_gate_fused.cu): blocks of spb = rows*k slots.  scan -> place -> gather.
int launch_plan_from_counts(const uint32_t* expert, const uint8_t* finished, int64_t T, int k,
                            int64_t E, int64_t spb, const PlanWork& w, uint32_t* perm,
                            uint32_t* inv, uint32_t* offsets, uint32_t* problems,
                            uint32_t* active, const uint16_t* gather_src, int64_t cols,
                            uint16_t* gather_dst, cudaStream_t st) {
  const int64_t S = T * k;
  if (S == 0) return MOE_OK;
  if (E + 1 > 1024) return set_error(MOE_EINVAL, "routing plan: at most 1023 experts");
  const int64_t nblk = (S + spb - 1) / spb;
  static const int64_t fused_max =
      std::getenv("MOE_PLAN_FUSED_MAX") ? std::atoll(std::getenv("MOE_PLAN_FUSED_MAX")) : kFusedScanMax;
  if ((E + 1) * nblk <= fused_max && (cols % 8) == 0 && spb <= 1024) {
    const int threads = (int)std::max<int64_t>(kPlaceThreads, (spb + 31) / 32 * 32);
    // tot | base | wcnt[warps] | pos | staged histogram [(E+1) x nblk]
    const size_t smem0 = ((E + 1) * 2 + 1 + (threads / 32) * (E + 1) + threads +
                          std::max<int64_t>((E + 1) * (nblk + 1), threads)) * 4;
    // + the block's source rows, staged by bulk copies (when they fit)
    const size_t rows_bytes = (size_t)spb * cols * 2;
    static const bool no_stage = std::getenv("MOE_PLAN_NO_STAGE") != nullptr;  // dev A/B
    const int stage_rows = !no_stage && gather_dst != nullptr && rows_bytes <= 64 * 1024 ? 1 : 0;
    const size_t smem = smem0 + (stage_rows ? 16 + 16 + rows_bytes : 0);
    if (smem > 48 * 1024) {
      static size_t attr = 0;
      if (smem > attr) {
        MOE_CUDA_TRY(cudaFuncSetAttribute(plan_place_fused_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = smem;
      }
    }
    static long long* dtr = nullptr;
    const bool tr = std::getenv("MOE_GATE_TRACE") != nullptr && nblk <= 65536;
    if (tr && !dtr) MOE_CUDA_TRY(cudaMalloc(&dtr, 8 * (16 + 2 * 65536)));
    MOE_CUDA_TRY(launch_k(0, plan_place_fused_kernel, dim3((unsigned)nblk), dim3(threads), smem, st,
                          (int)spb, expert, finished, S, k, E, (const uint32_t*)w.blockcnt, perm,
                          inv, offsets, problems, active, gather_src, cols, gather_dst, w.bad,
                          tr ? dtr : nullptr, stage_rows));
    note_launch();
    if (tr) {
      std::vector<long long> h(16 + 2 * nblk);
      cudaStreamSynchronize(st);
      cudaMemcpy(h.data(), dtr, h.size() * 8, cudaMemcpyDeviceToHost);
      long long lo = h[16], hi = h[17], sum = 0;
      for (int64_t i = 0; i < nblk; ++i) {
        lo = std::min(lo, h[16 + 2 * i]);
        hi = std::max(hi, h[17 + 2 * i]);
        sum += h[17 + 2 * i] - h[16 + 2 * i];
      }
      std::fprintf(stderr, "plan_place_fused grid=%lld threads=%d spb=%lld: span=%lld ns cta mean=%lld ns; "
                   "cta0 clocks counts=%lld scan=%lld place=%lld gather=%lld\n",
                   (long long)nblk, threads, (long long)spb, hi - lo, sum / nblk, h[1] - h[0],
                   h[2] - h[1], h[3] - h[2], h[5] - h[3]);
    }
    return check_launch("plan_place_fused");
  }
  if (w.keytot == nullptr) return set_error(MOE_EINVAL, "plan_from_counts: no key-total workspace");
  plan_keyscan_kernel<<<(unsigned)(E + 1), 256, 0, st>>>(w.blockcnt, nblk, w.blockbase, w.keytot);
  note_launch();
  const int threads = (int)((spb + 31) / 32 * 32);
  const size_t smem = ((threads / 32) * (E + 1) + threads + (E + 1)) * 4;
  plan_place_kernel<<<(unsigned)nblk, threads, smem, st>>>(
      (int)spb, expert, finished, S, k, E, w.blockbase, perm, inv, nullptr, 0, nullptr, w.bad,
      w.keytot, offsets, problems, active);
  note_launch();
  const int s1 = check_launch("plan_from_counts");
  if (s1 != MOE_OK || gather_dst == nullptr) return s1;
  return launch_permute(gather_src, cols, perm, S, k, gather_dst, st);
}

// ------------------------------------------------------------------ permute
__global__ void permute_kernel(const uint16_t* __restrict__ x, int64_t cols,
                               const uint32_t* __restrict__ perm, int64_t S, int k,
                               uint16_t* __restrict__ xp) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= S) return;
  const uint16_t* a = x + (int64_t)(perm[row] / k) * cols;
  uint16_t* b = xp + row * cols;
  if (cols % 8 == 0) {
    for (int64_t c = lane; c < cols / 8; c += 32)
      reinterpret_cast<uint4*>(b)[c] = reinterpret_cast<const uint4*>(a)[c];
  } else {
    for (int64_t c = lane; c < cols; c += 32) b[c] = a[c];
  }
}

int launch_permute(const uint16_t* x, int64_t cols, const uint32_t* perm, int64_t S, int k,
                   uint16_t* xp, cudaStream_t st) {
  if (S == 0) return MOE_OK;
  permute_kernel<<<(unsigned)((S + 7) / 8), 256, 0, st>>>(x, cols, perm, S, k, xp);
  note_launch();
  return check_launch("permute");
}

// ---------------------------------------------------------------- unpermute
// out[perm[i]] = half_mul(y[i], scale[perm[i]]) for i < active, other rows 0
// (routing.cpp:99-116).  Rows are zeroed by the caller.
__global__ void unpermute_kernel(const uint16_t* __restrict__ y, int64_t T, int64_t cols,
                                 const uint32_t* __restrict__ perm,
                                 const uint32_t* __restrict__ active,
                                 const uint16_t* __restrict__ scale, uint16_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= T || i >= (int64_t)*active) return;
  const uint32_t r = perm[i];
  const uint16_t s = scale[r];
  for (int64_t c = lane; c < cols; c += 32) out[(int64_t)r * cols + c] = hmul(y[i * cols + c], s);
}

int launch_unpermute_scale(const uint16_t* y, int64_t T, int64_t cols, const uint32_t* perm,
                           const uint32_t* active, const uint16_t* scale, uint16_t* out,
                           cudaStream_t st) {
  if (T == 0) return MOE_OK;
  MOE_CUDA_TRY(cudaMemsetAsync(out, 0, (size_t)T * cols * 2, st));
  unpermute_kernel<<<(unsigned)((T + 7) / 8), 256, 0, st>>>(y, T, cols, perm, active, scale, out);
  note_launch();
  return check_launch("unpermute");
}

// ------------------------------------------------------------------ combine
// out[r] = finished[r] ? x[r]
//        : (((x[r] (+) y[inv[r,0]]*s0) (+) y[inv[r,1]]*s1) ...)  fp16 RN each op
// (model.cpp:334-346 with routing.cpp:106-114; slot order for k > 1).
__global__ void combine_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ y,
                               const uint32_t* __restrict__ inv,
                               const uint16_t* __restrict__ scale,
                               const uint8_t* __restrict__ finished, int64_t T, int64_t d, int k,
                               uint16_t* __restrict__ out) {
  griddep_launch();
  griddep_wait();
  const int64_t chunks = d / 8;
  const int64_t total = T * chunks;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / chunks, c = i % chunks;
    uint4 acc = reinterpret_cast<const uint4*>(x + r * d)[c];
    if (finished == nullptr || finished[r] == 0) {
      // slots in groups of up to 4: every index / scale load, then every y
      // row load of the group in flight before the (slot-ordered) folds
      for (int s0 = 0; s0 < k; s0 += 4) {
        const int ns = k - s0 < 4 ? k - s0 : 4;
        uint32_t p[4], sc[4];
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s < ns) {
            p[s] = inv[r * k + s0 + s];
            sc[s] = scale[r * k + s0 + s];
          }
        uint4 yv[4];
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s < ns) yv[s] = reinterpret_cast<const uint4*>(y + (int64_t)p[s] * d)[c];
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (s < ns) {
            const uint32_t s2 = sc[s] | (sc[s] << 16);
            uint32_t* a = reinterpret_cast<uint32_t*>(&acc);
            const uint32_t* b = reinterpret_cast<const uint32_t*>(&yv[s]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t prod, sum;
              asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(prod) : "r"(b[q]), "r"(s2));
              asm("add.rn.f16x2 %0, %1, %2;" : "=r"(sum) : "r"(a[q]), "r"(prod));
              a[q] = sum;
            }
          }
      }
    }
    reinterpret_cast<uint4*>(out + r * d)[c] = acc;
  }
}

__global__ void combine_scalar_kernel(const uint16_t* __restrict__ x,
                                      const uint16_t* __restrict__ y,
                                      const uint32_t* __restrict__ inv,
                                      const uint16_t* __restrict__ scale,
                                      const uint8_t* __restrict__ finished, int64_t T, int64_t d,
                                      int k, uint16_t* __restrict__ out) {
  const int64_t total = T * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d, c = i % d;
    uint16_t acc = x[i];
    if (finished == nullptr || finished[r] == 0)
      for (int s = 0; s < k; ++s)
        acc = hadd(acc, hmul(y[(int64_t)inv[r * k + s] * d + c], scale[r * k + s]));
    out[i] = acc;
  }
}

int launch_combine(const uint16_t* x, const uint16_t* y, const uint32_t* inv,
                   const uint16_t* scale, const uint8_t* finished, int64_t T, int64_t d, int k,
                   uint16_t* out, cudaStream_t st) {
  if (T == 0) return MOE_OK;
  // 16-byte vector path only when every row start is 16-byte aligned
  const bool vec = d % 8 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                                   reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t work = vec ? T * d / 8 : T * d;
  const unsigned blocks = (unsigned)std::min<int64_t>((work + 255) / 256, 148 * 16);
  if (vec)
    MOE_CUDA_TRY(launch_k(3, combine_kernel, dim3(blocks), dim3(256), 0, st, x, y, inv, scale, finished,
                          T, d, k, out));
  else
    combine_scalar_kernel<<<blocks, 256, 0, st>>>(x, y, inv, scale, finished, T, d, k, out);
  note_launch();
  return check_launch("combine");
}

// --------------------------------------------------------------- EP counts
__global__ void ep_counts_kernel(const uint32_t* __restrict__ offsets, int64_t E, int G,
                                 int64_t* __restrict__ counts) {
  const int g = threadIdx.x;
  if (g >= G) return;
  const int64_t per = E / G;
  counts[g] = (int64_t)offsets[(g + 1) * per] - (int64_t)offsets[g * per];
}

int launch_ep_rank_counts(const uint32_t* offsets, int64_t E, int G, int64_t* counts,
                          cudaStream_t st) {
  if (G < 1 || G > 1024 || E % G != 0)
    return set_error(MOE_EINVAL, "ep: n_experts must be divisible by the world size");
  ep_counts_kernel<<<1, 1024, 0, st>>>(offsets, E, G, counts);
  note_launch();
  return check_launch("ep_rank_counts");
}

}  // namespace moecu
