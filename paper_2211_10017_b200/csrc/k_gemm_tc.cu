// k_gemm_tc.cu -- FAST-mode grouped expert GEMM on the 5th-gen tensor cores.
//
// Replaces the per-expert panel loop of proj/src/grouped_gemm.cpp:165-214
// (fused dequant) with one persistent, warp-specialised sm_100a kernel:
//
//   D[feature, token] = sum_k  Wq[k, feature] * X[token, k]
//
// * MMA M = 128 output features of one expert, N = BN tokens (up to 224),
//   K = 16 per instruction, kind::f16 with f32 accumulation in TMEM
//   (double-buffered: 2 x BN columns).  A = the dequantised weight tile lives
//   in TENSOR MEMORY (2 stages x 32 columns; "TS" MMA), B = the activation
//   tile in shared memory (TMA, 128-byte swizzle, K-major).  Keeping A out of
//   shared memory removes the A-tile stores and the MMA's A reads from the
//   shared-memory pipe, which ncu showed ~80% busy in the SS form.
// * Dequant warps (one per 32-feature TMEM lane quarter, two groups
//   alternating k-blocks) turn each feature's 64 codes -- bulk-copied into
//   shared memory packed -- into fp16 with the magic I2F trick
//   (proj/include/moeinfer/dequant.hpp:39-63; 9 ops per 8 int4 codes) and
//   write them to TMEM with one tcgen05.st.32x32b.x32 per thread.  The
//   per-channel scale is applied to
//   the f32 accumulator in the epilogue instead of to each weight (the
//   reference rounds q*s to fp16 first; both stay inside the tolerance,
//   DESIGN.md §4).
// * ONE thread runs the MMA loop.  Measured on this B200
//   (scripts/mma_bench{2,3}.cu): issuing a tcgen05.mma costs ~90 cycles of
//   the issuing thread, so an instruction must carry >= 128 tensor cycles
//   (M=128 x N=256) to stay tensor-bound; a warp-wide wait + lane-0 issue
//   costs ~650 cycles per 4-MMA k-block; and SS-mode N=256 MMAs keep full
//   rate while shared memory also absorbs ~130 B/clk of stores plus ~60
//   B/clk of TMA fills (this kernel needs ~100 B/clk).
// * Shared-memory stages (TMA + bulk) and A stages are separate rings.
//
// Roles (512 threads): warp 0 TMA/bulk producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warp 3 tile-table builder, warps 4-11 dequant (two groups
// of four), warps 12-15 epilogue.  Tiles: (problem, token tile of BN,
// feature tile of 128), token-tile major so concurrently running CTAs share
// activation tiles in L2.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace moecu {

namespace tc {

constexpr int kDqGroups = 2;                            // dequant warp groups
constexpr int kEpiGroups = 2;                           // epilogue warp groups
constexpr int kThreads = 32 * (4 + 4 * kDqGroups + 4 * kEpiGroups);
constexpr int kMaxProblems = 1024;

// TS = true: A (dequantised weights) in TMEM, 2 x BN accumulator columns
// (BN <= 224).  TS = false: A in shared memory (SS MMA), which frees TMEM for
// two 256-column accumulators -- chosen when 256-token tiles fit one wave.
template <int BITS, int BN, bool TS, int CL = 1, int NSX = 8>
struct Cfg {
  static constexpr int WBYTES = wblock_bytes(BITS);
  static constexpr int BBYTES = BN / CL * 128;   // this CTA's BN / CL rows x 64 fp16
  static constexpr int ABYTES = TS ? 0 : 128 * 128;  // SS: 128 features x 64 fp16 per A stage
  static constexpr int STAGE = BBYTES + WBYTES;
  static constexpr int EPI_WBUF = 32 * 32 * 2;                   // per warp: [32][32] fp16
  static constexpr int EPI = kEpiGroups * 4 * EPI_WBUF;
  // A stages: TS keeps as many 32-column stages as TMEM leaves beside the
  // accumulators (each dequant group then has >= 2 stages to run ahead)
  // accumulators: double-buffered (the epilogue of tile i overlaps the
  // mainloop of tile i+1) except TS with 256-token tiles, whose A ring
  // needs the TMEM -- chosen for launches of at most one wave, where there
  // is no next tile to overlap
  static constexpr int NACC = (TS && BN > 224) ? 1 : 2;
  static constexpr int NA = TS ? ((512 - NACC * BN) / 32 >= 4 ? 4 : 2) : 2;
  static constexpr int BUDGET = 220 * 1024 - EPI - NA * ABYTES;  // TMA stages
  static constexpr int NS0 = BUDGET / STAGE;
  // TMA stages, an EVEN count (root cause of the round-1 fault at NS = 3 / 7,
  // fp16 weights): the two dequant groups take alternate k-blocks, and
  // stage s serves k-blocks it, it + NS, it + 2NS, ...  With NS odd those
  // alternate between the groups, so each group waits on every SECOND phase
  // of full[s]; an mbarrier parity wait only tells adjacent phases apart, so
  // a group waiting for phase n + 2 returned as soon as phase n had
  // completed (the barrier still in phase n + 1) and dequantised stale or
  // not-yet-landed weights.  With NS even a group owns every phase of its
  // stages.  (The A ring is even for the same reason.)
  // at most NSX = 8 (16 measured no faster for C5's 96-token pair tiles,
  // 12 no faster for C2 / C4's 192-token pair tiles)
  static constexpr int NS = NS0 > NSX ? NSX : (NS0 & ~1);
  // [TMA stages][B | W] | [SS: A stages] | epilogue staging | barriers | table
  static constexpr int OFF_A = NS * STAGE;
  static constexpr int OFF_EPI = OFF_A + NA * ABYTES;
  static constexpr int OFF_BAR = OFF_EPI + EPI;
  static constexpr int NBAR = 2 * NS + 2 * NA + 4;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
  static constexpr int OFF_TABLE = OFF_TMEMPTR + 16;
  static constexpr int SMEM = OFF_TABLE + (kMaxProblems + 1) * 4 + 1024;  // + align slack
  static constexpr int A_COL = NACC * BN;                        // TMEM: acc0 | acc1 | [TS: A ring]
  static_assert(NS >= 2, "pipeline too shallow");
  static_assert(NACC * BN + (TS ? NA * 32 : 0) <= 512, "TMEM overflow");
  static_assert(BBYTES % 1024 == 0 && WBYTES % 1024 == 0, "stage alignment");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

struct Tile {
  int p;
  int64_t e, r0, r1, row0, row1, ft;  // problem rows [r0, r1); this tile's [row0, row1)
};

// t indexes (token tile, feature-tile group of CL); CTA `rank` of a CL-CTA
// cluster takes feature tile group*CL + rank of the same token tile
__device__ __forceinline__ Tile decode(const uint32_t* table, int np, const uint32_t* problems,
                                       uint32_t t, int64_t nftg, int BN, int CL = 1,
                                       int rank = 0) {
  const uint32_t g = t / (uint32_t)nftg;  // global token-tile index
  int lo = 0, hi = np - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (table[mid] <= g) lo = mid; else hi = mid - 1;
  }
  Tile x;
  x.p = lo;
  x.e = problems[3 * lo];
  x.r0 = problems[3 * lo + 1];
  x.r1 = problems[3 * lo + 2];
  // a problem's ceil(len / BN) token tiles split its rows evenly (sizes
  // differ by at most one): no 224 + 32 tails whose MMAs would be issue-bound
  const int64_t nt = table[lo + 1] - table[lo], j = g - table[lo], len = x.r1 - x.r0;
  x.row0 = x.r0 + (j * len) / nt;
  x.row1 = x.r0 + ((j + 1) * len) / nt;
  x.ft = (int64_t)(t % (uint32_t)nftg) * CL + rank;
  return x;
}

// MMA N of a tile: a problem's last token tile is usually partial, so N
// follows its live rows (multiple of 16: the pair form splits N in halves of
// whole 8-row swizzle atoms) and padding costs no tensor time
template <int BN, int CL>
__device__ __forceinline__ int tile_n(const Tile& T) {
  const int64_t live = T.row1 - T.row0;
  return live >= BN ? BN : (int)((live + 15) / 16 * 16);
}

struct Params {
  const uint8_t* tiled;
  const uint16_t* scales;
  const uint16_t* bias;
  const uint32_t* problems;
  uint16_t* out;
  const uint16_t* cx;        // fused k = 1 combine (GemmArgs::cout), else null
  const uint32_t* cperm;
  const uint16_t* cscale;
  uint16_t* cout;
  int64_t m, n, np, nft, nkb;
  int relu;
  uint32_t debias2;
  uint32_t hibias2;  // -(64 + debias - 1024) in both halves (i2f_u4_fast)
  unsigned long long* trace;  // dev-only role timestamps of CTA 0 (MOE_TC_TRACE), else null
  int dbg;  // dev-only ablation bits (MOE_TC_DBG): 1 no epilogue, 2 no A stores, 4 no W load
};

constexpr int kTraceN = 1024;  // events per role slot
#define TC_TRACE(slot, idx)                                                      \
  do {                                                                           \
    if (P.trace != nullptr && blockIdx.x == 0 && (idx) < kTraceN)               \
      P.trace[(slot) * kTraceN + (idx)] = clock64();                             \
  } while (0)

// CL = 2: CTA pairs (a 2-CTA cluster on one TPC) run cta_group::2 MMAs of
// M = 256 features x N = BN tokens.  Each CTA dequantises its own 128
// features (adjacent feature tiles) into its own A stage and TMA-loads HALF
// of the token tile (columns [0, N/2) in rank 0, [N/2, N) in rank 1, same
// shared-memory offset); rank 0's thread issues the MMA for both.  Versus
// single CTAs this halves each SM's activation fill and shared-memory reads
// and halves the MMA instructions per output -- the two limits measured on
// the single-CTA kernel.  Barriers the MMA waits on live in
// rank 0: `full` counts both halves' TMA bytes, `afull` / `tempty` take the
// peer's dequant / epilogue arrivals remotely; commits multicast to both.
template <int BITS, int BN, bool TS, int CL, int NSX = 8>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params P) {
  using C = Cfg<BITS, BN, TS, CL, NSX>;
  constexpr bool PAIR = CL == 2;
  const int rank = CL > 1 ? (int)cluster_ctarank() : 0;
  const uint32_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;  // cluster id / count
  const int64_t nftg = P.nft / CL;                               // feature-tile groups
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzle atoms, by pointer arithmetic on
  // the shared array so the compiler keeps shared-space (LDS/STS) accesses.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;                 // smem stage landed  (1 arrive + tx)
  uint64_t* empty = full + C::NS;        // smem stage free    (MMA commit)
  uint64_t* afull = empty + C::NS;       // A stage written    (4 dequant warps)
  uint64_t* aempty = afull + C::NA;      // A stage free       (MMA commit)
  uint64_t* tfull = aempty + C::NA;      // accumulator ready  (MMA commit)
  uint64_t* tempty = tfull + 2;          // accumulator drained (4 epilogue warps)
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);
  uint32_t* table = reinterpret_cast<uint32_t*>(smem + C::OFF_TABLE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = (int)P.np;
  griddep_launch();

  if (warp == 0) {
    if (lane == 0) tma_prefetch_desc(&tmap_x);
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < C::NS; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < C::NA; ++i) {
        mbar_init(&afull[i], 4 * CL);  // pair: both CTAs' dequant warps (rank 0's copy)
        mbar_init(&aempty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 4 * kEpiGroups * CL);
      }
      fence_barrier_init();
    }
  } else if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_ptr, 512);
    else tmem_alloc(tmem_ptr, 512);
  } else if (warp == 3) {
    griddep_wait();  // problems (and the activations) come from the previous kernels
    // token-tile prefix over problems: table[p] = sum_{q<p} ceil(len_q / BN)
    uint32_t carry = 0;
    for (int base = 0; base < np; base += 32) {
      const int p = base + lane;
      uint32_t c = 0;
      if (p < np) c = (P.problems[3 * p + 2] - P.problems[3 * p + 1] + BN - 1) / BN;
      uint32_t incl = c;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (p < np) table[p] = carry + incl - c;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) table[np] = carry;
  }
  griddep_wait();  // every thread: the previous kernels' outputs are visible past here
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // peer barriers initialised before remote use
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  const uint32_t ntiles = table[np] * (uint32_t)nftg;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    // converged warp, one elected lane issues (see the MMA issuer below)
    {
      uint32_t it = 0;
      for (uint32_t t = cid; t < ntiles; t += ncl) {
        const Tile T = decode(table, np, P.problems, t, nftg, BN, CL, rank);
        const uint8_t* wsrc = P.tiled + ((T.e * P.nft + T.ft) * P.nkb) * (int64_t)C::WBYTES;
        const int row = __shfl_sync(0xffffffffu, (int)(T.row0 + rank * (tile_n<BN, CL>(T) / 2)), 0);
        for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
          const int s = it % C::NS;
          mbar_wait_warp(&empty[s], ((it / C::NS) & 1) ^ 1);
          TC_TRACE(0, it);
          uint8_t* sb = smem + s * C::STAGE;
          const uint32_t wb = (P.dbg & 4) ? 0u : (uint32_t)C::WBYTES;
          if (elect_one()) {
            if constexpr (PAIR) {
              // rank 0's full[s] counts both token halves plus its weights;
              // rank 1's counts only its weights (read by its own dequant)
              mbar_arrive_expect_tx(&full[s], rank == 0 ? 2 * C::BBYTES + wb : wb);
              tma_load_2d_pair(sb, &tmap_x, mapa_shared(smem_u32(&full[s]), 0), (int)(kb * 64),
                               row);
            } else {
              mbar_arrive_expect_tx(&full[s], C::BBYTES + wb);
              tma_load_2d(sb, &tmap_x, &full[s], (int)(kb * 64), row);
            }
            if (!(P.dbg & 4))
              bulk_load(sb + C::BBYTES, wsrc + kb * C::WBYTES, C::WBYTES, &full[s]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs the loop converged, so the tile bookkeeping and
    // the descriptors stay warp-uniform (uniform registers feed UTCHMMA
    // directly); one elected lane issues.  A loop run by lane 0 alone makes
    // ptxas re-uniformise every operand per instruction (ELECT + 6 x
    // R2UR.BROADCAST waterfall, ~100 cycles per MMA).
    if (rank == 0) {
      const uint32_t smem_base = smem_u32(smem);
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
      uint32_t it = 0, local = 0;
      for (uint32_t t = cid; t < ntiles; t += ncl, ++local) {
        const int acc = (int)(local % C::NACC);
        // a problem's last token tile is usually partial: the MMA N follows
        // the live rows (multiple of 16) so padding costs no tensor time
        const Tile Tt = decode(table, np, P.problems, t, nftg, BN, CL, rank);
        const uint32_t idesc =
            __shfl_sync(0xffffffffu, umma_idesc_f16(128 * CL, tile_n<BN, CL>(Tt)), 0);
        mbar_wait_warp(&tempty[acc], ((local / C::NACC) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tm + acc * BN;
        for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
          const int s = it % C::NS, a = it % C::NA;
          // one barrier per k-block: every dequant warp waited on full[s]
          // (rank 0's counts both token halves) before arriving on afull[a],
          // so afull also orders the activation tile (each try_wait costs
          // ~90 cycles of this thread even when already complete)
          TC_TRACE(1, it);
          mbar_wait_warp(&afull[a], (it / C::NA) & 1);
          tc_fence_after();
          TC_TRACE(2, it);
          const uint64_t bdesc = umma_desc_sw128(smem_base + s * C::STAGE);
          if (elect_one()) {
            if constexpr (TS) {
              const uint32_t a_tmem = tm + C::A_COL + a * 32;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {  // K advance of 16: B 32 bytes (2 desc units), A 8 TMEM cols
                if constexpr (PAIR)
                  tc_mma_ts_pair(d_tmem, a_tmem + kk * 8, bdesc + (uint64_t)(kk * 2), idesc,
                                 (kb | kk) != 0 ? 1u : 0u);
                else
                  tc_mma_ts(d_tmem, a_tmem + kk * 8, bdesc + (uint64_t)(kk * 2), idesc,
                            (kb | kk) != 0 ? 1u : 0u);
              }
            } else {
              const uint64_t adesc = umma_desc_sw128(smem_base + C::OFF_A + a * C::ABYTES);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {  // K advance of 16 fp16 = 32 bytes = 2 desc units
                if constexpr (PAIR)
                  tc_mma_ss_pair(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2),
                                 idesc, (kb | kk) != 0 ? 1u : 0u);
                else
                  tc_mma_ss(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2),
                            idesc, (kb | kk) != 0 ? 1u : 0u);
              }
            }
            if constexpr (PAIR) {  // both CTAs' stages are released by the pair's MMAs
              tc_commit_pair_mc(&empty[s], 3);
              tc_commit_pair_mc(&aempty[a], 3);
            } else {
              tc_commit(&empty[s]);
              tc_commit(&aempty[a]);
            }
          }
          __syncwarp();
          TC_TRACE(3, it);
        }
        if (elect_one()) {
          if constexpr (PAIR) tc_commit_pair_mc(&tfull[acc], 3);
          else tc_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 4 + 4 * kDqGroups) {
    // ------------------------------------------------------------ dequant
    // kDqGroups groups of 4 warps (one warp per TMEM sub-partition) take
    // alternate k-blocks, so one group's shared-memory/ALU latency overlaps
    // the other's tcgen05.st.
    const int q = (warp - 4) & 3, grp = (warp - 4) >> 2;
    const int feat = q * 32 + lane;
    uint32_t it = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl) {
      for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
        if ((int)(it % kDqGroups) != grp) continue;
        const int s = it % C::NS, a = it % C::NA;
        mbar_wait_warp(&full[s], (it / C::NS) & 1);
        mbar_wait_warp(&aempty[a], ((it / C::NA) & 1) ^ 1);
        if (lane == 0 && q == 0) TC_TRACE(4, it);
        const uint4* wblk = reinterpret_cast<const uint4*>(smem + s * C::STAGE + C::BBYTES);
        uint32_t v[32];
        if constexpr (BITS == 4) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 c = wblk[h * 128 + feat];
            const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int w = 0; w < 4; ++w)
              i2f_u4_fast(wd[w], P.debias2, P.hibias2, &v[h * 16 + w * 4]);
          }
        } else if constexpr (BITS == 8) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const uint4 c = wblk[c4 * 128 + feat];
            const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) i2f_u8(wd[w], P.debias2, &v[c4 * 8 + w * 2]);
          }
        } else {
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint4 c = wblk[c8 * 128 + feat];
            v[c8 * 4 + 0] = c.x;
            v[c8 * 4 + 1] = c.y;
            v[c8 * 4 + 2] = c.z;
            v[c8 * 4 + 3] = c.w;
          }
        }
        if constexpr (TS) {
          // A row `feat` = TMEM lane feat: 64 fp16 = 32 columns (k pairs), one
          // 32x32b.x32 store per thread into this warp's lane quarter
          if (!(P.dbg & 2))
            tmem_st_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + C::A_COL + a * 32, v);
          tc_wait_st();
          tc_fence_before();  // TMEM stores -> ordered before the mbarrier arrive
        } else {
          // A tile row `feat`: 128 bytes, 16-byte chunk c (k = 8c..8c+7) stored at
          // chunk position c ^ (feat & 7) -- the 128B-swizzle K-major atom layout
          if (!(P.dbg & 2)) {
            uint8_t* arow = smem + C::OFF_A + a * C::ABYTES + feat * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<uint4*>(arow + ((c ^ (feat & 7)) << 4)) =
                  make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          }
          fence_proxy_async_smem();  // generic-proxy stores -> visible to tcgen05.mma
        }
        __syncwarp();
        if (lane == 0) {
          if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&afull[a]), 0));
          else mbar_arrive(&afull[a]);
        }
        if (lane == 0 && q == 0) TC_TRACE(5, it);
      }
    }
  } else if (warp >= 4 + 4 * kDqGroups) {
    // ----------------------------------------------------------- epilogue
    // kEpiGroups groups of 4 warps take alternate 32-token chunks of a tile.
    // Every warp works alone: it drains its 32 features x 32 tokens from TMEM,
    // stages them as [token][32 features] fp16 (one 64-byte row per token) in
    // its private staging buffer, and reads them back as 16-byte row chunks
    // (8 features) that it stores directly.  Each chunk is guarded by its
    // row (a problem's last chunk never writes the next expert's rows) and by
    // its column (n % 8 == 0, so a chunk is entirely inside or outside the
    // row when n % 32 != 0).  No cross-warp barriers.
    const int q = warp & 3, ew = warp - 4 - 4 * kDqGroups, eg = ew >> 2;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint16_t* stage0 = reinterpret_cast<uint16_t*>(smem + C::OFF_EPI + ew * C::EPI_WBUF);
    uint32_t cc = 0;  // chunks processed by this warp
    uint32_t local = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++local) {
      const int acc = (int)(local % C::NACC);
      const Tile T = decode(table, np, P.problems, t, nftg, BN, CL, rank);
      const int64_t col = T.ft * 128 + q * 32 + lane;
      float sc = 1.0f, bi = 0.0f;
      if (col < P.n) {
        if (BITS != 16) sc = h2f(P.scales[T.e * P.n + col]);
        bi = h2f(P.bias[T.e * P.n + col]);
      }
      mbar_wait_warp(&tfull[acc], (local / C::NACC) & 1);
      tc_fence_after();
      if (lane == 0 && ew == 0) TC_TRACE(6, local);
      // only the columns holding this tile's rows need draining
      const int64_t live = T.row1 - T.row0;
      const int ncols = (int)(live < BN ? (live + 31) / 32 * 32 : BN);
#pragma unroll 1
      for (int c0 = eg * 32; c0 < ((P.dbg & 1) ? 0 : ncols); c0 += 32 * kEpiGroups, ++cc) {
        uint16_t* stg = stage0;  // read back before the next chunk overwrites it
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_addr + acc * BN + c0, v);
        tc_wait_ld();
        if (lane == 0 && ew == 0) TC_TRACE(9, cc);
        // two tokens per cvt (f16x2, ReLU folded in), then a 2x2 transpose with
        // the neighbour lane so each 32-bit store holds two adjacent features
        // of one token: even lanes write row j, odd lanes row j+1.
        uint32_t* srow = reinterpret_cast<uint32_t*>(stg + (lane & 1) * 32 + (lane & ~1));
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float h0 = fmaf(__uint_as_float(v[j]), sc, bi);
          const float h1 = fmaf(__uint_as_float(v[j + 1]), sc, bi);
          uint32_t own;
          if (P.relu)
            asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(own) : "f"(h1), "f"(h0));
          else
            asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(own) : "f"(h1), "f"(h0));
          const uint32_t other = __shfl_xor_sync(0xffffffffu, own, 1);
          srow[j * 16] = (lane & 1) ? __byte_perm(other, own, 0x7632)
                                    : __byte_perm(own, other, 0x5410);
        }
        __syncwarp();
        if (lane == 0 && ew == 0) TC_TRACE(10, cc);
        // read back as 16-byte vectors: lane -> (row lane/4 + 8i, 8 features)
        const int nrow = (int)::min((int64_t)32, T.row1 - (T.row0 + c0));
        const int64_t col = T.ft * 128 + q * 32 + (lane & 3) * 8;
        const bool col_live = col < P.n;  // whole 8-feature chunk (n % 8 == 0)
        if (P.cout == nullptr) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = i * 8 + (lane >> 2);
            const uint4 val = *reinterpret_cast<const uint4*>(stg + row * 32 + (lane & 3) * 8);
            if (row < nrow && col_live)
              *reinterpret_cast<uint4*>(P.out + (T.row0 + c0 + row) * P.n + col) = val;
          }
        } else {
          // fused k = 1 combine: out[token] = x[token] (+) y * scale[token];
          // the four rows' loads are issued together (two L2 round trips)
          uint32_t tok[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = i * 8 + (lane >> 2);
            tok[i] = row < nrow && col_live ? P.cperm[T.row0 + c0 + row] : 0xFFFFFFFFu;
          }
          uint4 xv[4];
          uint16_t sv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (tok[i] != 0xFFFFFFFFu) {
              xv[i] = *reinterpret_cast<const uint4*>(P.cx + (int64_t)tok[i] * P.n + col);
              sv[i] = P.cscale[tok[i]];
            }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (tok[i] != 0xFFFFFFFFu) {
              const int row = i * 8 + (lane >> 2);
              const uint4 val = *reinterpret_cast<const uint4*>(stg + row * 32 + (lane & 3) * 8);
              *reinterpret_cast<uint4*>(P.cout + (int64_t)tok[i] * P.n + col) =
                  combine8(xv[i], val, sv[i]);
            }
        }
        __syncwarp();
        if (lane == 0 && ew == 0) TC_TRACE(11, cc);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (lane == 0 && ew == 0) TC_TRACE(7, local);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no peer commit / arrive still in flight
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem, 512);
    else tmem_dealloc(tmem, 512);
  }
}

}  // namespace tc

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int BITS, int BN, bool TS, int CL = 1, int NSX = 8>
static int run_tc(const GemmArgs& a, cudaStream_t st) {
  using C = tc::Cfg<BITS, BN, TS, CL, NSX>;
  auto encode = get_encode();
  if (!encode) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)a.m, (cuuint64_t)a.rows};
  const cuuint64_t strides[1] = {(cuuint64_t)a.m * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)(BN / CL)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(a.x), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  tc::Params P;
  P.tiled = static_cast<const uint8_t*>(a.tiled);
  P.scales = a.scales;
  P.bias = a.bias;
  P.problems = a.problems;
  P.out = a.out;
  P.cx = a.cx;
  P.cperm = a.cperm;
  P.cscale = a.cscale;
  P.cout = a.cout;
  P.m = a.m;
  P.n = a.n;
  P.np = a.np;
  P.nft = (a.n + 127) / 128;
  P.nkb = (a.m + 63) / 64;
  P.relu = a.relu;
  P.debias2 = (uint32_t)a.debias | ((uint32_t)a.debias << 16);
  {
    // value of the debias constant minus 1024 (8 healthy, 9 under MOE_FAULT_INJECT)
    const int off = (int)(a.debias & 0x3FF);
    const uint16_t hb = (uint16_t)(0x8000 | (21 << 10) | (off << 4));  // -(64 + off), 2^6 binade
    P.hibias2 = (uint32_t)hb | ((uint32_t)hb << 16);
  }
  static bool attr_set = false;
  if (!attr_set) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(tc::gemm_tc_kernel<BITS, BN, TS, CL, NSX>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  const char* trace_path = std::getenv("MOE_TC_TRACE");  // development instrumentation
  P.trace = nullptr;
  P.dbg = std::getenv("MOE_TC_DBG") ? std::atoi(std::getenv("MOE_TC_DBG")) : 0;
  if (trace_path) MOE_CUDA_TRY(cudaMalloc(&P.trace, 12 * tc::kTraceN * 8));
  if (P.trace) MOE_CUDA_TRY(cudaMemset(P.trace, 0, 12 * tc::kTraceN * 8));
  if constexpr (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sm_count() / CL * CL));
    cfg.blockDim = dim3(tc::kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled(a.second ? 2 : 1) ? 2 : 1;
    if (trace_path) {
      int nc = 0;
      cudaOccupancyMaxActiveClusters(&nc, tc::gemm_tc_kernel<BITS, BN, TS, CL, NSX>, &cfg);
      std::fprintf(stderr, "gemm_tc pair BN=%d TS=%d: max active clusters %d\n", BN, (int)TS, nc);
    }
    MOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc::gemm_tc_kernel<BITS, BN, TS, CL, NSX>, tmap, P));
  } else {
    MOE_CUDA_TRY(launch_k(a.second ? 2 : 1, tc::gemm_tc_kernel<BITS, BN, TS, CL, NSX>, dim3(sm_count()), dim3(tc::kThreads),
                          C::SMEM, st, tmap, P));
  }
  note_launch();
  const int rc = check_launch("gemm_tc");
  if (P.trace) {
    std::vector<unsigned long long> h(12 * tc::kTraceN);
    cudaStreamSynchronize(st);
    cudaMemcpy(h.data(), P.trace, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(P.trace);
    if (FILE* f = std::fopen(trace_path, "ab")) {
      const int64_t hdr[4] = {BITS, BN, C::NS * 100 + C::NA, P.nkb};
      std::fwrite(hdr, 8, 4, f);
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  return rc;
}

template <int BITS>
static int run_tc_bits(const GemmArgs& a, cudaStream_t st) {
  // Large problems run on CTA pairs (cta_group::2, M = 256 features) when
  // the feature tiles pair up.  Token-tile width, from B200 measurements
  // (bench.py sweeps with MOE_TC_BN / MOE_TC_BNM, C2 and C4, routed and uniform):
  //   * at most one wave of 256-token tiles: TS-256 with a single
  //     accumulator (A in TMEM, MMA-bound k-blocks; nothing to overlap);
  //   * otherwise TS-192 (4 A stages; the evenly split tiles of ~128-190
  //     rows absorb the spread of routed expert sizes; at C2's 1024-row
  //     experts it edges out SS-256, whose k-blocks are bound by the
  //     shared-memory traffic of A).
  // Single CTAs below that (MOE_TC_PAIR=0 forces them; MOE_TC_BN forces a
  // width: 128/160/192/224 TS, 256 SS, 257 TS single-accumulator).
  const int64_t nft = (a.n + 127) / 128;
  static const int force = std::getenv("MOE_TC_BN") ? std::atoi(std::getenv("MOE_TC_BN")) : 0;
  static const bool small_pairs =
      !(std::getenv("MOE_TC_SMALL_PAIR") && std::atoi(std::getenv("MOE_TC_SMALL_PAIR")) == 0);
  if (a.rows_hint >= 32 && a.rows_hint < 96 && small_pairs && nft % 2 == 0 && force == 0) {
    // few rows per expert (C5's 64): every weight tile serves one short token
    // tile, and a single CTA re-reads 2 B of activations from L2 per weight
    // byte; the pair halves that stream and the MMA issues per SM
    return run_tc<BITS, 96, true, 2>(a, st);
  }
  if (a.rows_hint >= 96) {
    static const bool pair_ok = !(std::getenv("MOE_TC_PAIR") && std::atoi(std::getenv("MOE_TC_PAIR")) == 0);
    if (pair_ok && nft % 2 == 0) {
      const int64_t pairs = sm_count() / 2;
      const int64_t tiles256 = a.np * ((a.rows_hint + 255) / 256) * (nft / 2);
      int bn = force;
      static const int multi = std::getenv("MOE_TC_BNM") ? std::atoi(std::getenv("MOE_TC_BNM")) : 192;
      if (bn == 0) bn = tiles256 <= pairs ? 257 : multi;  // MOE_TC_BNM: dev A/B of the multi-wave width
      switch (bn) {
        case 128: return run_tc<BITS, 128, true, 2>(a, st);
        case 160: return run_tc<BITS, 160, true, 2>(a, st);
        case 192: return run_tc<BITS, 192, true, 2>(a, st);
        case 224: return run_tc<BITS, 224, true, 2>(a, st);
        case 257: return run_tc<BITS, 256, true, 2>(a, st);
        default: return run_tc<BITS, 256, false, 2>(a, st);
      }
    }
  }
  if (a.rows_hint >= 160) {
    const int64_t tiles256 = a.np * ((a.rows_hint + 255) / 256) * nft;
    if (tiles256 <= sm_count() || force == 256) return run_tc<BITS, 256, false>(a, st);
    return run_tc<BITS, 224, true>(a, st);
  }
  if (a.rows_hint >= 96) return run_tc<BITS, 128, true>(a, st);
  if (a.rows_hint >= 40) return run_tc<BITS, 64, true>(a, st);
  return run_tc<BITS, 32, true>(a, st);
}

int launch_gemm_tc(const GemmArgs& a, cudaStream_t st) {
  if (a.np == 0 || a.rows == 0) return MOE_OK;
  if (a.np > tc::kMaxProblems)
    return set_error(MOE_EINVAL, "grouped_gemm(fast): at most %d problems", tc::kMaxProblems);
  if (a.m % 8 != 0 || a.n % 8 != 0)
    return set_error(MOE_EINVAL, "grouped_gemm(fast): m and n must be multiples of 8");
  if ((reinterpret_cast<uintptr_t>(a.x) & 15) != 0)
    return set_error(MOE_EINVAL, "grouped_gemm(fast): activations must be 16-byte aligned");
  switch (a.bits) {
    case 4: return run_tc_bits<4>(a, st);
    case 8: return run_tc_bits<8>(a, st);
    default: return run_tc_bits<16>(a, st);
  }
}

}  // namespace moecu
