// k_gemm_tc.cu -- FAST-mode grouped expert GEMM on the 5th-gen tensor cores.
//
// Replaces the per-expert panel loop of proj/src/grouped_gemm.cpp:165-214
// (fused dequant) with one persistent, warp-specialised sm_100a kernel:
//
//   D[feature, token] = sum_k  Wq[k, feature] * X[token, k]
//
// * The MMA's M side is 128 output features of one expert; A = dequantised
//   weights living in TMEM (tcgen05 "TS" form), B = a BN-token x 64-k
//   activation tile in shared memory (TMA, 128-byte swizzle, K-major).
//   Putting the weights in TMEM keeps the dequantised tile out of shared
//   memory entirely: shared memory only carries the packed int4/int8 codes
//   (bulk copies) and the activation tile.
// * Dequant warps (one per TMEM sub-partition) turn each feature's 64 codes
//   into 32 fp16x2 registers with the magic I2F trick (lop3 + hsub2 per 2
//   values; proj/include/moeinfer/dequant.hpp:39-63) and tcgen05.st them.
//   The per-channel scale is NOT applied here -- the MMA runs on the exact
//   small integers (code - offset) and the epilogue multiplies the f32
//   accumulator by s[feature] (the reference instead rounds q*s to fp16
//   before the dot product; both are within the stated tolerance, see
//   DESIGN.md §4).
// * One elected thread issues tcgen05.mma kind::f16 (M=128, N=BN, K=16)
//   into a double-buffered TMEM accumulator; epilogue warps tcgen05.ld it,
//   apply scale, bias, ReLU, round to fp16 and store through a shared-memory
//   transpose (16-byte global stores).
//
// Roles (384 threads): warp 0 TMA/bulk producer, warp 1 MMA issuer, warp 2
// TMEM allocator, warp 3 tile-table builder, warps 4-7 dequant, warps 8-11
// epilogue.  Tiles: (problem, token tile of BN, feature tile of 128), token
// tile major so concurrently running CTAs share activation tiles in L2.
#include <cudaTypedefs.h>

#include "kernels.cuh"

namespace moecu {

namespace tc {

constexpr int kThreads = 384;
constexpr int kMaxProblems = 1024;

template <int BITS, int BN>
struct Cfg {
  static constexpr int WBYTES = wblock_bytes(BITS);
  static constexpr int BBYTES = BN * 128;  // BN rows x 64 fp16
  static constexpr int STAGE = BBYTES + WBYTES;
  static constexpr int BUDGET = 176 * 1024;
  static constexpr int NST_SMEM = BUDGET / STAGE;
  static constexpr int NST_TMEM = (512 - 2 * BN) / 32;
  static constexpr int NST0 = NST_SMEM < NST_TMEM ? NST_SMEM : NST_TMEM;
  static constexpr int NST = NST0 > 12 ? 12 : NST0;
  static constexpr int ACOL0 = 2 * BN;  // first TMEM column of the A stages
  static constexpr int EPI = 4 * 32 * 32 * 2;
  // [stages][B | W] | epilogue staging | barriers | tile table
  static constexpr int OFF_EPI = NST * STAGE;
  static constexpr int OFF_BAR = OFF_EPI + EPI;
  static constexpr int NBAR = 3 * NST + 4;
  static constexpr int OFF_TMEMPTR = OFF_BAR + NBAR * 8;
  static constexpr int OFF_TABLE = OFF_TMEMPTR + 16;
  static constexpr int SMEM = OFF_TABLE + (kMaxProblems + 1) * 4 + 1024;  // + align slack
  static_assert(NST >= 2, "pipeline too shallow");
  static_assert(2 * BN + NST * 32 <= 512, "TMEM overflow");
};

struct Tile {
  int p;
  int64_t e, r0, r1, row0, ft;
};

__device__ __forceinline__ Tile decode(const uint32_t* table, int np, const uint32_t* problems,
                                       uint32_t t, int64_t nft, int BN) {
  const uint32_t g = t / (uint32_t)nft;  // global token-tile index
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
  x.row0 = x.r0 + (int64_t)(g - table[lo]) * BN;
  x.ft = t % (uint32_t)nft;
  return x;
}

struct Params {
  const uint8_t* tiled;
  const uint16_t* scales;
  const uint16_t* bias;
  const uint32_t* problems;
  uint16_t* out;
  int64_t m, n, np, nft, nkb;
  int relu;
  uint32_t debias2;
};

template <int BITS, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const Params P) {
  using C = Cfg<BITS, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* full = bars;               // TMA+bulk landed      (count 1 + tx)
  uint64_t* afull = bars + C::NST;     // A stage in TMEM      (count 4)
  uint64_t* empty = bars + 2 * C::NST; // MMA done with stage  (count 1, commit)
  uint64_t* tfull = bars + 3 * C::NST; // accumulator ready    (count 1, commit)
  uint64_t* tempty = tfull + 2;        // accumulator drained  (count 4)
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + C::OFF_TMEMPTR);
  uint32_t* table = reinterpret_cast<uint32_t*>(smem + C::OFF_TABLE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int np = (int)P.np;

  if (warp == 0) {
    if (lane == 0) tma_prefetch_desc(&tmap_x);
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < C::NST; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&afull[i], 4);
        mbar_init(&empty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], 4);
      }
      fence_barrier_init();
    }
  } else if (warp == 2) {
    tmem_alloc(tmem_ptr, 512);
  } else if (warp == 3) {
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  const uint32_t ntiles = table[np] * (uint32_t)P.nft;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = decode(table, np, P.problems, t, P.nft, BN);
        const uint8_t* wsrc = P.tiled + ((T.e * P.nft + T.ft) * P.nkb) * (int64_t)C::WBYTES;
        for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
          const int s = it % C::NST;
          const uint32_t ph = (it / C::NST) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sb = smem + s * C::STAGE;
          mbar_arrive_expect_tx(&full[s], C::STAGE);
          tma_load_2d(sb, &tmap_x, &full[s], (int)(kb * 64), (int)T.row0);
          bulk_load(sb + C::BBYTES, wsrc + kb * C::WBYTES, C::WBYTES, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_f16(128, BN);
    uint32_t it = 0, local = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * BN;
      for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
        const int s = it % C::NST;
        const uint32_t ph = (it / C::NST) & 1;
        mbar_wait(&full[s], ph);
        mbar_wait(&afull[s], ph);
        tc_fence_after();
        if (lane == 0) {  // the same thread issues and commits (commit tracks its own MMAs)
          const uint64_t bdesc = umma_desc_sw128(smem_u32(smem + s * C::STAGE));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_ts(d_tmem, tmem + C::ACOL0 + s * 32 + kk * 8, bdesc + (uint64_t)(kk * 2),
                      idesc, (kb | kk) != 0 ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ dequant
    const int q = warp - 4;
    const int feat = q * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int64_t kb = 0; kb < P.nkb; ++kb, ++it) {
        const int s = it % C::NST;
        const uint32_t ph = (it / C::NST) & 1;
        mbar_wait(&full[s], ph);
        const uint4* wblk = reinterpret_cast<const uint4*>(smem + s * C::STAGE + C::BBYTES);
        uint32_t a[32];
        if constexpr (BITS == 4) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 c = wblk[h * 128 + feat];
            const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) i2f_u4(wd[w], P.debias2, &a[h * 16 + w * 4]);
          }
        } else if constexpr (BITS == 8) {
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const uint4 c = wblk[c4 * 128 + feat];
            const uint32_t wd[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int w = 0; w < 4; ++w) i2f_u8(wd[w], P.debias2, &a[c4 * 8 + w * 2]);
          }
        } else {
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint4 c = wblk[c8 * 128 + feat];
            a[c8 * 4 + 0] = c.x;
            a[c8 * 4 + 1] = c.y;
            a[c8 * 4 + 2] = c.z;
            a[c8 * 4 + 3] = c.w;
          }
        }
        tmem_st_32x32b_x32(tmem + lane_addr + C::ACOL0 + s * 32, a);
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[s]);
      }
    }
  } else if (warp >= 8) {
    // ----------------------------------------------------------- epilogue
    const int q = warp - 8;
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    uint16_t* stage = reinterpret_cast<uint16_t*>(smem + C::OFF_EPI) + q * 32 * 32;
    uint32_t local = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      const Tile T = decode(table, np, P.problems, t, P.nft, BN);
      const int64_t col = T.ft * 128 + q * 32 + lane;
      float sc = 1.0f, bi = 0.0f;
      if (col < P.n) {
        if (BITS != 16) sc = h2f(P.scales[T.e * P.n + col]);
        bi = h2f(P.bias[T.e * P.n + col]);
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem + lane_addr + acc * BN + c0, v);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float h = fmaf(__uint_as_float(v[j]), sc, bi);
          if (P.relu && !(h > 0.0f)) h = 0.0f;
          stage[j * 32 + lane] = f2h(h);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 8 + (lane >> 2), ch = lane & 3;
          const int64_t pos = T.row0 + c0 + row;
          const int64_t c8 = T.ft * 128 + q * 32 + ch * 8;
          const uint4 val = *reinterpret_cast<const uint4*>(stage + row * 32 + ch * 8);
          if (pos < T.r1 && c8 < P.n) *reinterpret_cast<uint4*>(P.out + pos * P.n + c8) = val;
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
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

template <int BITS, int BN>
static int run_tc(const GemmArgs& a, cudaStream_t st) {
  using C = tc::Cfg<BITS, BN>;
  auto encode = get_encode();
  if (!encode) return set_error(MOE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)a.m, (cuuint64_t)a.rows};
  const cuuint64_t strides[1] = {(cuuint64_t)a.m * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)BN};
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
  P.m = a.m;
  P.n = a.n;
  P.np = a.np;
  P.nft = (a.n + 127) / 128;
  P.nkb = (a.m + 63) / 64;
  P.relu = a.relu;
  P.debias2 = (uint32_t)a.debias | ((uint32_t)a.debias << 16);
  static bool attr_set = false;
  if (!attr_set) {
    MOE_CUDA_TRY(cudaFuncSetAttribute(tc::gemm_tc_kernel<BITS, BN>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  tc::gemm_tc_kernel<BITS, BN><<<sm_count(), tc::kThreads, C::SMEM, st>>>(tmap, P);
  note_launch();
  return check_launch("gemm_tc");
}

template <int BITS>
static int run_tc_bits(const GemmArgs& a, cudaStream_t st) {
  if (a.rows_hint >= 96) return run_tc<BITS, 128>(a, st);
  if (a.rows_hint >= 40) return run_tc<BITS, 64>(a, st);
  return run_tc<BITS, 32>(a, st);
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
