// kernels.cuh -- internal launch interface between the C-ABI (abi.cu) and the
// kernel translation units.  Every launcher returns a moe_cuda.h status.
#pragma once

#include <algorithm>
#include <utility>

#include "../../include/moe_cuda.h"
#include "common.cuh"

namespace moecu {

constexpr int kFeatTile = 128;  // output columns per GEMM tile (MMA M)
constexpr int kKBlock = 64;     // inputs per k-block (one 128-byte fp16 row)

__host__ __device__ constexpr int wblock_bytes(int bits) {
  return bits == 4 ? 4096 : bits == 8 ? 8192 : 16384;
}

int sm_count();

// Programmatic dependent launch for the layer-path kernels: each is
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, calls
// griddep_launch() as it starts (its dependent may be scheduled and run its
// independent prologue -- barrier init, TMEM alloc, weight prefetch) and
// griddep_wait() before it reads anything the previous kernel wrote.  In a
// CUDA graph the edges become programmatic, so each kernel's launch latency
// overlaps its predecessor.  Default MOE_PDL=4 (the second GEMM of an FFN
// pair and the combine); the other modes are A/B switches (abi.cu
// pdl_enabled).
// kind 0: routing kernels, 1: the grouped GEMMs, 2: the second GEMM of an
// FFN pair, 3: the combine, 4: the decode GEMVs, 5: the fused gate (MOE_PDL=
// 1: all, 2: GEMMs, 3: the second GEMM, 4: the second GEMM and the combine,
// 5: 4 + GEMVs, 6: 4 + the gate)
bool pdl_enabled(int kind = 0);
template <typename... KArgs, typename... Args>
cudaError_t launch_k(int pdl_kind, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(pdl_kind) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// k_quant.cu
int launch_quantize(const uint16_t* w, int64_t e, int64_t m, int64_t n, int bits,
                    uint8_t* packed, uint16_t* scales, unsigned long long* bad,
                    cudaStream_t st);
int launch_pack_int4(const uint8_t* v, int64_t count, uint8_t* out, unsigned long long* bad,
                     cudaStream_t st);
int launch_unpack_int4(const uint8_t* p, int64_t count, uint8_t* out, cudaStream_t st);
int launch_dequantize(const uint8_t* packed, const uint16_t* scales, int64_t e, int64_t m,
                      int64_t n, int bits, int fast, uint16_t debias, uint16_t* out,
                      cudaStream_t st);
int64_t tiled_bytes(int64_t e, int64_t m, int64_t n, int bits);
int launch_tile_weights(const void* src, int64_t e, int64_t m, int64_t n, int bits,
                        void* tiled, cudaStream_t st);

// k_gate.cu
int launch_layer_norm(const uint16_t* x, int64_t T, int64_t d, const uint16_t* g,
                      const uint16_t* b, uint16_t* out, cudaStream_t st);
int launch_gate_logits(const uint16_t* xn, int64_t T, int64_t d, const uint16_t* gw,
                       const uint16_t* gb, int64_t E, float* logits, cudaStream_t st);
int launch_gate_topk(const float* logits, int64_t T, int64_t E, int k, uint32_t* expert,
                     uint16_t* scale, uint32_t* bad_row, cudaStream_t st);

// k_gate_fused.cu: LN + logits + top-k + per-block key histogram
struct GateFusedArgs {
  const uint16_t* x;
  int64_t T, d;
  const uint16_t *g, *b;
  const float* gw32;  // (d/2, gwp, 2) f32 k-pair interleaved, zero-padded experts
  int64_t gwp;
  const uint16_t* gb;
  int64_t E;
  int k;
  const uint8_t* finished;
  uint16_t* xn;
  uint32_t* expert;
  uint16_t* scale;
  uint32_t* blockcnt;  // ceil(T/rows) * (E+1)
  uint32_t* bad_row;
  int rows;            // ln_gate_rows(T, d, E, k)
  uint16_t* out_fin = nullptr;  // non-null: write out[r] = x[r] for finished rows (fused combine)
};
int64_t gate_fused_pitch(int64_t E);  // f32 gate weight pitch (multiple of 8)
// k_ln_gate.cu: LN + logits + top-k + routing-key histogram, one kernel
bool ln_gate_supported(int64_t T, int64_t d, int64_t E, int k);
int ln_gate_rows(int64_t T, int64_t d, int64_t E, int k);  // rows per block (GateFusedArgs::rows)
int launch_ln_gate(const GateFusedArgs& a, cudaStream_t st);
int launch_widen_gate(const uint16_t* gw, int64_t d, int64_t E, int64_t gwp, float* out,
                      cudaStream_t st);
// LN only (the ln_gate kernel's LayerNorm, xn to global + finished-row
// passthrough), for the wide-gate path below
int launch_ln_rows(const GateFusedArgs& a, cudaStream_t st);
// k_gate_tile.cu: wide gates (E = 64 / 128, T*E >= 2^18): logits as a
// register-tiled GEMM over xn + top-k + key histogram per tile of rows
bool gate_tile_supported(int64_t T, int64_t d, int64_t E, int k);
int gate_tile_rows(int64_t T, int64_t E);  // rows per tile (the plan's slots per block / k)
int launch_gate_tile(const GateFusedArgs& a, int tile_rows, cudaStream_t st);

// k_route.cu
struct PlanWork {
  uint32_t* blockcnt;   // nblk * (E+1)
  uint32_t* blockbase;  // nblk * (E+1)
  uint32_t* bad;        // 1 (expert out of range: lowest slot)
  uint32_t* keytot = nullptr;  // E+1 per-key totals (plan_keyscan path)
};
int64_t plan_blocks(int64_t S);
int launch_routing_plan(const uint32_t* expert, const uint8_t* finished, int64_t T, int k,
                        int64_t E, uint32_t* perm, uint32_t* inv, uint32_t* offsets,
                        uint32_t* problems, uint32_t* active, const PlanWork& w,
                        const uint16_t* gather_src, int64_t cols, uint16_t* gather_dst,
                        cudaStream_t st);
int launch_plan_from_counts(const uint32_t* expert, const uint8_t* finished, int64_t T, int k,
                            int64_t E, int64_t spb, const PlanWork& w, uint32_t* perm,
                            uint32_t* inv, uint32_t* offsets, uint32_t* problems,
                            uint32_t* active, const uint16_t* gather_src, int64_t cols,
                            uint16_t* gather_dst, cudaStream_t st);
int launch_permute(const uint16_t* x, int64_t cols, const uint32_t* perm, int64_t S, int k,
                   uint16_t* xp, cudaStream_t st);
int launch_unpermute_scale(const uint16_t* y, int64_t T, int64_t cols, const uint32_t* perm,
                           const uint32_t* active, const uint16_t* scale, uint16_t* out,
                           cudaStream_t st);
int launch_combine(const uint16_t* x, const uint16_t* y, const uint32_t* inv,
                   const uint16_t* scale, const uint8_t* finished, int64_t T, int64_t d, int k,
                   uint16_t* out, cudaStream_t st);
int launch_ep_rank_counts(const uint32_t* offsets, int64_t E, int G, int64_t* counts,
                          cudaStream_t st);

// k_gemm_exact.cu / k_gemm_tc.cu
struct GemmArgs {
  const uint16_t* x;
  int64_t rows, m;
  const uint32_t* problems;
  int64_t np;
  const void* tiled;
  const uint16_t* scales;
  int bits;
  int64_t E, n;
  const uint16_t* bias;
  int relu;
  uint16_t* out;
  uint16_t debias;  // 0x6408 (W4) / 0x6480 (W8), MOE_FAULT_INJECT aware
  int64_t rows_hint;  // expected rows per problem (tile-size choice)
  int second = 0;     // the second GEMM of an FFN pair (MOE_PDL=3: PDL on this launch only)
  // k = 1 combine fused into the epilogue (tcgen05 kernel only): output row r
  // (slot position) goes to token t = cperm[r] as
  //   cout[t] = cx[t] (+) (y_r (*) cscale[t])   (fp16 RN each, = combine_kernel)
  // and `out` is not written.  Null cout: plain output rows.
  const uint16_t* cx = nullptr;
  const uint32_t* cperm = nullptr;
  const uint16_t* cscale = nullptr;
  uint16_t* cout = nullptr;
};
int launch_gemm_exact(const GemmArgs& a, cudaStream_t st);

// k_gemv.cu: decode-sized FAST path (mma.sync over the same weight tiles)
constexpr int64_t kGemvMaxRows = 256;  // routed rows (T*k) up to which the layer uses it
struct GemvWork {
  float* part;       // split-K partials, nsplit * rows * n
  uint32_t* ticket;  // E * ceil(n/128), zero-initialised, self-resetting
  int nsplit;
};
int gemv_splits(int64_t m, int64_t n, double active_experts);
int launch_gemv(const GemmArgs& a, const GemvWork& w, cudaStream_t st);
// both GEMMs of a decode FFN pair in one persistent launch (a2.x == a1.out);
// w1 / w2 need distinct split-K workspaces; ready: E * ceil(a1.n / 128)
// words, ctl: 2 words, both zero-initialised and self-resetting
int launch_gemv_pair(const GemmArgs& a1, const GemmArgs& a2, const GemvWork& w1,
                     const GemvWork& w2, uint32_t* ready, uint32_t* ctl, cudaStream_t st);
bool gemv_pair_supported(int64_t rows, int64_t np, int64_t d, int64_t f, int bits);
// splits whose k range fits the pair kernel's rows buffers (rows: routed rows)
int gemv_pair_splits(int64_t m, int64_t n, double active_experts, int64_t rows);
int launch_gemm_tc(const GemmArgs& a, cudaStream_t st);

}  // namespace moecu
