/* include/moe_cuda.h -- C-ABI of libmoe_cuda.so, the B200 (sm_100a) MoE-layer
 * hot path.
 *
 * Plain pointers, int64 sizes, cudaStream_t passed as void*, int status.
 * Every *device* argument is a device pointer unless the name ends in _host.
 * No torch types.  Status codes:
 *   MOE_OK 0, MOE_EINVAL 1 (argument / data validation; message mirrors the
 *   reference's std::invalid_argument text), MOE_ECUDA 2, MOE_ENCCL 3,
 *   MOE_ERANGE 4 (index out of range, reference std::out_of_range),
 *   MOE_EIO 5 (checkpoint file errors, reference std::runtime_error).
 * moe_cuda_last_error() returns the thread-local message of the last failure.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).  The C++ drop-in
 * (include/moeinfer/*.hpp, libmoeinfer_b200.so) and the Python module
 * (_moeinfer) are thin layers over these.
 *
 * Numerics modes:
 *   MOE_MODE_EXACT -- CUDA-core kernels that reproduce the reference bit for
 *                     bit (k-sequential f32 accumulation, RN16(q*s) weights).
 *   MOE_MODE_FAST  -- tensor-core grouped GEMM (f32 accumulate, per-channel
 *                     scale applied in the epilogue): tcgen05/TMEM tiles for
 *                     prefill-sized batches, the K5 dequant-GEMV (mma.sync
 *                     over the same weight tiles) when a layer routes at most
 *                     256 rows; gating, routing and combine stay bit-exact.
 */
#ifndef MOE_CUDA_H
#define MOE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_OK 0
#define MOE_EINVAL 1
#define MOE_ECUDA 2
#define MOE_ENCCL 3
#define MOE_ERANGE 4
#define MOE_EIO 5 /* checkpoint file errors (reference std::runtime_error "checkpoint: ...") */

#define MOE_MODE_EXACT 0
#define MOE_MODE_FAST 1
#define MOE_MODE_GEMV 2 /* moe_grouped_gemm only: force the decode (K5) kernel */

/* weight formats: fp16 experts, or reference-quantized codes */
#define MOE_W16 16
#define MOE_W8 8
#define MOE_W4 4

typedef void* moe_stream_t; /* a cudaStream_t */

const char* moe_cuda_last_error(void);
/* library / device info: 0 ok; fills sm count and compute capability */
int moe_cuda_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* Number of this library's kernels launched since load (all entry points).
 * bench.py reports the delta as gpu_launches. */
uint64_t moe_cuda_launch_count(void);

/* Memory / stream plumbing for host-side callers that do not link the CUDA
 * runtime themselves (the C++ drop-in, ctypes).  kind: 0 H2D, 1 D2H, 2 D2D. */
int moe_cuda_malloc(void** ptr, size_t bytes);
int moe_cuda_free(void* ptr);
int moe_cuda_host_alloc(void** ptr, size_t bytes); /* pinned */
/* Write-combined pinned host memory for streaming INPUTS (host writes,
 * device reads): measured on the B200 boxes 41.8 GB/s H2D (35.6 for default
 * pinned memory, 9.1 for a framework's registered pinned buffers), and 32.8 GB/s each way with a
 * concurrent D2H (12.4 for default pinned).  Host reads of it are slow. */
int moe_cuda_host_alloc_wc(void** p, size_t bytes);
int moe_cuda_host_free(void* ptr);
int moe_cuda_memcpy(void* dst, const void* src, size_t bytes, int kind, moe_stream_t stream);
int moe_cuda_memset(void* dst, int value, size_t bytes, moe_stream_t stream);
int moe_cuda_sync(moe_stream_t stream);

/* Debias constants of the magic I2F path (include/moeinfer/dequant.hpp:35-36,
 * src/dequant.cpp:45-53).  Initialised from MOE_FAULT_INJECT exactly like
 * src/dequant.cpp:12-30 ("i2f4" -> 0x6409 for u4, other non-empty -> 0x6481
 * for u8); tests may override. */
void moe_cuda_debias(uint16_t* u8c, uint16_t* u4c);
void moe_cuda_set_debias(uint16_t u8c, uint16_t u4c);

/* ---- K1: quantizer -- replaces moe::quantize (include/moeinfer/quantize.hpp:56-57,
 * src/quantize.cpp:74-122).  w: (e,m,n) fp16; packed: reference layout
 * (e*m*n bytes for 8-bit, e*m*n/2 interleaved nibbles for 4-bit);
 * scales: (e,n) fp16.  Synchronises the stream (validation result). */
int moe_quantize(const uint16_t* w, int64_t e, int64_t m, int64_t n, int bits,
                 uint8_t* packed, uint16_t* scales, moe_stream_t stream);

/* pack_int4_interleaved / unpack_int4_interleaved
 * (include/moeinfer/quantize.hpp:62-65, src/quantize.cpp:34-72). */
int moe_pack_int4(const uint8_t* values, int64_t count, uint8_t* packed,
                  moe_stream_t stream);
int moe_unpack_int4(const uint8_t* packed, int64_t count, uint8_t* values,
                    moe_stream_t stream);

/* ---- K0: dequantizer -- replaces dequantize_naive / dequantize_fast
 * (include/moeinfer/dequant.hpp:73-74, src/dequant.cpp:55-112). */
int moe_dequantize(const uint8_t* packed, const uint16_t* scales, int64_t e,
                   int64_t m, int64_t n, int bits, int fast, uint16_t* out,
                   moe_stream_t stream);

/* ---- device weight tiles (new) ----
 * Re-tiles one expert tensor (e,m,n) from the reference layout into the
 * GEMM layout: [e][n/128][m/64][block], block = 128 output columns x 64
 * inputs, each column's 64 codes contiguous (16-byte chunks).  Sizes are
 * padded to 128 (n) and 64 (m) with zero codes. */
int64_t moe_tiled_bytes(int64_t e, int64_t m, int64_t n, int bits);
int moe_tile_weights(const void* src, int64_t e, int64_t m, int64_t n, int bits,
                     void* tiled, moe_stream_t stream);

/* ---- K2: gating ----
 * layer_norm (src/model.cpp:175-205); gate_logits_f32 (src/model.cpp:273-297);
 * gate_top1 (src/routing.cpp:11-41) generalised to top-k. */
int moe_layer_norm(const uint16_t* x, int64_t T, int64_t d, const uint16_t* gamma,
                   const uint16_t* beta, uint16_t* out, moe_stream_t stream);
int moe_gate_logits(const uint16_t* xn, int64_t T, int64_t d, const uint16_t* gw,
                    const uint16_t* gb, int64_t E, float* logits, moe_stream_t stream);
/* expert, scale: (T,k).  Non-finite logits are reported (lowest bad row) and
 * the call synchronises to raise MOE_EINVAL with the reference's message. */
int moe_gate_topk(const float* logits, int64_t T, int64_t E, int k, uint32_t* expert,
                  uint16_t* scale, moe_stream_t stream);

/* ---- K3: routing plan -- build_routing_plan (src/routing.cpp:43-87) over
 * S = T*k slots.  finished may be NULL (no finished rows).  offsets: E+1.
 * problems (may be NULL): E triples (expert, row_begin, row_end).
 * active (device u32, may be NULL).  Validates expert < E (synchronises). */
int moe_routing_plan(const uint32_t* expert, const uint8_t* finished, int64_t T,
                     int k, int64_t E, uint32_t* perm, uint32_t* inv,
                     uint32_t* offsets, uint32_t* problems, uint32_t* active,
                     moe_stream_t stream);
/* permute_rows (src/routing.cpp:89-97): xp[p] = x[perm[p]/k]. */
int moe_permute_rows(const uint16_t* x, int64_t cols, const uint32_t* perm,
                     int64_t S, int k, uint16_t* xp, moe_stream_t stream);
/* unpermute_and_scale (src/routing.cpp:99-116), top-1 plan. */
int moe_unpermute_scale(const uint16_t* y, int64_t T, int64_t cols,
                        const uint32_t* perm, const uint32_t* active,
                        const uint16_t* scale, uint16_t* out, moe_stream_t stream);
/* K6 combine: out[r] = finished ? x[r] : fold_s half_add(., half_mul(y[inv[r*k+s]], scale[r,s]))
 * (src/model.cpp:334-346 + src/routing.cpp:106-114, slot-ordered for k>1). */
int moe_combine(const uint16_t* x, const uint16_t* y, const uint32_t* inv,
                const uint16_t* scale, const uint8_t* finished, int64_t T,
                int64_t d, int k, uint16_t* out, moe_stream_t stream);

/* ---- K4/K5: grouped expert GEMM -- grouped_gemm_f16 / grouped_gemm_quant
 * (include/moeinfer/grouped_gemm.hpp:65-82, src/grouped_gemm.cpp:140-214).
 * x: (rows, m) fp16 row-major (expert-sorted).  problems: np triples on the
 * device.  tiled: moe_tile_weights output; scales (E,n) fp16 (NULL for W16).
 * bias (E,n) fp16.  out (rows, n): rows outside every problem are left
 * untouched (callers zero them when the reference semantics need it). */
int moe_grouped_gemm(const uint16_t* x, int64_t rows, int64_t m,
                     const uint32_t* problems, int64_t np, const void* tiled,
                     const uint16_t* scales, int bits, int64_t E, int64_t n,
                     const uint16_t* bias, int relu, int mode, uint16_t* out,
                     moe_stream_t stream);

/* ---- whole MoE layer -- replaces moe::moe_ffn_forward
 * (include/moeinfer/model.hpp:154-156, src/model.cpp:299-349) with a
 * device-resident layer object (weights uploaded and tiled once). */
typedef struct moe_layer moe_layer;

typedef struct {
  int64_t d, f, E;
  int bits;                       /* 16, 8 or 4 */
  /* host pointers, reference layouts (model.hpp:73-84) */
  const uint16_t *ln_g, *ln_b;    /* d */
  const uint16_t *gate_w;         /* (d, E) */
  const uint16_t *gate_b;         /* E */
  const uint16_t *b1, *b2;        /* (E, f), (E, d) */
  const uint16_t *w1, *w2;        /* bits 16: (E,d,f), (E,f,d) */
  const uint8_t *q1, *q2;         /* bits 8/4: quantize() payloads */
  const uint16_t *s1, *s2;        /* (E,f), (E,d) scales */
  /* expert parallelism: when e_count > 0 the expert tensors above (w/q, s,
   * b1, b2) hold only experts [e_begin, e_begin + e_count); the gate still
   * covers all E.  0 = every expert (single-GPU layer). */
  int64_t e_begin, e_count;
} moe_layer_desc;

int moe_layer_create(const moe_layer_desc* desc, moe_layer** out);
/* Same, with every pointer in desc a DEVICE pointer (e.g. quantized on the
 * GPU by moe_quantize); weights are still copied/tiled into the layer. */
int moe_layer_create_device(const moe_layer_desc* desc, moe_layer** out);
int moe_layer_destroy(moe_layer* L);
/* Device-resident forward: x, finished (nullable), out on the device.
 * Graph-capturable (no host synchronisation, no allocation once the
 * workspace for (T,k) exists -- call moe_layer_reserve first).
 * Non-finite gate logits are flagged on the device; see moe_layer_status. */
int moe_layer_reserve(moe_layer* L, int64_t T, int k);
int moe_layer_forward(moe_layer* L, const uint16_t* x, const uint8_t* finished,
                      int64_t T, int k, int mode, uint16_t* out, moe_stream_t stream);
/* Same as moe_layer_forward, through a CUDA graph: the launch sequence for
 * this exact argument set (pointers, T, k, mode) is captured once and
 * replayed on later calls (no per-kernel launch cost).  Any stream, including
 * the legacy default stream. */
int moe_layer_forward_graph(moe_layer* L, const uint16_t* x, const uint8_t* finished,
                            int64_t T, int k, int mode, uint16_t* out, moe_stream_t stream);
/* Host-buffer forward (the drop-in / e2e path): copies x and finished in,
 * runs, copies out back, synchronises, and raises validation errors.  With
 * pinned host buffers the whole sequence (H2D, kernels, D2H, status
 * readback) is one cached CUDA graph. */
int moe_layer_forward_host(moe_layer* L, const uint16_t* x_host,
                           const uint8_t* finished_host, int64_t T, int k, int mode,
                           uint16_t* out_host, moe_stream_t stream);
/* Expert-parallel building blocks (orchestrated over NCCL by
 * paper_2211_10017_b200/ep.py).  route: stages LN..gather of the layer into
 * its workspace (expert-sorted rows at *xp, plan via moe_layer_routing).
 * experts: FFN1 (ReLU) + FFN2 of the layer's LOCAL experts over `rows`
 * expert-sorted rows (problems: np device triples, expert ids local).
 * combine: residual + gate-scaled un-permute of y (sorted order) using the
 * last route's plan. */
int moe_layer_route(moe_layer* L, const uint16_t* x, const uint8_t* finished, int64_t T, int k,
                    moe_stream_t stream);
int moe_layer_buffers(moe_layer* L, const uint16_t** xp, uint16_t** y);
/* Re-run only FFN1 + FFN2 over the last forward's routed rows (kernel timing:
 * bench.py captures back-to-back calls in a graph between two events). */
int moe_layer_ffn(moe_layer* L, int mode, moe_stream_t stream);
int moe_layer_experts(moe_layer* L, const uint16_t* xin, int64_t rows, const uint32_t* problems,
                      int64_t np, int mode, uint16_t* out, moe_stream_t stream);
int moe_layer_combine(moe_layer* L, const uint16_t* x, const uint16_t* y,
                      const uint8_t* finished, int64_t T, int k, uint16_t* out,
                      moe_stream_t stream);
/* Synchronises and reports device-side validation (non-finite logits). */
int moe_layer_status(moe_layer* L, moe_stream_t stream);
/* Routing diagnostics of the last forward (device pointers owned by L):
 * expert/scale (T,k), perm/inv (T*k), offsets (E+1), active (1). */
int moe_layer_routing(moe_layer* L, const uint32_t** expert, const uint16_t** scale,
                      const uint32_t** perm, const uint32_t** inv,
                      const uint32_t** offsets, const uint32_t** active);
/* Stage timing with CUDA events recorded on the forward's own stream
 * (bench.py's roofline).  enable = 1 records only the grouped-GEMM
 * boundaries (ffn1, ffn2), enable = 2 every stage, 0 stops; enabling resets
 * the record (up to 512 forwards; a graph replays its captured slot).  read
 * returns the summed milliseconds of the 7 stages {gate (fused LN+logits+
 * top-k, or layer_norm), gate_logits, gate_topk, routing_plan+gather, ffn1,
 * ffn2, combine} (unrecorded stages read 0) over the recorded forwards. */
int moe_layer_profile(moe_layer* L, int enable);
int moe_layer_profile_read(moe_layer* L, double* stage_ms, int* forwards);
/* Analytic traffic of the last forward, reference accounting
 * (src/grouped_gemm.cpp:155-160, 201-211; src/model.cpp:303-347):
 * out6 = {expert.weight, expert.activation, expert.written,
 *         other.weight, other.activation, other.written}.  Synchronises. */
int moe_layer_traffic(moe_layer* L, uint64_t* out6, moe_stream_t stream);

/* ---- expert-parallel helpers (new) ----
 * Per-destination-rank slot counts for EP dispatch: experts are owned in
 * contiguous blocks of E/G; counts[g] = #active slots routed to rank g. */
int moe_ep_rank_counts(const uint32_t* offsets, int64_t E, int G, int64_t* counts,
                       moe_stream_t stream);

/* ---- expert parallelism (new; csrc/ep.cu) ----
 * The layer of proj/src/model.cpp:299-349 with its experts sharded over G
 * ranks: rank g's layer holds experts [g*E/G, (g+1)*E/G) (moe_layer_desc
 * e_begin / e_count) and the full gate; each rank brings its own tokens.
 * Transport: NCCL point-to-point (ncclGroupStart + ncclSend/ncclRecv per
 * (peer, local expert) segment), one process per GPU; or an in-process
 * loopback of G ranks on one device (tests).  NCCL is resolved at run time
 * from the process's libnccl.so.2 (status MOE_ENCCL if absent). */
typedef struct moe_ep moe_ep;
#define MOE_EP_ID_BYTES 128
/* ncclGetUniqueId on the root rank; broadcast the bytes to every rank */
int moe_ep_unique_id(uint8_t* id);
/* ncclCommInitRank: a communicator of nranks processes, this one = rank
 * (call with the CUDA device of this rank current) */
int moe_ep_create(const uint8_t* id, int nranks, int rank, moe_ep** out);
/* all nranks ranks held by this process (device-to-device copies) */
int moe_ep_create_loopback(int nranks, moe_ep** out);
int moe_ep_destroy(moe_ep* ep);
int moe_ep_world(const moe_ep* ep, int* nranks, int* rank, int* local_ranks);
/* One EP layer forward.  Arrays hold one entry per LOCAL rank (1 for an
 * NCCL communicator, nranks for loopback): that rank's layer, its T[i]
 * tokens x[i] (device, T x d fp16), finished flags (finished may be NULL, or
 * entries NULL) and its output rows out[i].  One host synchronisation per
 * call (the exchanged counts size the NCCL transfers); routing status
 * (non-finite logits) is reported after the collective sequence completes. */
int moe_ep_forward(moe_ep* ep, moe_layer* const* layers, const uint16_t* const* x,
                   const uint8_t* const* finished, const int64_t* T, int k, int mode,
                   uint16_t* const* out, moe_stream_t stream);
/* Counts of the last forward on local rank `local`: rows sent to (peer p,
 * local expert j) at [p*el + j], rows received from (source s, j), total
 * received rows (expert-capacity bookkeeping across ranks). */
int moe_ep_counts(const moe_ep* ep, int local, uint32_t* send_cnt, uint32_t* recv_cnt,
                  int64_t* recv_rows);
/* Pure host arithmetic of the exchange (no device needed): from the sent and
 * received counts [G*el], the sorted-buffer offset of each sent segment,
 * the expert-major destination row of each received segment, the local
 * grouped-GEMM problems (el x {expert, row_begin, row_end}) and the rows
 * received. */
int moe_ep_segments(int G, int64_t el, const uint32_t* send_cnt, const uint32_t* recv_cnt,
                    int64_t* send_off, int64_t* recv_dst, uint32_t* problems, int64_t* rows);

/* ---- expert-capacity bookkeeping (north_star item 1; new) ----
 * Load report of the layer's last routed forward, computed on the device
 * (no host sync, graph-capturable) into `report` (device, E + 8 u32):
 *   report[0..E)  rows routed to each expert (live slots; finished excluded)
 *   report[E+0]   capacity  = ceil(capacity_factor * live_slots / E)
 *   report[E+1]   max expert load
 *   report[E+2]   live slots (T*k minus finished)
 *   report[E+3]   experts over capacity
 *   report[E+4]   overflow rows = sum max(0, load - capacity)
 *   report[E+5]   active (non-empty) experts
 * Nothing is dropped: the reference routes every live slot (routing.cpp:55-71);
 * the report states what a capacity-bounded dispatch would have to drop. */
int moe_layer_load_report(moe_layer* L, float capacity_factor, uint32_t* report,
                          moe_stream_t stream);

/* ---- decode with batch pruning (new; csrc/decode.cu) ----
 * The MoE blocks of beam-search decoding (proj/src/decode.cpp:104-345): for
 * every step s < steps and every block l < n_layers, one layer forward over
 * the step's rows (x_steps[s], steps x rows x d device), block l's output
 * feeding block l+1, the last block's output written to out_steps[s]; the
 * finished mask of step s (finished_steps[s], steps x rows, may be NULL) is
 * routed iff prune (decode.cpp:167-169, 216): finished rows leave the expert
 * workload and pass through bit for bit.  work: rows x d device scratch.  One
 * stream, no host synchronisation (graph-capturable). */
int moe_decode_run(moe_layer* const* layers, int n_layers, const uint16_t* x_steps,
                   const uint8_t* finished_steps, int steps, int64_t rows, int k, int mode,
                   int prune, uint16_t* out_steps, uint16_t* work, moe_stream_t stream);

/* ---- .moec checkpoint -> device layers (new; csrc/moec.cu) ----
 * Parses the reference checkpoint format (proj/src/checkpoint.cpp:35-446:
 * magic, version, config, precision, FNV-1a checksum, every record in the
 * reference's order, same "checkpoint: ..." messages, status MOE_EIO) and,
 * if create_layers, builds one device layer per MoE block (enc.i.ffn /
 * dec.i.ffn, i % moe_every == 0) straight from the file's int4 / int8 / fp16
 * payloads -- no host dequantization; re-tiled on the device. */
typedef struct moe_moec moe_moec;
int moe_moec_load(const char* path, int create_layers, moe_moec** out);
/* cfg9: d_model, d_ffn, n_enc_layers, n_dec_layers, n_experts, n_heads,
 * vocab_size, moe_every, max_seq_len; precision 0 f16, 1 int8, 2 int4 */
int moe_moec_info(const moe_moec* m, uint32_t* cfg9, int* precision, int* n_moe_blocks);
/* i-th MoE block in file order: its layer (NULL unless created) and name */
int moe_moec_block(const moe_moec* m, int i, moe_layer** layer, char* name, size_t name_len);
int moe_moec_destroy(moe_moec* m);

/* ---- encoder_forward on the device (new; csrc/encoder.cu) ----
 * proj/src/model.cpp:351-398 over a checkpoint loaded with create_layers:
 * embeddings, every encoder layer (attention: LN, Q/K/V/O projections,
 * per-sentence softmax attention; then the MoE block or the dense FFN),
 * final LayerNorm.  tokens: HOST int32 [batch][len] (the reference's range
 * checks and messages); out: device (batch * len, d_model) fp16.  EXACT
 * mode is bit-identical to encoder_forward; FAST runs the projections and
 * experts on the tensor cores (layer tolerance).  Synchronises once (token
 * range check). */
/* A synthetic .moec in the reference's format (random fp16 tensors, random
 * int4/int8 codes with per-column scales) for benchmarks at model sizes no
 * fixture covers (C4: 24 encoder layers, E = 64, d 1024 / 4096).  Host-only. */
int moe_moec_write_synthetic(const char* path, const uint32_t* cfg9, int bits, uint64_t seed);
int moe_encoder_forward(moe_moec* m, const int32_t* tokens, int64_t batch, int64_t len, int mode,
                        uint16_t* out, moe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
