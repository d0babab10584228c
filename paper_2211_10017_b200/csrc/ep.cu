// ep.cu -- expert parallelism: the MoE layer
// (proj/src/model.cpp:299-349) with its experts sharded over G ranks, one
// process per GPU, the token exchange over NCCL (NVLink / NVSwitch).
//
// Partition: expert e lives on rank e / (E/G) (contiguous slices), every rank
// holds the full gate and its own contiguous range of tokens.  One forward,
// per rank, all on the caller's stream:
//
//   1. route    LN -> gate -> top-k -> plan -> gather (layer_route): the
//               expert-sorted rows are also sorted by owner rank
//   2. counts   ep_counts_kernel: rows per (owner rank, local expert) from the
//               plan offsets; exchanged device-to-device (G x E/G u32 each way)
//   3. one D2H of the sent + received counts (the only host synchronisation:
//               NCCL point-to-point sizes are host arguments)
//   4. dispatch ONE ncclSend per peer (the sorted rows owned by that peer are
//               contiguous) and one ncclRecv per source into a staging buffer
//               ((source, local expert)-major); a segment-copy kernel regroups
//               the rows EXPERT-major for the grouped GEMMs (one message per
//               peer: NCCL point-to-point costs ~5 us per operation, so
//               per-(peer, expert) messages -- E of them -- cost more than the
//               extra on-device copy)
//   5. experts  FFN1 + FFN2 of the local experts over the received rows
//               (layer_ffn: tcgen05 grouped GEMM, or the decode GEMV)
//   6. combine  the inverse segment copy puts the results back in
//               (source, expert) order, one ncclSend per source returns them
//               straight to their sorted positions in the sender's y; then the
//               local residual + gate-scaled un-permute (combine_kernel)
//
// Rows are independent in every kernel, so with the same kernel choices an
// EP forward is bit-identical to the single-GPU layer on the same tokens
// (tests/test_gpu_ep.py).  Two transports share this orchestration: NCCL
// (one local rank per process) and an in-process loopback (all G ranks in one
// process on one device; segments become device-to-device copies) used to
// test G = 2..8 on one GPU.  Only the segment arithmetic is host logic; it is
// exported as the pure function moe_ep_segments (tested on CPU with gloo).
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <type_traits>
#include <vector>

#include "layer.cuh"

// ----------------------------------------------------------------- NCCL (dlopen)
// The library does not link NCCL: the symbols are resolved at first use from
// the libnccl.so.2 already in the process (torch's), else the system one.
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess
constexpr int kNcclUint8 = 1;

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) return r;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    r.ok = sym(r.GetUniqueId, "ncclGetUniqueId") && sym(r.CommInitRank, "ncclCommInitRank") &&
           sym(r.CommDestroy, "ncclCommDestroy") && sym(r.GroupStart, "ncclGroupStart") &&
           sym(r.GroupEnd, "ncclGroupEnd") && sym(r.Send, "ncclSend") &&
           sym(r.Recv, "ncclRecv") && sym(r.GetErrorString, "ncclGetErrorString") &&
           sym(r.GetVersion, "ncclGetVersion");
    return r;
  }();
  return n;
}

int nccl_error(ncclResult_t r, const char* what) {
  const Nccl& n = nccl();
  return moecu::set_error(MOE_ENCCL, "NCCL error %d (%s) at %s", r,
                          n.GetErrorString ? n.GetErrorString(r) : "?", what);
}

#define NCCL_TRY(expr)                                    \
  do {                                                    \
    const ncclResult_t r__ = (expr);                      \
    if (r__ != 0) return nccl_error(r__, #expr);          \
  } while (0)
}  // namespace

// ------------------------------------------------------------------- state
// Per local rank: device + pinned-host exchange state of the last forward.
struct EpRank {
  // device: send counts [G*el] | recv counts [G*el] | problems [el*3] | segments [G*el*3]
  uint32_t* dcnt = nullptr;
  // pinned: send | recv | bad_row, bad_expert | problems [el*3] | segments [G*el*3]
  uint32_t* hcnt = nullptr;
  uint16_t *xr = nullptr;     // received rows, (source, expert)-major; reused for the results
  uint16_t *xe = nullptr, *ye = nullptr;  // received rows (expert-major) and their FFN output
  int64_t cap = 0;            // rows xr / xe / ye hold
  int64_t rows = 0;           // rows received in the last forward
  int nseg = 0;               // non-empty (source, expert) segments of the last forward
  std::vector<int64_t> send_off, recv_dst;
};

struct moe_ep {
  int G = 1, rank = 0;    // world size; this process's rank (NCCL) / 0 (loopback)
  bool loopback = false;  // all G ranks in this process
  ncclComm_t comm = nullptr;
  int64_t el = 0, E = 0;  // bound at the first forward
  std::vector<EpRank> r;  // one per local rank
  ~moe_ep() {
    for (auto& x : r) {
      if (x.dcnt) cudaFree(x.dcnt);
      if (x.hcnt) cudaFreeHost(x.hcnt);
      if (x.xr) cudaFree(x.xr);
      if (x.xe) cudaFree(x.xe);
      if (x.ye) cudaFree(x.ye);
    }
    if (comm && nccl().ok) nccl().CommDestroy(comm);
  }
  int local() const { return loopback ? G : 1; }
  int global_rank(int i) const { return loopback ? i : rank; }
};

namespace moecu {

// send counts per (owner rank, local expert) = plan offsets differences
__global__ void ep_counts_kernel(const uint32_t* __restrict__ offsets, int64_t E,
                                 uint32_t* __restrict__ cnt) {
  for (int64_t e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = offsets[e + 1] - offsets[e];
}

// Row moves between the staging order ((source, expert)-major) and the
// expert-major GEMM order: one CTA per segment {staging row, expert-major
// row, rows}; inverse swaps source and destination.
__global__ void ep_regroup_kernel(const uint32_t* __restrict__ seg, const uint16_t* __restrict__ src,
                                  uint16_t* __restrict__ dst, int64_t d, int inverse) {
  const uint32_t a = seg[3 * blockIdx.x], b = seg[3 * blockIdx.x + 1], nr = seg[3 * blockIdx.x + 2];
  // blockIdx.y splits the segment's rows (large segments over several CTAs)
  const uint32_t r0 = (uint32_t)((uint64_t)nr * blockIdx.y / gridDim.y);
  const uint32_t n = (uint32_t)((uint64_t)nr * (blockIdx.y + 1) / gridDim.y) - r0;
  const int64_t from = (int64_t)(inverse ? b : a) + r0, to = (int64_t)(inverse ? a : b) + r0;
  if (d % 8 == 0) {
    const int64_t q = d / 8, total = (int64_t)n * q;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + from * d);
    uint4* d4 = reinterpret_cast<uint4*>(dst + to * d);
    for (int64_t i = threadIdx.x; i < total; i += blockDim.x) d4[i] = s4[i];
  } else {
    const int64_t total = (int64_t)n * d;
    for (int64_t i = threadIdx.x; i < total; i += blockDim.x) dst[to * d + i] = src[from * d + i];
  }
}

// Sends issued by local rank i and receives posted by local rank i, in
// issue order.  NCCL matches the sends and receives of one rank pair in
// order; the loopback pairs them the same way.
struct Xfer {
  struct Op {
    int peer;
    void* ptr;
    size_t bytes;
  };
  std::vector<std::vector<Op>> send, recv;
  explicit Xfer(int n) : send(n), recv(n) {}
};

static int run_xfer(moe_ep* ep, Xfer& x, cudaStream_t st) {
  if (!ep->loopback) {
    const Nccl& n = nccl();
    NCCL_TRY(n.GroupStart());
    for (auto& o : x.send[0]) NCCL_TRY(n.Send(o.ptr, o.bytes, kNcclUint8, o.peer, ep->comm, st));
    for (auto& o : x.recv[0]) NCCL_TRY(n.Recv(o.ptr, o.bytes, kNcclUint8, o.peer, ep->comm, st));
    NCCL_TRY(n.GroupEnd());
    return MOE_OK;
  }
  // loopback: the k-th send of rank s to rank p lands in the k-th receive
  // of rank p from rank s
  const int G = ep->G;
  for (int s = 0; s < G; ++s)
    for (int p = 0; p < G; ++p) {
      std::vector<const Xfer::Op*> a, b;
      for (auto& o : x.send[s])
        if (o.peer == p) a.push_back(&o);
      for (auto& o : x.recv[p])
        if (o.peer == s) b.push_back(&o);
      if (a.size() != b.size())
        return set_error(MOE_EINVAL, "ep: unmatched exchange %d -> %d", s, p);
      for (size_t i = 0; i < a.size(); ++i) {
        if (a[i]->bytes != b[i]->bytes)
          return set_error(MOE_EINVAL, "ep: exchange size mismatch %d -> %d", s, p);
        MOE_CUDA_TRY(cudaMemcpyAsync(b[i]->ptr, a[i]->ptr, a[i]->bytes, cudaMemcpyDeviceToDevice, st));
      }
    }
  return MOE_OK;
}

static int ep_bind(moe_ep* ep, moe_layer* const* layers) {
  const int n = ep->local();
  for (int i = 0; i < n; ++i) {
    moe_layer* L = layers[i];
    if (!L) return set_error(MOE_EINVAL, "ep: null layer");
    if (L->E % ep->G != 0) return set_error(MOE_EINVAL, "ep: n_experts must be divisible by the world size");
    const int64_t el = L->E / ep->G;
    if (L->El != el || L->e0 != (int64_t)ep->global_rank(i) * el)
      return set_error(MOE_EINVAL, "ep: rank %d's layer must hold experts [%lld, %lld)",
                       ep->global_rank(i), (long long)(ep->global_rank(i) * el),
                       (long long)((ep->global_rank(i) + 1) * el));
    if (ep->E != 0 && ep->E != L->E) return set_error(MOE_EINVAL, "ep: layer shape changed");
  }
  if (ep->E == 0) {
    ep->E = layers[0]->E;
    ep->el = ep->E / ep->G;
    ep->r.resize(n);
    const int64_t G = ep->G, el = ep->el;
    for (auto& x : ep->r) {
      MOE_CUDA_TRY(cudaMalloc(&x.dcnt, (2 * G * el + 3 * el + 3 * G * el) * 4));
      MOE_CUDA_TRY(cudaMallocHost(&x.hcnt, (2 * G * el + 2 + 3 * el + 3 * G * el) * 4));
      x.send_off.resize(G * el);
      x.recv_dst.resize(G * el);
    }
  }
  return MOE_OK;
}

}  // namespace moecu

using namespace moecu;

extern "C" {

int moe_ep_segments(int G, int64_t el, const uint32_t* send_cnt, const uint32_t* recv_cnt,
                    int64_t* send_off, int64_t* recv_dst, uint32_t* problems, int64_t* rows) {
  if (G < 1 || el < 1 || !send_cnt || !recv_cnt)
    return set_error(MOE_EINVAL, "ep: bad segment arguments");
  // send: the plan sorts rows by global expert p*el + j, so the segment of
  // (p, j) starts at the running sum in that order (= plan offsets)
  int64_t acc = 0;
  for (int64_t i = 0; i < (int64_t)G * el; ++i) {
    if (send_off) send_off[i] = acc;
    acc += send_cnt[i];
  }
  // receive: expert-major, sources in rank order inside an expert
  int64_t pos = 0;
  for (int64_t j = 0; j < el; ++j) {
    const int64_t start = pos;
    for (int s = 0; s < G; ++s) {
      if (recv_dst) recv_dst[(int64_t)s * el + j] = pos;
      pos += recv_cnt[(int64_t)s * el + j];
    }
    if (problems) {
      problems[3 * j] = (uint32_t)j;
      problems[3 * j + 1] = (uint32_t)start;
      problems[3 * j + 2] = (uint32_t)pos;
    }
  }
  if (rows) *rows = pos;
  return MOE_OK;
}

int moe_ep_unique_id(uint8_t* id) {
  if (!id) return set_error(MOE_EINVAL, "ep: null id");
  if (!nccl().ok) return set_error(MOE_ENCCL, "ep: libnccl.so.2 not found");
  ncclUniqueId u;
  NCCL_TRY(nccl().GetUniqueId(&u));
  std::memcpy(id, u.internal, sizeof u.internal);
  return MOE_OK;
}

int moe_ep_create(const uint8_t* id, int nranks, int rank, moe_ep** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(MOE_EINVAL, "ep: bad communicator arguments");
  if (!nccl().ok) return set_error(MOE_ENCCL, "ep: libnccl.so.2 not found");
  auto ep = std::make_unique<moe_ep>();
  ep->G = nranks;
  ep->rank = rank;
  ncclUniqueId u;
  std::memcpy(u.internal, id, sizeof u.internal);
  NCCL_TRY(nccl().CommInitRank(&ep->comm, nranks, u, rank));
  *out = ep.release();
  return MOE_OK;
}

int moe_ep_create_loopback(int nranks, moe_ep** out) {
  if (!out || nranks < 1) return set_error(MOE_EINVAL, "ep: bad loopback arguments");
  auto ep = std::make_unique<moe_ep>();
  ep->G = nranks;
  ep->loopback = true;
  *out = ep.release();
  return MOE_OK;
}

int moe_ep_destroy(moe_ep* ep) {
  delete ep;
  return MOE_OK;
}

int moe_ep_world(const moe_ep* ep, int* nranks, int* rank, int* local_ranks) {
  if (!ep) return set_error(MOE_EINVAL, "ep: null");
  if (nranks) *nranks = ep->G;
  if (rank) *rank = ep->rank;
  if (local_ranks) *local_ranks = ep->local();
  return MOE_OK;
}

int moe_ep_forward(moe_ep* ep, moe_layer* const* layers, const uint16_t* const* x,
                   const uint8_t* const* finished, const int64_t* T, int k, int mode,
                   uint16_t* const* out, moe_stream_t stream) {
  if (!ep || !layers || !x || !T || !out) return set_error(MOE_EINVAL, "ep: null argument");
  TRY(ep_bind(ep, layers));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n = ep->local(), G = ep->G;
  const int64_t el = ep->el, E = ep->E, d = layers[0]->d;
  if (k < 1 || k > E) return set_error(MOE_EINVAL, "moe_ffn: k must be in [1, n_experts]");
  for (int i = 0; i < n; ++i)
    if (T[i] < 0) return set_error(MOE_EINVAL, "moe_ffn: negative row count");
  // 1. route + 2. counts (a rank without tokens still serves its experts)
  for (int i = 0; i < n; ++i) {
    moe_layer* L = layers[i];
    TRY(layer_reserve(L, std::max<int64_t>(T[i], 1), k));
    if (T[i] == 0) {
      MOE_CUDA_TRY(cudaMemsetAsync(ep->r[i].dcnt, 0, (size_t)G * el * 4, st));
      MOE_CUDA_TRY(cudaMemsetAsync(L->bad_row, 0xFF, 8, st));
      continue;
    }
    Marks mark(L, st, false);
    TRY(layer_route(L, x[i], finished ? finished[i] : nullptr, T[i], k, st, mark));
    ep_counts_kernel<<<1, 256, 0, st>>>(L->offsets, E, ep->r[i].dcnt);
    note_launch();
    TRY(check_launch("ep_counts"));
  }
  {
    Xfer xc(n);
    for (int i = 0; i < n; ++i)
      for (int p = 0; p < G; ++p) {
        xc.send[i].push_back({p, ep->r[i].dcnt + p * el, (size_t)el * 4});
        xc.recv[i].push_back({p, ep->r[i].dcnt + G * el + p * el, (size_t)el * 4});
      }
    TRY(run_xfer(ep, xc, st));
  }
  // 3. counts -> host (with the gate / plan status words)
  for (int i = 0; i < n; ++i) {
    EpRank& R = ep->r[i];
    MOE_CUDA_TRY(cudaMemcpyAsync(R.hcnt, R.dcnt, 2 * G * el * 4, cudaMemcpyDeviceToHost, st));
    MOE_CUDA_TRY(cudaMemcpyAsync(R.hcnt + 2 * G * el, layers[i]->bad_row, 8, cudaMemcpyDeviceToHost, st));
  }
  MOE_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i < n; ++i) {
    EpRank& R = ep->r[i];
    uint32_t* prob = R.hcnt + 2 * G * el + 2;
    uint32_t* segt = prob + 3 * el;
    TRY(moe_ep_segments(G, el, R.hcnt, R.hcnt + G * el, R.send_off.data(), R.recv_dst.data(),
                        prob, &R.rows));
    // staging order: source-major, experts in order inside a source
    const uint32_t* rc = R.hcnt + G * el;
    int64_t pos = 0;
    R.nseg = 0;
    for (int s2 = 0; s2 < G; ++s2)
      for (int64_t j = 0; j < el; ++j) {
        const uint32_t c = rc[s2 * el + j];
        if (c == 0) continue;
        segt[3 * R.nseg] = (uint32_t)pos;
        segt[3 * R.nseg + 1] = (uint32_t)R.recv_dst[s2 * el + j];
        segt[3 * R.nseg + 2] = c;
        ++R.nseg;
        pos += c;
      }
    if (R.rows > R.cap) {  // grow the receive buffers (rows of the exchange)
      for (uint16_t** b : {&R.xr, &R.xe, &R.ye})
        if (*b) {
          cudaFree(*b);
          *b = nullptr;
        }
      const int64_t cap = R.rows + R.rows / 4 + 64;
      MOE_CUDA_TRY(cudaMalloc(&R.xr, cap * d * 2));
      MOE_CUDA_TRY(cudaMalloc(&R.xe, cap * d * 2));
      MOE_CUDA_TRY(cudaMalloc(&R.ye, cap * d * 2));
      R.cap = cap;
    }
    TRY(layer_grow_hidden(layers[i], std::max<int64_t>(R.rows, 1)));
    MOE_CUDA_TRY(cudaMemcpyAsync(R.dcnt + 2 * G * el, prob, (3 * el + 3 * (int64_t)R.nseg) * 4,
                                 cudaMemcpyHostToDevice, st));
  }
  // one message per (rank pair): rows [send_off[p*el], +sum_j sent[p][j]) of
  // the sorted buffer <-> staging rows [base_s, +sum_j recv[s][j])
  const size_t rb = (size_t)d * 2;
  auto pairs = [&](bool forward) {
    Xfer xd(n);
    for (int i = 0; i < n; ++i) {
      EpRank& R = ep->r[i];
      const uint32_t *sc = R.hcnt, *rc = R.hcnt + G * el;
      uint16_t* sorted = forward ? layers[i]->xp : layers[i]->y;
      for (int p = 0; p < G; ++p) {
        int64_t c = 0;
        for (int64_t j = 0; j < el; ++j) c += sc[p * el + j];
        if (c) (forward ? xd.send : xd.recv)[i].push_back({p, sorted + R.send_off[p * el] * d, c * rb});
      }
      int64_t base = 0;
      for (int s2 = 0; s2 < G; ++s2) {
        int64_t c = 0;
        for (int64_t j = 0; j < el; ++j) c += rc[s2 * el + j];
        if (c) (forward ? xd.recv : xd.send)[i].push_back({s2, R.xr + base * d, c * rb});
        base += c;
      }
    }
    return xd;
  };
  auto regroup = [&](int i, int inverse) -> int {
    EpRank& R = ep->r[i];
    if (R.nseg == 0) return MOE_OK;
    // ~2 CTAs per SM over all segments
    const int ys = (int)std::max<int64_t>(1, std::min<int64_t>(32, (2 * sm_count() + R.nseg - 1) / R.nseg));
    ep_regroup_kernel<<<dim3(R.nseg, ys), 256, 0, st>>>(R.dcnt + 2 * G * el + 3 * el, inverse ? R.ye : R.xr,
                                              inverse ? R.xr : R.xe, d, inverse);
    note_launch();
    return check_launch("ep_regroup");
  };
  // 4. dispatch + regroup
  {
    Xfer xd = pairs(true);
    TRY(run_xfer(ep, xd, st));
  }
  for (int i = 0; i < n; ++i) TRY(regroup(i, 0));
  // 5. local experts
  for (int i = 0; i < n; ++i) {
    EpRank& R = ep->r[i];
    if (R.rows == 0) continue;
    moe_layer* L = layers[i];
    Marks mark(L, st, false);
    TRY(layer_ffn(L, R.xe, R.rows, R.dcnt + 2 * G * el, el, mode, L->ep_h, R.ye, st, mark));
  }
  // 6. results back in staging order, one message per rank pair, then residual
  for (int i = 0; i < n; ++i) TRY(regroup(i, 1));
  {
    Xfer xb = pairs(false);
    TRY(run_xfer(ep, xb, st));
  }
  for (int i = 0; i < n; ++i) {
    moe_layer* L = layers[i];
    if (T[i] == 0) continue;
    TRY(launch_combine(x[i], L->y, L->inv, L->scale, finished ? finished[i] : nullptr, T[i], d, k,
                       out[i], st));
  }
  // the gate / plan status of this forward (read with the counts; reported
  // only now so that every rank completes the collective sequence)
  for (int i = 0; i < n; ++i) {
    const uint32_t* h = ep->r[i].hcnt + 2 * G * el;
    if (h[0] != 0xFFFFFFFFu) return set_error(MOE_EINVAL, "gate_top1: non-finite logit at row %u", h[0]);
    if (h[1] != 0xFFFFFFFFu) return set_error(MOE_EINVAL, "build_routing_plan: expert out of range");
  }
  return MOE_OK;
}

int moe_ep_counts(const moe_ep* ep, int local, uint32_t* send_cnt, uint32_t* recv_cnt,
                  int64_t* recv_rows) {
  if (!ep || local < 0 || local >= (int)ep->r.size())
    return set_error(MOE_EINVAL, "ep: no forward on this local rank yet");
  const EpRank& R = ep->r[local];
  const int64_t n = (int64_t)ep->G * ep->el;
  if (send_cnt) std::memcpy(send_cnt, R.hcnt, n * 4);
  if (recv_cnt) std::memcpy(recv_cnt, R.hcnt + n, n * 4);
  if (recv_rows) *recv_rows = R.rows;
  return MOE_OK;
}

}  // extern "C"
