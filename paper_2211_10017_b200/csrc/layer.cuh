// layer.cuh -- the device-resident MoE layer object shared by the C-ABI
// (abi.cu: single-GPU forward) and expert parallelism (ep.cu).
#pragma once

#include <vector>

#include "kernels.cuh"

struct moe_layer {
  int64_t d = 0, f = 0, E = 0;
  int64_t El = 0, e0 = 0;  // experts whose FFN weights live here: [e0, e0 + El)
  int bits = 16;
  // weights (device)
  uint16_t *ln_g = nullptr, *ln_b = nullptr, *gw = nullptr, *gb = nullptr;
  uint16_t *b1 = nullptr, *b2 = nullptr, *s1 = nullptr, *s2 = nullptr;
  void *w1t = nullptr, *w2t = nullptr;
  float* gw32 = nullptr;  // gate weights widened to f32, (d, gwp) (fused gate kernel)
  int64_t gwp = 0;
  // workspace, sized for (cap_S slots, cap_T rows)
  int64_t cap_T = 0, cap_S = 0;
  uint16_t *xn = nullptr, *xp = nullptr, *h = nullptr, *y = nullptr;
  float* logits = nullptr;
  uint32_t *expert = nullptr, *perm = nullptr, *inv = nullptr, *offsets = nullptr,
           *problems = nullptr, *active = nullptr, *bad_row = nullptr;
  uint16_t* scale = nullptr;
  uint32_t *blockcnt = nullptr, *blockbase = nullptr, *bad_expert = nullptr, *keytot = nullptr;
  // EP: hidden activations of rows received from peers
  uint16_t* ep_h = nullptr;
  int64_t ep_cap = 0;
  // decode GEMV split-K workspace (routed rows <= kGemvMaxRows)
  float* gv_part = nullptr;
  uint32_t* gv_ticket = nullptr;
  // host-path staging
  uint16_t *dx = nullptr, *dout = nullptr;
  uint8_t* dfin = nullptr;
  int64_t last_T = 0;
  int last_k = 1;
  std::vector<void*> allocs;
  // stage profiling (moe_layer_profile): kStages+1 events per forward
  static constexpr int kStages = 7, kProfCap = 512;
  bool prof = false;
  int prof_level = 0;
  int prof_n = 0;
  std::vector<cudaEvent_t> ev;
  // CUDA-graph cache (moe_layer_forward_graph / pinned-buffer host path):
  // the launch sequence of one argument set, captured once, replayed after.
  struct GraphKey {
    const void *x = nullptr, *fin = nullptr, *out = nullptr;
    int64_t T = 0;
    int k = 0, mode = -1, host = 0, prof = 0;
    bool operator==(const GraphKey& o) const {
      return x == o.x && fin == o.fin && out == o.out && T == o.T && k == o.k && mode == o.mode &&
             host == o.host && prof == o.prof;
    }
  };
  struct Graph {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    uint64_t nlaunch = 0;  // kernels in the graph (moe_cuda_launch_count on replay)
  };
  std::vector<Graph> graphs;  // small LRU-less cache
  cudaStream_t cap_stream = nullptr;
  uint32_t* hstatus = nullptr;  // pinned: (bad_row, bad_expert) per chunk of the last host-path forward
  // chunked host path: copy-in / copy-out streams forked from the capture
  // stream, fork/join events, per-chunk status words (device)
  cudaStream_t io_in = nullptr, io_out = nullptr;
  std::vector<cudaEvent_t> io_ev;
  uint32_t* dstatus = nullptr;
  static constexpr int kMaxChunks = 8;

  void drop_graphs() {
    for (auto& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  ~moe_layer() {
    drop_graphs();
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (io_in) cudaStreamDestroy(io_in);
    if (io_out) cudaStreamDestroy(io_out);
    for (cudaEvent_t e : io_ev) cudaEventDestroy(e);
    if (hstatus) cudaFreeHost(hstatus);
    for (void* p : allocs) cudaFree(p);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
  template <class T>
  int alloc(T** p, size_t bytes) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
    if (e != cudaSuccess) return moecu::set_cuda_error(e, "layer alloc");
    allocs.push_back(q);
    *p = static_cast<T*>(q);
    return MOE_OK;
  }
  void release(void* p) {
    for (auto& q : allocs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
};

// Stage-event recorder of one forward (profiling only): ev[slot*(kStages+1)+i]
// before stage i.  Inside a graph capture only an *external* record becomes a
// real event-record node (readable after each replay).  Level 1 records only
// the GEMM boundaries (marks 4..6): every event node costs ~2-3 us of pipeline
// drain, so the cheap level is the one used for kernel timing.
struct Marks {
  moe_layer* L;
  cudaStream_t st;
  cudaEvent_t* evs = nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  int stage = 0;
  Marks(moe_layer* l, cudaStream_t s, bool on) : L(l), st(s) {
    if (on && L->prof && L->prof_n < moe_layer::kProfCap) {
      evs = &L->ev[(size_t)L->prof_n * (moe_layer::kStages + 1)];
      cudaStreamIsCapturing(st, &cap);
    }
  }
  int operator()() {
    if (evs && (L->prof_level >= 2 || (stage >= 4 && stage <= 6)))
      MOE_CUDA_TRY(cudaEventRecordWithFlags(
          evs[stage], st, cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
    ++stage;
    return MOE_OK;
  }
  void done() {
    if (evs) ++L->prof_n;
  }
};


namespace moecu {
int layer_reserve(moe_layer* L, int64_t T, int k);
int layer_route(moe_layer* L, const uint16_t* x, const uint8_t* fin, int64_t T, int k,
                cudaStream_t st, Marks& mark, uint16_t* out_fin = nullptr);
int layer_ffn(moe_layer* L, const uint16_t* xin, int64_t rows, const uint32_t* problems,
              int64_t np, int mode, uint16_t* h, uint16_t* out, cudaStream_t st, Marks& mark,
              const GemmArgs* comb = nullptr);
int layer_grow_hidden(moe_layer* L, int64_t rows);  // EP: L->ep_h holds >= rows x f
// the whole layer (moe_ffn_forward) on one stream, no host synchronisation
int layer_forward(moe_layer* L, const uint16_t* x, const uint8_t* fin, int64_t T, int k, int mode,
                  uint16_t* out, cudaStream_t st);
}  // namespace moecu

#define TRY(x)                     \
  do {                             \
    const int s__ = (x);           \
    if (s__ != MOE_OK) return s__; \
  } while (0)
