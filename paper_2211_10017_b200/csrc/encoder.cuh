// encoder.cuh -- device copy of a .moec checkpoint's encoder (SURVEY §8f
// row 3): the attention and dense-FFN weights next to the MoE blocks, so
// encoder_forward (proj/src/model.cpp:351-398) runs end to end on the GPU.
#pragma once
#include <vector>

#include "layer.cuh"

namespace moecu {

// a dense fp16 projection y = x W + b, W (m, n) tiled once for every GEMM
// kernel (k_quant.cu tile_weights, bits = 16, one "expert")
struct DevLinear {
  void* tiled = nullptr;
  uint16_t* bias = nullptr;
  int64_t m = 0, n = 0;
};

struct EncLayerDev {
  uint16_t *ln_g = nullptr, *ln_b = nullptr;  // attention LayerNorm
  DevLinear qkv, o;  // Q | K | V concatenated (n = 3 d)
  int moe_block = -1;                         // index into moe_moec::layers, or -1: dense FFN
  uint16_t *fln_g = nullptr, *fln_b = nullptr;
  DevLinear w1, w2;
};

struct EncoderDev {
  int64_t d = 0, f = 0, heads = 0, vocab = 0, maxlen = 0;
  uint16_t *tok = nullptr, *pos = nullptr, *ln_g = nullptr, *ln_b = nullptr;
  std::vector<EncLayerDev> layers;
  std::vector<void*> allocs;  // everything above, freed with the checkpoint
  // forward workspace (grown on demand)
  int64_t cap_t = 0;
  uint16_t *x = nullptr, *x2 = nullptr, *xn = nullptr, *q = nullptr, *k = nullptr, *v = nullptr,
           *ctx = nullptr, *o = nullptr, *h = nullptr;
  int32_t* tokens = nullptr;
  uint32_t* problem = nullptr;  // {0, 0, t}: one-problem grouped GEMM
  uint32_t* bad = nullptr;      // token range check
  uint32_t* ident = nullptr;    // FAST residuals in the GEMM epilogue: identity row map
  uint16_t* ones = nullptr;     //   and unit scales (x (+) y (*) 1 == x (+) y)
  ~EncoderDev();
};

// upload one fp16 (m, n) weight + (n) bias from the file image
int enc_linear(EncoderDev* E, const uint16_t* w, const uint16_t* b, int64_t m, int64_t n,
               DevLinear* out);
int enc_upload(EncoderDev* E, const uint16_t* host, int64_t count, uint16_t** out);

}  // namespace moecu
