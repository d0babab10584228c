// tests/native/dropin_quantize_model.cpp -- the C++ drop-in's quantize_model
// (include/moeinfer/model.hpp; reference model.hpp:118, model.cpp:153-173)
// on a two-block fp16 MoeModel: precision tag, per-block codes/scales equal
// to quantize() of the same tensors, masters dropped, biases kept, and the
// reference's rejection of a non-fp16 source.  Needs a GPU (the quantizer
// runs there); built and run by tests/test_gpu_dropin.py.
#include <cstdio>
#include <random>
#include <stdexcept>

#include "moeinfer/model.hpp"

using namespace moe;

static HalfTensor3 rnd3(size_t e, size_t m, size_t n, std::mt19937& g) {
  std::normal_distribution<float> nd(0.f, 0.3f);
  HalfTensor3 t(e, m, n);
  for (auto& h : t.data) h = f32_to_half(nd(g));
  return t;
}
static HalfMat rnd2(size_t r, size_t c, std::mt19937& g) {
  std::normal_distribution<float> nd(0.f, 0.05f);
  HalfMat t(r, c);
  for (auto& h : t.data) h = f32_to_half(nd(g));
  return t;
}

int main() {
  std::mt19937 g(7);
  const size_t d = 64, f = 128, E = 4;
  MoeModel m;
  for (int b = 0; b < 2; ++b) {
    MoeFfn blk;
    blk.ln.gamma.assign(d, f32_to_half(1.f));
    blk.ln.beta.assign(d, f32_to_half(0.f));
    blk.gate_w = rnd2(d, E, g);
    blk.gate_b.assign(E, f32_to_half(0.f));
    blk.w1 = rnd3(E, d, f, g);
    blk.w2 = rnd3(E, f, d, g);
    blk.b1 = rnd2(E, f, g);
    blk.b2 = rnd2(E, d, g);
    m.blocks.push_back(blk);
  }
  int bad = 0;
  for (QuantBits bits : {QuantBits::b4, QuantBits::b8}) {
    const MoeModel q = quantize_model(m, bits);
    bad += q.precision != (bits == QuantBits::b8 ? Precision::int8 : Precision::int4);
    for (size_t b = 0; b < m.blocks.size(); ++b) {
      const auto& src = m.blocks[b];
      const auto& dst = q.blocks[b];
      const QuantizedExpertWeights w1 = quantize(src.w1, bits), w2 = quantize(src.w2, bits);
      bad += !dst.quantized() || dst.qw1->packed != w1.packed || dst.qw2->packed != w2.packed;
      bad += dst.qw1->scales != w1.scales || dst.qw2->scales != w2.scales;
      bad += !dst.w1.data.empty() || !dst.w2.data.empty();
      bad += dst.b1.data != src.b1.data || dst.b2.data != src.b2.data;
    }
    try {
      quantize_model(q, bits);
      ++bad;  // must throw: source is not fp16
    } catch (const std::invalid_argument& e) {
      bad += std::string(e.what()) != "quantize_model: source must be an fp16 model";
    }
  }
  std::printf("dropin_quantize_model: %s\n", bad ? "FAIL" : "ok");
  return bad != 0;
}
