// include/moeinfer/model.hpp -- the MoE-layer slice of the reference's
// proj/include/moeinfer/model.hpp (MoeFfn :73-84, ModelTraffic :124-133,
// layer_norm :138-140, moe_ffn_forward :154-156, gate_logits_f32 :159-161).
// Attention, the dense FFN, the encoder/decoder stack and beam search are
// outside the hot path and are not part of this library.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "moeinfer/grouped_gemm.hpp"
#include "moeinfer/quantize.hpp"
#include "moeinfer/routing.hpp"
#include "moeinfer/tensor.hpp"

namespace moe {

struct LayerNormWeights {
  std::vector<Half> gamma, beta;
};

struct MoeFfn {
  LayerNormWeights ln;
  HalfMat gate_w;  // (d_model, E)
  std::vector<Half> gate_b;
  HalfTensor3 w1;  // (E, d_model, d_ffn); empty when quantized
  HalfTensor3 w2;  // (E, d_ffn, d_model); empty when quantized
  HalfMat b1;      // (E, d_ffn)
  HalfMat b2;      // (E, d_model)
  std::optional<QuantizedExpertWeights> qw1, qw2;
  bool quantized() const { return qw1.has_value(); }
};

struct ModelTraffic {
  TrafficCounter expert;
  TrafficCounter other;
  ModelTraffic& operator+=(const ModelTraffic& o) {
    expert += o.expert;
    other += o.other;
    return *this;
  }
  friend bool operator==(const ModelTraffic&, const ModelTraffic&) = default;
};

HalfMat layer_norm(const HalfMat& x, const LayerNormWeights& ln);
std::vector<float> gate_logits_f32(const HalfMat& xn, const HalfMat& gate_w,
                                   std::span<const Half> gate_b, TrafficCounter* tc = nullptr);
// Pre-norm MoE FFN block with residual; finished rows pass through exactly.
// Uploads the block on every call (value semantics); use moe::cuda::
// DeviceMoeFfn (moeinfer/device.hpp) to keep weights resident.
HalfMat moe_ffn_forward(const HalfMat& x, const MoeFfn& w, std::span<const uint8_t> finished,
                        ModelTraffic* tr = nullptr, int threads = 1);
// quantize both expert tensors of a block (model.cpp:153-173, per block)
MoeFfn quantize_moe_ffn(const MoeFfn& w, QuantBits bits, int threads = 1);

// Model precision tag (model.hpp:52)
enum class Precision : uint8_t { f16 = 0, int8 = 1, int4 = 2 };

// The hot-path slice of moe::Model (model.hpp:97-112): its MoE blocks in
// file order (encoder, then decoder) and the precision tag.
struct MoeModel {
  Precision precision = Precision::f16;
  std::vector<MoeFfn> blocks;
};

// quantize_model (model.hpp:118, model.cpp:153-173): every MoE block's
// expert tensors quantized (on the GPU, codes bit-identical to quantize()),
// everything else -- biases included -- stays FP16; the source must be an
// fp16 model.
MoeModel quantize_model(const MoeModel& m, QuantBits bits, int threads = 1);

}  // namespace moe
