// include/moeinfer/device.hpp -- additive device-resident API (no reference
// counterpart): the MoE block uploaded and tiled once, forward on device or
// host buffers, top-k gating extension, numerics switch for the value API.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "moeinfer/model.hpp"

struct moe_layer;  // include/moe_cuda.h

namespace moe::cuda {

enum class Numerics : int { exact = 0, fast = 1 };
// Numerics of the value-semantics API (grouped_gemm_*, moe_ffn_forward).
// Default exact (bit-identical to the reference).
void set_numerics(Numerics n);
Numerics numerics();

class DeviceMoeFfn {
 public:
  explicit DeviceMoeFfn(const MoeFfn& w);
  ~DeviceMoeFfn();
  DeviceMoeFfn(const DeviceMoeFfn&) = delete;
  DeviceMoeFfn& operator=(const DeviceMoeFfn&) = delete;

  size_t d_model() const { return d_; }
  size_t n_experts() const { return e_; }
  // host buffers (copies in/out, synchronises, raises the reference errors)
  HalfMat forward(const HalfMat& x, std::span<const uint8_t> finished, int top_k = 1,
                  Numerics n = Numerics::fast);
  // device pointers on a cudaStream_t (graph-capturable, no host sync)
  void forward_device(const uint16_t* x, const uint8_t* finished, int64_t T, int top_k,
                      Numerics n, uint16_t* out, void* stream);
  ModelTraffic last_traffic();
  moe_layer* handle() { return h_; }

 private:
  moe_layer* h_ = nullptr;
  size_t d_ = 0, e_ = 0;
};

}  // namespace moe::cuda
