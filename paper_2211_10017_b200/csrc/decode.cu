// decode.cu -- the MoE side of incremental beam-search decoding with batch
// pruning (proj/src/decode.cpp:104-345).
//
// The reference decodes rows = batch x beam one token per step through the
// decoder stack; at every MoE block it calls
//   moe_ffn_forward(x, moe, route_finished, ...)            (decode.cpp:216)
// with route_finished = finished_rows when opts.prune, else all zeros
// (decode.cpp:167-169): rows of sentences that already emitted EOS leave the
// expert workload (their output is x, bit for bit) -- the paper's "batch
// pruning".  Because rows never interact, pruning is
// output-transparent for the live rows.
//
// moe_decode_run replays exactly that contract on the device for a whole
// decode: for every step s and every MoE block l of the stack, one layer
// forward (LN -> gate -> plan -> expert FFNs -> combine, layer_forward) on the
// step's rows, the finished mask of step s routed iff prune, the output of
// block l feeding block l+1.  Everything stays device-resident and is issued
// on one stream with no host synchronisation (capturable in one CUDA graph);
// the attention and embedding halves of the decoder (not on the MoE path,
// DESIGN.md §7) are represented by the per-step inputs x_steps.
#include "layer.cuh"

using namespace moecu;

extern "C" int moe_decode_run(moe_layer* const* layers, int n_layers, const uint16_t* x_steps,
                              const uint8_t* finished_steps, int steps, int64_t rows, int k,
                              int mode, int prune, uint16_t* out_steps, uint16_t* work,
                              moe_stream_t stream) {
  if (!layers || n_layers < 1 || !x_steps || !out_steps || !work)
    return set_error(MOE_EINVAL, "decode: null argument");
  if (steps < 1 || rows < 1) return set_error(MOE_EINVAL, "decode: empty decode");
  const int64_t d = layers[0]->d;
  for (int l = 0; l < n_layers; ++l) {
    if (!layers[l] || layers[l]->d != d) return set_error(MOE_EINVAL, "decode: layer width mismatch");
    if (layers[l]->El != layers[l]->E)
      return set_error(MOE_EINVAL, "decode: layers must hold all experts");
    TRY(layer_reserve(layers[l], rows, k));
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int s = 0; s < steps; ++s) {
    const uint16_t* in = x_steps + (int64_t)s * rows * d;
    const uint8_t* fin = prune && finished_steps ? finished_steps + (int64_t)s * rows : nullptr;
    uint16_t* last = out_steps + (int64_t)s * rows * d;
    for (int l = 0; l < n_layers; ++l) {
      // ping-pong so that the last block of the step lands in out_steps[s]
      uint16_t* dst = ((n_layers - 1 - l) & 1) == 0 ? last : work;
      TRY(layer_forward(layers[l], in, fin, rows, k, mode, dst, st));
      in = dst;
    }
  }
  return MOE_OK;
}
