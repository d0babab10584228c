// k_gate_fused.cu -- one-time preparation of the gate weights for K2
// (k_ln_gate.cu): widened to f32 and blocked by (input pair, expert pair),
//   [k/2][e/2][k%2][e%2]  i.e.  w[2j][2p], w[2j][2p+1], w[2j+1][2p], w[2j+1][2p+1]
// (experts zero-padded to gwp).  A thread owning experts e0..e0+EPG-1 (e0
// even) reads inputs 2j, 2j+1 of all of them as one contiguous 8*EPG-byte
// piece, and each FFMA2 operand pair (two experts, one input) is two
// adjacent floats of it -- no register shuffling between load and FMA.
// Shared-memory load issue, not bandwidth, is what the single-warp logit
// chains at decode sizes pay for.  Chunks of whole input pairs stay
// contiguous, so the kernel's weight ring copies inputs [k0, k0 + kc) as one
// bulk copy of kc * gwp floats.
#include "kernels.cuh"

namespace moecu {

__global__ void widen_gate_kernel(const uint16_t* __restrict__ gw, int64_t d, int64_t E,
                                  int64_t gwp, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d * gwp) return;
  const int64_t blk = i / 4, r = i % 4;
  const int64_t k = 2 * (blk / (gwp / 2)) + (r >> 1), e = 2 * (blk % (gwp / 2)) + (r & 1);
  out[i] = e < E ? h2f(gw[k * E + e]) : 0.f;
}

int launch_widen_gate(const uint16_t* gw, int64_t d, int64_t E, int64_t gwp, float* out,
                      cudaStream_t st) {
  if (d % 2 != 0) return set_error(MOE_EINVAL, "widen_gate: d must be even");
  const int64_t n = d * gwp;
  widen_gate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gw, d, E, gwp, out);
  note_launch();
  return check_launch("widen_gate");
}

// f32 gate weight row pitch: EPG <= 8 expert groups never straddle a row
int64_t gate_fused_pitch(int64_t E) { return (E + 7) / 8 * 8; }

}  // namespace moecu
