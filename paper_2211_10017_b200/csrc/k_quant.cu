// k_quant.cu -- K1 quantizer, K0 dequantizer, int4 pack/unpack and the
// device weight tiling used by the grouped GEMMs.
//
// Reference: proj/src/quantize.cpp:14-122 (quantizer, packing),
//            proj/src/dequant.cpp:55-112 + include/moeinfer/dequant.hpp:39-63.
// All of this is HBM-bound byte/integer work: one thread per output channel
// (column) so the m-loop reads are coalesced across the warp; int4 nibbles
// are packed in-register with warp shuffles (8 lanes -> one 32-bit word).
#include "kernels.cuh"

namespace moecu {

// ------------------------------------------------------------- quantize (K1)
// One thread per (expert, column).  Pass 1: channel max |w| (f32, exactly as
// quantize.cpp:100-102) + non-finite detection (lowest flat index wins, the
// order quantize.cpp:81-86 reports).  Pass 2: encode with IEEE f64 division
// and round-half-away-from-zero (quantize.cpp:26-32), pack.
template <int BITS>
__global__ void __launch_bounds__(256) quantize_kernel(const uint16_t* __restrict__ w, int64_t e,
                                                       int64_t m, int64_t n,
                                                       uint8_t* __restrict__ packed,
                                                       uint16_t* __restrict__ scales,
                                                       unsigned long long* bad) {
  const int64_t cols_per_e = (n + 255) / 256 * 256;
  const int64_t g = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const int64_t ei = g / cols_per_e;
  const int64_t ni = g % cols_per_e;
  const bool live = ei < e && ni < n;
  constexpr int qmax = BITS == 8 ? 127 : 7;
  constexpr int offset = BITS == 8 ? 128 : 8;

  float mx = 0.0f;
  if (live) {
    const uint16_t* col = w + ei * m * n + ni;
    for (int64_t mi = 0; mi < m; ++mi) {
      const uint16_t h = __ldg(col + mi * n);
      if ((h & 0x7C00) == 0x7C00) {
        atomicMin(bad, (unsigned long long)((ei * m + mi) * n + ni));
        break;
      }
      mx = fmaxf(mx, fabsf(h2f(h)));
    }
  }
  // quant_scale_from_maxabs (quantize.cpp:14-24)
  uint16_t s = 0x3C00;
  if (mx != 0.0f) {
    s = f2h(__fdiv_rn(mx, (float)qmax));
    if ((s & 0x7FFF) == 0) s = 0x0001;
  }
  if (live) scales[ei * n + ni] = s;
  const double sd = (double)h2f(s);
  const uint16_t* col = w + (live ? ei * m * n + ni : 0);
  for (int64_t mi = 0; mi < m; ++mi) {
    uint32_t code = offset;
    if (live) {
      const double q = round(__ddiv_rn((double)h2f(__ldg(col + mi * n)), sd));
      const double qc = fmin(fmax(q, (double)-qmax), (double)qmax);
      code = (uint32_t)((int)qc + offset);
    }
    if constexpr (BITS == 8) {
      if (live) packed[(ei * m + mi) * n + ni] = (uint8_t)code;
    } else {
      // nibble for logical position j = ni % 8 inside its group of 8:
      // word = v0 | v2<<4 | v4<<8 | v6<<12 | v1<<16 | v3<<20 | v5<<24 | v7<<28
      const int j = (int)(ni & 7);
      uint32_t word = code << ((j & 1) * 16 + (j >> 1) * 4);
      word |= __shfl_xor_sync(0xffffffffu, word, 1);
      word |= __shfl_xor_sync(0xffffffffu, word, 2);
      word |= __shfl_xor_sync(0xffffffffu, word, 4);
      if (live && j == 0)
        *reinterpret_cast<uint32_t*>(packed + ((ei * m + mi) * n + ni) / 2) = word;
    }
  }
}

// Vector form (n % 8 == 0, 16-byte aligned rows).  A CTA owns 128 columns
// of one expert: 16 column groups of 8 (one 16-byte load per row; a
// half-warp reads 256 contiguous bytes of a row) x 16 row slices.  Pass 1:
// per-thread channel max |w| and first non-finite weight (lowest flat index,
// no early exit) over its slice, reduced over the slices in shared memory;
// pass 2 (same rows, mostly L2): codes with an f32 division and
// round-half-away -- identical to the reference's llround(f64 w / f64 s) for
// every fp16 pair (exhaustive proof: tests/native/quant_div_check.c) --
// packed in registers: one 32-bit word (int4) or 8 bytes (int8) per row.
constexpr int kQCols = 16, kQSlices = 16;
template <int BITS>
__global__ void __launch_bounds__(256) quantize8_kernel(const uint16_t* __restrict__ w, int64_t e,
                                                        int64_t m, int64_t n,
                                                        uint8_t* __restrict__ packed,
                                                        uint16_t* __restrict__ scales,
                                                        unsigned long long* bad) {
  __shared__ float smx[kQSlices][kQCols * 8];
  const int64_t cpb = (n + 8 * kQCols - 1) / (8 * kQCols);  // CTAs per expert
  const int64_t ei = blockIdx.x / cpb;
  const int cg = threadIdx.x % kQCols, sl = threadIdx.x / kQCols;
  const int64_t c0 = (blockIdx.x % cpb) * 8 * kQCols + cg * 8;
  const bool live = c0 < n;
  constexpr int qmax = BITS == 8 ? 127 : 7;
  constexpr int offset = BITS == 8 ? 128 : 8;
  const uint4* col = reinterpret_cast<const uint4*>(w + ei * m * n + (live ? c0 : 0));
  const int64_t rs = n / 8;  // row stride in uint4
  const int64_t r0 = m * sl / kQSlices, r1 = m * (sl + 1) / kQSlices;
  float mx[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) mx[j] = 0.f;
  unsigned long long first_bad = ~0ull;
  auto scan = [&](const uint4& v, int64_t mi) {
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint16_t h = (uint16_t)(wd[j >> 1] >> ((j & 1) * 16));
      if ((h & 0x7C00) == 0x7C00)
        first_bad = ::min(first_bad, (unsigned long long)((ei * m + mi) * n + c0 + j));
      mx[j] = fmaxf(mx[j], fabsf(h2f(h)));
    }
  };
  if (live) {
    int64_t mi = r0;
    for (; mi + 4 <= r1; mi += 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(col + (mi + u) * rs);
#pragma unroll
      for (int u = 0; u < 4; ++u) scan(v[u], mi + u);
    }
    for (; mi < r1; ++mi) scan(__ldg(col + mi * rs), mi);
    if (first_bad != ~0ull) atomicMin(bad, first_bad);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) smx[sl][cg * 8 + j] = mx[j];
  __syncthreads();
  // quant_scale_from_maxabs (quantize.cpp:14-24), max over the slices
  float sf[8];
  uint16_t sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float v = 0.f;
    for (int q = 0; q < kQSlices; ++q) v = fmaxf(v, smx[q][cg * 8 + j]);
    uint16_t s = 0x3C00;
    if (v != 0.0f) {
      s = f2h(__fdiv_rn(v, (float)qmax));
      if ((s & 0x7FFF) == 0) s = 0x0001;
    }
    sh[j] = s;
    sf[j] = h2f(s);
  }
  if (!live) return;
  if (sl == 0)
    *reinterpret_cast<uint4*>(scales + ei * n + c0) =
        make_uint4(sh[0] | (uint32_t)sh[1] << 16, sh[2] | (uint32_t)sh[3] << 16,
                   sh[4] | (uint32_t)sh[5] << 16, sh[6] | (uint32_t)sh[7] << 16);
  auto emit = [&](const uint4& v, int64_t mi) {
    const uint32_t wd[4] = {v.x, v.y, v.z, v.w};
    uint32_t code[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float q = roundf(__fdiv_rn(h2f((uint16_t)(wd[j >> 1] >> ((j & 1) * 16))), sf[j]));
      code[j] = (uint32_t)((int)fminf(fmaxf(q, (float)-qmax), (float)qmax) + offset);
    }
    const int64_t flat = (ei * m + mi) * n + c0;
    if constexpr (BITS == 8) {
      *reinterpret_cast<uint2*>(packed + flat) =
          make_uint2(code[0] | code[1] << 8 | code[2] << 16 | code[3] << 24,
                     code[4] | code[5] << 8 | code[6] << 16 | code[7] << 24);
    } else {
      // quantize.cpp:44-47: v0|v2<<4, v4|v6<<4, v1|v3<<4, v5|v7<<4
      *reinterpret_cast<uint32_t*>(packed + flat / 2) =
          code[0] | code[2] << 4 | code[4] << 8 | code[6] << 12 | code[1] << 16 |
          code[3] << 20 | code[5] << 24 | code[7] << 28;
    }
  };
  int64_t mi = r0;
  for (; mi + 4 <= r1; mi += 4) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(col + (mi + u) * rs);
#pragma unroll
    for (int u = 0; u < 4; ++u) emit(v[u], mi + u);
  }
  for (; mi < r1; ++mi) emit(__ldg(col + mi * rs), mi);
}

int launch_quantize(const uint16_t* w, int64_t e, int64_t m, int64_t n, int bits,
                    uint8_t* packed, uint16_t* scales, unsigned long long* bad,
                    cudaStream_t st) {
  const bool vec = n % 8 == 0 && ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(scales) |
                                   reinterpret_cast<uintptr_t>(packed)) & 15) == 0;
  if (vec) {
    const unsigned blocks = (unsigned)(e * ((n + 8 * kQCols - 1) / (8 * kQCols)));
    if (bits == 8)
      quantize8_kernel<8><<<blocks, 256, 0, st>>>(w, e, m, n, packed, scales, bad);
    else
      quantize8_kernel<4><<<blocks, 256, 0, st>>>(w, e, m, n, packed, scales, bad);
    note_launch();
    return check_launch("quantize");
  }
  const int64_t cols_per_e = (n + 255) / 256 * 256;
  const int64_t blocks = e * cols_per_e / 256;
  if (bits == 8)
    quantize_kernel<8><<<(unsigned)blocks, 256, 0, st>>>(w, e, m, n, packed, scales, bad);
  else
    quantize_kernel<4><<<(unsigned)blocks, 256, 0, st>>>(w, e, m, n, packed, scales, bad);
  note_launch();
  return check_launch("quantize");
}

// ------------------------------------------------------- int4 pack / unpack
__global__ void pack_int4_kernel(const uint8_t* __restrict__ v, int64_t groups,
                                 uint8_t* __restrict__ out, unsigned long long* bad) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  const uint8_t* s = v + 8 * g;
  uint32_t word = 0;
  for (int j = 0; j < 8; ++j) {
    if (s[j] >= 16) atomicMin(bad, (unsigned long long)(8 * g + j));
    word |= (uint32_t)(s[j] & 15) << ((j & 1) * 16 + (j >> 1) * 4);
  }
  reinterpret_cast<uint32_t*>(out)[g] = word;
}

__global__ void unpack_int4_kernel(const uint8_t* __restrict__ p, int64_t groups,
                                   uint8_t* __restrict__ out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  const uint32_t word = reinterpret_cast<const uint32_t*>(p)[g];
  for (int j = 0; j < 8; ++j) out[8 * g + j] = (word >> ((j & 1) * 16 + (j >> 1) * 4)) & 15;
}

int launch_pack_int4(const uint8_t* v, int64_t count, uint8_t* out, unsigned long long* bad,
                     cudaStream_t st) {
  const int64_t groups = count / 8;
  if (groups == 0) return MOE_OK;
  pack_int4_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(v, groups, out, bad);
  note_launch();
  return check_launch("pack_int4");
}
int launch_unpack_int4(const uint8_t* p, int64_t count, uint8_t* out, cudaStream_t st) {
  const int64_t groups = count / 8;
  if (groups == 0) return MOE_OK;
  unpack_int4_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(p, groups, out);
  note_launch();
  return check_launch("unpack_int4");
}

// logical stored code (ei, mi, ni) of a reference-layout payload
__device__ __forceinline__ uint32_t ref_code(const uint8_t* __restrict__ packed, int bits,
                                             int64_t m, int64_t n, int64_t ei, int64_t mi,
                                             int64_t ni) {
  const int64_t flat = (ei * m + mi) * n + ni;
  if (bits == 8) return packed[flat];
  const uint32_t word = __ldg(reinterpret_cast<const uint32_t*>(packed) + flat / 8);
  const int j = (int)(flat & 7);
  return (word >> ((j & 1) * 16 + (j >> 1) * 4)) & 15;
}

// ----------------------------------------------------------- dequantize (K0)
// out = RN16(v * s), v = (code - offset) exactly: naive via int->half
// (dequant.cpp:61-65), fast via the mantissa composition
// (0x6400 | code) - debias (dequant.hpp:40-63).
__global__ void dequant_kernel(const uint8_t* __restrict__ packed,
                               const uint16_t* __restrict__ scales, int64_t e, int64_t m,
                               int64_t n, int bits, int fast, uint16_t debias,
                               uint16_t* __restrict__ out) {
  const int64_t total = e * m * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ni = i % n, mi = (i / n) % m, ei = i / (m * n);
    const uint32_t code = ref_code(packed, bits, m, n, ei, mi, ni);
    const int offset = bits == 8 ? 128 : 8;
    uint16_t v;
    if (fast)
      v = hsub((uint16_t)(0x6400 | code), debias);
    else
      v = __half_as_ushort(__int2half_rn((int)code - offset));
    out[i] = hmul(v, scales[ei * n + ni]);
  }
}

int launch_dequantize(const uint8_t* packed, const uint16_t* scales, int64_t e, int64_t m,
                      int64_t n, int bits, int fast, uint16_t debias, uint16_t* out,
                      cudaStream_t st) {
  const int64_t total = e * m * n;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  dequant_kernel<<<(unsigned)blocks, 256, 0, st>>>(packed, scales, e, m, n, bits, fast, debias,
                                                   out);
  note_launch();
  return check_launch("dequantize");
}

// -------------------------------------------------------------- weight tiles
// tiled[e][ft][kb][chunk][feat][16B]: feature tile ft = 128 output columns,
// k-block kb = 64 inputs, each feature's 64 codes in 16-byte chunks.
//   W4 : 2 chunks, chunk h holds k = 32h..32h+31 as 4 interleaved words
//        (word w: k = 32h+8w..+7, nibble order of quantize.cpp:44-47)
//   W8 : 4 chunks, chunk c holds k = 16c..16c+15, one byte each
//   W16: 8 chunks, chunk c holds k = 8c..8c+7, fp16 each
// Padding (k >= m or feature >= n) is the zero code (8 / 128 / 0x0000).
__global__ void tile_weights_kernel(const void* __restrict__ src, int64_t e, int64_t m,
                                    int64_t n, int bits, uint4* __restrict__ tiled) {
  const int64_t nft = (n + 127) / 128, nkb = (m + 63) / 64;
  const int chunks = bits == 4 ? 2 : bits == 8 ? 4 : 8;
  const int64_t total = e * nft * nkb * chunks * 128;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int feat = (int)(i % 128);
    const int c = (int)((i / 128) % chunks);
    const int64_t blk = i / (128 * chunks);
    const int64_t kb = blk % nkb, ft = (blk / nkb) % nft, ei = blk / (nkb * nft);
    const int64_t ni = ft * 128 + feat;
    uint32_t wds[4];
    if (bits == 16) {
      const uint16_t* w = static_cast<const uint16_t*>(src);
      for (int q = 0; q < 4; ++q) {
        uint32_t pr = 0;
        for (int h = 0; h < 2; ++h) {
          const int64_t k = kb * 64 + c * 8 + q * 2 + h;
          const uint16_t v = (k < m && ni < n) ? w[(ei * m + k) * n + ni] : 0;
          pr |= (uint32_t)v << (16 * h);
        }
        wds[q] = pr;
      }
    } else if (bits == 8) {
      const uint8_t* p = static_cast<const uint8_t*>(src);
      for (int q = 0; q < 4; ++q) {
        uint32_t wd = 0;
        for (int b = 0; b < 4; ++b) {
          const int64_t k = kb * 64 + c * 16 + q * 4 + b;
          const uint32_t code = (k < m && ni < n) ? ref_code(p, 8, m, n, ei, k, ni) : 128;
          wd |= code << (8 * b);
        }
        wds[q] = wd;
      }
    } else {
      const uint8_t* p = static_cast<const uint8_t*>(src);
      for (int q = 0; q < 4; ++q) {
        uint32_t wd = 0;
        for (int j = 0; j < 8; ++j) {
          const int64_t k = kb * 64 + c * 32 + q * 8 + j;
          const uint32_t code = (k < m && ni < n) ? ref_code(p, 4, m, n, ei, k, ni) : 8;
          wd |= code << ((j & 1) * 16 + (j >> 1) * 4);
        }
        wds[q] = wd;
      }
    }
    tiled[i] = make_uint4(wds[0], wds[1], wds[2], wds[3]);
  }
}

int64_t tiled_bytes(int64_t e, int64_t m, int64_t n, int bits) {
  const int64_t nft = (n + 127) / 128, nkb = (m + 63) / 64;
  return e * nft * nkb * (int64_t)wblock_bytes(bits);
}

int launch_tile_weights(const void* src, int64_t e, int64_t m, int64_t n, int bits,
                        void* tiled, cudaStream_t st) {
  const int64_t total = tiled_bytes(e, m, n, bits) / 16;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 64);
  tile_weights_kernel<<<(unsigned)blocks, 256, 0, st>>>(src, e, m, n, bits,
                                                        static_cast<uint4*>(tiled));
  note_launch();
  return check_launch("tile_weights");
}

}  // namespace moecu
