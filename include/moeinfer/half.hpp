// include/moeinfer/half.hpp -- binary16 value type of the drop-in C++ API.
//
// Same names and semantics as the reference's software FP16
// (proj/include/moeinfer/half.hpp:20-146): a Half is a raw IEEE binary16 bit
// pattern; every arithmetic helper rounds the exact result once to nearest
// even (subnormals kept, no FTZ).  Implemented here with the compiler's
// _Float16 (GCC >= 12, correctly rounded conversions) instead of the
// reference's hand-written f64 narrowing; results are bit-identical for all
// finite inputs, and NaN results use the reference's canonical 0x7E00.
#pragma once

#include <cstdint>
#include <cstring>

namespace moe {

struct Half {
  uint16_t bits = 0;
  constexpr Half() = default;
  constexpr explicit Half(uint16_t b) : bits(b) {}
  friend constexpr bool operator==(Half a, Half b) { return a.bits == b.bits; }
  friend constexpr bool operator!=(Half a, Half b) { return a.bits != b.bits; }
};

inline constexpr Half kHalfZero{0x0000};
inline constexpr Half kHalfOne{0x3C00};
inline constexpr Half kHalfMinSubnormal{0x0001};

namespace detail {
inline _Float16 as_f16(Half h) {
  _Float16 f;
  std::memcpy(&f, &h.bits, 2);
  return f;
}
inline Half from_f16(_Float16 f) {
  Half h;
  std::memcpy(&h.bits, &f, 2);
  if ((h.bits & 0x7C00u) == 0x7C00u && (h.bits & 0x03FFu) != 0) h.bits = 0x7E00;  // canonical NaN
  return h;
}
}  // namespace detail

// 0x6400 | y : the I2F "magic" composition (value 1024 + y for y < 1024)
inline constexpr Half compose_magic(uint16_t y) { return Half(static_cast<uint16_t>(0x6400u | y)); }

inline float half_to_f32(Half h) { return static_cast<float>(detail::as_f16(h)); }
inline double half_to_f64(Half h) { return static_cast<double>(detail::as_f16(h)); }
// one RNE rounding from f64 (f64 -> f16 is a single correctly-rounded step)
inline Half f64_to_half(double x) { return detail::from_f16(static_cast<_Float16>(x)); }
// f32 -> f16 directly is also a single RNE step (no double rounding)
inline Half f32_to_half(float x) { return detail::from_f16(static_cast<_Float16>(x)); }

// exact op in f64 (fp16 operands: sums/products are exact in f64), then RN16
inline Half half_add(Half a, Half b) { return f64_to_half(half_to_f64(a) + half_to_f64(b)); }
inline Half half_sub(Half a, Half b) { return f64_to_half(half_to_f64(a) - half_to_f64(b)); }
inline Half half_mul(Half a, Half b) { return f64_to_half(half_to_f64(a) * half_to_f64(b)); }

}  // namespace moe
