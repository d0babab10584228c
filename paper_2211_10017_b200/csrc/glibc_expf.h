// glibc_expf.h -- bit-exact restatement of the host libm `expf` the reference
// gate calls (proj/src/routing.cpp:34, std::exp(float)).
//
// Third-party dependency: GNU C Library 2.39 (Ubuntu 2.39-0ubuntu8.5), libm
// `expf`, algorithm from sysdeps/ieee754/flt-32/e_expf.c + e_exp2f_data.c
// (Szabolcs Nagy's table method: x*N/ln2 = k + r, N = 32, 2^(k/N) from a
// 32-entry table, degree-3 polynomial in double).  On x86_64 hosts with
// AVX2+FMA the ifunc selects the variant compiled with -mfma; GCC contracts
// four of its mul/add pairs into FMAs (read off the shipped libm.so.6
// machine code: vfmadd132sd / vfmsub132sd / vfmadd213sd / vfmadd132sd /
// vfmadd132sd).  The constants below are the values shipped in that libm
// (__exp2f_data: shift, invln2_scaled, poly_scaled, tab).
//
// Usable from host C/C++ and CUDA device code: every step is an IEEE double
// operation (fma() is exact-then-round on both), so host and device agree
// bit-for-bit.  Verified exhaustively against the host libm over all 2^32
// float inputs by tests/test_expf_port.py (CPU) and spot-checked on device
// by tests/test_gpu_gate.py.
#pragma once

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define MOE_HD __host__ __device__ __forceinline__
// global (L1-cached), not __constant__: lanes index the table divergently
#define MOE_EXPF_TAB_QUAL __device__ const
#else
#define MOE_HD static inline
#define MOE_EXPF_TAB_QUAL static const
#include <math.h>
#endif

// tab[i] = asuint64(2^(i/32)) - (i << 47)
#define MOE_EXPF_TAB_INIT                                                     \
  {0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full,     \
   0x3fef9301d0125b51ull, 0x3fef72b83c7d517bull, 0x3fef54873168b9aaull,     \
   0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, 0x3fef06fe0a31b715ull,     \
   0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,     \
   0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull,     \
   0x3feea47eb03a5585ull, 0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull,     \
   0x3feea11473eb0187ull, 0x3feea589994cce13ull, 0x3feeace5422aa0dbull,     \
   0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,     \
   0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull,     \
   0x3fef3720dcef9069ull, 0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full,     \
   0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull}

#ifdef __CUDACC__
MOE_EXPF_TAB_QUAL uint64_t moe_expf_tab_dev[32] = MOE_EXPF_TAB_INIT;
#endif
static const uint64_t moe_expf_tab_host[32] = MOE_EXPF_TAB_INIT;

MOE_HD double moe_u2d(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
MOE_HD uint64_t moe_d2u(double d) {
#ifdef __CUDA_ARCH__
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}
MOE_HD uint32_t moe_f2u(float f) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
#endif
}
MOE_HD float moe_u2f(uint32_t u) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

// tab: the 32-entry table (a shared-memory copy on the device avoids an L2
// round trip on the first call of a CTA)
MOE_HD float moe_glibc_expf_t(float x, const uint64_t* tab) {
  const uint32_t ux = moe_f2u(x);
  const uint32_t abstop = (ux >> 20) & 0x7ff;
  if (abstop >= 0x42b) {                      // |x| >= 88 or x is nan
    if (ux == 0xff800000u) return 0.0f;       // -inf
    if (abstop >= 0x7f8) return x + x;        // inf, nan
    if (x > moe_u2f(0x42b17217u)) return moe_u2f(0x7f800000u);  // overflow
    if (x < moe_u2f(0xc2cff1b4u)) return 0.0f;                  // underflow
    if (x < moe_u2f(0xc2ce8ecfu)) return moe_u2f(0x00000001u);  // may-underflow
  }
  const double xd = (double)x;
  const double invln2n = moe_u2d(0x40471547652b82feull);
  const double shift = moe_u2d(0x4338000000000000ull);
  const double kd_sh = fma(invln2n, xd, shift);
  const uint64_t ki = moe_d2u(kd_sh);
  const double kd = kd_sh - shift;
  const double r = fma(invln2n, xd, -kd);
  uint64_t t = tab[ki & 31];
  t += ki << 47;
  const double s = moe_u2d(t);
  const double z = fma(moe_u2d(0x3ebc6af84b912394ull), r, moe_u2d(0x3f2ebfce50fac4f3ull));
  const double r2 = r * r;
  double y = fma(r, moe_u2d(0x3f962e42ff0c52d6ull), 1.0);
  y = fma(z, r2, y);
  y = y * s;
  return (float)y;
}

MOE_HD float moe_glibc_expf(float x) {
#ifdef __CUDA_ARCH__
  return moe_glibc_expf_t(x, moe_expf_tab_dev);
#else
  return moe_glibc_expf_t(x, moe_expf_tab_host);
#endif
}
