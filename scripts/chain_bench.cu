// dev microbenchmark: serial logit-chain loop variants on one warp (16
// active lanes), operands in shared memory.  Prints cycles per input k.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ float2 ffma2(float a, float2 b, float2 c) {
  uint64_t r;
  const uint64_t bb = (uint64_t)__float_as_uint(b.x) | ((uint64_t)__float_as_uint(b.y) << 32);
  const uint64_t cc = (uint64_t)__float_as_uint(c.x) | ((uint64_t)__float_as_uint(c.y) << 32);
  const uint64_t aa = (uint64_t)__float_as_uint(a) | ((uint64_t)__float_as_uint(a) << 32);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(aa), "l"(bb), "l"(cc));
  return make_float2(__uint_as_float((uint32_t)r), __uint_as_float((uint32_t)(r >> 32)));
}
constexpr int D = 1024, GWP = 32;
struct Step { float x[8]; float2 w[8]; };
template <int V>
__global__ void kern(const float* gw, float* out, long long* cyc, int active) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* ws = reinterpret_cast<float*>(sm);                  // pair-blocked [D/2][GWP/2][2][2]
  float* xf = ws + D * GWP + 256;                            // [D + 64]
  for (int i = threadIdx.x; i < D * GWP; i += blockDim.x) ws[i] = gw[i];
  for (int i = threadIdx.x; i < D + 64; i += blockDim.x) xf[i] = 0.001f * (i % 97);
  __syncthreads();
  const int t = threadIdx.x;
  float2 acc = make_float2(0.f, 0.f), acc2 = acc;
  long long t0 = clock64();
  if (t < active) {
    const float* wg = ws + 4 * t;  // expert pair t
    auto load = [&](Step& o, int kk) {
      const float4 a = *reinterpret_cast<const float4*>(xf + kk);
      const float4 b = *reinterpret_cast<const float4*>(xf + kk + 4);
      o.x[0] = a.x; o.x[1] = a.y; o.x[2] = a.z; o.x[3] = a.w;
      o.x[4] = b.x; o.x[5] = b.y; o.x[6] = b.z; o.x[7] = b.w;
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const float4 w4 = *reinterpret_cast<const float4*>(wg + ((kk + q) >> 1) * 2 * GWP);
        o.w[q] = make_float2(w4.x, w4.y);
        o.w[q + 1] = make_float2(w4.z, w4.w);
      }
    };
    auto fma8 = [&](const Step& o, float2& c) {
#pragma unroll
      for (int q = 0; q < 8; ++q) c = ffma2(o.x[q], o.w[q], c);
    };
    if constexpr (V == 0) {  // naive: load then use
      for (int kk = 0; kk < D; kk += 8) { Step s; load(s, kk); fma8(s, acc); }
    } else if constexpr (V == 1) {  // 2-step ring
      Step a, b;
      load(a, 0); load(b, 8);
      for (int kk = 0; kk < D; kk += 16) {
        fma8(a, acc); load(a, kk + 16);
        fma8(b, acc); load(b, kk + 24);
      }
    } else if constexpr (V == 2) {  // 4-step ring
      Step a, b, c, d;
      load(a, 0); load(b, 8); load(c, 16); load(d, 24);
      for (int kk = 0; kk < D; kk += 32) {
        fma8(a, acc); load(a, kk + 32);
        fma8(b, acc); load(b, kk + 40);
        fma8(c, acc); load(c, kk + 48);
        fma8(d, acc); load(d, kk + 56);
      }
    } else if constexpr (V == 3) {  // no loads in the loop: operands from registers
      Step a; load(a, 0);
      for (int kk = 0; kk < D; kk += 8) fma8(a, acc);
    } else if constexpr (V == 4) {  // two independent chains (2 expert pairs), 2-step ring
      Step a, b;
      load(a, 0); load(b, 8);
      for (int kk = 0; kk < D; kk += 16) {
        fma8(a, acc); fma8(a, acc2); load(a, kk + 16);
        fma8(b, acc); fma8(b, acc2); load(b, kk + 24);
      }
    } else {  // pure chain, constant operands
      const float2 w = *reinterpret_cast<const float2*>(wg);
      const float xv = xf[t];
      for (int kk = 0; kk < D; ++kk) acc = ffma2(xv, w, acc);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc.x + acc.y + acc2.x + acc2.y;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float *gw, *out;
  long long* cyc;
  cudaMalloc(&gw, D * GWP * 4);
  cudaMemset(gw, 0, D * GWP * 4);
  cudaMalloc(&out, 4096);
  cudaMallocManaged(&cyc, 8);
  const size_t smem = (D * GWP + 256 + D + 128) * 4;
  auto run = [&](const char* name, auto k, int act, double per) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 2; ++i) { k<<<1, 256, smem>>>(gw, out, cyc, act); cudaDeviceSynchronize(); }
    printf("%-44s active=%3d: %.2f cycles/k\n", name, act, (double)*cyc / (D * per));
  };
  run("V0 load-then-use", kern<0>, 16, 1);
  run("V1 2-step ring", kern<1>, 16, 1);
  run("V2 4-step ring", kern<2>, 16, 1);
  run("V3 register operands (no loads)", kern<3>, 16, 1);
  run("V4 2 chains/thread, 2-step ring (per chain-k)", kern<4>, 16, 2);
  run("V5 constant operands", kern<5>, 16, 1);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
