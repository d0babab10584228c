// dev microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) latency and throughput on sm_100a
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t f2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
template <int CH>
__global__ void k_ffma(float* out, float x, long long* cyc, int iters) {
  float a[CH];
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 0.001f + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fmaf(a[i], x, 0.5f * i + x);
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; ++i) s += a[i];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
__global__ void k_ffma2(float* out, float x, long long* cyc, int iters) {
  uint64_t a[CH];
  for (int i = 0; i < CH; ++i) { float lo = threadIdx.x * 0.001f + i, hi = lo + 1; a[i] = (uint64_t)__float_as_uint(lo) | ((uint64_t)__float_as_uint(hi) << 32); }
  uint64_t xx = (uint64_t)__float_as_uint(x) | ((uint64_t)__float_as_uint(x) << 32);
  uint64_t cc = (uint64_t)__float_as_uint(0.5f) | ((uint64_t)__float_as_uint(0.25f) << 32);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = f2(a[i], xx, cc);
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < CH; ++i) s += __uint_as_float((uint32_t)a[i]) + __uint_as_float((uint32_t)(a[i] >> 32));
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 24); cudaMallocManaged(&cyc, 8);
  const int iters = 4096;
  auto run = [&](const char* name, auto kern, int chains, int warps) {
    kern<<<1, 32 * warps>>>(out, 1.0001f, cyc, iters); cudaDeviceSynchronize();
    kern<<<1, 32 * warps>>>(out, 1.0001f, cyc, iters); cudaDeviceSynchronize();
    printf("%-6s chains=%d warps=%2d: %.2f cycles per instruction per warp-chain-step (%.2f cyc/inst/SMSP)\n",
           name, chains, warps, (double)*cyc / (iters * chains), (double)*cyc / (iters * chains) / (warps > 4 ? warps / 4.0 : 1.0));
  };
  run("FFMA", k_ffma<1>, 1, 1);  run("FFMA2", k_ffma2<1>, 1, 1);
  run("FFMA", k_ffma<8>, 8, 1);  run("FFMA2", k_ffma2<8>, 8, 1);
  run("FFMA", k_ffma<8>, 8, 4);  run("FFMA2", k_ffma2<8>, 8, 4);
  run("FFMA", k_ffma<8>, 8, 16); run("FFMA2", k_ffma2<8>, 8, 16);
  run("FFMA", k_ffma<8>, 8, 32); run("FFMA2", k_ffma2<8>, 8, 32);
  return 0;
}
