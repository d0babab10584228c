// Dev microbenchmark: raw tcgen05.mma kind::f16 issue rate on one SM per CTA
// (no loads): TS (A in TMEM) vs SS (A in smem), N = 64/128/256, M = 128.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2211_10017_b200/csrc mma_bench.cu
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace moecu;
namespace moecu {
void note_launch() {}
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, unsigned long long* out, int rnd) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t* bt = base;              // N x 64 fp16, SW128 K-major
  uint8_t* at = base + 256 * 128;  // 128 x 64 fp16
  __shared__ uint64_t bar;
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (256 * 128 + 128 * 128) / 4; i += 128)
    reinterpret_cast<uint32_t*>(base)[i] = rnd ? ((i * 2654435761u) & 0x3BFF3BFFu) : 0u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tptr, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(128, N);
    const uint64_t bdesc = umma_desc_sw128(smem_u32(bt));
    const uint64_t adesc = umma_desc_sw128(smem_u32(at));
    // warm-up
    for (int kk = 0; kk < 4; ++kk) {
      if (TS)
        tc_mma_ts(tmem, tmem + 256 + kk * 8, bdesc + kk * 2, idesc, kk);
      else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(adesc + kk * 2), "l"(bdesc + kk * 2), "r"(idesc), "r"(kk));
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          tc_mma_ts(tmem, tmem + 256 + kk * 8, bdesc + kk * 2, idesc, 1);
        else
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(adesc + kk * 2), "l"(bdesc + kk * 2), "r"(idesc), "r"(1));
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 1);
    const unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N, bool TS>
void run(int nsm, int rnd) {
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  const int smem = 256 * 128 + 128 * 128 + 1024;
  cudaFuncSetAttribute(mma_bench<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mma_bench<N, TS><<<nsm, 128, smem>>>(iters, d, rnd);
  cudaEventRecord(a);
  mma_bench<N, TS><<<nsm, 128, smem>>>(iters, d, rnd);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (auto v : h) cyc += v;
  cyc /= nsm;
  const double per = cyc / (iters * 4.0);
  const double macs = 128.0 * N * 16;
  const double flops = 2.0 * macs * iters * 4 * nsm;
  printf("rnd=%d %s N=%3d: %.1f cycles/MMA (ideal %d), %.0f MAC/clk/SM, %.0f TFLOP/s, clk=%.0f MHz  err=%s\n",
         rnd, TS ? "TS" : "SS", N, per, 128 * N / 256, macs / per, flops / (ms * 1e-3) / 1e12,
         cyc / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int rnd = 0; rnd < 2; ++rnd) {
    run<128, true>(nsm, rnd);
    run<256, true>(nsm, rnd);
    run<128, false>(nsm, rnd);
    run<256, false>(nsm, rnd);
  }
  return 0;
}
