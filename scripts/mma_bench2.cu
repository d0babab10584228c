// Dev microbenchmark 2: what slows tcgen05.mma inside a pipelined loop?
//   mode 0: back-to-back MMAs (4 per "k-block"), no sync
//   mode 1: + per k-block tcgen05.commit to an mbarrier (never waited)
//   mode 2: + per k-block wait on a pre-completed mbarrier + fence::after
//   mode 3: + concurrent 1-D bulk copies (warp 2) into a separate smem region
//   mode 4: + per k-block commit and WAIT for that commit (serialises MMA)
//   mode 5: like 2 but the waiting is done by the whole warp, lane 0 issues
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace moecu;
namespace moecu {
void note_launch() {}
}

template <int N>
__global__ void __launch_bounds__(128, 1) bench(int iters, int mode, const uint8_t* gsrc,
                                                unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t* bt = base;                // N x 64 fp16
  uint8_t* cp_dst = base + 32768;    // 64 KB landing zone for bulk copies
  __shared__ uint64_t bar, bar2, cbar;
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 32768 / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&cbar, 1);
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tptr, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  if (threadIdx.x == 0) mbar_arrive(&bar2);  // bar2 phase 0 complete
  __syncthreads();
  constexpr uint32_t idesc = umma_idesc_f16(128, N);
  const uint64_t bdesc = umma_desc_sw128(smem_u32(bt));
  if (warp == 1 && (mode == 2 || mode == 5 || mode == 3 || mode == 4)) {
    // issuer in warp 1 (like the GEMM kernel)
  }
  if ((mode != 5 && threadIdx.x == 32) || (mode == 5 && warp == 1)) {
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      if (mode >= 2 && mode != 4) {
        mbar_wait(&bar2, 0);
        tc_fence_after();
      }
      if (mode != 5 || lane == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_ts(tmem, tmem + 256 + kk * 8, bdesc + kk * 2, idesc, 1);
        if (mode >= 1) tc_commit(mode == 4 ? &cbar : &bar);
      }
      if (mode == 5) __syncwarp();
      if (mode == 4) {
        mbar_wait(&cbar, ph);
        ph ^= 1;
      }
    }
    if (lane == 0) {
      tc_commit(&cbar);
      mbar_wait(&cbar, ph);
      out[blockIdx.x] = clock64() - t0;
    }
    stop = 1;
  }
  if (mode == 3 && warp == 2 && lane == 0) {
    uint32_t ph = 0;
    int n = 0;
    while (!stop && n < 100000) {
      mbar_arrive_expect_tx(&bar, 0);  // keep bar's phase moving harmlessly
      mbar_arrive_expect_tx(&cbar, 0);
      uint64_t b3;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], 16384;"
                   : "=l"(b3) : "r"(smem_u32(&bar2)));
      bulk_load(cp_dst + (n & 3) * 16384, gsrc + (size_t)(n % 512) * 16384, 16384, &bar2);
      ++n;
      (void)ph;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N>
void run(int nsm, int mode, const uint8_t* g) {
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  const int smem = 32768 + 65536 + 1024;
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  bench<N><<<nsm, 128, smem>>>(iters, mode, g, d);
  cudaDeviceSynchronize();
  bench<N><<<nsm, 128, smem>>>(iters, mode, g, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(nsm);
  cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (auto v : h) cyc += v;
  cyc /= nsm;
  printf("N=%d mode=%d: %.1f cycles per k-block of 4 MMAs (ideal %d)  err=%s\n", N, mode,
         cyc / iters, 4 * 128 * N / 256, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* g;
  cudaMalloc(&g, 512 * 16384);
  cudaMemset(g, 0, 512 * 16384);
  for (int mode : {0, 1, 2, 5, 4}) run<128>(nsm, mode, g);
  for (int mode : {0, 2, 5}) run<256>(nsm, mode, g);
  return 0;
}
