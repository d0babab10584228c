// Dev microbenchmark 3: does SS-mode tcgen05.mma (N=256) keep full rate while
// shared memory also absorbs (a) STS.128 stores from 8 warps and/or (b) 1-D
// bulk (TMA) copies from global?  Thread 0 issues 4 MMAs per "k-block" with a
// single-thread wait on a pre-completed barrier + commit, like the GEMM loop.
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace moecu;
namespace moecu {
void note_launch() {}
}

constexpr int kThreads = 384;

__global__ void __launch_bounds__(kThreads, 1) bench(int iters, int mode, const uint8_t* gsrc,
                                                     unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t* bt = base;               // 256 x 64 fp16 (32 KB)
  uint8_t* at = base + 32768;       // 128 x 64 fp16 (16 KB)
  uint8_t* sts_dst = base + 49152;  // 16 KB STS target
  uint8_t* cp_dst = base + 65536;   // 4 x 16 KB bulk-copy target
  __shared__ uint64_t bar, cbar, cpbar[4];
  __shared__ uint32_t tptr;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 49152 / 4; i += kThreads) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&cbar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&cpbar[i], 1);
    stop = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tptr, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  if (threadIdx.x == 0) mbar_arrive(&bar);
  __syncthreads();
  unsigned long long sts_bytes = 0, cp_bytes = 0;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_f16(128, 256);
    const uint64_t bdesc = umma_desc_sw128(smem_u32(bt));
    const uint64_t adesc = umma_desc_sw128(smem_u32(at));
    const unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&bar, 0);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (it & 1) * 256),
            "l"(adesc + kk * 2), "l"(bdesc + kk * 2), "r"(idesc), "r"(1));
      tc_commit(&cbar);
    }
    tc_commit(&cbar);
    // drain: wait for the last commit's phase
    asm volatile("tcgen05.fence::before_thread_sync;");
    (void)ph;
    unsigned long long t1 = clock64();
    // crude completion wait: poll until barrier count settles
    for (int i = 0; i < 4096; ++i) __nanosleep(64);
    out[blockIdx.x * 4 + 0] = t1 - t0;
    stop = 1;
  } else if (warp >= 4 && (mode & 1)) {
    // 8 warps of STS.128 into a 16 KB region
    uint4 v = make_uint4(lane, warp, 1, 2);
    int n = 0;
    while (!stop) {
#pragma unroll 8
      for (int i = 0; i < 8; ++i) {
        const int idx = ((warp - 4) * 32 + lane + i * 256) & 1023;
        reinterpret_cast<uint4*>(sts_dst)[idx] = v;
      }
      n += 8;
    }
    sts_bytes = (unsigned long long)n * 16;
  } else if (warp == 2 && lane == 0 && (mode & 2)) {
    int n = 0;
    while (!stop) {
      const int b = n & 3;
      if (n >= 4) mbar_wait(&cpbar[b], ((n >> 2) - 1) & 1);
      mbar_arrive_expect_tx(&cpbar[b], 16384);
      bulk_load(cp_dst + b * 16384, gsrc + (size_t)(n % 4096) * 16384, 16384, &cpbar[b]);
      ++n;
    }
    for (int b = 0; b < 4 && b < n; ++b) {
      const int last = n - 1 - ((n - 1 - b) & 3);
      (void)last;
    }
    cp_bytes = (unsigned long long)n * 16384;
    for (int i = 0; i < 4096; ++i) __nanosleep(64);  // let copies land
  }
  if (sts_bytes) atomicAdd(&out[blockIdx.x * 4 + 1], sts_bytes);
  if (cp_bytes) atomicAdd(&out[blockIdx.x * 4 + 2], cp_bytes);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* g;
  cudaMalloc(&g, (size_t)4096 * 16384);
  cudaMemset(g, 0, (size_t)4096 * 16384);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 32);
  const int smem = 65536 + 65536 + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int mode : {0, 1, 2, 3}) {
    cudaMemset(d, 0, nsm * 32);
    bench<<<nsm, kThreads, smem>>>(iters, mode, g, d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(nsm * 4);
    cudaMemcpy(h.data(), d, nsm * 32, cudaMemcpyDeviceToHost);
    double cyc = 0, sts = 0, cp = 0;
    for (int i = 0; i < nsm; ++i) {
      cyc += h[i * 4];
      sts += h[i * 4 + 1];
      cp += h[i * 4 + 2];
    }
    cyc /= nsm;
    sts /= nsm;
    cp /= nsm;
    printf("mode=%d (1=STS 2=TMA): %.1f cycles per 4 SS-MMAs N=256 (ideal 512); STS %.1f B/clk, TMA %.1f B/clk  %s\n",
           mode, cyc / iters, sts / cyc, cp / cyc, cudaGetErrorString(e));
  }
  return 0;
}
