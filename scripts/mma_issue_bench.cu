// Dev microbenchmark: tcgen05.mma (kind::f16, SS, M=128, cta_group::1)
// issue/execute rate vs N and vs the number of issuing warps.  Each issuing
// warp (converged, one elected lane) issues `iters` MMAs back to back into
// its own TMEM accumulator, then commits to its own mbarrier; the clock runs
// until every commit has completed.  Reports cycles per MMA (all warps) and
// the tensor-bound ideal (M*N*K*2 / 8192 flop per clock per SM).
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace moecu;
namespace moecu {
void note_launch() {}
}

template <int N>
__global__ void __launch_bounds__(128, 1) bench(int iters, int nwarps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t* at = base;              // 128 x 64 fp16 (16 KB)
  uint8_t* bt = base + 16384;      // N x 64 fp16
  __shared__ uint64_t done[4];
  __shared__ uint32_t tptr;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += 128) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&done[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tptr, 512);
  asm volatile("fence.proxy.async.shared::cta;");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tptr;
  constexpr uint32_t idesc = umma_idesc_f16(128, N);
  const uint64_t adesc = umma_desc_sw128(smem_u32(at));
  const uint64_t bdesc = umma_desc_sw128(smem_u32(bt));
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t d = tmem + (uint32_t)(warp * (512 / 4 >= N ? 128 : N)) % 512;
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) tc_mma_ss(d, adesc + (it & 3) * 2, bdesc + (it & 3) * 2, idesc, 1u);
      __syncwarp();
    }
    if (elect_one()) tc_commit(&done[warp]);
    __syncwarp();
    mbar_wait_warp(&done[warp], 0);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N>
void run(unsigned long long* d, int nsm) {
  const int smem = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int nw : {1, 2, 4}) {
    bench<N><<<nsm, 128, smem>>>(iters, nw, d);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<unsigned long long> h(nsm);
    cudaMemcpy(h.data(), d, nsm * 8, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (auto v : h) cyc += v;
    cyc /= nsm;
    printf("N=%3d issuers=%d: %.1f cycles per MMA (tensor ideal %.0f)  %s\n", N, nw,
           cyc / (iters * nw), 128.0 * N * 16 * 2 / 8192, cudaGetErrorString(e));
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* d;
  cudaMalloc(&d, nsm * 8);
  run<16>(d, nsm);
  run<32>(d, nsm);
  run<64>(d, nsm);
  run<128>(d, nsm);
  run<256>(d, nsm);
  return 0;
}
