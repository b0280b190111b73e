// tcgen05 issue-rate probe: one CTA per SM, one thread issues `iters` k-blocks of 4 MMAs
// (M=128, N=n, K=16, bf16 SS, smem resident), optionally committing to an mbarrier after each
// k-block and waiting `lag` k-blocks behind (like a smem ring of `lag` stages).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include "../../paper_2505_14468_b200/csrc/tc_ptx.cuh"
using namespace slx::tc;

__global__ void mma_probe(int n, int iters, int commit_every, int lag, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(buf + 64 * 1024);
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tslot, 256);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, n);
    const uint32_t a = smem_u32(buf), b = smem_u32(buf + 32 * 1024);
    for (int i = 0; i < iters; ++i) {
      if (commit_every && i >= lag) mbar_wait(&bars[(i - lag) % 16], ((i - lag) / 16) & 1);
      for (int ks = 0; ks < 4; ++ks)
        mma_bf16_ss(t, smem_desc_sw128(a + ks * 32), smem_desc_sw128(b + ks * 32), idesc, (i | ks) ? 1u : 0u);
      if (commit_every) mma_commit(&bars[i % 16]);
    }
    mma_commit(&bars[15]);
  }
  __syncthreads();
  fence_before_sync();
  __syncthreads();
  if (warp == 0) { fence_after_sync(); tmem_dealloc(t, 256); }
  if (threadIdx.x == 0 && iters < 0) sink[0] = 1.f;
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  for (int n = 64; n <= 256; n *= 2)
    for (int ce = 0; ce <= 1; ++ce)
      for (int lag = 1; lag <= (ce ? 8 : 1); lag *= 2) {
        mma_probe<<<sms, 128, 100 * 1024>>>(n, iters, ce, lag, sink);
        cudaEventRecord(e0);
        mma_probe<<<sms, 128, 100 * 1024>>>(n, iters, ce, lag, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double cyc = ms * 1e-3 * 1.9e9 / (iters * 4.0);
        printf("{\"N\": %d, \"commit\": %d, \"lag\": %d, \"us\": %.1f, \"ns_per_mma\": %.1f, \"cyc_per_mma@1.9GHz\": %.1f, \"err\": \"%s\"}\n",
               n, ce, lag, ms * 1e3, ms * 1e6 / (iters * 4.0), cyc, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
