// Can two CTAs that use tcgen05 (TMEM) share an SM?  grid = 2 x #SMs CTAs, each allocating
// COLS TMEM columns and SMEM_KB of shared memory, busy WORK ns: total time ~WORK when two CTAs
// run per SM, ~2 WORK when one.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_cores tmem_cores.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

template <int COLS, bool USE>
__global__ void k(int work_ns, float* out) {
  extern __shared__ float sm[];
  __shared__ uint32_t slot;
  if (USE && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "n"(COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  __syncthreads();
  float v = 1.f;
  const unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)work_ns) v = v * 0.999f + 1.f;
  sm[threadIdx.x] = v;
  __syncthreads();
  if (USE && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "n"(COLS) : "memory");
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

template <int COLS, bool USE>
void run(const char* name, int smem_kb, int sms, float* out) {
  auto f = k<COLS, USE>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) f<<<2 * sms, 192, smem_kb * 1024>>>(20000, out);
  cudaEventRecord(e0);
  f<<<2 * sms, 192, smem_kb * 1024>>>(20000, out);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 192, smem_kb * 1024);
  printf("%-28s smem %3d KB: %.1f us for 2x%d CTAs of 20 us (occupancy API says %d/SM) %s\n", name,
         smem_kb, ms * 1000, sms, occ, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096 * 4);
  run<256, false>("no tcgen05", 96, sms, out);
  run<256, true>("tcgen05 alloc 256 cols", 96, sms, out);
  run<128, true>("tcgen05 alloc 128 cols", 96, sms, out);
  run<512, true>("tcgen05 alloc 512 cols", 96, sms, out);
  run<256, true>("tcgen05 alloc 256 cols", 40, sms, out);
  return 0;
}
