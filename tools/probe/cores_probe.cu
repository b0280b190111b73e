// Co-residency probe: primary A (192 threads, 160 KB smem, busy WORK ns, launch_dependents at
// entry; with or without a tcgen05 TMEM allocation) followed by a PDL dependent B (64 threads,
// optional cluster of 8, 512 CTAs).  Prints A's first entry / last exit and B's first entry,
// last entry and last wait-release, relative to A's first entry: shows whether B's CTAs can
// occupy SMs that hold an A CTA, and how long B's release takes after A ends.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cores_probe cores_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

template <bool TM>
__global__ void kA(int work_ns, unsigned long long* st) {
  extern __shared__ float sm[];
  __shared__ uint32_t slot;
  if (threadIdx.x == 0) st[blockIdx.x * 2] = gt();
  if (TM && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float v = 1.f;
  const unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)work_ns) v = v * 0.999f + 1.f;
  sm[threadIdx.x] = v;
  __syncthreads();
  if (TM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
  if (threadIdx.x == 0) st[blockIdx.x * 2 + 1] = gt();
}

__global__ void kB(unsigned long long* st) {
  if (threadIdx.x == 0) st[blockIdx.x * 2] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) st[blockIdx.x * 2 + 1] = gt();
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *sa, *sb;
  cudaMalloc(&sa, 4096 * 8); cudaMalloc(&sb, 4096 * 8);
  cudaFuncSetAttribute(kA<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kA<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaFuncSetAttribute(kB, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int acl : {1, 2}) {
    unsigned long long ha[4096], hb[4096];
    for (int rep = 0; rep < 3; ++rep) {
      cudaLaunchConfig_t c = {};
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      at[1].id = cudaLaunchAttributeClusterDimension;
      at[1].val.clusterDim.x = acl; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
      c.gridDim = dim3(108); c.blockDim = dim3(192); c.dynamicSmemBytes = 200 * 1024; c.stream = s;
      c.attrs = at; c.numAttrs = acl > 1 ? 2 : 1;
      cudaLaunchKernelEx(&c, kA<true>, 10000, sa);
      cudaLaunchConfig_t d = {};
      d.gridDim = dim3(148); d.blockDim = dim3(288); d.dynamicSmemBytes = 200 * 1024; d.stream = s;
      d.attrs = at; d.numAttrs = 1;
      cudaLaunchKernelEx(&d, kB, sb);
      cudaStreamSynchronize(s);
    }
    cudaError_t e = cudaGetLastError();
    cudaMemcpy(ha, sa, 108 * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb, sb, 148 * 16, cudaMemcpyDeviceToHost);
    unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b1 = 0;
    int early = 0;
    for (int i = 0; i < 108; ++i) { a0 = ha[2 * i] < a0 ? ha[2 * i] : a0; a1 = ha[2 * i + 1] > a1 ? ha[2 * i + 1] : a1; }
    for (int i = 0; i < 148; ++i) { b0 = hb[2 * i] < b0 ? hb[2 * i] : b0; b1 = hb[2 * i + 1] > b1 ? hb[2 * i + 1] : b1; }
    for (int i = 0; i < 148; ++i) early += hb[2 * i] < a1;
    printf("A cluster %d (108 CTAs, tcgen05, 200 KB) -> B (148 x 288, 200 KB): A end %.2f | B first entry %.2f, CTAs entered before A end %d, last release %.2f us %s\n",
           acl, (a1 - a0) / 1e3, ((long long)(b0 - a0)) / 1e3, early, ((long long)(b1 - a0)) / 1e3,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  for (int co : {-1, 100})
  for (int tm = 0; tm < 2; ++tm)
    for (int cl : {1, 8})
      for (int gA : {144, 148}) {
        cudaFuncSetAttribute(kB, cudaFuncAttributePreferredSharedMemoryCarveout, co);
        unsigned long long ha[4096], hb[4096];
        for (int rep = 0; rep < 3; ++rep) {
          cudaLaunchConfig_t c = {};
          cudaLaunchAttribute at[2];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1;
          c.gridDim = dim3(gA); c.blockDim = dim3(192); c.dynamicSmemBytes = 160 * 1024; c.stream = s;
          c.attrs = at; c.numAttrs = 1;
          if (tm) cudaLaunchKernelEx(&c, kA<true>, 10000, sa);
          else cudaLaunchKernelEx(&c, kA<false>, 10000, sa);
          cudaLaunchConfig_t d = {};
          d.gridDim = dim3(512); d.blockDim = dim3(64); d.dynamicSmemBytes = 0; d.stream = s;
          at[1].id = cudaLaunchAttributeClusterDimension;
          at[1].val.clusterDim.x = cl; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
          d.attrs = at; d.numAttrs = cl > 1 ? 2 : 1;
          cudaLaunchKernelEx(&d, kB, sb);
          cudaStreamSynchronize(s);
        }
        cudaError_t e = cudaGetLastError();
        cudaMemcpy(ha, sa, gA * 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(hb, sb, 512 * 16, cudaMemcpyDeviceToHost);
        unsigned long long a0 = ~0ull, a1 = 0, b0 = ~0ull, b0max = 0, b1 = 0;
        for (int i = 0; i < gA; ++i) { a0 = ha[2 * i] < a0 ? ha[2 * i] : a0; a1 = ha[2 * i + 1] > a1 ? ha[2 * i + 1] : a1; }
        for (int i = 0; i < 512; ++i) {
          b0 = hb[2 * i] < b0 ? hb[2 * i] : b0;
          b0max = hb[2 * i] > b0max ? hb[2 * i] : b0max;
          b1 = hb[2 * i + 1] > b1 ? hb[2 * i + 1] : b1;
        }
        printf("B carveout %4d | A tcgen05=%d grid %d | B cluster %d: A end %.2f | B first entry %.2f, last entry %.2f, last release %.2f us %s\n",
               co, tm, gA, cl, (a1 - a0) / 1e3, ((long long)(b0 - a0)) / 1e3, ((long long)(b0max - a0)) / 1e3,
               ((long long)(b1 - a0)) / 1e3, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
