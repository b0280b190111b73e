// Kernel-boundary latency probe: a CUDA graph of NK dependent PDL kernels (148 CTAs each, a
// fixed busy-wait of WORK ns per CTA) with the features our decode kernels carry toggled one by
// one: TMEM alloc/dealloc of 512 columns, an L2 bulk prefetch of PF MB at the end (split over the
// CTAs), cluster launch (2 or 8), 200 KB of shared memory, a stream-ordered (non-PDL) launch.
// Per-boundary overhead = (graph time - NK * WORK) / NK.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_probe sync_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

template <bool TM>
__global__ void k(int tmem, long long pf_bytes, const char* pf_src, int work_ns, float* buf) {
  extern __shared__ float sm[];
  __shared__ uint32_t slot;
  const int n = gridDim.x;
  if (TM && tmem && threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float v = buf[(blockIdx.x * 128 + threadIdx.x + 1) % (n * 128)];
  const unsigned long long t0 = gt();
  while (gt() - t0 < (unsigned long long)work_ns) v = v * 0.999f + 1.f;
  sm[threadIdx.x] = v;
  buf[blockIdx.x * 128 + threadIdx.x] = v;
  if (pf_bytes > 0 && threadIdx.x == 0) {
    const long long per = (pf_bytes / n) & ~4095LL;
    const char* p = pf_src + per * blockIdx.x;
    for (long long o = 0; o < per; o += 65536) {
      const uint32_t sz = (uint32_t)min(65536LL, per - o);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(sz) : "memory");
    }
  }
  __syncthreads();
  if (TM && tmem && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot) : "memory");
}

int main() {
  const int NK = 200;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf;
  char* big;
  const size_t BIG = (size_t)4 << 30;
  cudaMalloc(&buf, 1024 * 128 * 4);
  cudaMalloc(&big, BIG);
  cudaMemset(buf, 0, 1024 * 128 * 4);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  struct V { const char* name; int pdl, tmem, pf_mb, cl, smem_kb; int grid = 0; int thr = 0; };
  const V vs[] = {
      {"stream", 0, 0, 0, 1, 1},        {"pdl", 1, 0, 0, 1, 1},
      {"pdl smem200", 1, 0, 0, 1, 200}, {"pdl tmem", 1, 1, 0, 1, 200},
      {"pdl pf16", 1, 0, 16, 1, 200},   {"pdl pf4", 1, 0, 4, 1, 200},
      {"pdl cl2", 1, 0, 0, 2, 200},     {"pdl cl8", 1, 0, 0, 8, 1},
      {"pdl tmem cl2 pf16", 1, 1, 16, 2, 200},
      {"pdl cl8 g64", 1, 0, 0, 8, 1, 64},  {"pdl cl8 g128", 1, 0, 0, 8, 1, 128},
      {"pdl cl8 g512", 1, 0, 0, 8, 1, 512}, {"pdl cl4 g512", 1, 0, 0, 4, 1, 512},
      {"pdl cl2 g512", 1, 0, 0, 2, 1, 512}, {"pdl g512", 1, 0, 0, 1, 1, 512},
      {"pdl g64", 1, 0, 0, 1, 1, 64},
      {"pdl cl8 g512 t64", 1, 0, 0, 8, 1, 512, 64}, {"pdl g512 t64", 1, 0, 0, 1, 1, 512, 64},
  };
  for (int work : {2000, 5000}) {
    for (const V& v : vs) {
      const int grid = v.grid ? v.grid : v.cl > 1 ? sms / v.cl * v.cl - (v.cl == 8 ? 16 : 0) : sms;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < NK; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid); cfg.blockDim = dim3(v.thr ? v.thr : 128);
        cfg.dynamicSmemBytes = v.smem_kb * 1024; cfg.stream = s;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (v.pdl) {
          at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[na].val.programmaticStreamSerializationAllowed = 1;
          ++na;
        }
        if (v.cl > 1) {
          at[na].id = cudaLaunchAttributeClusterDimension;
          at[na].val.clusterDim.x = v.cl; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1;
          ++na;
        }
        cfg.attrs = at; cfg.numAttrs = na;
        const char* src = big + ((size_t)i * (64 << 20)) % (BIG - (64 << 20));
        if (v.tmem) cudaLaunchKernelEx(&cfg, k<true>, v.tmem, (long long)v.pf_mb << 20, src, work, buf);
        else cudaLaunchKernelEx(&cfg, k<false>, v.tmem, (long long)v.pf_mb << 20, src, work, buf);
      }
      cudaStreamEndCapture(s, &g);
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("%s: instantiate failed\n", v.name); continue; }
      for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
      const int R = 10;
      for (int r = 0; r < R; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(e1, s);
      cudaError_t err = cudaStreamSynchronize(s);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double per = ms * 1e3 / R / NK;
      printf("work %5d ns  %-20s grid %3d: %.2f us per kernel, boundary overhead %.2f us %s\n", work,
             v.name, grid, per, per - work / 1e3, err == cudaSuccess ? "" : cudaGetErrorString(err));
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  return 0;
}
