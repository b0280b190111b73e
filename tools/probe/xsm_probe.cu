// Cross-SM exchange latency probe: G CTAs each write a 64 KB fp32 "piece", arrive on a counter
// (red.release), wait for all (ld.acquire), then read a peer's piece.  Variants of the load path.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xsm_probe xsm_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

template <int MODE>
__global__ void __launch_bounds__(128) probe(float* part, unsigned* cnt, unsigned long long* tr, int G,
                                             float* sink) {
  const int c = blockIdx.x, t = threadIdx.x;
  float* mine = part + (size_t)c * 16384;
  unsigned base = 0;
  if (t == 0) { asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(base) : "l"(cnt + 1)); tr[c * 8 + 0] = gt(); }
  // write 64 KB: thread t writes 128 float4 (warp-coalesced 512 B rows)
  for (int i = 0; i < 32; ++i) {
    float4 v = make_float4(c + i, t, 1.f, 2.f);
    if (MODE == 2) __stcg(reinterpret_cast<float4*>(mine) + i * 128 + t, v);
    else reinterpret_cast<float4*>(mine)[i * 128 + t] = v;
  }
  __syncthreads();
  if (t == 0) {
    tr[c * 8 + 1] = gt();
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
    tr[c * 8 + 2] = gt();
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v - base < (unsigned)G);
    tr[c * 8 + 3] = gt();
  }
  __syncthreads();
  const float* peer = part + (size_t)((c + 37) % G) * 16384;
  float acc = 0.f;
  float4 q[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float4* p = reinterpret_cast<const float4*>(peer) + i * 128 + t;
    if (MODE == 1) q[i] = *p; else q[i] = __ldcg(p);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += q[i].x + q[i].y + q[i].z + q[i].w;
  if (t == 0) tr[c * 8 + 4] = gt();
  // second read of the same data (now warm)
#pragma unroll
  for (int i = 0; i < 32; ++i) q[i] = __ldcg(reinterpret_cast<const float4*>(peer) + i * 128 + t);
#pragma unroll
  for (int i = 0; i < 32; ++i) acc += q[i].x;
  if (t == 0) tr[c * 8 + 5] = gt();
  sink[c * 128 + t] = acc;
  __syncthreads();
  if (t == 0) { atomicAdd(cnt + 1, 1u); tr[c * 8 + 6] = gt(); }
}

int main() {
  const int G = 148;
  float *part, *sink; unsigned* cnt; unsigned long long* tr;
  cudaMalloc(&part, (size_t)G * 65536); cudaMalloc(&sink, G * 128 * 4);
  cudaMalloc(&cnt, 64); cudaMemset(cnt, 0, 64);
  cudaMalloc(&tr, G * 8 * 8);
  unsigned long long h[G * 8];
  const char* names[] = {"ldcg", "ld.ca", "stcg+ldcg"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(tr, 0, G * 64);
      if (mode == 0) probe<0><<<G, 128>>>(part, cnt, tr, G, sink);
      if (mode == 1) probe<1><<<G, 128>>>(part, cnt, tr, G, sink);
      if (mode == 2) probe<2><<<G, 128>>>(part, cnt, tr, G, sink);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, tr, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < G; ++c) t0 = h[c * 8] < t0 ? h[c * 8] : t0;
    double mx[7] = {0}, sm[7] = {0};
    for (int c = 0; c < G; ++c)
      for (int k = 0; k < 7; ++k) { double v = (h[c * 8 + k] - t0) / 1000.0; sm[k] += v / G; mx[k] = v > mx[k] ? v : mx[k]; }
    printf("%-10s", names[mode]);
    const char* ph[] = {"start", "written", "arrived", "allin", "read1", "read2", "depart"};
    for (int k = 0; k < 7; ++k) printf(" %s %.2f/%.2f", ph[k], sm[k], mx[k]);
    printf("   (mean/max us)\n");
  }
  return 0;
}
