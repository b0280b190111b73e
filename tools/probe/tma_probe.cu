// Streaming-bandwidth probe on B200: how fast can CTAs pull a large buffer into shared memory
// with (a) 2D tensor TMA boxes of 128x64 bf16 (16 KB), (b) 1D cp.async.bulk of 16 KB,
// (c) plain 16-byte ld.global; consumer releases each stage immediately.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(dst)), "l"(m), "r"(su32(b)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(su32(dst)), "l"(src), "r"(n), "r"(su32(b)) : "memory");
}

// mode 0: tensor TMA, mode 1: 1D bulk.  Each CTA streams boxes b = cta, cta+grid, ...
__global__ void stream_tma(const __grid_constant__ CUtensorMap map, const uint8_t* base, long n_boxes,
                           int stages, int mode, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(buf + stages * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long i = 0;
  float acc = 0.f;
  long my = 0;
  for (long b = blockIdx.x; b < n_boxes; b += gridDim.x) ++my;
  // prime
  long issued = 0, done = 0;
  long next_box = blockIdx.x;
  auto issue = [&](long k) {
    const int s = k % stages;
    expect_tx(&full[s], 16384);
    if (mode == 0) tma2d(buf + s * 16384, &map, &full[s], 0, (int)(next_box * 128));
    else bulk1d(buf + s * 16384, base + next_box * 16384, 16384, &full[s]);
    next_box += gridDim.x;
  };
  for (; issued < my && issued < stages; ++issued) issue(issued);
  for (; done < my; ++done) {
    const int s = done % stages;
    mwait(&full[s], (done / stages) & 1);
    acc += ((volatile float*)(buf + s * 16384))[0];
    if (issued < my) { issue(issued); ++issued; }
  }
  (void)i;
  if (acc == 12345.f) sink[0] = acc;
}

__global__ void stream_ldg(const uint4* p, long n16, float* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc.x ^= v.x;
  }
  if (acc.x == 0x12345) sink[0] = 1.f;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = 2ull << 30;  // 2 GiB
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  float* sink;
  cudaMalloc(&sink, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  Enc enc = (Enc)fp;
  CUtensorMap map;
  const long rows = bytes / 128;
  cuuint64_t dims[2] = {64, (cuuint64_t)rows};
  cuuint64_t str[1] = {128};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  cudaFuncSetAttribute(stream_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(stream_tma, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  const long n_boxes = bytes / 16384;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 2; ++mode)
    for (int ctas = 1; ctas <= 4; ctas *= 2)
      for (int stages = 2; stages <= 12; stages += 2) {
        const size_t smem = (size_t)stages * 16384 + 1024 + 256;
        if (smem * ctas > 220 * 1024) continue;
        const int grid = sms * ctas;
        stream_tma<<<grid, 32, smem>>>(map, buf, n_boxes, stages, mode, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) stream_tma<<<grid, 32, smem>>>(map, buf, n_boxes, stages, mode, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"stages\": %d, \"GB/s\": %.1f, \"err\": \"%s\"}\n",
               mode ? "bulk1d" : "tma2d", ctas, stages, 3.0 * bytes / (ms * 1e6),
               cudaGetErrorString(cudaGetLastError()));
      }
  for (int tpb = 256; tpb <= 1024; tpb *= 2) {
    const int grid = sms * (2048 / tpb);
    stream_ldg<<<grid, tpb>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) stream_ldg<<<grid, tpb>>>((const uint4*)buf, bytes / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"mode\": \"ldg128\", \"tpb\": %d, \"GB/s\": %.1f}\n", tpb, 3.0 * bytes / (ms * 1e6));
  }
  return 0;
}
