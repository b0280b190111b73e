// Probe: where does a tcgen05.mma M=64 (cta_group::1, kind::f16) accumulator land in TMEM?
// A = 64 x 64 bf16 (row r = r + 1 at column 0, else 0), B = 256 x 64 bf16 (row n: 1 at column 0,
// else 0) -> D[r][n] = r + 1.  Four warps dump lanes 0..127, column 0 with 32x32b loads.
// nvcc -gencode arch=compute_100a,code=sm_100a -o m64 m64_layout.cu && ./m64
#include <cuda.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include "../../paper_2505_14468_b200/csrc/tc_ptx.cuh"
using namespace slx::tc;

__global__ void probe(float* out, int M) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __nv_bfloat16* A = (__nv_bfloat16*)buf;             // [128][64] SW128 (rows >= M zero)
  __nv_bfloat16* B = (__nv_bfloat16*)(buf + 16384);   // [256][64] SW128
  uint64_t* bar = (uint64_t*)(buf + 16384 + 32768);
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fill with the 128B swizzle: element (row, col) at row*128 + ((col/8) ^ (row%8))*16 + (col%8)*2
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    const float av = (c == 0 && r < M) ? (float)(r + 1) : 0.f;
    *(__nv_bfloat16*)((uint8_t*)A + r * 128 + (((c / 8) ^ (r % 8)) * 16) + (c % 8) * 2) = __float2bfloat16(av);
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64, c = i % 64;
    *(__nv_bfloat16*)((uint8_t*)B + r * 128 + (((c / 8) ^ (r % 8)) * 16) + (c % 8) * 2) = __float2bfloat16(c == 0 ? 1.f : 0.f);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&tslot, 256);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t t = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_bf16_f32(M, 256);
    for (int ks = 0; ks < 4; ++ks)
      mma_bf16_ss(t, smem_desc_sw128(smem_u32(A) + ks * 32), smem_desc_sw128(smem_u32(B) + ks * 32), idesc, ks ? 1u : 0u);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  fence_after_sync();
  float v[16];
  tmem_ld16(t + ((uint32_t)(warp * 32) << 16), v);
  out[warp * 32 + lane] = v[0];
  out[128 + warp * 32 + lane] = v[5];
  fence_before_sync();
  __syncthreads();
  if (warp == 0) { fence_after_sync(); tmem_dealloc(t, 256); }
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int M : {128, 64}) {
    cudaMemset(d, 0, 256 * 4);
    probe<<<1, 128, 64 * 1024>>>(d, M);
    float h[256];
    cudaError_t e = cudaMemcpy(h, d, 256 * 4, cudaMemcpyDeviceToHost);
    printf("M=%d (%s): lane -> D[.,0] (D[.,5])\n", M, cudaGetErrorString(e));
    for (int w = 0; w < 4; ++w) {
      printf("  warp %d:", w);
      for (int l = 0; l < 32; ++l) printf(" %g", h[w * 32 + l]);
      printf("   |5: %g %g\n", h[128 + w * 32], h[128 + w * 32 + 16]);
    }
  }
  return 0;
}
