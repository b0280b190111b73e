// Host-side helpers shared by the tcgen05 GEMM translation units (gemm_tc.cu, gemm_sk.cu).
#pragma once

#include <cuda.h>
#include <stddef.h>

#include "../../include/slora_b200.h"

namespace slx {
// K-major bf16 matrix [rows, cols] with row stride ld (elements); TMA box = box_rows x 64,
// SWIZZLE_128B (the tcgen05 smem descriptor layout).
bool make_tmap(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, int box_rows);
// Max dynamic smem opt-in + smem-heavy carveout for a kernel (idempotent).
void configure_kernel(const void* k);

// Stream-K decode GEMM (gemm_sk.cu).  Returns SLX_ERR_UNSUPPORTED when the shape is outside
// its envelope (M > 64, row-major W, workspace too small, tuning->tile_kernel), so the caller
// can use gemm_tc.
struct SkCall {
  const void* A; int lda; const void* W; void* C; int ldc; int c_dtype;
  const void* R; int ldr; int M, N, K, epilogue, n_main; void* C2; int ldc2;
  void* ws; size_t ws_bytes; void* stream; unsigned long long* trace;
  const slx_l2_prefetch* pf;
  float* part_out;    // slx_gemm_bf16_splitk: pieces out (no epilogue), `splits` per tile
  int splits;
  size_t part_bytes;
  const slx_gemm_tuning* tuning;   // explicit tiling (tests / tools); nullptr = planner
};
int gemm_sk_launch(const SkCall& c);
// Debug timeline window for the next traced launch (nullptr when tracing is off); kinds:
// 1-3 GEMM (epilogue + 1), 4 split-K GEMM, 5 decode attention.
unsigned long long* next_trace_window(int kind);
size_t gemm_sk_workspace_bytes(int M, int N, int K);
size_t gemm_sk_splitk_bytes(int M, int N, int splits);
}  // namespace slx
