// K1: backbone projection GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C[M,N] = A[M,K] . W[N,K]^T  (+ residual | SiLU*mul epilogue), bf16 in, fp32 accumulate.
//
// Two tilings of one warp-specialised kernel (warp 0 lane 0: TMA producer, warp 1 lane 0:
// MMA issuer, all 4 warps: TMEM -> register epilogue):
//  * NORMAL (prefill, M > 128): D tile = 128 rows of A x BN rows of W, TMEM lane = token.
//  * SWAP   (decode,  M <= 128): D tile = 128 rows of W x BN(=M padded to 16) tokens,
//    TMEM lane = output feature.  The weight stream is split along K over `splits` CTAs
//    so that all 148 SMs pull weights; partial tiles are reduced deterministically by the
//    last-arriving CTA (tile counter, split order 0..S-1), which applies the epilogue.
// SiLU*mul: W rows are blocked [gate 128 | up 128] per 128 output features, so one TMEM
// row (NORMAL) or two accumulators of one CTA (SWAP, nsub = 2) hold gate and up together.
//
// Replaces the modelled prefill/decode time of the reference (batching.py:17-21 T0+alpha(b-1);
// engine.py:832 prefill work, engine.py:888,909 decode_ms_per_token) with the real projections.
#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace slx {

constexpr int TC_THREADS = 128;
constexpr int TC_BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int TC_MAX_STAGES = 8;
constexpr int P_TILE_BYTES = 128 * TC_BK * 2;  // 16 KB
constexpr size_t TC_CNT_BYTES = 64 * 1024;     // split-K tile counters (<= 16384 tiles)

struct GemmArgs {
  int M, N, K;
  int bn;       // UMMA N
  int nsub;     // P sub-tiles per CTA (SWAP SiLU: 2)
  int stages;
  int kblocks;
  int splits;
  int n_tiles;
  void* C;
  int ldc;
  const void* R;
  int ldr;
  float* part;
  int* cnt;
};

template <typename OutT>
__device__ __forceinline__ void store_out(OutT* p, float v) {
  *p = from_f32<OutT>(v);
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

template <bool SWAP, int EPI, typename OutT>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_p, const __grid_constant__ CUtensorMap tmap_q,
               GemmArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int q_tile_bytes = g.bn * TC_BK * 2;
  const int stage_bytes = g.nsub * P_TILE_BYTES + q_tile_bytes;
  uint64_t* full = (uint64_t*)(smem + g.stages * stage_bytes);
  uint64_t* empty = full + TC_MAX_STAGES;
  uint64_t* accum = empty + TC_MAX_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(accum + 1);
  __shared__ int is_last_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int split = SWAP ? blockIdx.y : 0;
  const int kb_per = (g.kblocks + g.splits - 1) / g.splits;
  const int kb_lo = split * kb_per;
  const int kb_hi = min(g.kblocks, kb_lo + kb_per);
  const int n_kb = kb_hi - kb_lo;
  // P rows (TMEM lanes) and Q rows (TMEM columns) of this tile
  const int p_row0 = SWAP ? tile * 128 * g.nsub : blockIdx.y * 128;
  const int q_row0 = SWAP ? 0 : tile * g.bn;
  const uint32_t tmem_cols_alloc = (g.nsub * g.bn <= 32) ? 32 : (g.nsub * g.bn <= 64) ? 64
                                   : (g.nsub * g.bn <= 128) ? 128 : (g.nsub * g.bn <= 256) ? 256 : 512;

  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmap_p);
    tc::tma_prefetch_desc(&tmap_q);
    for (int s = 0; s < g.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(accum, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, tmem_cols_alloc);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t pol_p = SWAP ? tc::policy_evict_first() : tc::policy_evict_last();
    const uint64_t pol_q = SWAP ? tc::policy_evict_last() : tc::policy_evict_first();
    for (int i = 0; i < n_kb; ++i) {
      const int s = i % g.stages;
      tc::mbar_wait(&empty[s], ((i / g.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int kc = (kb_lo + i) * TC_BK;
      for (int sub = 0; sub < g.nsub; ++sub)
        tc::tma_load_2d(st + sub * P_TILE_BYTES, &tmap_p, &full[s], kc, p_row0 + sub * 128, pol_p);
      tc::tma_load_2d(st + g.nsub * P_TILE_BYTES, &tmap_q, &full[s], kc, q_row0, pol_q);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread)
    const uint32_t idesc = tc::idesc_bf16_f32(128, g.bn);
    for (int i = 0; i < n_kb; ++i) {
      const int s = i % g.stages;
      tc::mbar_wait(&full[s], (i / g.stages) & 1);
      tc::fence_after_sync();
      const uint32_t st = tc::smem_u32(smem + s * stage_bytes);
      const uint32_t q_addr = st + g.nsub * P_TILE_BYTES;
#pragma unroll
      for (int ks = 0; ks < TC_BK / 16; ++ks) {
        const uint64_t bdesc = tc::smem_desc_sw128(q_addr + ks * 32);
        for (int sub = 0; sub < g.nsub; ++sub) {
          const uint64_t adesc = tc::smem_desc_sw128(st + sub * P_TILE_BYTES + ks * 32);
          tc::mma_bf16_ss(tmem_base + sub * g.bn, adesc, bdesc, idesc, (i > 0 || ks > 0) ? 1u : 0u);
        }
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(accum);
  }

  // ---------------- epilogue: all 4 warps; warp w owns TMEM lanes [32w, 32w+32)
  tc::mbar_wait(accum, 0);
  __syncwarp();
  tc::fence_after_sync();
  const int r = warp * 32 + lane;
  const uint32_t t_row = tmem_base + ((uint32_t)(warp * 32) << 16);
  OutT* C = reinterpret_cast<OutT*>(g.C);
  const OutT* R = reinterpret_cast<const OutT*>(g.R);

  if (!SWAP) {
    const int m = p_row0 + r;
    if (EPI == SLX_EPI_SILU_MUL) {
      for (int c0 = 0; c0 < 128; c0 += 16) {
        float gv[16], uv[16];
        tc::tmem_ld16(t_row + c0, gv);
        tc::tmem_ld16(t_row + 128 + c0, uv);
        const int f0 = tile * 128 + c0;
        if (m < g.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (f0 + j < g.N / 2) store_out(C + (size_t)m * g.ldc + f0 + j, silu_f(gv[j]) * uv[j]);
        }
      }
    } else {
      for (int c0 = 0; c0 < g.bn; c0 += 16) {
        float v[16];
        tc::tmem_ld16(t_row + c0, v);
        const int n0 = q_row0 + c0;
        if (m < g.M) {
          if (EPI == SLX_EPI_RESIDUAL) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + j < g.N) v[j] += to_f32(R[(size_t)m * g.ldr + n0 + j]);
          }
          if (n0 + 16 <= g.N && sizeof(OutT) == 2) {
            Vec8<bf16>::store((bf16*)(C + (size_t)m * g.ldc + n0), v);
            Vec8<bf16>::store((bf16*)(C + (size_t)m * g.ldc + n0 + 8), v + 8);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + j < g.N) store_out(C + (size_t)m * g.ldc + n0 + j, v[j]);
          }
        }
      }
    }
  } else {
    // SWAP: TMEM lane r = output feature row, column c = token
    const int nrows_total = g.nsub * 128;
    if (g.splits > 1) {
      float* part = g.part + ((size_t)(split * g.n_tiles + tile) * g.nsub) * g.bn * 128;
      for (int sub = 0; sub < g.nsub; ++sub)
        for (int c0 = 0; c0 < g.bn; c0 += 16) {
          float v[16];
          tc::tmem_ld16(t_row + sub * g.bn + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) part[((size_t)sub * g.bn + c0 + j) * 128 + r] = v[j];
        }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int old = atomicAdd(&g.cnt[tile], 1);
        is_last_s = (old == g.splits - 1);
      }
      __syncthreads();
      if (!is_last_s) goto teardown;
      __threadfence();
    }
    for (int c0 = 0; c0 < g.bn; c0 += 16) {
      float v[2][16];
      for (int sub = 0; sub < g.nsub; ++sub) {
        if (g.splits == 1) {
          tc::tmem_ld16(t_row + sub * g.bn + c0, v[sub]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[sub][j] = 0.f;
          for (int s = 0; s < g.splits; ++s) {
            const float* p = g.part + ((size_t)(s * g.n_tiles + tile) * g.nsub + sub) * g.bn * 128;
#pragma unroll
            for (int j = 0; j < 16; ++j) v[sub][j] += __ldcg(p + (size_t)(c0 + j) * 128 + r);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = c0 + j;
        if (m >= g.M) break;
        if (EPI == SLX_EPI_SILU_MUL) {
          const int f = tile * 128 + r;
          if (f < g.N / 2) store_out(C + (size_t)m * g.ldc + f, silu_f(v[0][j]) * v[1][j]);
        } else {
          const int n = tile * nrows_total + r;
          if (n < g.N) {
            float o = v[0][j];
            if (EPI == SLX_EPI_RESIDUAL) o += to_f32(R[(size_t)m * g.ldr + n]);
            store_out(C + (size_t)m * g.ldc + n, o);
          }
        }
      }
    }
    if (g.splits > 1 && threadIdx.x == 0) g.cnt[tile] = 0;  // self-cleaning for replay
  }

teardown:
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem_base, tmem_cols_alloc);
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

// K-major bf16 matrix [rows, cols] with row stride ld (elements); box = box_rows x 64.
static bool make_tmap(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct GemmPlan {
  bool swap;
  int bn, nsub, stages, kblocks, splits, n_tiles;
  size_t smem, part_bytes, cnt_bytes;
};

static GemmPlan plan_gemm(int M, int N, int K, int epi) {
  GemmPlan p{};
  p.kblocks = ceil_div(K, TC_BK);
  p.swap = M <= 128;
  const size_t bar_bytes = 2 * TC_MAX_STAGES * 8 + 8 + 16;
  if (p.swap) {
    p.bn = ((M + 15) / 16) * 16;
    if (p.bn < 16) p.bn = 16;
    p.nsub = (epi == SLX_EPI_SILU_MUL) ? 2 : 1;
    const int stage = p.nsub * P_TILE_BYTES + p.bn * TC_BK * 2;
    p.n_tiles = ceil_div(N, 128 * p.nsub);
    if (p.n_tiles > (int)(TC_CNT_BYTES / 4)) {  // rejected by the caller
      p.n_tiles = -1;
      return p;
    }
    const size_t two_cta_budget = 112 * 1024 - 1024 - bar_bytes;
    int st2 = (int)(two_cta_budget / stage);
    int ctas_per_sm;
    if (st2 >= 2) {
      p.stages = st2 > 6 ? 6 : st2;
      ctas_per_sm = 2;
    } else {
      int st1 = (int)((220 * 1024 - bar_bytes) / stage);
      p.stages = st1 > TC_MAX_STAGES ? TC_MAX_STAGES : st1;
      ctas_per_sm = 1;
    }
    const int slots = ctas_per_sm * sm_count();
    int s = slots / p.n_tiles;
    const int max_s = p.kblocks / 4 > 1 ? p.kblocks / 4 : 1;
    s = s < 1 ? 1 : (s > max_s ? max_s : s);
    // every split must own >= 1 k-block
    while (s > 1 && (s - 1) * ceil_div(p.kblocks, s) >= p.kblocks) --s;
    p.splits = s;
    p.smem = (size_t)p.stages * stage + bar_bytes + 1024;
    p.part_bytes = p.splits > 1 ? (size_t)p.splits * p.n_tiles * p.nsub * p.bn * 128 * 4 : 0;
    // fixed-size counter region at the head of ws, independent of the shape, so counters of
    // one call are never overlapped by another call's partial tiles (they stay zero)
    p.cnt_bytes = p.splits > 1 ? TC_CNT_BYTES : 0;
  } else {
    p.bn = 256;
    p.nsub = 1;
    p.stages = 4;
    p.n_tiles = ceil_div(N, p.bn);
    p.splits = 1;
    p.smem = (size_t)p.stages * (P_TILE_BYTES + p.bn * TC_BK * 2) + bar_bytes + 1024;
    p.part_bytes = 0;
    p.cnt_bytes = 0;
  }
  return p;
}

template <bool SWAP, int EPI, typename OutT>
static int launch_tc(const CUtensorMap& mp, const CUtensorMap& mq, const GemmArgs& a, dim3 grid,
                     size_t smem, cudaStream_t s) {
  auto k = gemm_tc_kernel<SWAP, EPI, OutT>;
  static size_t configured = 0;  // per instantiation: largest dynamic smem opted into so far
  if (smem > configured) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SLX_ERR_CUDA;
    configured = smem;
  }
  SLX_CLEAR_STALE();
  k<<<grid, TC_THREADS, smem, s>>>(mp, mq, a);
  SLX_LAUNCH_CHECK();
  return SLX_OK;
}

template <bool SWAP>
static int dispatch_tc(int epi, int c_dtype, const CUtensorMap& mp, const CUtensorMap& mq,
                       const GemmArgs& a, dim3 grid, size_t smem, cudaStream_t s) {
  if (c_dtype == SLX_DT_BF16) {
    if (epi == SLX_EPI_NONE) return launch_tc<SWAP, SLX_EPI_NONE, bf16>(mp, mq, a, grid, smem, s);
    if (epi == SLX_EPI_RESIDUAL) return launch_tc<SWAP, SLX_EPI_RESIDUAL, bf16>(mp, mq, a, grid, smem, s);
    return launch_tc<SWAP, SLX_EPI_SILU_MUL, bf16>(mp, mq, a, grid, smem, s);
  }
  if (epi == SLX_EPI_NONE) return launch_tc<SWAP, SLX_EPI_NONE, float>(mp, mq, a, grid, smem, s);
  if (epi == SLX_EPI_RESIDUAL) return launch_tc<SWAP, SLX_EPI_RESIDUAL, float>(mp, mq, a, grid, smem, s);
  return launch_tc<SWAP, SLX_EPI_SILU_MUL, float>(mp, mq, a, grid, smem, s);
}

}  // namespace slx

using namespace slx;

extern "C" size_t slx_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  GemmPlan p = plan_gemm(M, N, K, epilogue);
  return p.cnt_bytes + p.part_bytes;
}

extern "C" int slx_gemm_bf16(const void* A, int lda, const void* W, void* C, int ldc, int c_dtype,
                             const void* R, int ldr, int M, int N, int K, int epilogue, void* ws,
                             size_t ws_bytes, void* stream) {
  SLX_CHECK_ARG(A && W && C && M >= 0 && N > 0 && K > 0 && lda >= K && K % 8 == 0 &&
                lda % 8 == 0 && ldc % 8 == 0);
  SLX_CHECK_ARG(c_dtype == SLX_DT_BF16 || c_dtype == SLX_DT_F32);
  SLX_CHECK_ARG(epilogue == SLX_EPI_NONE || epilogue == SLX_EPI_RESIDUAL ||
                epilogue == SLX_EPI_SILU_MUL);
  SLX_CHECK_ALIGN(A, 16);
  SLX_CHECK_ALIGN(W, 16);
  SLX_CHECK_ALIGN(C, 16);
  if (epilogue == SLX_EPI_SILU_MUL) {
    SLX_CHECK_ARG(N % 256 == 0 && ldc >= N / 2);
  } else {
    SLX_CHECK_ARG(N % 16 == 0 && ldc >= N);
  }
  if (epilogue == SLX_EPI_RESIDUAL) SLX_CHECK_ARG(R != nullptr && ldr >= N);
  if (M == 0) return SLX_OK;
  GemmPlan p = plan_gemm(M, N, K, epilogue);
  if (p.n_tiles <= 0) return SLX_ERR_UNSUPPORTED;
  const size_t need = p.cnt_bytes + p.part_bytes;
  if (need > 0) {
    if (!ws || ws_bytes < need) return SLX_ERR_WORKSPACE;
    SLX_CHECK_ALIGN(ws, 256);
  }
  CUtensorMap mp, mq;
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.bn = p.bn; a.nsub = p.nsub; a.stages = p.stages; a.kblocks = p.kblocks;
  a.splits = p.splits; a.n_tiles = p.n_tiles;
  a.C = C; a.ldc = ldc; a.R = R; a.ldr = ldr;
  a.cnt = need ? (int*)ws : nullptr;
  a.part = need ? (float*)((char*)ws + p.cnt_bytes) : nullptr;
  cudaStream_t s = (cudaStream_t)stream;
  if (p.swap) {
    if (!make_tmap(&mp, W, N, K, K, 128) || !make_tmap(&mq, A, M, K, lda, p.bn)) return SLX_ERR_CUDA;
    dim3 grid((unsigned)p.n_tiles, (unsigned)p.splits);
    return dispatch_tc<true>(epilogue, c_dtype, mp, mq, a, grid, p.smem, s);
  }
  if (!make_tmap(&mp, A, M, K, lda, 128) || !make_tmap(&mq, W, N, K, K, p.bn)) return SLX_ERR_CUDA;
  dim3 grid((unsigned)p.n_tiles, (unsigned)ceil_div(M, 128));
  return dispatch_tc<false>(epilogue, c_dtype, mp, mq, a, grid, p.smem, s);
}
