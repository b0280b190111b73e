// K1: backbone projection GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C[M,N] = A[M,K] . W[N,K]^T  (+ residual | SiLU*mul epilogue), bf16 in, fp32 accumulate.
//
// Two tilings of one warp-specialised kernel (warp 0 lane 0: TMA producer, warp 1 lane 0:
// MMA issuer, all 4 warps: TMEM -> register epilogue):
//  * NORMAL (prefill, M > 128): D tile = 128 rows of A x BN rows of W, TMEM lane = token.
//  * SWAP   (decode,  M <= 128): D tile = 128 rows of W x BN (= M padded to 16) tokens;
//    TMEM lane = output feature.  The weight stream of one tile is split along K over the
//    S CTAs of a thread-block CLUSTER (S <= 8) so that every SM pulls weights; the S fp32
//    partial tiles are reduced through distributed shared memory (DSMEM) in a fixed order
//    (deterministic), each CTA finishing 1/S of the tile's columns with the epilogue.
//    No global workspace, no atomics, no serial last-CTA tail.
// PDL: the weight tiles of the first pipeline stages are fetched BEFORE griddepcontrol.wait,
// overlapping the previous kernel's tail; activations are loaded after it.
// SiLU*mul: W rows are blocked [gate 128 | up 128] per 128 output features, so one TMEM
// row (NORMAL) or two accumulators of one CTA (SWAP, nsub = 2) hold gate and up together.
//
// Replaces the modelled prefill/decode time of the reference (batching.py:17-21 T0+alpha(b-1);
// engine.py:832 prefill work, engine.py:888,909 decode_ms_per_token) with the real projections.
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace slx {

constexpr int TC_THREADS = 128;
constexpr int TC_BK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int TC_MAX_STAGES = 8;
constexpr int P_TILE_BYTES = 128 * TC_BK * 2;  // 16 KB
constexpr int TC_MAX_CLUSTER = 8;

struct GemmArgs {
  int M, N, K;
  int bn;       // UMMA N
  int nsub;     // P sub-tiles per CTA (SWAP SiLU: 2)
  int stages;
  int kblocks;
  int splits;   // SWAP: cluster size along K
  int n_tiles;
  void* C;
  int ldc;
  const void* R;
  int ldr;
  int w_tiled;  // W packed as [N/128][kblocks][128][64] (SLX_W_TILED)
};

template <typename OutT>
__device__ __forceinline__ void store_out(OutT* p, float v) {
  *p = from_f32<OutT>(v);
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + expf(-g)); }

// TMA coordinates of the 128-row weight block `row0` (multiple of 128) at k-block `kb`.
__device__ __forceinline__ void w_coord(const GemmArgs& g, int row0, int kb, int& c0, int& c1) {
  if (g.w_tiled) {
    c0 = 0;
    c1 = ((row0 >> 7) * g.kblocks + kb) * 128;
  } else {
    c0 = kb * TC_BK;
    c1 = row0;
  }
}

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

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = SWAP ? g.splits : 1;
  const int tile = SWAP ? blockIdx.x / S : blockIdx.x;
  const int split = SWAP ? blockIdx.x % S : 0;   // == cluster rank (cluster dims (S,1,1))
  const int kb_per = (g.kblocks + S - 1) / S;
  const int kb_lo = split * kb_per;
  const int kb_hi = min(g.kblocks, kb_lo + kb_per);
  const int n_kb = max(0, kb_hi - kb_lo);
  const int p_row0 = SWAP ? tile * 128 * g.nsub : blockIdx.y * 128;
  const int q_row0 = SWAP ? 0 : tile * g.bn;
  const int cols = g.nsub * g.bn;
  const uint32_t tmem_cols_alloc = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128
                                   : cols <= 256 ? 256 : 512;

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
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t pol_w = tc::policy_evict_first();  // weights: streamed once
    const uint64_t pol_x = tc::policy_evict_last();   // activations: re-read by every tile
    const int npre = min(n_kb, g.stages);
    // weight operand: SWAP -> P (nsub blocks of 128 rows), NORMAL -> Q (bn/128 blocks)
    auto load_w = [&](uint8_t* st, uint64_t* bar, int kb) {
      const int nblk = SWAP ? g.nsub : g.bn / 128;
      uint8_t* dst = SWAP ? st : st + P_TILE_BYTES;
      const int row0 = SWAP ? p_row0 : q_row0;
      for (int b = 0; b < nblk; ++b) {
        int c0, c1;
        w_coord(g, row0 + b * 128, kb, c0, c1);
        tc::tma_load_2d(dst + b * P_TILE_BYTES, SWAP ? &tmap_p : &tmap_q, bar, c0, c1, pol_w);
      }
    };
    auto load_x = [&](uint8_t* st, uint64_t* bar, int kb) {
      if (SWAP)
        tc::tma_load_2d(st + g.nsub * P_TILE_BYTES, &tmap_q, bar, kb * TC_BK, q_row0, pol_x);
      else
        tc::tma_load_2d(st, &tmap_p, bar, kb * TC_BK, p_row0, pol_x);
    };
    // the weight operand of the first stages does not depend on the previous kernel
    for (int i = 0; i < npre; ++i) {
      tc::mbar_arrive_expect_tx(&full[i], stage_bytes);
      load_w(smem + i * stage_bytes, &full[i], kb_lo + i);
    }
    pdl_wait();
    for (int i = 0; i < npre; ++i) load_x(smem + i * stage_bytes, &full[i], kb_lo + i);
    for (int i = npre; i < n_kb; ++i) {
      const int s = i % g.stages;
      tc::mbar_wait(&empty[s], ((i / g.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
      load_w(st, &full[s], kb_lo + i);
      load_x(st, &full[s], kb_lo + i);
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
  pdl_wait();
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
          if (f0 + 16 <= g.N / 2 && sizeof(OutT) == 2) {
            float o[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) o[j] = silu_f(gv[j]) * uv[j];
            Vec8<bf16>::store((bf16*)(C + (size_t)m * g.ldc + f0), o);
            Vec8<bf16>::store((bf16*)(C + (size_t)m * g.ldc + f0 + 8), o + 8);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (f0 + j < g.N / 2) store_out(C + (size_t)m * g.ldc + f0 + j, silu_f(gv[j]) * uv[j]);
          }
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
  } else if (S == 1) {
    // SWAP, whole K in this CTA: TMEM lane r = output feature, column c = token.
    // Non-SiLU: sub-tile `sub` covers W rows tile*128*nsub + sub*128.  SiLU: sub pair
    // (2p, 2p+1) = (gate, up) of feature block tile*nsub/2 + p.
    const int npair = EPI == SLX_EPI_SILU_MUL ? g.nsub / 2 : g.nsub;
    for (int p = 0; p < npair; ++p)
      for (int c0 = 0; c0 < g.bn && c0 < g.M; c0 += 16) {
        float v0[16], v1[16];
        if (EPI == SLX_EPI_SILU_MUL) {
          tc::tmem_ld16(t_row + (2 * p) * g.bn + c0, v0);
          tc::tmem_ld16(t_row + (2 * p + 1) * g.bn + c0, v1);
        } else {
          tc::tmem_ld16(t_row + p * g.bn + c0, v0);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = c0 + j;
          if (m >= g.M) break;
          if (EPI == SLX_EPI_SILU_MUL) {
            const int f = (tile * npair + p) * 128 + r;
            if (f < g.N / 2) store_out(C + (size_t)m * g.ldc + f, silu_f(v0[j]) * v1[j]);
          } else {
            const int n = (tile * npair + p) * 128 + r;
            if (n < g.N) {
              float o = v0[j];
              if (EPI == SLX_EPI_RESIDUAL) o += to_f32(R[(size_t)m * g.ldr + n]);
              store_out(C + (size_t)m * g.ldc + n, o);
            }
          }
        }
      }
  } else {
    // SWAP split-K over the cluster: stage this CTA's partial tile in its (now idle) pipeline
    // smem as red[sub][c][r], then reduce 1/S of the columns across the cluster via DSMEM.
    float* red = reinterpret_cast<float*>(smem);
    for (int sub = 0; sub < g.nsub; ++sub)
      for (int c0 = 0; c0 < g.bn && c0 < g.M; c0 += 16) {
        float v[16];
        tc::tmem_ld16(t_row + sub * g.bn + c0, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) red[(sub * g.bn + c0 + j) * 128 + r] = v[j];
      }
    tc::cluster_sync();
    const uint32_t red_base = tc::smem_u32(red);
    const int npair = EPI == SLX_EPI_SILU_MUL ? g.nsub / 2 : g.nsub;
    const int per = EPI == SLX_EPI_SILU_MUL ? 2 : 1;
    // work items (p, m): this CTA takes m = split, split + S, ...
    for (int p = 0; p < npair; ++p)
      for (int m = split; m < g.M && m < g.bn; m += S) {
        float acc[2] = {0.f, 0.f};
        for (int u = 0; u < per; ++u) {
          const int sub = p * per + u;
          const uint32_t off = red_base + (uint32_t)(((sub * g.bn + m) * 128 + r) * 4);
          float part[TC_MAX_CLUSTER];
#pragma unroll
          for (int s = 0; s < TC_MAX_CLUSTER; ++s)
            part[s] = s < S ? tc::ld_dsmem(tc::mapa(off, (uint32_t)s)) : 0.f;
          float a = 0.f;
#pragma unroll
          for (int s = 0; s < TC_MAX_CLUSTER; ++s) a += part[s];   // fixed order: deterministic
          acc[u] = a;
        }
        const int n = (tile * npair + p) * 128 + r;
        if (EPI == SLX_EPI_SILU_MUL) {
          if (n < g.N / 2) store_out(C + (size_t)m * g.ldc + n, silu_f(acc[0]) * acc[1]);
        } else if (n < g.N) {
          float o = acc[0];
          if (EPI == SLX_EPI_RESIDUAL) o += to_f32(R[(size_t)m * g.ldr + n]);
          store_out(C + (size_t)m * g.ldc + n, o);
        }
      }
    tc::cluster_sync();  // keep our smem alive until every peer finished reading it
  }

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
  size_t smem;
};

static constexpr size_t BAR_BYTES = 2 * TC_MAX_STAGES * 8 + 8 + 16;

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

static void configure_kernel(const void* k, size_t smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // without this the driver may pick an L1-heavy carveout that fits only one CTA per SM
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

// Max co-resident clusters of `cluster` CTAs with `smem` bytes each (cached; queried on the
// swap-AB kernel, whose resource footprint is the same for every epilogue instantiation).
static int max_active_clusters(size_t smem, int cluster) {
  struct Key { size_t smem; int cluster; int value; };
  static Key cache[64];
  static int n_cache = 0;
  for (int i = 0; i < n_cache; ++i)
    if (cache[i].smem == smem && cache[i].cluster == cluster) return cache[i].value;
  const void* k = (const void*)gemm_tc_kernel<true, SLX_EPI_NONE, bf16>;
  configure_kernel(k, 227 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cluster * 64);
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (unsigned)cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<true, SLX_EPI_NONE, bf16>, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    n = sm_count() / cluster;  // conservative fallback
  }
  if (n_cache < 64) cache[n_cache++] = Key{smem, cluster, n};
  return n;
}

// SWAP (decode) tiling: one CTA streams nsub x 128 weight rows over a k-range; the k-range
// of a tile is split over a cluster of S CTAs.  The planner picks, among nsub in {1,2}
// (SiLU: 2) and 2 or 1 CTAs per SM, the split S that puts the most CTAs in flight while all
// clusters stay co-resident (one wave, cudaOccupancyMaxActiveClusters) and every split keeps
// >= 4 k-blocks.  SLX_GEMM_{NSUB,CTAS,STAGES,SPLITS} override for tuning (tools/gemm_sweep.py).

static GemmPlan plan_gemm(int M, int N, int K, int epi) {
  GemmPlan p{};
  p.kblocks = ceil_div(K, TC_BK);
  p.swap = M <= 128;
  if (!p.swap) {
    p.bn = 256;
    p.nsub = 1;
    p.stages = 4;
    p.n_tiles = ceil_div(N, p.bn);
    p.splits = 1;
    p.smem = (size_t)p.stages * (P_TILE_BYTES + p.bn * TC_BK * 2) + BAR_BYTES + 1024;
    return p;
  }
  p.bn = ((M + 15) / 16) * 16;
  if (p.bn < 16) p.bn = 16;
  const bool silu = epi == SLX_EPI_SILU_MUL;
  const int e_nsub = env_int("SLX_GEMM_NSUB", 0), e_ctas = env_int("SLX_GEMM_CTAS", 0);
  const int e_st = env_int("SLX_GEMM_STAGES", 0), e_s = env_int("SLX_GEMM_SPLITS", 0);
  double best_score = -1.0;
  for (int nsub = 1; nsub <= 4; nsub *= 2) {
    if (silu && nsub == 1) continue;
    if (nsub * p.bn > 512) continue;
    // measured on B200 (tools/gemm_sweep.py): nsub 1 for plain projections, 2 for SiLU pairs
    if (e_nsub ? nsub != e_nsub : nsub != (silu ? 2 : 1)) continue;
    const size_t stage = (size_t)nsub * P_TILE_BYTES + (size_t)p.bn * TC_BK * 2;
    const size_t red = (size_t)nsub * p.bn * 128 * 4;
    const int n_tiles = ceil_div(N, 128 * nsub);
    for (int ctas = 2; ctas >= 1; --ctas) {
      if (e_ctas && ctas != e_ctas) continue;
      const size_t budget = ctas == 2 ? 112 * 1024 - 1024 - BAR_BYTES : 225 * 1024 - 1024 - BAR_BYTES;
      int st = (int)(budget / stage);
      st = st > (ctas == 2 ? 6 : TC_MAX_STAGES) ? (ctas == 2 ? 6 : TC_MAX_STAGES) : st;
      if (e_st >= 2 && e_st < st) st = e_st;
      if (st < 2) continue;
      const size_t smem = (size_t)st * stage + BAR_BYTES + 1024;
      for (int s = TC_MAX_CLUSTER; s >= 1; --s) {
        if (e_s && s != e_s) continue;
        if (s > 1 && (size_t)st * stage < red) continue;            // partials must fit in smem
        if (s > 1 && ceil_div(p.kblocks, s) < 4 && !e_s) continue;   // >= 4 k-blocks per split
        if ((s - 1) * ceil_div(p.kblocks, s) >= p.kblocks) continue; // no empty split
        const int cap = max_active_clusters(smem, s);
        if (n_tiles > cap && !e_s) continue;                         // single wave only
        // score: independent weight pipelines in flight (2 CTAs/SM preferred), then stages
        const double score = (double)n_tiles * s * (ctas == 2 ? 1.0 : 0.75) + 0.01 * st;
        if (score > best_score) {
          best_score = score;
          p.nsub = nsub; p.stages = st; p.splits = s; p.n_tiles = n_tiles; p.smem = smem;
        }
        break;   // the largest feasible split for this (nsub, ctas)
      }
    }
  }
  if (best_score < 0) {   // nothing fits in one wave: smallest footprint, no split
    p.nsub = silu ? 2 : 1;
    const size_t stage = (size_t)p.nsub * P_TILE_BYTES + (size_t)p.bn * TC_BK * 2;
    p.stages = (int)((225 * 1024 - 1024 - BAR_BYTES) / stage);
    if (p.stages > TC_MAX_STAGES) p.stages = TC_MAX_STAGES;
    p.splits = 1;
    p.n_tiles = ceil_div(N, 128 * p.nsub);
    p.smem = (size_t)p.stages * stage + BAR_BYTES + 1024;
  }
  return p;
}

template <bool SWAP, int EPI, typename OutT>
static int launch_tc(const CUtensorMap& mp, const CUtensorMap& mq, const GemmArgs& a, dim3 grid,
                     size_t smem, unsigned cluster, cudaStream_t s) {
  auto k = gemm_tc_kernel<SWAP, EPI, OutT>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    configure_kernel((const void*)k, 227 * 1024);
    configured = true;
  }
  return launch_ex(k, grid, dim3(TC_THREADS), smem, s, cluster, mp, mq, a);
}

template <bool SWAP>
static int dispatch_tc(int epi, int c_dtype, const CUtensorMap& mp, const CUtensorMap& mq,
                       const GemmArgs& a, dim3 grid, size_t smem, unsigned cl, cudaStream_t s) {
  if (c_dtype == SLX_DT_BF16) {
    if (epi == SLX_EPI_NONE) return launch_tc<SWAP, SLX_EPI_NONE, bf16>(mp, mq, a, grid, smem, cl, s);
    if (epi == SLX_EPI_RESIDUAL)
      return launch_tc<SWAP, SLX_EPI_RESIDUAL, bf16>(mp, mq, a, grid, smem, cl, s);
    return launch_tc<SWAP, SLX_EPI_SILU_MUL, bf16>(mp, mq, a, grid, smem, cl, s);
  }
  if (epi == SLX_EPI_NONE) return launch_tc<SWAP, SLX_EPI_NONE, float>(mp, mq, a, grid, smem, cl, s);
  if (epi == SLX_EPI_RESIDUAL)
    return launch_tc<SWAP, SLX_EPI_RESIDUAL, float>(mp, mq, a, grid, smem, cl, s);
  return launch_tc<SWAP, SLX_EPI_SILU_MUL, float>(mp, mq, a, grid, smem, cl, s);
}

}  // namespace slx

using namespace slx;

extern "C" size_t slx_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
  (void)M; (void)N; (void)K; (void)epilogue;
  return 0;  // split-K partials live in cluster shared memory
}

extern "C" int slx_gemm_bf16(const void* A, int lda, const void* W, void* C, int ldc, int c_dtype,
                             const void* R, int ldr, int M, int N, int K, int epilogue,
                             int w_layout, void* stream) {
  SLX_CHECK_ARG(w_layout == SLX_W_ROWMAJOR || w_layout == SLX_W_TILED);
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
  if (env_int("SLX_GEMM_DEBUG", 0))
    fprintf(stderr, "[slx_gemm] M=%d N=%d K=%d epi=%d swap=%d bn=%d nsub=%d stages=%d splits=%d tiles=%d smem=%zu\n",
            M, N, K, epilogue, (int)p.swap, p.bn, p.nsub, p.stages, p.splits, p.n_tiles, p.smem);
  CUtensorMap mp, mq;
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.bn = p.bn; a.nsub = p.nsub; a.stages = p.stages; a.kblocks = p.kblocks;
  a.splits = p.splits; a.n_tiles = p.n_tiles;
  a.C = C; a.ldc = ldc; a.R = R; a.ldr = ldr;
  a.w_tiled = w_layout == SLX_W_TILED;
  cudaStream_t s = (cudaStream_t)stream;
  // tiled W: a [n_blocks * kblocks * 128, 64] matrix of contiguous 16 KB boxes
  const int w_rows = a.w_tiled ? ceil_div(N, 128) * p.kblocks * 128 : N;
  const int w_cols = a.w_tiled ? TC_BK : K;
  if (p.swap) {
    if (!make_tmap(&mp, W, w_rows, w_cols, w_cols, 128) || !make_tmap(&mq, A, M, K, lda, p.bn))
      return SLX_ERR_CUDA;
    dim3 grid((unsigned)(p.n_tiles * p.splits), 1);
    return dispatch_tc<true>(epilogue, c_dtype, mp, mq, a, grid, p.smem, (unsigned)p.splits, s);
  }
  if (!make_tmap(&mp, A, M, K, lda, 128) || !make_tmap(&mq, W, w_rows, w_cols, w_cols, 128))
    return SLX_ERR_CUDA;
  dim3 grid((unsigned)p.n_tiles, (unsigned)ceil_div(M, 128));
  return dispatch_tc<false>(epilogue, c_dtype, mp, mq, a, grid, p.smem, 1u, s);
}

// ------------------------------------------------------------------ weight packing
namespace slx {
__global__ void pack_weight_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, int N,
                                   int K, int ld, int kblocks) {
  pdl_trigger();
  pdl_wait();
  // one thread per 16-byte chunk of the packed tensor
  const size_t chunk = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)ceil_div(N, 128) * kblocks * 128 * 8;
  if (chunk >= total) return;
  const int c8 = (int)(chunk % 8);
  const size_t row = chunk / 8;           // row of the [blocks*kblocks*128, 64] view
  const int r = (int)(row % 128);
  const size_t bk = row / 128;
  const int kb = (int)(bk % kblocks);
  const int nb = (int)(bk / kblocks);
  const int n = nb * 128 + r, k = kb * TC_BK + c8 * 8;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (n < N && k < K) v = *reinterpret_cast<const uint4*>(src + (size_t)n * ld + k);  // K % 8 == 0
  *reinterpret_cast<uint4*>(dst + row * TC_BK + c8 * 8) = v;
}
}  // namespace slx

extern "C" size_t slx_packed_weight_elems(int N, int K) {
  if (N <= 0 || K <= 0) return 0;
  return (size_t)ceil_div(N, 128) * 128 * (size_t)ceil_div(K, TC_BK) * TC_BK;
}

extern "C" int slx_pack_weight(void* dst, const void* src, int N, int K, int ld, void* stream) {
  SLX_CHECK_ARG(dst && src && N > 0 && K > 0 && K % 8 == 0 && ld >= K && ld % 8 == 0);
  SLX_CHECK_ALIGN(dst, 16);
  SLX_CHECK_ALIGN(src, 16);
  const int kb = ceil_div(K, TC_BK);
  const size_t total = (size_t)ceil_div(N, 128) * kb * 128 * 8;
  return launch_ex(pack_weight_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0,
                   (cudaStream_t)stream, 1u, (bf16*)dst, (const bf16*)src, N, K, ld, kb);
}
