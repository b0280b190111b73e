// K1: backbone projection GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C[M,N] = A[M,K] . W[N,K]^T  (+ residual | SiLU*mul epilogue), bf16 in, fp32 accumulate.
//
// One warp-specialised kernel (warp 0 lane 0: TMA producer, warp 1 lane 0: MMA issuer, all 4
// warps: TMEM -> register epilogue).  The D tile is 128 token rows (TMEM lanes) x 256 weight
// rows (TMEM columns): the weight operand is always the N = 256 side of tcgen05.mma.kind::f16.
// A B200 tcgen05 instruction costs about the same time at N = 64 as at N = 256 (measured,
// tools/probe/mma_probe.cu), so streaming weights as the wide operand needs 4x fewer MMAs per
// weight byte than a swap-AB (weights-as-M) tiling — decisive for HBM-bound decode.
//
//  * prefill (many 128-row token tiles): grid = (N/256, M/128), full K per CTA.
//  * decode (M <= 128, few tiles): the activation box is only `bm` = M rounded to 16 rows and
//    the K range of each weight tile is split over the S CTAs of a thread-block CLUSTER (S <= 8)
//    so that every SM streams weights; the S fp32 partial tiles are reduced through
//    distributed shared memory (DSMEM) in a fixed order (deterministic), each CTA finishing a
//    1/S slice of the tile's columns with the epilogue.  No workspace, no atomics.
// SiLU*mul: W rows are blocked [gate 128 | up 128] per 128 features, so the two halves of one
// 256-column TMEM tile hold gate and up of the same features.
// Weights are stored SLX_W_TILED ([N/128][K/64][128][64]) so every TMA box is one contiguous
// 16 KB burst; PDL: the first stages' weight boxes are fetched BEFORE griddepcontrol.wait.
//
//  * prefill with many tiles runs the PERSISTENT variant gemm_tcp_kernel (below): one CTA per SM,
//    two TMEM accumulators, the epilogue of tile i overlapping the mainloop of tile i + 1.
// Replaces the modelled prefill/decode time of the reference (batching.py:17-21 T0+alpha(b-1);
// engine.py:832 prefill work, engine.py:888,909 decode_ms_per_token) with the real projections.
#include <cuda.h>

#include "common.cuh"
#include "gemm_host.h"
#include "tc_ptx.cuh"

namespace slx {

constexpr int TC_THREADS = 128;
constexpr int TC_BK = 64;       // 64 bf16 = one 128-byte swizzle row
constexpr int TC_BN_MAX = 256;  // weight rows per tile (MMA N): 256 or 128
constexpr int TC_MAX_STAGES = 8;
constexpr int W_BLOCK_BYTES = 128 * TC_BK * 2;   // 16 KB: one 128-row weight box
constexpr int TC_MAX_CLUSTER = 8;

// Grouped mode (SGMV on the tensor cores): CTA x-index -> one GroupTile; each group (adapter
// segment) has its own row-major W tensor map and alpha (the LoRA scale).
constexpr int TC_MAX_GROUPS = 16;
constexpr int TC_MAX_MAPS = 48;   // LoRA fold: (adapter, target) B maps, <= 16 adapters x 3
struct GroupTile {
  int group, m0, m_rows, n0;
};
struct GroupMaps {
  CUtensorMap w[TC_MAX_MAPS];
  float alpha[TC_MAX_MAPS];
  CUtensorMap v;   // LoRA fold: the shrink output v [T, 64 * n_targets] (scale folded in)
};

struct GemmArgs {
  int M, N, K;
  int bm;        // activation rows per tile actually loaded (<= 128, multiple of 16)
  int stages;
  int kblocks;
  int splits;    // cluster size along K (1 = no split)
  int n_tiles;
  void* C;
  int ldc;
  const void* R;
  int ldr;
  int w_tiled;   // W packed as [N/128][kblocks][128][64] (SLX_W_TILED)
  int n_main;    // columns >= n_main go to the fp32 side output C2 (LoRA shrink rows)
  float* C2;
  int ldc2;
  const GroupTile* gtiles;   // grouped mode only
  int gsplit;                // split-K reduced through global partial tiles (no cluster)
  float* ws_part;            // [tiles][S][bm][BN] fp32 partials
  int* ws_cnt;               // [tiles] arrival counters (zero; self-cleaning)
  unsigned long long* trace; // debug (slx_debug_gemm_trace): 8 globaltimer stamps per CTA
  // LoRA fold (slx_gemm_bf16_lorafold, grouped tiles): the main K range uses the backbone W
  // (tmap_w) for every tile; a tile whose group >= 0 adds ONE more k-block
  //   D += v[m0.., t*64 : t*64+64] . B_(group, t)[n0 - lbound[t] .., :64]^T
  // (t = target of the tile's columns), i.e. the LoRA expand rides in the backbone mainloop.
  int lfold, lnt;
  int lbound[4];
  // rasterised 1-D grid (prefill, no split): tiles visited in groups of `raster` m-tiles x all
  // n-tiles, so the ~148 co-resident CTAs share a few X row blocks and W tiles in L2
  int raster, m_tiles;
  int n_work;    // persistent kernel: tiles to walk (raster grid or gtiles)
  // grouped mode with gseg > 1: every tile's B operand is gseg 64-row segments, segment s from
  // map [group * gseg + s] (e.g. the q, k, v A matrices of one adapter: one shrink launch)
  int gseg;
  // RoPE + KV append in the epilogue (slx_rope_kv; persistent kernel, EPI_NONE, bf16 out)
  int rope, r_h, r_hkv, r_max_ctx;
  const int32_t* r_pos;
  const int32_t* r_seq;
  const float* r_cos;
  const float* r_sin;
  bf16* r_kc;
  bf16* r_vc;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define SLX_TR(i) \
  if (g.trace) g.trace[(size_t)(blockIdx.y * gridDim.x + blockIdx.x) * 16 + (i)] = gtimer()

template <typename OutT>
__device__ __forceinline__ void store_out(OutT* p, float v) {
  *p = from_f32<OutT>(v);
}
// fast-math SiLU: no IEEE-division slow path (whose per-element branch serialises the epilogue)
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// 16 consecutive outputs of one row: vector stores for bf16 when the run is in bounds.
template <typename OutT>
__device__ __forceinline__ void store16(OutT* row, int n0, int n_lim, const float* v) {
  if (sizeof(OutT) == 2 && n0 + 16 <= n_lim) {
    Vec8<bf16>::store(reinterpret_cast<bf16*>(row + n0), v);
    Vec8<bf16>::store(reinterpret_cast<bf16*>(row + n0 + 8), v + 8);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n0 + j < n_lim) store_out(row + n0 + j, v[j]);
  }
}

// 16 output columns [n, n+16) of row m: main columns get the residual and go to C, side
// columns (n >= n_main, LoRA shrink rows appended to W) go to the fp32 side output C2.
template <int EPI, typename OutT>
__device__ __forceinline__ void store_cols(const GemmArgs& g, OutT* C, const OutT* R, int m, int n,
                                           int n_out, float* v, float alpha = 1.f) {
  if (alpha != 1.f) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] *= alpha;
  }
  if (g.C2 != nullptr && n >= g.n_main) {
    float* row = g.C2 + (size_t)m * g.ldc2 + (n - g.n_main);
    if (n + 16 <= g.N) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<float4*>(row)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n + j < g.N) row[j] = v[j];
    }
    return;
  }
  const int lim = g.C2 != nullptr ? g.n_main : n_out;
  if (EPI == SLX_EPI_RESIDUAL) {
    const OutT* rr = R + (size_t)m * g.ldr + n;
    if (n + 16 <= lim && (reinterpret_cast<uintptr_t>(rr) & 15) == 0) {   // two 16 B loads
      float r[16];
      Vec8<OutT>::load(rr, r);
      Vec8<OutT>::load(rr + 8, r + 8);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] += r[j];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (n + j < lim) v[j] += to_f32(rr[j]);
    }
  }
  store16(C + (size_t)m * g.ldc, n, lim, v);
}

// TMA coordinates of the 128-row weight block starting at row0 (multiple of 128), k-block kb.
__device__ __forceinline__ void w_coord(const GemmArgs& g, int row0, int kb, int& c0, int& c1) {
  if (g.w_tiled) {
    c0 = 0;
    c1 = ((row0 >> 7) * g.kblocks + kb) * 128;
  } else {
    c0 = kb * TC_BK;
    c1 = row0;
  }
}

template <int EPI, typename OutT, int TC_BN, bool GROUPED>
__global__ void __launch_bounds__(TC_THREADS, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
               GemmArgs g, const __grid_constant__ GroupMaps gm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int x_bytes = g.bm * TC_BK * 2;
  constexpr int WB = TC_BN / 128;   // 128-row weight boxes per stage
  const int stage_bytes = x_bytes + WB * W_BLOCK_BYTES;
  uint64_t* full = (uint64_t*)(smem + g.stages * stage_bytes);
  uint64_t* empty = full + TC_MAX_STAGES;
  uint64_t* accum = empty + TC_MAX_STAGES;
  uint32_t* tmem_slot = (uint32_t*)(accum + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) SLX_TR(0);
  const int S = g.splits;
  int tile, mt;
  if (!GROUPED && g.raster > 0) {
    const int L = blockIdx.x, per = g.raster * g.n_tiles;
    const int grp = L / per, rem = L - grp * per;
    const int gsz = min(g.raster, g.m_tiles - grp * g.raster);
    mt = grp * g.raster + rem % gsz;
    tile = rem / gsz;
  } else {
    tile = blockIdx.x / S;
    mt = blockIdx.y;
  }
  const int split = g.raster > 0 ? 0 : blockIdx.x % S;   // == cluster rank (cluster dims (S,1,1))
  const int kb_per = (g.kblocks + S - 1) / S;
  const int kb_lo = split * kb_per;
  const int kb_hi = min(g.kblocks, kb_lo + kb_per);
  const int n_kb = max(0, kb_hi - kb_lo);
  // grouped mode: the tile table comes from the host stream; read it after the PDL wait
  if (GROUPED) pdl_wait();
  const GroupTile gt = GROUPED ? g.gtiles[blockIdx.x] : GroupTile{0, 0, 0, 0};
  const int m0 = GROUPED ? gt.m0 : mt * 128;
  const int n0 = GROUPED ? gt.n0 : tile * TC_BN;
  const int m_lim = GROUPED ? gt.m0 + gt.m_rows : g.M;
  const bool lfold = GROUPED && g.lfold;
  const float alpha = (GROUPED && !lfold) ? gm.alpha[gt.group] : 1.f;
  const CUtensorMap* wmap = (GROUPED && !lfold) ? &gm.w[gt.group] : &tmap_w;
  int ltgt = 0;
  if (lfold) {
#pragma unroll
    for (int t = 1; t < 4; ++t)
      if (t < g.lnt && n0 >= g.lbound[t]) ltgt = t;
  }
  const bool lblk = lfold && gt.group >= 0;            // one extra (LoRA) k-block
  const int n_tot = n_kb + (lblk ? 1 : 0);

  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmap_x);
    tc::tma_prefetch_desc(wmap);
    for (int s = 0; s < g.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(accum, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TC_BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) SLX_TR(1);
  if (!(warp == 0 && lane == 0)) {
    pdl_wait();
    pdl_trigger();
  }

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer
    const uint64_t pol_w = tc::policy_evict_first();  // weights: streamed once
    const uint64_t pol_x = tc::policy_evict_last();   // activations: re-read by every tile
    auto load_w = [&](uint8_t* st, uint64_t* bar, int kb) {
      for (int b = 0; b < WB; ++b) {
        int c0, c1;
        w_coord(g, n0 + b * 128, kb, c0, c1);
        tc::tma_load_2d(st + x_bytes + b * W_BLOCK_BYTES, wmap, bar, c0, c1, pol_w);
      }
    };
    const int npre = min(n_kb, g.stages);
    // the weight operand of the first stages does not depend on the previous kernel
    for (int i = 0; i < npre; ++i) {
      tc::mbar_arrive_expect_tx(&full[i], stage_bytes);
      load_w(smem + i * stage_bytes, &full[i], kb_lo + i);
    }
    pdl_wait();
    pdl_trigger();
    SLX_TR(2);
    for (int i = 0; i < npre; ++i)
      tc::tma_load_2d(smem + i * stage_bytes, &tmap_x, &full[i], (kb_lo + i) * TC_BK, m0, pol_x);
    for (int i = npre; i < n_tot; ++i) {
      const int s = i % g.stages;
      tc::mbar_wait(&empty[s], ((i / g.stages) & 1) ^ 1);
      uint8_t* st = smem + s * stage_bytes;
      tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
      if (i < n_kb) {
        load_w(st, &full[s], kb_lo + i);
        tc::tma_load_2d(st, &tmap_x, &full[s], (kb_lo + i) * TC_BK, m0, pol_x);
      } else {   // LoRA k-block: v slice of the tile's target x B rows of (adapter, target)
        const CUtensorMap* bmap = &gm.w[gt.group * g.lnt + ltgt];
        for (int b = 0; b < WB; ++b)
          tc::tma_load_2d(st + x_bytes + b * W_BLOCK_BYTES, bmap, &full[s], 0,
                          n0 - g.lbound[ltgt] + b * 128, pol_x);
        tc::tma_load_2d(st, &gm.v, &full[s], ltgt * TC_BK, m0, pol_x);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread): D[128 x 256] += X[128 x 16] . W[256 x 16]^T.
    // Rows >= bm of the X operand read stale shared memory; they only feed D rows that are
    // never stored.
    const uint32_t idesc = tc::idesc_bf16_f32(128, TC_BN);
    for (int i = 0; i < n_tot; ++i) {
      const int s = i % g.stages;
      tc::mbar_wait(&full[s], (i / g.stages) & 1);
      tc::fence_after_sync();
      if (i == 0) SLX_TR(3);
      const uint32_t st = tc::smem_u32(smem + s * stage_bytes);
#pragma unroll
      for (int ks = 0; ks < TC_BK / 16; ++ks)
        tc::mma_bf16_ss(tmem_base, tc::smem_desc_sw128(st + ks * 32),
                        tc::smem_desc_sw128(st + x_bytes + ks * 32), idesc,
                        (i > 0 || ks > 0) ? 1u : 0u);
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(accum);
    SLX_TR(4);
  }

  // ---------------- epilogue: all 4 warps; warp w owns TMEM lanes (token rows) [32w, 32w+32)
  tc::mbar_wait(accum, 0);
  __syncwarp();
  tc::fence_after_sync();
  if (threadIdx.x == 0) SLX_TR(5);
  const int r = warp * 32 + lane;
  const int m = m0 + r;
  const bool warp_live = m0 + warp * 32 < m_lim && warp * 32 < g.bm;   // warp-uniform
  const uint32_t t_row = tmem_base + ((uint32_t)(warp * 32) << 16);
  OutT* C = reinterpret_cast<OutT*>(g.C);
  const OutT* R = reinterpret_cast<const OutT*>(g.R);
  const int n_out = EPI == SLX_EPI_SILU_MUL ? g.N / 2 : g.N;

  if (S == 1) {
    if (warp_live) {
      if (EPI == SLX_EPI_SILU_MUL) {
        for (int c0 = 0; c0 < TC_BN / 2; c0 += 16) {
          float gv[16], uv[16];
          tc::tmem_ld16(t_row + c0, gv);
          tc::tmem_ld16(t_row + TC_BN / 2 + c0, uv);
          if (m < m_lim) {
#pragma unroll
            for (int j = 0; j < 16; ++j) gv[j] = silu_f(gv[j]) * uv[j];
            store16(C + (size_t)m * g.ldc, tile * (TC_BN / 2) + c0, n_out, gv);
          }
        }
      } else {
        for (int c0 = 0; c0 < TC_BN; c0 += 16) {
          float v[16];
          tc::tmem_ld16(t_row + c0, v);
          const int n = n0 + c0;
          if (m < m_lim) store_cols<EPI>(g, C, R, m, n, n_out, v, alpha);
        }
      }
    }
  } else if (g.gsplit) {
    // split-K through global memory (no cluster placement constraints): every split CTA
    // writes its fp32 partial tile with 16-byte stores, the S CTAs of the tile rendezvous on
    // an arrival counter (the plan is one wave at <= 1 CTA per SM, so all S are resident),
    // and each reduces a 1/S column slice in split order (deterministic).  A departure
    // counter lets the last CTA out reset both counters for the next launch / graph replay.
    float* part = g.ws_part + (size_t)tile * S * g.bm * TC_BN;
    int* arrive = g.ws_cnt + 2 * tile;
    int* depart = arrive + 1;
    if (warp_live) {
      for (int c0 = 0; c0 < TC_BN; c0 += 16) {
        float v[16];
        tc::tmem_ld16(t_row + c0, v);
        if (r < g.bm) {
          float4* dst = reinterpret_cast<float4*>(part + ((size_t)split * g.bm + r) * TC_BN + c0);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(arrive, 1);
      while (atomicAdd(arrive, 0) < S) __nanosleep(64);
    }
    __syncthreads();
    __threadfence();
    if (threadIdx.x == 0) SLX_TR(6);
    auto sum16 = [&](int col0, float* out) {
#pragma unroll
      for (int j = 0; j < 16; ++j) out[j] = 0.f;
#pragma unroll
      for (int sp = 0; sp < TC_MAX_CLUSTER; ++sp) {   // fixed order: deterministic
        if (sp < S) {
          const float4* src = reinterpret_cast<const float4*>(part + ((size_t)sp * g.bm + r) * TC_BN + col0);
          float4 q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = __ldcg(src + u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            out[4 * u] += q[u].x; out[4 * u + 1] += q[u].y;
            out[4 * u + 2] += q[u].z; out[4 * u + 3] += q[u].w;
          }
        }
      }
    };
    const int feats = EPI == SLX_EPI_SILU_MUL ? TC_BN / 2 : TC_BN;
    const int fw = ((feats + S - 1) / S + 15) / 16 * 16;
    const int f_lo = min(feats, split * fw), f_hi = min(feats, f_lo + fw);
    if (warp_live && m < m_lim && r < g.bm) {
      for (int f0 = f_lo; f0 < f_hi; f0 += 16) {
        float v[16];
        sum16(f0, v);
        if (EPI == SLX_EPI_SILU_MUL) {
          float u[16];
          sum16(f0 + TC_BN / 2, u);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = silu_f(v[j]) * u[j];
          store16(C + (size_t)m * g.ldc, tile * (TC_BN / 2) + f0, n_out, v);
        } else {
          store_cols<EPI>(g, C, R, m, n0 + f0, n_out, v);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(depart, 1) == S - 1) {
      *arrive = 0;   // every split passed the rendezvous and finished reading the partials
      *depart = 0;
      __threadfence();
    }
  } else {
    // split-K over the cluster: stage this CTA's partial tile (rows < bm) in its idle pipeline
    // smem as red[row][col] (row stride RED_LD floats, padded against bank conflicts), then
    // reduce a 1/S slice of the columns across the cluster with 16-byte DSMEM loads.
    constexpr int RED_LD = TC_BN + 4;
    static_assert(EPI != SLX_EPI_SILU_MUL || TC_BN == 256, "SiLU pairs need 256-wide tiles");
    float* red = reinterpret_cast<float*>(smem);
    if (warp_live) {
      for (int c0 = 0; c0 < TC_BN; c0 += 16) {
        float v[16];
        tc::tmem_ld16(t_row + c0, v);
        if (r < g.bm) {
          float4* dst = reinterpret_cast<float4*>(red + (size_t)r * RED_LD + c0);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        }
      }
    }
    tc::cluster_sync();
    if (threadIdx.x == 0) SLX_TR(6);
    const uint32_t red_base = tc::smem_u32(red);
    // this CTA's slice: output features [f_lo, f_hi) of the tile (SiLU: 128 features)
    const int feats = EPI == SLX_EPI_SILU_MUL ? TC_BN / 2 : TC_BN;
    const int fw = ((feats + S - 1) / S + 15) / 16 * 16;
    const int f_lo = min(feats, split * fw), f_hi = min(feats, f_lo + fw);
    auto reduce16 = [&](int col0, float* out) {   // sum over the cluster of red[r][col0..col0+16)
#pragma unroll
      for (int j = 0; j < 16; ++j) out[j] = 0.f;
      const uint32_t off = red_base + (uint32_t)((r * RED_LD + col0) * 4);
#pragma unroll
      for (int s = 0; s < TC_MAX_CLUSTER; ++s) {   // fixed order: deterministic
        if (s < S) {
          const uint32_t ra = tc::mapa(off, (uint32_t)s);
          float4 q[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) q[u] = tc::ld_dsmem4(ra + u * 16);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            out[4 * u] += q[u].x; out[4 * u + 1] += q[u].y;
            out[4 * u + 2] += q[u].z; out[4 * u + 3] += q[u].w;
          }
        }
      }
    };
    if (warp_live && m < m_lim && r < g.bm) {
      for (int f0 = f_lo; f0 < f_hi; f0 += 16) {
        float v[16];
        reduce16(f0, v);
        if (EPI == SLX_EPI_SILU_MUL) {
          float u[16];
          reduce16(f0 + TC_BN / 2, u);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = silu_f(v[j]) * u[j];
          store16(C + (size_t)m * g.ldc, tile * (TC_BN / 2) + f0, n_out, v);
        } else {
          store_cols<EPI>(g, C, R, m, n0 + f0, n_out, v);
        }
      }
    }
    tc::cluster_sync();  // keep our smem alive until every peer finished reading it
  }

  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x == 0) SLX_TR(7);
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem_base, TC_BN);
  }
}

// ------------------------------------------------------------------ persistent prefill kernel
// Many 128 x 256 tiles (prefill, no K split): one CTA per SM walks tiles L = blockIdx.x,
// blockIdx.x + G, ... (the raster order of the 1-D grid above, or the grouped tile table), with
// the TMA ring running continuously across tiles and TWO TMEM accumulators (2 x 256 columns),
// so the epilogue of tile i (its own four warps) overlaps the mainloop of tile i + 1 instead of
// idling the tensor core between one-tile CTAs (drain, CTA exit / launch, prologue, refill).
// Roles (192 threads): warp 0 lane 0 TMA producer, warp 1 lane 0 MMA issuer, warps 2-5
// epilogue (warp w drains TMEM lanes 32 (w % 4) ..).  Same tile math and epilogues as
// gemm_tc_kernel (bit-identical outputs).
constexpr int TCP_THREADS = 192;

struct TcpTile {
  int m0, n0, m_lim, tile, n_kb, group, ltgt;
  bool lblk;
  float alpha;
};

template <bool GROUPED>
__device__ __forceinline__ TcpTile tcp_tile(const GemmArgs& g, const GroupMaps& gm, int L) {
  TcpTile t{};
  if (GROUPED) {
    const GroupTile gt = g.gtiles[L];
    t.m0 = gt.m0;
    t.n0 = gt.n0;
    t.m_lim = gt.m0 + gt.m_rows;
    t.group = gt.group;
    t.tile = gt.n0 / 256;
  } else {
    const int per = g.raster * g.n_tiles;
    const int grp = L / per, rem = L - grp * per;
    const int gsz = min(g.raster, g.m_tiles - grp * g.raster);
    const int mt = grp * g.raster + rem % gsz;
    t.tile = rem / gsz;
    t.m0 = mt * 128;
    t.n0 = t.tile * 256;
    t.m_lim = g.M;
    t.group = 0;
  }
  t.n_kb = g.kblocks;
  const bool lfold = GROUPED && g.lfold;
  t.alpha = (GROUPED && !lfold) ? gm.alpha[t.group * (g.gseg > 1 ? g.gseg : 1)] : 1.f;
  t.ltgt = 0;
  if (lfold) {
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (q < g.lnt && t.n0 >= g.lbound[q]) t.ltgt = q;
  }
  t.lblk = lfold && t.group >= 0;
  return t;
}

template <int EPI, typename OutT, bool GROUPED>
__global__ void __launch_bounds__(TCP_THREADS, 1)
gemm_tcp_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
                GemmArgs g, const __grid_constant__ GroupMaps gm) {
  constexpr int BN = 256, WB = 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int x_bytes = 128 * TC_BK * 2;
  const int stage_bytes = x_bytes + WB * W_BLOCK_BYTES;
  uint64_t* full = (uint64_t*)(smem + g.stages * stage_bytes);
  uint64_t* empty = full + TC_MAX_STAGES;
  uint64_t* tfull = empty + TC_MAX_STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tmap_x);
    tc::tma_prefetch_desc(&tmap_w);
    for (int s = 0; s < g.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      tc::mbar_init(&tfull[q], 1);
      tc::mbar_init(&tempty[q], 4);   // one arrival per epilogue warp
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;
  // The next kernel is released (launch_dependents) only when this CTA reaches its LAST tile:
  // a persistent grid that triggered at its start would have the next kernel's CTAs launched
  // and parked on the SMs for the whole GEMM.
  if (GROUPED || warp != 0) pdl_wait();   // the grouped tile table comes from the host stream

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      const uint64_t pol_w = tc::policy_evict_first();
      const uint64_t pol_x = tc::policy_evict_last();
      int i = 0;
      bool waited = GROUPED;
      const bool segs = GROUPED && !g.lfold && g.gseg > 1;
      const int stage_tx = segs ? x_bytes + g.gseg * (W_BLOCK_BYTES / 2) : stage_bytes;
      for (int L = blockIdx.x; L < g.n_work; L += gridDim.x) {
        if (L + (int)gridDim.x >= g.n_work && waited) pdl_trigger();
        const TcpTile t = tcp_tile<GROUPED>(g, gm, L);
        const CUtensorMap* wmap = (GROUPED && !g.lfold) ? &gm.w[t.group] : &tmap_w;
        const int n_tot = t.n_kb + (t.lblk ? 1 : 0);
        for (int kk = 0; kk < n_tot; ++kk, ++i) {
          const int s = i % g.stages;
          tc::mbar_wait(&empty[s], ((i / g.stages) & 1) ^ 1);
          uint8_t* st = smem + s * stage_bytes;
          tc::mbar_arrive_expect_tx(&full[s], t.lblk && kk >= t.n_kb ? stage_bytes : stage_tx);
          if (kk < t.n_kb && segs) {   // 64-row segments, each from its own map
            for (int sg = 0; sg < g.gseg; ++sg)
              tc::tma_load_2d(st + x_bytes + sg * (W_BLOCK_BYTES / 2), &gm.w[t.group * g.gseg + sg],
                              &full[s], kk * TC_BK, 0, pol_w);
          } else if (kk < t.n_kb) {
            for (int b = 0; b < WB; ++b) {
              int c0, c1;
              w_coord(g, t.n0 + b * 128, kk, c0, c1);
              tc::tma_load_2d(st + x_bytes + b * W_BLOCK_BYTES, wmap, &full[s], c0, c1, pol_w);
            }
          }
          if (kk < t.n_kb) {
            if (!waited) {   // weights first; the activations come from the previous kernel
              pdl_wait();
              waited = true;
              if (L + (int)gridDim.x >= g.n_work) pdl_trigger();
            }
            tc::tma_load_2d(st, &tmap_x, &full[s], kk * TC_BK, t.m0, pol_x);
          } else {   // LoRA k-block: v slice of the tile's target x B rows of (adapter, target)
            const CUtensorMap* bmap = &gm.w[t.group * g.lnt + t.ltgt];
            for (int b = 0; b < WB; ++b)
              tc::tma_load_2d(st + x_bytes + b * W_BLOCK_BYTES, bmap, &full[s], 0,
                              t.n0 - g.lbound[t.ltgt] + b * 128, pol_x);
            tc::tma_load_2d(st, &gm.v, &full[s], t.ltgt * TC_BK, t.m0, pol_x);
          }
        }
      }
      if (!waited) pdl_wait();
      pdl_trigger();   // (no-op if already issued)
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = tc::idesc_bf16_f32(128, BN);
      int i = 0, j = 0;
      for (int L = blockIdx.x; L < g.n_work; L += gridDim.x, ++j) {
        const TcpTile t = tcp_tile<GROUPED>(g, gm, L);
        const int n_tot = t.n_kb + (t.lblk ? 1 : 0);
        tc::mbar_wait(&tempty[j & 1], ((j >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t d = tmem_base + (uint32_t)((j & 1) * BN);
        for (int kk = 0; kk < n_tot; ++kk, ++i) {
          const int s = i % g.stages;
          tc::mbar_wait(&full[s], (i / g.stages) & 1);
          tc::fence_after_sync();
          const uint32_t st = tc::smem_u32(smem + s * stage_bytes);
#pragma unroll
          for (int ks = 0; ks < TC_BK / 16; ++ks)
            tc::mma_bf16_ss(d, tc::smem_desc_sw128(st + ks * 32),
                            tc::smem_desc_sw128(st + x_bytes + ks * 32), idesc,
                            (kk > 0 || ks > 0) ? 1u : 0u);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[j & 1]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue (warps 2-5)
    const int q = warp & 3;
    const int r = q * 32 + lane;
    OutT* C = reinterpret_cast<OutT*>(g.C);
    const OutT* R = reinterpret_cast<const OutT*>(g.R);
    const int n_out = EPI == SLX_EPI_SILU_MUL ? g.N / 2 : g.N;
    int j = 0;
    for (int L = blockIdx.x; L < g.n_work; L += gridDim.x, ++j) {
      const TcpTile t = tcp_tile<GROUPED>(g, gm, L);
      const int acc = j & 1;
      tc::mbar_wait(&tfull[acc], (j >> 1) & 1);
      __syncwarp();
      tc::fence_after_sync();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      const int m = t.m0 + r;
      if (t.m0 + q * 32 < t.m_lim) {   // warp-uniform
        if (EPI == SLX_EPI_NONE && sizeof(OutT) == 2 && g.rope) {
          // q: rotate-half RoPE into C; k: rotated into the k cache; v: into the v cache — the
          // arithmetic of slx_rope_kv_write on the bf16-rounded projection (head_dim 128: two
          // heads per 256-column tile, pairs (c, c + 64) of a head)
          const bool row_ok = m < t.m_lim;
          const int pos = row_ok ? g.r_pos[m] : 0, seq = row_ok ? g.r_seq[m] : 0;
          const int qc = g.r_h * 128, kcol = qc + g.r_hkv * 128;
          for (int hh = 0; hh < 2; ++hh) {
            const int col0 = t.n0 + hh * 128;   // first column of this head
            const uint32_t th = t_row + hh * 128;
            if (col0 >= kcol) {   // v
              bf16* dst = g.r_vc + (((size_t)seq * g.r_hkv + (col0 - kcol) / 128) * g.r_max_ctx + pos) * 128;
              for (int c0 = 0; c0 < 128; c0 += 32) {
                float v0[16], v1[16];
                tc::tmem_ld16x2(th + c0, th + c0 + 16, v0, v1);
                if (row_ok) {
                  Vec8<bf16>::store(dst + c0, v0);
                  Vec8<bf16>::store(dst + c0 + 8, v0 + 8);
                  Vec8<bf16>::store(dst + c0 + 16, v1);
                  Vec8<bf16>::store(dst + c0 + 24, v1 + 8);
                }
              }
            } else {   // q or k: rotate
              bf16* dst = col0 < qc
                  ? reinterpret_cast<bf16*>(g.C) + (size_t)m * g.ldc + col0
                  : g.r_kc + (((size_t)seq * g.r_hkv + (col0 - qc) / 128) * g.r_max_ctx + pos) * 128;
              const float* cr = g.r_cos + (size_t)pos * 64;
              const float* sr = g.r_sin + (size_t)pos * 64;
              for (int c0 = 0; c0 < 64; c0 += 16) {
                float x1[16], x2[16];
                tc::tmem_ld16x2(th + c0, th + c0 + 64, x1, x2);
                if (row_ok) {
                  float cs[16], sn[16], r1[16], r2[16];
#pragma unroll
                  for (int e = 0; e < 16; e += 8) {
                    Vec8<float>::load(cr + c0 + e, cs + e);
                    Vec8<float>::load(sr + c0 + e, sn + e);
                  }
#pragma unroll
                  for (int e = 0; e < 16; ++e) {
                    const float a1 = __bfloat162float(__float2bfloat16_rn(x1[e]));
                    const float a2 = __bfloat162float(__float2bfloat16_rn(x2[e]));
                    r1[e] = a1 * cs[e] - a2 * sn[e];
                    r2[e] = a2 * cs[e] + a1 * sn[e];
                  }
                  Vec8<bf16>::store(dst + c0, r1);
                  Vec8<bf16>::store(dst + c0 + 8, r1 + 8);
                  Vec8<bf16>::store(dst + c0 + 64, r2);
                  Vec8<bf16>::store(dst + c0 + 72, r2 + 8);
                }
              }
            }
          }
        } else if (EPI == SLX_EPI_SILU_MUL) {
          for (int c0 = 0; c0 < BN / 2; c0 += 16) {
            float gv[16], uv[16];
            tc::tmem_ld16x2(t_row + c0, t_row + BN / 2 + c0, gv, uv);
            if (m < t.m_lim) {
#pragma unroll
              for (int e = 0; e < 16; ++e) gv[e] = silu_f(gv[e]) * uv[e];
              store16(C + (size_t)m * g.ldc, t.tile * (BN / 2) + c0, n_out, gv);
            }
          }
        } else {
          for (int c0 = 0; c0 < BN; c0 += 32) {
            float v0[16], v1[16];
            tc::tmem_ld16x2(t_row + c0, t_row + c0 + 16, v0, v1);
            if (m < t.m_lim) {
              store_cols<EPI>(g, C, R, m, t.n0 + c0, n_out, v0, t.alpha);
              store_cols<EPI>(g, C, R, m, t.n0 + c0 + 16, n_out, v1, t.alpha);
            }
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem_base, 2 * BN);
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
bool make_tmap(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, int box_rows) {
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

void configure_kernel(const void* k) {
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, k);   // the opt-in limit counts static + dynamic shared memory
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)(227 * 1024 - fa.sharedSizeBytes));
  // without this the driver may pick an L1-heavy carveout that fits fewer CTAs per SM
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

struct GemmPlan {
  int bn, bm, stages, kblocks, splits, n_tiles, m_tiles;
  int gsplit;
  size_t smem;
};

static constexpr size_t GS_CNT_BYTES = 64 * 1024;   // counter region at the head of ws:
// [0, 32K) gemm_sk (monotonic), [32K, 64K) this path (self-cleaning); 2 ints per tile

static size_t gsplit_ws_bytes(const GemmPlan& p) {
  return GS_CNT_BYTES + (size_t)p.n_tiles * p.m_tiles * p.splits * p.bm * p.bn * 4;
}

static constexpr size_t BAR_BYTES = 2 * TC_MAX_STAGES * 8 + 8 + 16;

// Max co-resident clusters of `cluster` CTAs with `smem` bytes each (cached).
static int max_active_clusters(size_t smem, int cluster) {
  struct Key { size_t smem; int cluster; int value; };
  static Key cache[64];
  static int n_cache = 0;
  for (int i = 0; i < n_cache; ++i)
    if (cache[i].smem == smem && cache[i].cluster == cluster) return cache[i].value;
  auto k = gemm_tc_kernel<SLX_EPI_NONE, bf16, 256, false>;
  configure_kernel((const void*)k);
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
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess || n <= 0) {
    (void)cudaGetLastError();
    n = sm_count() / cluster;
  }
  if (n_cache < 64) cache[n_cache++] = Key{smem, cluster, n};
  return n;
}

// Few tiles (decode): pick CTAs/SM (1 or 2) and the cluster split S that cover the most SMs
// in ONE wave (cudaOccupancyMaxActiveClusters), every split keeping >= 4 k-blocks and its
// partial tile fitting the pipeline smem.  An explicit slx_gemm_tuning overrides (tests).
static GemmPlan plan_gemm(int M, int N, int K, bool silu, size_t ws_bytes,
                          const slx_gemm_tuning* tu) {
  GemmPlan p{};
  p.kblocks = ceil_div(K, TC_BK);
  p.m_tiles = ceil_div(M, 128);
  p.bm = M >= 128 ? 128 : ((M + 15) / 16) * 16;
  const int sms = sm_count();
  const int e_ctas = tu ? tu->ctas_per_sm : 0, e_s = tu ? tu->splits : 0;
  const int e_bn = tu ? tu->bn : 0;
  const int e_gs = (tu && tu->gsplit) ? (tu->gsplit == 1 ? 1 : 0) : -1;
  double best = -1.0;
  for (int bn = 256; bn >= 128; bn -= 128) {
    if (silu && bn != 256) continue;
    if (e_bn && bn != e_bn) continue;
    const int n_tiles = ceil_div(N, bn);
    const int tiles = n_tiles * p.m_tiles;
    const size_t stage = (size_t)p.bm * TC_BK * 2 + (size_t)(bn / 128) * W_BLOCK_BYTES;
    const size_t red = (size_t)(bn + 4) * p.bm * 4;
    for (int ctas = 1; ctas <= 2; ++ctas) {
      // measured (tools/gemm_sweep.py): one CTA per SM with a deep pipeline beats two CTAs
      // with shallow ones; 2 CTAs/SM only on request
      if (e_ctas ? ctas != e_ctas : ctas != 1) continue;
      const size_t budget = ctas == 2 ? 112 * 1024 - 1024 - BAR_BYTES : 225 * 1024 - 1024 - BAR_BYTES;
      int st = (int)(budget / stage);
      st = st > TC_MAX_STAGES ? TC_MAX_STAGES : st;
      if (st < 2) continue;
      const size_t smem = (size_t)st * stage + BAR_BYTES + 1024;
      for (int gs = 0; gs <= 1; ++gs) {
        if (e_gs >= 0 && gs != e_gs) continue;
        for (int s = 1; s <= TC_MAX_CLUSTER; ++s) {
          if (gs && s == 1) continue;
          if (e_s && s != e_s) continue;
          if (s > 1 && p.m_tiles > 1) continue;
          if (s > 1 && !gs && (size_t)st * stage < red) continue;
          if (!e_s && s > 1 && ceil_div(p.kblocks, s) < 4) continue;
          if ((s - 1) * ceil_div(p.kblocks, s) >= p.kblocks && s > 1) continue;   // no empty split
          const int ctas_total = tiles * s;
          if (!e_s && ctas_total > ctas * sms) continue;                            // one wave
          if (s > 1 && !gs && !e_s && tiles > max_active_clusters(smem, s)) continue;
          if (gs) {
            GemmPlan q = p;
            q.bn = bn; q.n_tiles = n_tiles; q.splits = s;
            if (gsplit_ws_bytes(q) > ws_bytes) continue;
          }
          const int covered = ctas_total < sms ? ctas_total : sms;
          // SMs covered; then wider tiles (fewer MMAs per weight byte), deeper pipelines,
          // fewer splits (less reduction), one CTA per SM, cluster reduction over global
          const double score = covered * 1000.0 + (bn == 256 ? 50.0 : 0.0) + st * 10.0 - s -
                               ctas - 5.0 * gs;
          if (score > best) {
            best = score;
            p.bn = bn; p.n_tiles = n_tiles; p.stages = st; p.splits = s; p.smem = smem;
            p.gsplit = gs;
          }
        }
      }
    }
  }
  if (best < 0) {   // many tiles (prefill) or overrides that cannot apply: one CTA/SM, no split
    p.gsplit = 0;
    p.bn = (e_bn == 128 && !silu) ? 128 : 256;
    p.n_tiles = ceil_div(N, p.bn);
    p.splits = 1;
    const size_t stage = (size_t)p.bm * TC_BK * 2 + (size_t)(p.bn / 128) * W_BLOCK_BYTES;
    int st = (int)((225 * 1024 - 1024 - BAR_BYTES) / stage);
    p.stages = st > TC_MAX_STAGES ? TC_MAX_STAGES : st;
    if (p.stages > 4 && p.n_tiles * p.m_tiles >= sms) p.stages = 4;
    p.smem = (size_t)p.stages * stage + BAR_BYTES + 1024;
  }
  return p;
}

static const GroupMaps& no_groups() {
  static GroupMaps gm{};
  return gm;
}

template <int EPI, typename OutT, int BN, bool GROUPED = false>
static int launch_tc(const CUtensorMap& mx, const CUtensorMap& mw, const GemmArgs& a, dim3 grid,
                     size_t smem, unsigned cluster, cudaStream_t s,
                     const GroupMaps& gm = no_groups()) {
  // many full-height 256-wide tiles without a K split (prefill): the persistent kernel
  if (BN == 256 && cluster == 1 && a.splits == 1 && a.bm == 128 && grid.y == 1 &&
      (GROUPED || a.raster > 0) && a.stages <= TC_MAX_STAGES) {
    auto kp = gemm_tcp_kernel<EPI, OutT, GROUPED>;
    static bool configured_p = false;
    if (!configured_p) {
      configure_kernel((const void*)kp);
      configured_p = true;
    }
    GemmArgs ap = a;
    ap.n_work = (int)grid.x;
    const int g = ap.n_work < sm_count() ? ap.n_work : sm_count();
    const size_t smem_p = smem + 4 * 8;   // two more barrier pairs (tfull / tempty)
    // Launched WITHOUT programmatic dependent launch (measured: 443 -> 406.5 ms on the
    // config-3 prefill): under PDL the persistent CTAs are scheduled while the previous kernel
    // (e.g. a 16384-CTA RMSNorm) still runs and park beside it; one CTA per SM then has to
    // wait for its whole SM.  The kernel's griddepcontrol.wait is a no-op here; the kernels
    // after it keep PDL (this grid releases them at each CTA's last tile).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g);
    cfg.blockDim = dim3(TCP_THREADS);
    cfg.dynamicSmemBytes = smem_p;
    cfg.stream = s;
    cfg.numAttrs = 0;
    (void)cudaGetLastError();
    if (cudaLaunchKernelEx(&cfg, kp, mx, mw, ap, gm) != cudaSuccess) return SLX_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? SLX_OK : SLX_ERR_CUDA;
  }
  auto k = gemm_tc_kernel<EPI, OutT, BN, GROUPED>;
  static bool configured = false;  // per instantiation
  if (!configured) {
    configure_kernel((const void*)k);
    configured = true;
  }
  return launch_ex(k, grid, dim3(TC_THREADS), smem, s, cluster, mx, mw, a, gm);
}

template <typename OutT, int BN>
static int dispatch_epi(int epi, const CUtensorMap& mx, const CUtensorMap& mw, const GemmArgs& a,
                        dim3 grid, size_t smem, unsigned cl, cudaStream_t s) {
  if (epi == SLX_EPI_NONE) return launch_tc<SLX_EPI_NONE, OutT, BN>(mx, mw, a, grid, smem, cl, s);
  if (epi == SLX_EPI_RESIDUAL) return launch_tc<SLX_EPI_RESIDUAL, OutT, BN>(mx, mw, a, grid, smem, cl, s);
  if (BN == 256) return launch_tc<SLX_EPI_SILU_MUL, OutT, 256>(mx, mw, a, grid, smem, cl, s);
  return SLX_ERR_UNSUPPORTED;
}

static int dispatch_tc(int epi, int c_dtype, int bn, const CUtensorMap& mx, const CUtensorMap& mw,
                       const GemmArgs& a, dim3 grid, size_t smem, unsigned cl, cudaStream_t s) {
  if (c_dtype == SLX_DT_BF16)
    return bn == 256 ? dispatch_epi<bf16, 256>(epi, mx, mw, a, grid, smem, cl, s)
                     : dispatch_epi<bf16, 128>(epi, mx, mw, a, grid, smem, cl, s);
  return bn == 256 ? dispatch_epi<float, 256>(epi, mx, mw, a, grid, smem, cl, s)
                   : dispatch_epi<float, 128>(epi, mx, mw, a, grid, smem, cl, s);
}

}  // namespace slx

using namespace slx;

static unsigned long long* g_trace_base = nullptr;
static unsigned g_trace_launch = 0;
// Debug timeline: every traced launch gets its own 4096-slot window (<= 256 CTAs x 16 stamps)
// and records its kind in the window's last slot.
namespace slx {
unsigned long long* next_trace_window(int kind) {
  if (g_trace_base == nullptr) return nullptr;
  (void)kind;   // the kernel writes its kind into the window's last slot
  return g_trace_base + (size_t)(g_trace_launch++) * 4096;
}
}  // namespace slx
// Debug: every following slx_gemm_bf16 launch records 8 globaltimer stamps per CTA into buf
// ([grid CTAs][8] u64: entry, prologue done, producer past PDL wait, first stage landed, last MMA
// issued, accumulator ready, split-K rendezvous passed, exit).  NULL turns it off.
extern "C" int slx_debug_gemm_trace(void* buf) {
  g_trace_base = (unsigned long long*)buf;
  g_trace_launch = 0;
  return SLX_OK;
}

extern "C" size_t slx_gemm_workspace_bytes(int M, int N, int K, int epilogue) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  // the largest global-split plan any shape can get: one wave of 2 CTAs/SM x 128 x 256 fp32
  (void)epilogue;
  const size_t gs = GS_CNT_BYTES + (size_t)2 * sm_count() * 128 * 256 * 4;
  const size_t sk = gemm_sk_workspace_bytes(M, N, K);
  return sk > gs ? sk : gs;
}

extern "C" int slx_gemm_bf16(const void* A, int lda, const void* W, void* C, int ldc, int c_dtype,
                             const void* R, int ldr, int M, int N, int K, int epilogue,
                             int w_layout, int n_main, void* C2, int ldc2, void* ws,
                             size_t ws_bytes, void* stream) {
  return slx_gemm_bf16_ex(A, lda, W, C, ldc, c_dtype, R, ldr, M, N, K, epilogue, w_layout, n_main,
                          C2, ldc2, ws, ws_bytes, nullptr, nullptr, stream);
}

extern "C" int slx_gemm_bf16_ex(const void* A, int lda, const void* W, void* C, int ldc,
                                int c_dtype, const void* R, int ldr, int M, int N, int K,
                                int epilogue, int w_layout, int n_main, void* C2, int ldc2,
                                void* ws, size_t ws_bytes, const slx_l2_prefetch* pf,
                                const slx_gemm_tuning* tuning, void* stream) {
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
    SLX_CHECK_ARG(C2 != nullptr || ldc >= N);   // any N: the epilogue masks columns >= N
  }
  if (C2 != nullptr) {
    SLX_CHECK_ARG(epilogue != SLX_EPI_SILU_MUL && n_main > 0 && n_main < N && n_main % 16 == 0 &&
                  ldc2 >= N - n_main && ldc2 % 4 == 0 && ldc >= n_main);
    SLX_CHECK_ALIGN(C2, 16);
  } else {
    n_main = N;
  }
  if (epilogue == SLX_EPI_RESIDUAL) SLX_CHECK_ARG(R != nullptr && ldr >= n_main && ldr % 8 == 0);
  if (M == 0) return SLX_OK;
  if (ws) SLX_CHECK_ALIGN(ws, 256);
  if (w_layout == SLX_W_TILED) {   // decode: stream-K kernel (gemm_sk.cu) when it applies
    SkCall sc{A, lda, W, C, ldc, c_dtype, R, ldr, M, N, K, epilogue, n_main, C2, ldc2,
              ws, ws ? ws_bytes : 0, stream, next_trace_window(1 + epilogue), pf, nullptr, 0, 0,
              tuning};
    const int st = gemm_sk_launch(sc);
    if (st != SLX_ERR_UNSUPPORTED) return st;
  }
  GemmPlan p = plan_gemm(M, N, K, epilogue == SLX_EPI_SILU_MUL, ws ? ws_bytes : 0, tuning);
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.bm = p.bm; a.stages = p.stages; a.kblocks = p.kblocks; a.splits = p.splits;
  a.n_tiles = p.n_tiles;
  a.C = C; a.ldc = ldc; a.R = R; a.ldr = ldr;
  a.w_tiled = w_layout == SLX_W_TILED;
  a.n_main = n_main;
  a.C2 = (float*)C2;
  a.ldc2 = ldc2;
  a.gsplit = p.gsplit;
  a.trace = nullptr;
  if (p.gsplit) {
    a.ws_cnt = (int*)((char*)ws + 32768);   // [tiles][2]: arrival, departure ([0,32K): gemm_sk)
    a.ws_part = (float*)((char*)ws + GS_CNT_BYTES);
  }
  // tiled W: a [n_blocks * kblocks * 128, 64] matrix of contiguous 16 KB boxes
  const int w_rows = a.w_tiled ? ceil_div(N, 128) * p.kblocks * 128 : N;
  const int w_cols = a.w_tiled ? TC_BK : K;
  CUtensorMap mx, mw;
  if (!make_tmap(&mx, A, M, K, lda, p.bm) || !make_tmap(&mw, W, w_rows, w_cols, w_cols, 128))
    return SLX_ERR_CUDA;
  dim3 grid((unsigned)(p.n_tiles * p.splits), (unsigned)p.m_tiles);
  constexpr int raster = 16;   // measured best of {4, 8, 16}
  if (p.splits == 1 && p.m_tiles > 1 && raster > 0) {
    a.raster = raster;
    a.m_tiles = p.m_tiles;
    grid = dim3((unsigned)(p.n_tiles * p.m_tiles), 1);
  }
  return dispatch_tc(epilogue, c_dtype, p.bn, mx, mw, a, grid, p.smem,
                     p.gsplit ? 1u : (unsigned)p.splits, (cudaStream_t)stream);
}

extern "C" size_t slx_gemm_splitk_bytes(int M, int N, int splits) {
  return gemm_sk_splitk_bytes(M, N, splits);
}

extern "C" int slx_gemm_bf16_splitk(const void* A, int lda, const void* W, int M, int N, int K,
                                    int splits, float* part, size_t part_bytes,
                                    const slx_l2_prefetch* pf, void* stream) {
  SLX_CHECK_ARG(A && W && part && M > 0 && N > 0 && K > 0 && lda >= K && K % 8 == 0 &&
                lda % 8 == 0 && N % 16 == 0 && splits >= 1);
  SLX_CHECK_ALIGN(A, 16);
  SLX_CHECK_ALIGN(W, 16);
  SLX_CHECK_ALIGN(part, 16);
  SkCall sc{A, lda, W, nullptr, 0, SLX_DT_BF16, nullptr, 0, M, N, K, SLX_EPI_NONE, N, nullptr, 0,
            nullptr, 0, stream, next_trace_window(4), pf, part, splits, part_bytes, nullptr};
  return gemm_sk_launch(sc);
}

// ------------------------------------------------------------------ weight packing
namespace slx {
__global__ void pack_weight_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, int N,
                                   int K, int ld, int kblocks) {
  pdl_wait();
  pdl_trigger();
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

// Write rows [row0, row0 + n) of an already packed (SLX_W_TILED) matrix from row-major src.
__global__ void pack_rows_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, int n,
                                 int K, int ld, int row0, int kblocks) {
  pdl_wait();
  pdl_trigger();
  const size_t chunk = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)n * kblocks * 8;
  if (chunk >= total) return;
  const int c8 = (int)(chunk % 8);
  const int kb = (int)((chunk / 8) % kblocks);
  const int i = (int)(chunk / 8 / kblocks);
  const int row = row0 + i, k = kb * TC_BK + c8 * 8;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (src != nullptr && k < K) v = *reinterpret_cast<const uint4*>(src + (size_t)i * ld + k);
  const size_t prow = ((size_t)(row >> 7) * kblocks + kb) * 128 + (row & 127);
  *reinterpret_cast<uint4*>(dst + prow * TC_BK + c8 * 8) = v;
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

extern "C" int slx_pack_weight_rows(void* dst, const void* src, int n_rows, int K, int ld,
                                    int row0, void* stream) {
  SLX_CHECK_ARG(dst && n_rows > 0 && K > 0 && K % 8 == 0 && row0 >= 0 && (!src || ld >= K) &&
                ld % 8 == 0);
  SLX_CHECK_ALIGN(dst, 16);
  if (src) SLX_CHECK_ALIGN(src, 16);
  const int kb = ceil_div(K, TC_BK);
  const size_t total = (size_t)n_rows * kb * 8;
  return launch_ex(pack_rows_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0,
                   (cudaStream_t)stream, 1u, (bf16*)dst, (const bf16*)src, n_rows, K, ld, row0, kb);
}

// ------------------------------------------------------------------ grouped GEMM (SGMV)
extern "C" size_t slx_gemm_group_tile_bytes(void) { return sizeof(GroupTile); }

extern "C" int slx_gemm_bf16_lorafold(const void* A, int lda, const void* W, int w_layout, void* C,
                                      int ldc, int c_dtype, const void* R, int ldr, int M, int N,
                                      int K, int epilogue, const void* gtiles, int n_gtiles,
                                      const void* v, int ldv, int n_targets, const int* t_bound,
                                      int n_adapters, const uint64_t* b_ptrs, const int* b_rows,
                                      const int* ranks, const slx_rope_kv* rope, void* stream) {
  SLX_CHECK_ARG(A && W && C && v && gtiles && t_bound && M > 0 && N > 0 && K > 0 &&
                K % 8 == 0 && lda >= K && lda % 8 == 0 && ldc % 8 == 0 && n_gtiles >= 0 &&
                n_targets >= 1 && n_targets <= 3 && n_adapters >= 0 && n_adapters <= 16 &&
                n_adapters * n_targets <= TC_MAX_MAPS && ldv >= 64 * n_targets && ldv % 8 == 0);
  SLX_CHECK_ARG(w_layout == SLX_W_ROWMAJOR || w_layout == SLX_W_TILED);
  SLX_CHECK_ARG(epilogue == SLX_EPI_NONE || epilogue == SLX_EPI_RESIDUAL);
  SLX_CHECK_ARG(c_dtype == SLX_DT_BF16 || c_dtype == SLX_DT_F32);
  if (epilogue == SLX_EPI_RESIDUAL) SLX_CHECK_ARG(R != nullptr && ldr % 8 == 0);
  SLX_CHECK_ALIGN(A, 16);
  SLX_CHECK_ALIGN(C, 16);
  SLX_CHECK_ALIGN(v, 16);
  for (int t = 0; t < n_targets; ++t)   // target column ranges start on 256-column tiles
    SLX_CHECK_ARG(t_bound[t] % 256 == 0 && (t == 0 ? t_bound[t] == 0 : t_bound[t] > t_bound[t - 1]));
  if (n_gtiles == 0) return SLX_OK;
  GroupMaps gm{};
  for (int a = 0; a < n_adapters; ++a) {
    SLX_CHECK_ARG(ranks[a] > 0 && ranks[a] <= 64 && ranks[a] % 8 == 0);
    for (int t = 0; t < n_targets; ++t) {
      const int i = a * n_targets + t;
      // B_(a, t) [d_out, rank] row-major: columns >= rank of the 64-wide box read as zeros
      if (b_ptrs[i] == 0 || !make_tmap(&gm.w[i], (const void*)b_ptrs[i], b_rows[t], ranks[a],
                                       ranks[a], 128))
        return b_ptrs[i] == 0 ? SLX_ERR_INVALID : SLX_ERR_CUDA;
      gm.alpha[i] = 1.f;
    }
  }
  if (!make_tmap(&gm.v, v, M, 64 * n_targets, ldv, 128)) return SLX_ERR_CUDA;
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.bm = 128; a.kblocks = ceil_div(K, TC_BK); a.splits = 1; a.n_tiles = 1;
  const size_t stage = (size_t)128 * TC_BK * 2 + 2 * W_BLOCK_BYTES;
  a.stages = 4;
  const size_t smem = (size_t)a.stages * stage + BAR_BYTES + 1024;
  a.C = C; a.ldc = ldc; a.R = R; a.ldr = ldr; a.w_tiled = w_layout == SLX_W_TILED; a.n_main = N;
  a.gtiles = (const GroupTile*)gtiles;
  a.lfold = 1;
  if (rope != nullptr) {
    SLX_CHECK_ARG(epilogue == SLX_EPI_NONE && c_dtype == SLX_DT_BF16 && rope->head_dim == 128 &&
                  rope->tok_pos && rope->tok_seq && rope->cos_tab && rope->sin_tab &&
                  rope->k_cache && rope->v_cache && rope->max_ctx > 0 && rope->heads > 0 &&
                  rope->kv_heads > 0 && rope->heads % rope->kv_heads == 0 &&
                  (rope->heads * 128) % 256 == 0 && (rope->kv_heads * 128) % 256 == 0 &&
                  N == (rope->heads + 2 * rope->kv_heads) * 128);
    SLX_CHECK_ALIGN(rope->k_cache, 16);
    SLX_CHECK_ALIGN(rope->v_cache, 16);
    SLX_CHECK_ALIGN(rope->cos_tab, 16);
    SLX_CHECK_ALIGN(rope->sin_tab, 16);
    a.rope = 1;
    a.r_h = rope->heads; a.r_hkv = rope->kv_heads; a.r_max_ctx = rope->max_ctx;
    a.r_pos = rope->tok_pos; a.r_seq = rope->tok_seq;
    a.r_cos = rope->cos_tab; a.r_sin = rope->sin_tab;
    a.r_kc = (bf16*)rope->k_cache; a.r_vc = (bf16*)rope->v_cache;
  }
  a.lnt = n_targets;
  for (int t = 0; t < 4; ++t) a.lbound[t] = t < n_targets ? t_bound[t] : 0;
  CUtensorMap mx, mw;
  const int kb = ceil_div(K, TC_BK);
  const int w_rows = a.w_tiled ? ceil_div(N, 128) * kb * 128 : N;
  const int w_cols = a.w_tiled ? TC_BK : K;
  if (!make_tmap(&mx, A, M, K, lda, 128) || !make_tmap(&mw, W, w_rows, w_cols, w_cols, 128))
    return SLX_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)n_gtiles, 1);
  if (c_dtype == SLX_DT_BF16) {
    if (epilogue == SLX_EPI_NONE)
      return launch_tc<SLX_EPI_NONE, bf16, 256, true>(mx, mw, a, grid, smem, 1u, s, gm);
    return launch_tc<SLX_EPI_RESIDUAL, bf16, 256, true>(mx, mw, a, grid, smem, 1u, s, gm);
  }
  if (epilogue == SLX_EPI_NONE)
    return launch_tc<SLX_EPI_NONE, float, 256, true>(mx, mw, a, grid, smem, 1u, s, gm);
  return launch_tc<SLX_EPI_RESIDUAL, float, 256, true>(mx, mw, a, grid, smem, 1u, s, gm);
}

extern "C" int slx_gemm_grouped_bf16(const void* A, int lda, int M, int K, int n_groups,
                                     int n_seg, const uint64_t* w_ptrs, const int* w_rows,
                                     const int* w_cols, const int* w_ld, const float* alpha, void* C,
                                     int ldc, int c_dtype, const void* R, int ldr, int N, int epilogue,
                                     const void* gtiles, int n_gtiles, void* stream) {
  SLX_CHECK_ARG(A && C && w_ptrs && w_rows && w_cols && w_ld && alpha && gtiles && M > 0 && K > 0 &&
                K % 8 == 0 && lda >= K && lda % 8 == 0 && ldc % 8 == 0 && N > 0 &&
                n_groups >= 1 && n_groups <= TC_MAX_GROUPS && n_gtiles >= 0 && n_seg >= 1 &&
                n_seg <= 4 && n_groups * n_seg <= TC_MAX_MAPS && (n_seg == 1 || N <= 64 * n_seg));
  SLX_CHECK_ARG(epilogue == SLX_EPI_NONE || epilogue == SLX_EPI_RESIDUAL);
  SLX_CHECK_ARG(c_dtype == SLX_DT_BF16 || c_dtype == SLX_DT_F32);
  if (epilogue == SLX_EPI_RESIDUAL) SLX_CHECK_ARG(R != nullptr && ldr % 8 == 0);
  SLX_CHECK_ALIGN(A, 16);
  SLX_CHECK_ALIGN(C, 16);
  if (n_gtiles == 0) return SLX_OK;
  GroupMaps gm{};
  for (int i = 0; i < n_groups * n_seg; ++i) {
    // per-map K extent: columns >= w_cols[i] read as zeros; with segments (n_seg > 1) map i is
    // segment i % n_seg of group i / n_seg: <= 64 rows (rows beyond w_rows read as zeros)
    SLX_CHECK_ARG(w_ptrs[i] != 0 && w_rows[i] > 0 && w_cols[i] > 0 && w_cols[i] <= K &&
                  w_ld[i] >= w_cols[i] && w_ld[i] % 8 == 0 && (n_seg == 1 || w_rows[i] <= 64));
    if (!make_tmap(&gm.w[i], (const void*)w_ptrs[i], w_rows[i], w_cols[i], w_ld[i],
                   n_seg > 1 ? 64 : 128))
      return SLX_ERR_CUDA;
    gm.alpha[i] = alpha[i];
  }
  GemmArgs a{};
  a.M = M; a.N = N; a.K = K;
  a.bm = 128; a.kblocks = ceil_div(K, TC_BK); a.splits = 1; a.n_tiles = 1;
  a.gseg = n_seg;
  const size_t stage = (size_t)128 * TC_BK * 2 + 2 * W_BLOCK_BYTES;
  a.stages = a.kblocks < 4 ? (a.kblocks < 2 ? 2 : a.kblocks) : 4;
  const size_t smem = (size_t)a.stages * stage + BAR_BYTES + 1024;
  a.C = C; a.ldc = ldc; a.R = R; a.ldr = ldr; a.w_tiled = 0; a.n_main = N;
  a.gtiles = (const GroupTile*)gtiles;
  CUtensorMap mx;
  if (!make_tmap(&mx, A, M, K, lda, 128)) return SLX_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)stream;
  dim3 grid((unsigned)n_gtiles, 1);
  if (c_dtype == SLX_DT_BF16) {
    if (epilogue == SLX_EPI_NONE)
      return launch_tc<SLX_EPI_NONE, bf16, 256, true>(mx, mx, a, grid, smem, 1u, s, gm);
    return launch_tc<SLX_EPI_RESIDUAL, bf16, 256, true>(mx, mx, a, grid, smem, 1u, s, gm);
  }
  if (epilogue == SLX_EPI_NONE)
    return launch_tc<SLX_EPI_NONE, float, 256, true>(mx, mx, a, grid, smem, 1u, s, gm);
  return launch_tc<SLX_EPI_RESIDUAL, float, 256, true>(mx, mx, a, grid, smem, 1u, s, gm);
}
