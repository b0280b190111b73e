// K1, decode path: stream-K tcgen05 GEMM for skinny activations (M <= 128 token rows).
//
//   C[M,N] = A[M,K] . W[N,K]^T (+ residual | SiLU*mul | fp32 side output), W in SLX_W_TILED.
//
// Decode projections stream 37-262 MB of weights per launch against 64 token rows, so they are
// HBM-bound and the whole game is keeping all 148 SMs streaming weights from the first to the
// last microsecond.  The weight tiles are 256 rows (the N = 256 side of tcgen05.mma, see
// gemm_tc.cu) and there are only 16-125 of them, so a tile-per-CTA grid leaves SMs idle and an
// integer split-K leaves stragglers.  Stream-K fixes both: the n_tiles x kblocks MMA units are
// cut into G (<= #SMs) equal contiguous ranges, one per persistent CTA; a range covers the tail
// of one tile, whole tiles, and the head of another ("segments").
//
// Roles (192 threads): warp 0 lane 0 TMA producer (weights are fetched before the PDL wait),
// warp 1 lane 0 MMA issuer (M = 64: the <= 64 token rows spread over all four TMEM lane
// quadrants) into one of TWO TMEM accumulators (2 x 256 columns), warps 2-5 epilogue, each
// draining 16 rows.  Because the epilogue has its own warps and the accumulator is double-buffered,
// draining segment j overlaps the MMAs of segment j+1.
//
// Split tiles are reduced deterministically without clusters: every piece is written in fp32
// to the workspace (coalesced [chunk][row][16] layout), the piece holders arrive on a per-tile
// counter, and — only after ALL of a CTA's pieces have arrived, so no CTA ever waits while
// holding an un-arrived piece — each of the np holders reduces a 1/np slice of the tile,
// summing pieces in piece order (bit-identical run to run), and applies the epilogue.  A
// departure counter lets the last holder re-zero both counters (self-cleaning workspace).
//
// Replaces the modelled decode step of the reference (engine.py:888,909 decode_ms_per_token;
// batching.py:17-21) with the real projections of the decode step.
#include <cuda.h>

#include "common.cuh"
#include "gemm_host.h"
#include "tc_ptx.cuh"

namespace slx {
namespace {

constexpr int SK_THREADS = 192;
constexpr int SK_BN = 256;
constexpr int SK_BK = 64;
constexpr int SK_MAX_STAGES = 8;
constexpr int SK_MAX_SEGS = 8;
constexpr int SK_MAX_M = 128;
constexpr int SK_PB = 8;                        // pieces loaded per batch in the reduction
constexpr int SK_WBOX = 128 * SK_BK * 2;        // one contiguous 16 KB weight box
constexpr size_t SK_CNT_BYTES = 32 * 1024;      // counters at the head of ws: 2 u32 per tile
constexpr size_t SK_PART_OFF = 64 * 1024;       // partials (gemm_tc's counters sit in [32K, 64K))
constexpr size_t SK_BAR_BYTES = (2 * SK_MAX_STAGES + 4) * 8 + 16 + 4 * SK_MAX_SEGS + 16;

struct SkArgs {
  int M, N, bm, stages, kblocks, n_tiles, G, pmax;
  int cs;        // > 1: cluster mode, G = n_tiles * cs, tile t's pieces are cluster t (DSMEM)
  int U;         // n_tiles * kblocks MMA units (one 64-wide k-block of one 256-row tile);
                 // U * G < 2^31 (planner), so all unit arithmetic is 32-bit
  void* C;
  int ldc;
  const void* R;
  int ldr;
  int n_main;    // columns >= n_main: fp32 side output C2 (stacked LoRA A rows)
  float* C2;
  int ldc2;
  float* part;   // [n_tiles][pmax][16 chunks][bm][16] fp32 pieces
  uint32_t* cnt; // [n_tiles][2]: arrivals, departures (monotonic; A == D between launches)
  unsigned long long* trace;
  PfArgs pf;     // L2 prefetch of the next kernel's first bytes, after our last TMA issue
  int part_only; // slx_gemm_bf16_splitk: every piece written to `part`, reduced by the consumer
};

__device__ __forceinline__ unsigned long long sk_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
#define SK_TR(i) \
  if (g.trace) g.trace[(size_t)blockIdx.x * 16 + (i)] = sk_timer()

__host__ __device__ __forceinline__ int sk_lo(int U, int G, int c) { return c * U / G; }
// CTA whose range holds unit u: the largest c with floor(c U / G) <= u.
__host__ __device__ __forceinline__ int sk_cta_of(int U, int G, int u) { return ((u + 1) * G - 1) / U; }

template <typename OutT>
__device__ __forceinline__ void sk_store16(OutT* row, int n0, int n_lim, const float* v) {
  if (sizeof(OutT) == 2 && n0 + 16 <= n_lim) {
    Vec8<bf16>::store(reinterpret_cast<bf16*>(row + n0), v);
    Vec8<bf16>::store(reinterpret_cast<bf16*>(row + n0 + 8), v + 8);
  } else if (sizeof(OutT) == 4 && n0 + 16 <= n_lim) {
    float4* p = reinterpret_cast<float4*>(row + n0);
#pragma unroll
    for (int q = 0; q < 4; ++q) p[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n0 + j < n_lim) row[j + n0] = from_f32<OutT>(v[j]);
  }
}

// Residual of 16 columns [n, n+16) of row m (bf16 / fp32, as OutT), zero beyond lim.
template <typename OutT>
__device__ __forceinline__ void sk_load_res(const SkArgs& g, int m, int n, int lim, float* r) {
  const OutT* R = reinterpret_cast<const OutT*>(g.R) + (size_t)m * g.ldr;
  if (n + 16 <= lim) {
    Vec8<OutT>::load(R + n, r);
    Vec8<OutT>::load(R + n + 8, r + 8);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = n + j < lim ? to_f32(R[n + j]) : 0.f;
  }
}

// Final values of 16 columns [n, n+16) of row m (not SiLU): side output or C (+ residual).
template <int EPI, typename OutT>
__device__ __forceinline__ void sk_finish(const SkArgs& g, int m, int n, float* v, const float* res) {
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
  const int lim = g.C2 != nullptr ? g.n_main : g.N;
  if (EPI == SLX_EPI_RESIDUAL) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] += res[j];
  }
  sk_store16(reinterpret_cast<OutT*>(g.C) + (size_t)m * g.ldc, n, lim, v);
}

// fast-math SiLU: no IEEE-division slow path (whose per-element branch serialises the epilogue)
__device__ __forceinline__ float sk_silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

// PO (part only, slx_gemm_bf16_splitk): every segment is written as an fp32 piece and nothing
// else — the reduction, cluster and direct-epilogue code is compiled out, which
// keeps the register footprint small enough for the consumer's CTAs to co-reside under PDL.
template <int EPI, typename OutT, bool PO = false>
__global__ void __launch_bounds__(SK_THREADS, 1)
gemm_sk_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_w,
               SkArgs g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int x_bytes = g.bm * SK_BK * 2;
  const int stage_bytes = x_bytes + 2 * SK_WBOX;
  uint64_t* full = (uint64_t*)(smem + g.stages * stage_bytes);
  uint64_t* empty = full + SK_MAX_STAGES;
  uint64_t* tfull = empty + SK_MAX_STAGES;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  const int kb = g.kblocks;
  const int lo = sk_lo(g.U, g.G, c), hi = sk_lo(g.U, g.G, c + 1);
  const int n_units = hi - lo;

  if (threadIdx.x == 0) {
    SK_TR(0);
    if (g.trace && blockIdx.x == 0) g.trace[4095] = PO ? 4 : 1 + EPI;
    tc::tma_prefetch_desc(&tmap_x);
    tc::tma_prefetch_desc(&tmap_w);
    for (int s = 0; s < g.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * SK_BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) SK_TR(1);
  if (threadIdx.x != 0) {
    pdl_wait();
    pdl_trigger();
  }

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = tc::policy_evict_first();   // weights: streamed once
      const uint64_t pol_x = tc::policy_evict_last();    // activations: re-read by every CTA
      auto load_w = [&](int i, uint8_t* st, uint64_t* bar) {
        const int u = lo + i;
        const int tile = u / kb, k = u - tile * kb;
#pragma unroll
        for (int b = 0; b < 2; ++b)
          tc::tma_load_2d(st + x_bytes + b * SK_WBOX, &tmap_w, bar, 0,
                          ((tile * 2 + b) * kb + k) * 128, pol_w);
      };
      auto load_x = [&](int i, uint8_t* st, uint64_t* bar) {
        tc::tma_load_2d(st, &tmap_x, bar, ((lo + i) % kb) * SK_BK, 0, pol_x);
      };
      const int npre = min(n_units, g.stages);
      // weights do not depend on the previous kernel: start streaming before the PDL wait
      for (int i = 0; i < npre; ++i) {
        tc::mbar_arrive_expect_tx(&full[i], stage_bytes);
        load_w(i, smem + i * stage_bytes, &full[i]);
      }
      pdl_wait();
      pdl_trigger();
      SK_TR(2);
      for (int i = 0; i < npre; ++i) load_x(i, smem + i * stage_bytes, &full[i]);
      for (int i = npre; i < n_units; ++i) {
        const int s = i % g.stages;
        tc::mbar_wait(&empty[s], ((i / g.stages) & 1) ^ 1);
        uint8_t* st = smem + s * stage_bytes;
        tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
        load_w(i, st, &full[s]);
        load_x(i, st, &full[s]);
      }
      l2_prefetch_part(g.pf, c, g.G);   // keep HBM busy across the kernel boundary
    }
    __syncwarp();   // reconverge before the CTA-wide barrier at the end
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      // D[128 tok x 256 w] (+)= X[128 x 16] . W[256 x 16]^T; X rows >= bm read stale smem and
      // only feed D rows that are never read.
      // M = 64 (bm <= 64 token rows): the accumulator's row r lands in lane r % 16 of TMEM lane
      // quadrant r / 16 (tools/probe/m64_layout.cu), so all four epilogue warps drain it;
      // M = 128 (65..128 rows): row r is lane r
      const uint32_t idesc = g.bm > 64 ? tc::idesc_bf16_f32(128, SK_BN) : tc::idesc_bf16_f32(64, SK_BN);
      int j = -1;
      uint32_t d = 0;
      bool first = true;
      for (int i = 0; i < n_units; ++i) {
        const int k = (lo + i) % kb;
        if (i == 0 || k == 0) {   // new segment -> next accumulator
          ++j;
          tc::mbar_wait(&tempty[j & 1], ((j >> 1) & 1) ^ 1);
          tc::fence_after_sync();
          d = tmem_base + (uint32_t)((j & 1) * SK_BN);
          first = true;
        }
        const int s = i % g.stages;
        tc::mbar_wait(&full[s], (i / g.stages) & 1);
        tc::fence_after_sync();
        if (i == 0) SK_TR(3);
        const uint32_t st = tc::smem_u32(smem + s * stage_bytes);
#pragma unroll
        for (int ks = 0; ks < SK_BK / 16; ++ks)
          tc::mma_bf16_ss(d, tc::smem_desc_sw128(st + ks * 32),
                          tc::smem_desc_sw128(st + x_bytes + ks * 32), idesc,
                          (first && ks == 0) ? 0u : 1u);
        first = false;
        tc::mma_commit(&empty[s]);
        if (k == kb - 1 || i == n_units - 1) tc::mma_commit(&tfull[j & 1]);
      }
      SK_TR(4);
    }
    __syncwarp();
  } else if (!PO && g.cs > 1) {
    // ------------------------------------------- epilogue, cluster mode (warps 2-5)
    // This CTA holds piece `rank` of tile c / cs (exactly one segment).  Pieces are staged in
    // each CTA's own (now idle) pipeline smem as [chunk][row][16] fp32 and reduced through
    // DSMEM: CTA `rank` sums a 1/cs slice of the tile over the cs peers in rank order.
    const bool m128 = g.bm > 64;
    const int q = warp & 3, r = m128 ? q * 32 + lane : q * 16 + (lane & 15), et = threadIdx.x - 64;
    const bool qlive = (m128 ? q * 32 : q * 16) < g.bm;   // warp-uniform
    const bool rv = m128 || lane < 16;   // M = 64: lanes 16-31 of the quadrant hold no row
    const bool silu = EPI == SLX_EPI_SILU_MUL;
    const int cs = g.cs, rank = c % cs, tile = c / cs;
    const int n_out = silu ? g.N / 2 : g.N;
    float* stg = reinterpret_cast<float*>(smem);
    tc::mbar_wait(&tfull[0], 0);
    if (et == 0) SK_TR(9);
    __syncwarp();
    tc::fence_after_sync();
    if (qlive) {
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16);
      for (int ch = 0; ch < 16; ch += 2) {
        float v0[16], v1[16];
        tc::tmem_ld16x2(tacc + ch * 16, tacc + ch * 16 + 16, v0, v1);
        if (rv && r < g.bm) {
          float4* p0 = reinterpret_cast<float4*>(stg + ((size_t)ch * g.bm + r) * 16);
          float4* p1 = reinterpret_cast<float4*>(stg + ((size_t)(ch + 1) * g.bm + r) * 16);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            p0[e] = make_float4(v0[4 * e], v0[4 * e + 1], v0[4 * e + 2], v0[4 * e + 3]);
            p1[e] = make_float4(v1[4 * e], v1[4 * e + 1], v1[4 * e + 2], v1[4 * e + 3]);
          }
        }
      }
    }
    tc::fence_before_sync();
    tc::cluster_sync();   // #1: every piece of the tile staged
    if (et == 0) SK_TR(6);
    const uint32_t stg_s = tc::smem_u32(stg);
    const int nfc = silu ? 8 : 16;
    const int items = nfc * g.bm;
    const int it_lo = rank * items / cs, it_hi = (rank + 1) * items / cs;
    for (int it = it_lo + et; it < it_hi; it += 128) {
      const int ch = it / g.bm, m = it % g.bm;
      const int n = tile * SK_BN + ch * 16;
      float res[16];
      if (EPI == SLX_EPI_RESIDUAL && m < g.M && n < g.N)
        sk_load_res<OutT>(g, m, n, g.C2 != nullptr ? g.n_main : g.N, res);
      const uint32_t oa = stg_s + (uint32_t)(((ch * g.bm + m) * 16) * 4);
      const uint32_t ob = stg_s + (uint32_t)((((ch + 8) * g.bm + m) * 16) * 4);
      float a[16], b[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) a[e] = b[e] = 0.f;
      constexpr int PB = EPI == SLX_EPI_SILU_MUL ? 4 : 8;   // register budget
      for (int p0 = 0; p0 < cs; p0 += PB) {
        float4 qa[PB][4], qb[silu ? PB : 1][4];
#pragma unroll
        for (int bi = 0; bi < PB; ++bi) {
          if (p0 + bi < cs) {
            const uint32_t ra = tc::mapa(oa, (uint32_t)(p0 + bi));
#pragma unroll
            for (int e = 0; e < 4; ++e) qa[bi][e] = tc::ld_dsmem4(ra + e * 16);
            if (silu) {
              const uint32_t rb = tc::mapa(ob, (uint32_t)(p0 + bi));
#pragma unroll
              for (int e = 0; e < 4; ++e) qb[silu ? bi : 0][e] = tc::ld_dsmem4(rb + e * 16);
            }
          }
        }
#pragma unroll
        for (int bi = 0; bi < PB; ++bi) {   // fixed rank order: deterministic
          if (p0 + bi < cs) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              a[4 * e] += qa[bi][e].x; a[4 * e + 1] += qa[bi][e].y;
              a[4 * e + 2] += qa[bi][e].z; a[4 * e + 3] += qa[bi][e].w;
              if (silu) {
                const float4 t = qb[silu ? bi : 0][e];
                b[4 * e] += t.x; b[4 * e + 1] += t.y; b[4 * e + 2] += t.z; b[4 * e + 3] += t.w;
              }
            }
          }
        }
      }
      if (m >= g.M) continue;
      if (silu) {
#pragma unroll
        for (int e = 0; e < 16; ++e) a[e] = sk_silu(a[e]) * b[e];
        sk_store16(reinterpret_cast<OutT*>(g.C) + (size_t)m * g.ldc, tile * 128 + ch * 16, n_out, a);
      } else if (n < g.N) {
        sk_finish<EPI, OutT>(g, m, n, a, res);
      }
    }
    if (et == 0) SK_TR(8);
    tc::cluster_sync();   // #2: keep our smem alive until every peer has read it
  } else {
    // -------------------------------------------------------------- epilogue (warps 2-5)
    const int q = warp & 3;              // TMEM lane quadrant this warp may access
    const bool m128 = g.bm > 64;         // M = 128 MMA: row r is TMEM lane r
    const int r = m128 ? q * 32 + lane : q * 16 + (lane & 15);   // token row of this thread
    const bool rv = m128 || lane < 16;   // M = 64: lanes 16-31 of the quadrant hold no row
    const int et = threadIdx.x - 64;     // 0..127
    const bool qlive = (m128 ? q * 32 : q * 16) < g.bm;   // warp-uniform
    const bool silu = EPI == SLX_EPI_SILU_MUL;
    const int piece_floats = g.bm * SK_BN;
    const int n_out = silu ? g.N / 2 : g.N;
    // Counters per tile: A (arrivals) and D (departures) only ever increase, and A == D whenever
    // no launch is in flight.  Reading D before arriving gives this launch's base: the tile is
    // complete once A - base == np.  No reset, so nothing is left to clean at the tail.
    uint32_t* base = reinterpret_cast<uint32_t*>(tmem_slot + 4);   // [SK_MAX_SEGS]
    if (et == 0) {
      int j = 0;
      for (int u = lo; u < hi; ++j) {
        const int tile = u / kb, k0 = u - tile * kb;
        const int k1 = min(kb, k0 + (hi - u));
        u += k1 - k0;
        if (!(k0 == 0 && k1 == kb) && !PO) base[j] = tc::ld_relaxed_gpu(&g.cnt[2 * tile + 1]);
      }
    }

    // phase 1: drain every segment (direct epilogue for whole tiles, fp32 piece otherwise)
    int j = 0;
    for (int u = lo; u < hi; ++j) {
      const int tile = u / kb, k0 = u - tile * kb;
      const int k1 = min(kb, k0 + (hi - u));
      u += k1 - k0;
      const int acc = j & 1;
      tc::mbar_wait(&tfull[acc], (j >> 1) & 1);
      if (et == 0) SK_TR(9 + (j < 2 ? j : 1));
      __syncwarp();
      tc::fence_after_sync();
      if (j == 0 && et == 0) SK_TR(5);
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * SK_BN);
      const bool whole = k0 == 0 && k1 == kb && !PO;
      if (whole) {
        if (qlive) {
          const int m = r;
          if (silu) {
            for (int ch = 0; ch < 8; ++ch) {
              float gv[16], uv[16];
              tc::tmem_ld16x2(tacc + ch * 16, tacc + 128 + ch * 16, gv, uv);
              if (rv && m < g.M) {
#pragma unroll
                for (int e = 0; e < 16; ++e) gv[e] = sk_silu(gv[e]) * uv[e];
                sk_store16(reinterpret_cast<OutT*>(g.C) + (size_t)m * g.ldc, tile * 128 + ch * 16,
                           n_out, gv);
              }
            }
          } else {
            for (int ch = 0; ch < 16; ch += 2) {
              float v0[16], v1[16], r0[16], r1[16];
              tc::tmem_ld16x2(tacc + ch * 16, tacc + ch * 16 + 16, v0, v1);
              const int n = tile * SK_BN + ch * 16;
              if (rv && m < g.M && n < g.N) {
                if (EPI == SLX_EPI_RESIDUAL) {
                  const int lim = g.C2 != nullptr ? g.n_main : g.N;
                  sk_load_res<OutT>(g, m, n, lim, r0);
                  sk_load_res<OutT>(g, m, n + 16, lim, r1);
                }
                sk_finish<EPI, OutT>(g, m, n, v0, r0);
                if (n + 16 < g.N) sk_finish<EPI, OutT>(g, m, n + 16, v1, r1);
              }
            }
          }
        }
      } else {
        const int piece = c - sk_cta_of(g.U, g.G, tile * kb);
        float* dst = g.part + (size_t)(tile * g.pmax + piece) * piece_floats;
        if (qlive) {
          for (int ch = 0; ch < 16; ch += 2) {
            float v0[16], v1[16];
            tc::tmem_ld16x2(tacc + ch * 16, tacc + ch * 16 + 16, v0, v1);
            if (rv && r < g.bm) {
              float4* p0 = reinterpret_cast<float4*>(dst + ((size_t)ch * g.bm + r) * 16);
              float4* p1 = reinterpret_cast<float4*>(dst + ((size_t)(ch + 1) * g.bm + r) * 16);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                p0[e] = make_float4(v0[4 * e], v0[4 * e + 1], v0[4 * e + 2], v0[4 * e + 3]);
                p1[e] = make_float4(v1[4 * e], v1[4 * e + 1], v1[4 * e + 2], v1[4 * e + 3]);
              }
            }
          }
        }
      }
      tc::fence_before_sync();
      tc::named_bar_sync(1, 128);
      if (et == 0) {
        tc::mbar_arrive(&tempty[acc]);
        // release at gpu scope after the CTA barrier publishes every thread's piece stores
        if (!whole && !PO) tc::red_release_gpu_add(&g.cnt[2 * tile], 1u);
      }
    }

    // phase 2: wait for every split tile held, then reduce this CTA's slice of each
    if (PO) {   // the consumer reduces the pieces (no rendezvous, no tail)
      if (et == 0) SK_TR(8);
    } else {
    if (et == 0) {
      SK_TR(6);
      int jj = 0;
      for (int u = lo; u < hi; ++jj) {
        const int tile = u / kb, k0 = u - tile * kb;
        const int k1 = min(kb, k0 + (hi - u));
        u += k1 - k0;
        if (k0 == 0 && k1 == kb) continue;
        const int t0 = tile * kb;
        const uint32_t np = (uint32_t)(sk_cta_of(g.U, g.G, t0 + kb - 1) - sk_cta_of(g.U, g.G, t0) + 1);
        while (tc::ld_acquire_gpu(&g.cnt[2 * tile]) - base[jj] < np) __nanosleep(20);
      }
      SK_TR(11);
    }
    tc::named_bar_sync(1, 128);
    int dbg_t = 0;
    for (int u = lo; u < hi;) {
      const int tile = u / kb, k0 = u - tile * kb;
      const int k1 = min(kb, k0 + (hi - u));
      u += k1 - k0;
      if (k0 == 0 && k1 == kb) continue;
      const int c_first = sk_cta_of(g.U, g.G, tile * kb);
      const int np = sk_cta_of(g.U, g.G, tile * kb + kb - 1) - c_first + 1;
      const int piece = c - c_first;
      const float* src = g.part + (size_t)tile * g.pmax * piece_floats;
      const int nfc = silu ? 8 : 16;   // feature chunks of 16 per tile
      const int items = nfc * g.bm;
      const int it_lo = (int)((long long)piece * items / np);
      const int it_hi = (int)((long long)(piece + 1) * items / np);
      for (int it = it_lo + et; it < it_hi; it += 128) {
        const int ch = it / g.bm, m = it % g.bm;
        float a[16], b[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) a[e] = b[e] = 0.f;
        float res[16];
        const int n = tile * SK_BN + ch * 16;
        if (EPI == SLX_EPI_RESIDUAL && m < g.M && n < g.N)
          sk_load_res<OutT>(g, m, n, g.C2 != nullptr ? g.n_main : g.N, res);
        const float* pa = src + ((size_t)ch * g.bm + m) * 16;
        const float* pb = src + ((size_t)(ch + 8) * g.bm + m) * 16;
        constexpr int PB = EPI == SLX_EPI_SILU_MUL ? SK_PB / 2 : SK_PB;   // register budget
        for (int p0 = 0; p0 < np; p0 += PB) {
          float4 qa[PB][4], qb[silu ? PB : 1][4];
#pragma unroll
          for (int bi = 0; bi < PB; ++bi) {
            if (p0 + bi < np) {
              const float4* s4 = reinterpret_cast<const float4*>(pa + (size_t)(p0 + bi) * piece_floats);
#pragma unroll
              for (int e = 0; e < 4; ++e) qa[bi][e] = __ldcg(s4 + e);
              if (silu) {
                const float4* t4 = reinterpret_cast<const float4*>(pb + (size_t)(p0 + bi) * piece_floats);
#pragma unroll
                for (int e = 0; e < 4; ++e) qb[silu ? bi : 0][e] = __ldcg(t4 + e);
              }
            }
          }
#pragma unroll
          for (int bi = 0; bi < PB; ++bi) {   // fixed piece order: deterministic
            if (p0 + bi < np) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                a[4 * e] += qa[bi][e].x; a[4 * e + 1] += qa[bi][e].y;
                a[4 * e + 2] += qa[bi][e].z; a[4 * e + 3] += qa[bi][e].w;
                if (silu) {
                  const float4 t = qb[silu ? bi : 0][e];
                  b[4 * e] += t.x; b[4 * e + 1] += t.y; b[4 * e + 2] += t.z; b[4 * e + 3] += t.w;
                }
              }
            }
          }
        }
        if (et == 0 && dbg_t == 0) SK_TR(12);
        if (m >= g.M) continue;
        if (silu) {
#pragma unroll
          for (int e = 0; e < 16; ++e) a[e] = sk_silu(a[e]) * b[e];
          sk_store16(reinterpret_cast<OutT*>(g.C) + (size_t)m * g.ldc, tile * 128 + ch * 16, n_out, a);
        } else if (n < g.N) {
          sk_finish<EPI, OutT>(g, m, n, a, res);
        }
      }
      if (et == 0 && dbg_t == 0) SK_TR(13);
      ++dbg_t;
      // departure: the next launch reads D as its base only after this grid has completed
      if (et == 0) atomicAdd(&g.cnt[2 * tile + 1], 1);
    }
    if (et == 0) SK_TR(8);
    }
  }

  if (!PO && warp < 2 && g.cs > 1) {   // producer / MMA warps join the epilogue's cluster barriers
    tc::cluster_sync();
    tc::cluster_sync();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x == 0) SK_TR(7);
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem_base, 2 * SK_BN);
  }
}

struct SkPlan {
  int bm, stages, kblocks, n_tiles, G, pmax, cs;
  long long U;
  size_t smem, ws;
};

int sk_max_clusters(size_t smem, int cluster);

bool sk_plan(int M, int N, int K, SkPlan* p, const slx_gemm_tuning* tu) {
  if (M <= 0 || M > SK_MAX_M) return false;
  p->bm = (M + 15) / 16 * 16;
  p->kblocks = ceil_div(K, SK_BK);
  p->n_tiles = ceil_div(N, SK_BN);
  p->U = (long long)p->n_tiles * p->kblocks;
  if ((size_t)p->n_tiles * 2 * sizeof(int) > SK_CNT_BYTES) return false;
  if (p->U * sm_count() >= (1ll << 31)) return false;   // 32-bit unit math in the kernel
  // Grid: every tile split into the same number s of equal pieces (G = n_tiles * s <= #SMs,
  // s <= 8, pieces >= 4 k-blocks), so no CTA straggles and whole tiles (s = 1) need no
  // reduction at all; measured (tools/gemm_bench.py) to beat an all-SM stream-K grid with uneven
  // pieces.  More tiles than SMs: plain stream-K over all SMs.
  const int sms = sm_count();
  const int min_units = (tu && tu->sk_min_units > 0) ? tu->sk_min_units : 4;
  long long G;
  if (p->n_tiles <= sms) {
    int s = sms / p->n_tiles;
    s = s > 8 ? 8 : s;
    while (s > 1 && p->kblocks / s < min_units) --s;
    G = (long long)p->n_tiles * s;
  } else {
    G = sms;
  }
  G = G < 1 ? 1 : G;
  const int e_g = tu ? tu->sk_ctas : 0;
  if (e_g > 0) {
    G = p->U / (min_units > 0 ? min_units : 1);
    G = G < 1 ? 1 : (G > sms ? sms : G);
    if (e_g < G) G = e_g;
  }
  p->G = (int)G;
  p->cs = 1;
  const long long upc = (p->U + G - 1) / G;
  if ((upc - 1) / p->kblocks + 2 > SK_MAX_SEGS) return false;
  int pmax = 1;
  for (int t = 0; t < p->n_tiles; ++t) {
    const int u0 = t * p->kblocks;
    const int np = sk_cta_of((int)p->U, p->G, u0 + p->kblocks - 1) - sk_cta_of((int)p->U, p->G, u0) + 1;
    pmax = np > pmax ? np : pmax;
  }
  p->pmax = pmax;
  const size_t stage = (size_t)p->bm * SK_BK * 2 + 2 * SK_WBOX;
  int st = (int)((227 * 1024 - 1024 - SK_BAR_BYTES) / stage);
  st = st > SK_MAX_STAGES ? SK_MAX_STAGES : st;
  p->stages = st;
  p->smem = (size_t)st * stage + SK_BAR_BYTES + 1024;
  p->ws = SK_PART_OFF + (size_t)p->n_tiles * pmax * p->bm * SK_BN * 4;
  // Uniform split (every CTA one piece, tile t = CTAs [t*s, t*s+s)): reduce through DSMEM in a
  // cluster of s when all n_tiles clusters are co-resident and the staged piece fits the
  // pipeline smem.
  const int s_split = p->G / p->n_tiles;
  if (!(tu && tu->sk_no_cluster) && s_split >= 2 && s_split <= 8 &&
      p->G == p->n_tiles * s_split && (size_t)p->bm * SK_BN * 4 <= (size_t)st * stage &&
      sk_max_clusters(p->smem, s_split) >= p->n_tiles) {
    p->cs = s_split;
    p->ws = SK_PART_OFF;
  }
  return true;
}

template <int EPI, typename OutT, bool PO = false>
int sk_launch_t(const CUtensorMap& mx, const CUtensorMap& mw, const SkArgs& a, const SkPlan& p,
                cudaStream_t s) {
  auto k = gemm_sk_kernel<EPI, OutT, PO>;
  static bool configured = false;
  if (!configured) {
    configure_kernel((const void*)k);
    configured = true;
  }
  return launch_ex(k, dim3((unsigned)p.G), dim3(SK_THREADS), p.smem, s, (unsigned)p.cs, mx, mw, a);
}

// Max co-resident clusters of `cluster` CTAs with `smem` bytes each (cached per device shape).
int sk_max_clusters(size_t smem, int cluster) {
  struct Key { size_t smem; int cluster, value; };
  static Key cache[32];
  static int n_cache = 0;
  for (int i = 0; i < n_cache; ++i)
    if (cache[i].smem == smem && cache[i].cluster == cluster) return cache[i].value;
  auto k = gemm_sk_kernel<SLX_EPI_NONE, bf16>;
  configure_kernel((const void*)k);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cluster * 64);
  cfg.blockDim = dim3(SK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (unsigned)cluster;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
    (void)cudaGetLastError();
    n = 0;
  }
  if (n_cache < 32) cache[n_cache++] = Key{smem, cluster, n};
  return n;
}

}  // namespace

size_t gemm_sk_splitk_bytes(int M, int N, int splits) {
  if (M <= 0 || M > SK_MAX_M || N <= 0 || splits < 1) return 0;
  return (size_t)ceil_div(N, SK_BN) * splits * ((M + 15) / 16 * 16) * SK_BN * 4;
}

size_t gemm_sk_workspace_bytes(int M, int N, int K) {
  SkPlan p{};
  return sk_plan(M, N, K, &p, nullptr) ? p.ws : 0;
}

int gemm_sk_launch(const SkCall& c) {
  SkPlan p{};
  if (c.part_out != nullptr) {
    // split-K pieces for the consumer: G = n_tiles * splits, every CTA exactly one piece
    if (!sk_plan(c.M, c.N, c.K, &p, nullptr)) return SLX_ERR_UNSUPPORTED;
    if (c.splits < 1 || c.splits > 16 || p.kblocks / c.splits < 1) return SLX_ERR_INVALID;
    p.G = p.n_tiles * c.splits;
    p.pmax = c.splits;
    p.cs = 1;
    if ((size_t)p.n_tiles * c.splits * p.bm * SK_BN * 4 > c.part_bytes) return SLX_ERR_WORKSPACE;
  } else {
    if ((c.tuning && c.tuning->tile_kernel) || c.ws == nullptr) return SLX_ERR_UNSUPPORTED;
    if (!sk_plan(c.M, c.N, c.K, &p, c.tuning) || p.ws > c.ws_bytes) return SLX_ERR_UNSUPPORTED;
  }
  SkArgs a{};
  a.M = c.M; a.N = c.N; a.bm = p.bm; a.stages = p.stages; a.kblocks = p.kblocks;
  a.n_tiles = p.n_tiles; a.G = p.G; a.pmax = p.pmax; a.U = (int)p.U; a.cs = p.cs;
  a.C = c.C; a.ldc = c.ldc; a.R = c.R; a.ldr = c.ldr;
  a.n_main = c.C2 != nullptr ? c.n_main : c.N;
  a.C2 = (float*)c.C2; a.ldc2 = c.ldc2;
  a.cnt = (uint32_t*)c.ws;
  a.part = (float*)((char*)c.ws + SK_PART_OFF);
  if (c.part_out != nullptr) {
    a.part = c.part_out;
    a.part_only = 1;
  }
  a.trace = c.trace;
  a.pf = pf_args(c.pf);
  CUtensorMap mx, mw;
  const int w_rows = ceil_div(c.N, 128) * p.kblocks * 128;
  if (!make_tmap(&mx, c.A, c.M, c.K, c.lda, p.bm) || !make_tmap(&mw, c.W, w_rows, SK_BK, SK_BK, 128))
    return SLX_ERR_CUDA;
  cudaStream_t s = (cudaStream_t)c.stream;
  const bool f32 = c.c_dtype == SLX_DT_F32;
  if (a.part_only) return sk_launch_t<SLX_EPI_NONE, bf16, true>(mx, mw, a, p, s);
  switch (c.epilogue) {
    case SLX_EPI_NONE:
      return f32 ? sk_launch_t<SLX_EPI_NONE, float>(mx, mw, a, p, s)
                 : sk_launch_t<SLX_EPI_NONE, bf16>(mx, mw, a, p, s);
    case SLX_EPI_RESIDUAL:
      return f32 ? sk_launch_t<SLX_EPI_RESIDUAL, float>(mx, mw, a, p, s)
                 : sk_launch_t<SLX_EPI_RESIDUAL, bf16>(mx, mw, a, p, s);
    case SLX_EPI_SILU_MUL:
      return f32 ? sk_launch_t<SLX_EPI_SILU_MUL, float>(mx, mw, a, p, s)
                 : sk_launch_t<SLX_EPI_SILU_MUL, bf16>(mx, mw, a, p, s);
    default:
      return SLX_ERR_INVALID;
  }
}

}  // namespace slx
