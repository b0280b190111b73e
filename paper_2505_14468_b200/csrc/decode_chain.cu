// K1 + norms, decode step: the projections and norms between two attention launches as ONE
// persistent launch ("chain") with grid-wide barriers between its phases.
//
//   o (split-K pieces) -> post-attention norm (+ pieces, + o LoRA delta) -> gate/up (SiLU*mul)
//   -> down (pieces) -> next layer's input norm (+ pieces) -> q/k/v (pieces, stacked LoRA
//   shrink rows) -> q/k/v reduction (bf16 q/k/v + fp32 shrink output for the attention kernel)
//
// Why: the separate-kernel decode step loses ~55 us per 7B layer at its kernel boundaries —
// each GEMM ramps up after the previous grid drained, split GEMMs end in reduction tails, and
// two latency-bound RMSNorm launches run with HBM idle.  Here every CTA (one per SM) runs every
// phase; the phases are separated by grid barriers (a monotonic arrival counter per barrier),
// and the TMA producer lane never waits for a barrier before issuing the WEIGHT boxes of its
// next GEMM phase: only the activation box of a stage waits (the stage's full-barrier expects
// both).  So the 200 KB smem ring of every SM keeps filling across the norms, the reductions
// and the barriers, and HBM keeps streaming weights.
//
// Roles (192 threads): warp 0 lane 0 TMA producer, warp 1 lane 0 tcgen05.mma issuer into one
// of two TMEM accumulators (2 x 256 columns), warps 2-5 ("epilogue group", 128 threads):
// accumulator drains, norms, reductions, barrier arrivals.  GEMM phases use the uniform split
// of the stream-K decode GEMM (gemm_sk.cu): CTA c < n_tiles * s holds piece c % s of tile c / s
// — the same K ranges and piece order, so the chain's results are bit-identical to the
// separate kernels' (the norm reproduces slx_rmsnorm_fused's summation tree).
//
// Barriers: `sync[b]` counts the CTAs that finished phase b.  The epilogue group arrives once
// its phase-b outputs are written (release at gpu scope after a group barrier); consumers poll
// with acquire loads (the producer before a stage's activation box, plus a proxy fence since
// TMA reads through the async proxy; the epilogue group before a norm / reduction).  The last
// CTA to leave zeroes the counters (a departure counter), so `sync` is left zeroed.
//
// Replaces the modelled decode step of the reference (engine.py:888,909 decode_ms_per_token).
#include <cuda.h>
#include <stdio.h>

#include "common.cuh"
#include "gemm_host.h"
#include "tc_ptx.cuh"

namespace slx {
namespace {

constexpr int CH_EPI_WARPS = 4;              // epilogue group: drains (first 4), norms, reductions
constexpr int CH_EPI = CH_EPI_WARPS * 32;
constexpr int CH_THREADS = 64 + CH_EPI;
constexpr int CH_NI = 4;                     // max norm items (token, 256-column block) per warp
constexpr int CH_BN = 256;
constexpr int CH_BK = 64;
constexpr int CH_MAX_STAGES = 8;
constexpr int CH_MAX_PH = 14;                // internal phases (a NORM is two)
constexpr int CH_NORM_A = 10, CH_NORM_B = 11; // internal kinds of a NORM's two halves
constexpr int CH_MAX_BLK = 32;                // 256-column blocks per row (d <= 8192)
constexpr int CH_WBOX = 128 * CH_BK * 2;     // one contiguous 16 KB weight box
constexpr int CH_PQ = 16;                    // pending activation boxes (>= stages)
constexpr int CH_SYNC_WORDS = 32;            // [0, MAX_PH): barriers, [16]: departures
constexpr int CH_DEP = 16;
// after the counters: the norms' per-(token, 256-column block) partial sums of squares
constexpr size_t CH_SYNC_BYTES = CH_SYNC_WORDS * 4 + 64 * CH_MAX_BLK * 4;

struct ChPhase {
  CUtensorMap tx;   // activations [M, K], box bm x 64, SW128
  CUtensorMap tw;   // tiled weight as [rows, 64], box 128 x 64
  const char* wptr; // the tiled weight (L2 prefetch addresses)
  int kind;
  int N, kblocks, n_tiles, splits, G;   // GEMM: G = n_tiles * splits CTAs work
  float* part;
  bf16* C;
  int ldc;
  float* C2;
  int ldc2;
  bf16* x;
  int ldx;
  bf16* out;
  int ldo;
  const bf16* nw;
  int d;
  float eps;
  int has_sk, has_lora;
  SplitArgs sk;
  DeltaArgs lora;
};

// Per-token LoRA metadata of the chain's (one) norm with a fused delta, resolved once at
// kernel start (the slot tables and the adapter pool are >= 2 launches old).
struct ChTokMeta {
  int slot, rank;
  float scale;
  int pad;
  const bf16* b[SLX_LORA_MAX_TARGETS];
};

struct ChArgs {
  ChPhase ph[CH_MAX_PH];
  int n_ph, M, bm, stages;
  int lora_ph;    // internal phase whose norm fuses a LoRA delta (-1: none)
  int pf_units;   // weight units the producer prefetches into L2 before it blocks on a barrier
  uint32_t* sync;
  float* ssp;   // [M][CH_MAX_BLK] partial sums of squares (NORM_A -> NORM_B)
  unsigned long long* trace;
  PfArgs pf;
};

__device__ __forceinline__ unsigned long long ch_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ bool is_gemm(int kind) {
  return kind == SLX_CHAIN_GEMM_PIECES || kind == SLX_CHAIN_GEMM_SILU;
}
// Wait until every CTA finished phase b (b = -1: the previous kernel, via PDL).
__device__ __forceinline__ void ch_wait_barrier(const ChArgs& a, int b) {
  if (b < 0) {
    pdl_wait();
    return;
  }
  const uint32_t need = gridDim.x;
  while (tc::ld_acquire_gpu(a.sync + b) < need) __nanosleep(32);
}
// fast-math SiLU (as gemm_sk.cu)
__device__ __forceinline__ float ch_silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

__device__ __forceinline__ void ch_store16_bf16(bf16* row, int n0, int n_lim, const float* v) {
  if (n0 + 16 <= n_lim) {
    Vec8<bf16>::store(row + n0, v);
    Vec8<bf16>::store(row + n0 + 8, v + 8);
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (n0 + j < n_lim) row[n0 + j] = __float2bfloat16_rn(v[j]);
  }
}

// --------------------------------------------------------------------------- norm phases
// slx_rmsnorm_fused semantics over ALL CTAs in two halves with a grid barrier between them.
// Work item = (token t, 256-column block b), one warp: lane l owns the 8-column unit u = 32 b + l.
//   NORM_A: x = round(x + pieces) (+ round(+ LoRA delta)), written back; the warp's partial
//           sum of squares (sequential per unit, xor-tree warp_sum) -> ssp[t][b];
//   NORM_B: total of the row's partials in the separate kernels' order — the cluster kernel's
//           (ranks of d/8 columns, warps in order within a rank, ranks in order) when pieces
//           are consumed and d % 2048 == 0, else the per-token kernel's / slx_rmsnorm's (d = 256,
//           4096) warp_sum over the partials — then out = (x * inv) * w.
// x is re-read through L2 (__ldcg): other SMs wrote it in this launch.
__device__ __forceinline__ void ldcg8_bf16(const bf16* p, float* f) {
  const uint4 u = __ldcg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// LoRA delta of one column from register B rows and v held by the warp's lanes: lane l holds
// v(target l >> 4, j = l & 15) in va and v(target 2 + (l >> 4), j) in vb (scale applied);
// sequential fmaf in j as delta_finish / slx_lora_expand.
__device__ __forceinline__ float ch_delta(const DeltaRow<2>& r, int rank, float va, float vb) {
  if (r.ti < 0) return 0.f;
  const float vsrc = r.ti < 2 ? va : vb;
  const int base = (r.ti & 1) * 16;
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (j * 8 < rank) {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&r.b[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __bfloat1622float2(h2[u]);
        acc = fmaf(__shfl_sync(0xffffffffu, vsrc, base + 8 * j + 2 * u), f.x, acc);
        acc = fmaf(__shfl_sync(0xffffffffu, vsrc, base + 8 * j + 2 * u + 1), f.y, acc);
      }
    } else {
      (void)__shfl_sync(0xffffffffu, vsrc, 0);   // keep the warp converged (rank uniform per item)
    }
  }
  return acc;
}

// NORM_A: the warp's items (item = gw, gw + n_gw, ...), one at a time.
__device__ void ch_norm_a(const ChArgs& a, const ChPhase& P, int gw, int n_gw, int lane,
                          const ChTokMeta* meta) {
  const int nb = P.d / 256;
#pragma unroll 1
  for (int item = gw; item < a.M * nb; item += n_gw) {
    const int t = item / nb, b = item - t * nb;
    const int i0 = (b * 32 + lane) * 8;
    int slot = -1, rank = 0;
    float scale = 0.f;
    if (P.has_lora) {
      slot = meta[t].slot;
      rank = meta[t].rank;
      scale = meta[t].scale;
    }
    const bool fast = slot >= 0 && rank > 0;
    unsigned long long* dtr = (a.trace && P.has_lora && lane == 0 && (gw & 3) == 0 && item == gw) ? a.trace + (size_t)(gw >> 2) * 64 : nullptr;
    if (dtr) dtr[48] = ch_timer();
    // every load of the item is independent: B rows, v (stacked piece columns), x, pieces
    DeltaRow<2> dr[8];
    float va = 0.f, vb = 0.f;
    if (fast) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        dr[j].ti = -1;
#pragma unroll
        for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
          const int n = i0 + j - P.lora.y_col_off[i];
          if (dr[j].ti < 0 && i < P.lora.n_targets && n >= 0 && n < P.lora.d_out[i] &&
              meta[t].b[i] != nullptr) {
            dr[j].ti = i;
            const uint4* src = reinterpret_cast<const uint4*>(meta[t].b[i] + (size_t)n * rank);
#pragma unroll
            for (int q = 0; q < 2; ++q) dr[j].b[q] = q * 8 < rank ? __ldg(src + q) : make_uint4(0, 0, 0, 0);
          }
        }
      }
      const int jj = lane & 15, i_a = lane >> 4, i_b = 2 + (lane >> 4);
      if (jj < rank && i_a < P.lora.n_targets)
        va = split_sum1(P.sk, t, P.sk.n_main + P.lora.v_col_off[i_a & 3] + slot * P.lora.v_slot_stride + jj) * scale;
      if (jj < rank && i_b < P.lora.n_targets)
        vb = split_sum1(P.sk, t, P.sk.n_main + P.lora.v_col_off[i_b & 3] + slot * P.lora.v_slot_stride + jj) * scale;
    }
    bf16* xr = P.x + (size_t)t * P.ldx;
    float f[8];
    ldcg8_bf16(xr + i0, f);
    if (dtr) dtr[49] = ch_timer() + (f[0] == 12345.f);
    if (P.has_sk) {
      float ps[8];
      split_sum8(P.sk, t, i0, ps);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = __bfloat162float(__float2bfloat16_rn(f[j] + ps[j]));
    }
    if (dtr) dtr[50] = ch_timer() + (f[0] == 12345.f) + (va == 12345.f);
    if (fast) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        f[j] = __bfloat162float(__float2bfloat16_rn(f[j] + ch_delta(dr[j], rank, va, vb)));
    }
    if (dtr) dtr[51] = ch_timer() + (f[0] == 12345.f);
    if (P.has_sk || fast) Vec8<bf16>::store(xr + i0, f);
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
    ss = warp_sum(ss);
    if (lane == 0) a.ssp[t * CH_MAX_BLK + b] = ss;
  }
}

// NORM_B: out = (x * inv) * w for the warp's items (partials, x and w loaded together).
__device__ void ch_norm_b(const ChArgs& a, const ChPhase& P, int gw, int n_gw, int lane) {
  const int nb = P.d / 256;
#pragma unroll 1
  for (int item = gw; item < a.M * nb; item += n_gw) {
    const int t = item / nb, b = item - t * nb;
    const int i0 = (b * 32 + lane) * 8;
    const float pl = lane < nb ? __ldcg(a.ssp + t * CH_MAX_BLK + lane) : 0.f;
    float f[8], g[8];
    ldcg8_bf16(P.x + (size_t)t * P.ldx + i0, f);
    Vec8<bf16>::load(P.nw + i0, g);
    float tot;
    if (P.has_sk && P.d % 2048 == 0) {   // the cluster kernel's order
      const int wpr = nb / 8;
      tot = 0.f;
      for (int rk = 0; rk < 8; ++rk) {
        float c = 0.f;
        for (int q = 0; q < wpr; ++q) c += __shfl_sync(0xffffffffu, pl, rk * wpr + q);
        tot += c;
      }
    } else {
      tot = warp_sum(pl);
    }
    const float inv = 1.0f / sqrtf(tot / (float)P.d + P.eps);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (f[j] * inv) * g[j];
    Vec8<bf16>::store(P.out + (size_t)t * P.ldo + i0, f);
  }
}

// --------------------------------------------------------------------------- reduce phase
// Pieces of an N-column projection -> bf16 C (columns < n_main) / fp32 C2 (columns >= n_main);
// item = (tile, 16-column chunk, row), summed in piece order from 0 (gemm_sk's reduction).
__device__ void ch_reduce(const ChPhase& P, int M, int c, int et) {
  const int bm = P.sk.bm, s = P.sk.splits;
  const int n_tiles = (P.N + CH_BN - 1) / CH_BN;
  const int items = n_tiles * 16 * bm;
  const size_t piece_floats = (size_t)bm * CH_BN;
  for (int it = c * CH_EPI + et; it < items; it += gridDim.x * CH_EPI) {
    const int tile = it / (16 * bm), rem = it - tile * 16 * bm;
    const int ch = rem / bm, m = rem - ch * bm;
    const int n = tile * CH_BN + ch * 16;
    if (m >= M || n >= P.N) continue;
    const float* src = P.sk.part + (size_t)tile * s * piece_floats + ((size_t)ch * bm + m) * 16;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    for (int p0 = 0; p0 < s; p0 += 4) {
      float4 q[4][4];
#pragma unroll
      for (int bi = 0; bi < 4; ++bi)
        if (p0 + bi < s) {
          const float4* s4 = reinterpret_cast<const float4*>(src + (size_t)(p0 + bi) * piece_floats);
#pragma unroll
          for (int e = 0; e < 4; ++e) q[bi][e] = __ldcg(s4 + e);
        }
#pragma unroll
      for (int bi = 0; bi < 4; ++bi)
        if (p0 + bi < s) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            acc[4 * e] += q[bi][e].x; acc[4 * e + 1] += q[bi][e].y;
            acc[4 * e + 2] += q[bi][e].z; acc[4 * e + 3] += q[bi][e].w;
          }
        }
    }
    if (P.C2 != nullptr && n >= P.sk.n_main) {
      float* row = P.C2 + (size_t)m * P.ldc2 + (n - P.sk.n_main);
      if (n + 16 <= P.N) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          reinterpret_cast<float4*>(row)[q4] =
              make_float4(acc[4 * q4], acc[4 * q4 + 1], acc[4 * q4 + 2], acc[4 * q4 + 3]);
      } else {
        for (int j = 0; j < 16; ++j)
          if (n + j < P.N) row[j] = acc[j];
      }
    } else {
      const int lim = P.C2 != nullptr ? P.sk.n_main : P.N;
      ch_store16_bf16(P.C + (size_t)m * P.ldc, n, lim, acc);
    }
  }
}

__global__ void __launch_bounds__(CH_THREADS, 1) decode_chain_kernel(const __grid_constant__ ChArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int x_bytes = a.bm * CH_BK * 2;
  const int stage_bytes = x_bytes + 2 * CH_WBOX;
  uint64_t* full = (uint64_t*)(smem + a.stages * stage_bytes);
  uint64_t* empty = full + CH_MAX_STAGES;
  uint64_t* tfull = empty + CH_MAX_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  ChTokMeta* meta = reinterpret_cast<ChTokMeta*>(tmem_slot + 4);   // [64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x;
  unsigned long long* tr = a.trace ? a.trace + (size_t)c * 64 : nullptr;
  if (threadIdx.x == 0) {
    if (tr) tr[62] = ch_timer();
    for (int p = 0; p < a.n_ph; ++p)
      if (is_gemm(a.ph[p].kind) && c < a.ph[p].G) {
        tc::tma_prefetch_desc(&a.ph[p].tx);
        tc::tma_prefetch_desc(&a.ph[p].tw);
      }
    for (int s = 0; s < a.stages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int q = 0; q < 2; ++q) {
      tc::mbar_init(&tfull[q], 1);
      tc::mbar_init(&tempty[q], 1);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * CH_BN);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA producer
      const uint64_t pol_w = tc::policy_evict_first();   // weights: streamed once
      const uint64_t pol_x = tc::policy_evict_last();    // activations: re-read by every CTA
      // activation boxes waiting for their barrier: (stage index, phase, k-block), oldest first
      int q_i[CH_PQ] = {}, q_p[CH_PQ] = {}, q_k[CH_PQ] = {};
      int qh = 0, qt = 0;
      int known = -2;   // highest barrier known passed (-1 = the previous kernel, PDL)
      int i = 0;        // next stage (unit) to load
      // L2 prefetch cursor over this CTA's units in load order: before the producer blocks on a
      // barrier it requests the weight boxes of its next pf_units units into L2, so HBM keeps
      // streaming past what the smem ring holds
      int pf_ph = 0, pf_k = -1, pf_i = 0;
      auto prefetch_to = [&](int target) {
        while (pf_i < target && pf_ph < a.n_ph) {
          const ChPhase& Q = a.ph[pf_ph];
          if (!is_gemm(Q.kind) || c >= Q.G) { ++pf_ph; pf_k = -1; continue; }
          const int kb = Q.kblocks, tile = c / Q.splits, piece = c - tile * Q.splits;
          if (pf_k < 0) pf_k = piece * kb / Q.splits;
          if (pf_k >= (piece + 1) * kb / Q.splits) { ++pf_ph; pf_k = -1; continue; }
          if (pf_i >= i) {
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const char* p = Q.wptr + ((size_t)(tile * 2 + b) * kb + pf_k) * CH_WBOX;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)CH_WBOX) : "memory");
            }
          }
          ++pf_k;
          ++pf_i;
        }
      };
      auto pass = [&](int b) {
        if (b <= known) return;
        if (b >= 0) prefetch_to(i + a.pf_units);
        if (known < -1) {   // every barrier poll comes after the PDL wait
          pdl_wait();
          pdl_trigger();
          known = -1;
        }
        if (b >= 0) {
          ch_wait_barrier(a, b);
          fence_proxy_async_global();   // other CTAs' generic writes -> our TMA reads
          known = b;
        }
      };
      int last_xp = -1;
      auto issue_x = [&](int e) {
        if (tr && q_p[e] != last_xp) {   // first activation box of a phase issued
          last_xp = q_p[e];
          tr[32 + last_xp] = ch_timer();
        }
        const int s = q_i[e] % a.stages;
        tc::tma_load_2d(smem + s * stage_bytes, &a.ph[q_p[e]].tx, &full[s], q_k[e] * CH_BK, 0, pol_x);
      };
      int first_pass = 1;
      for (int p = 0; p < a.n_ph; ++p) {
        const ChPhase& P = a.ph[p];
        if (!is_gemm(P.kind) || c >= P.G) continue;
        const int s_ = P.splits, kb = P.kblocks;
        const int tile = c / s_, piece = c - tile * s_;
        const int k0 = piece * kb / s_, k1 = (piece + 1) * kb / s_;
        for (int k = k0; k < k1; ++k, ++i) {
          // the slot's previous stage (i - stages) must have its activation box issued, or
          // nothing will ever free the slot: block on the oldest pending barriers first
          while (qh != qt && q_i[qh % CH_PQ] <= i - a.stages) {
            pass(q_p[qh % CH_PQ] - 1);
            issue_x(qh % CH_PQ);
            ++qh;
          }
          while (qh != qt && q_p[qh % CH_PQ] - 1 <= known) {   // opportunistic
            issue_x(qh % CH_PQ);
            ++qh;
          }
          const int s = i % a.stages;
          tc::mbar_wait(&empty[s], ((i / a.stages) & 1) ^ 1);
          uint8_t* st = smem + s * stage_bytes;
          tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
#pragma unroll
          for (int b = 0; b < 2; ++b)
            tc::tma_load_2d(st + x_bytes + b * CH_WBOX, &P.tw, &full[s], 0,
                            ((tile * 2 + b) * kb + k) * 128, pol_w);
          const int e = qt % CH_PQ;
          q_i[e] = i; q_p[e] = p; q_k[e] = k;
          ++qt;
          if (p - 1 <= known) {
            issue_x(e);
            ++qh;
          } else if (first_pass && qt - qh >= a.stages) {
            // the first ring-full of weights is in flight: now wait for the previous kernel
            pass(-1);
            first_pass = 0;
          }
        }
      }
      while (qh != qt) {
        pass(q_p[qh % CH_PQ] - 1);
        issue_x(qh % CH_PQ);
        ++qh;
      }
      if (known < -1) pass(-1);
      l2_prefetch_part(a.pf, c, gridDim.x);   // the next kernel's first bytes
    }
    __syncwarp();
  } else if (warp == 1) {
    pdl_wait();
    pdl_trigger();
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      const uint32_t idesc = tc::idesc_bf16_f32(128, CH_BN);
      int i = 0, j = 0;
      for (int p = 0; p < a.n_ph; ++p) {
        const ChPhase& P = a.ph[p];
        if (!is_gemm(P.kind) || c >= P.G) continue;
        const int s_ = P.splits, kb = P.kblocks;
        const int piece = c % s_;
        const int k0 = piece * kb / s_, k1 = (piece + 1) * kb / s_;
        tc::mbar_wait(&tempty[j & 1], ((j >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        const uint32_t dacc = tmem_base + (uint32_t)((j & 1) * CH_BN);
        for (int k = k0; k < k1; ++k, ++i) {
          const int s = i % a.stages;
          tc::mbar_wait(&full[s], (i / a.stages) & 1);
          tc::fence_after_sync();
          const uint32_t st = tc::smem_u32(smem + s * stage_bytes);
#pragma unroll
          for (int ks = 0; ks < CH_BK / 16; ++ks)
            tc::mma_bf16_ss(dacc, tc::smem_desc_sw128(st + ks * 32),
                            tc::smem_desc_sw128(st + x_bytes + ks * 32), idesc,
                            (k == k0 && ks == 0) ? 0u : 1u);
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[j & 1]);
        ++j;
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------------ epilogue group
    if (a.lora_ph >= 0) {
      const DeltaArgs& la = a.ph[a.lora_ph].lora;
      for (int t = threadIdx.x - 64; t < a.M; t += CH_EPI) {
        const DeltaTok dt = delta_tok(la, t);
        ChTokMeta mt{dt.slot, dt.rank, dt.scale, 0, {nullptr, nullptr, nullptr, nullptr}};
        if (dt.slot >= 0)
#pragma unroll
          for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i)
            if (i < la.n_targets) mt.b[i] = reinterpret_cast<const bf16*>(__ldg(&la.b_ptrs[i][dt.slot]));
        meta[t] = mt;
      }
      // the B rows this warp's norm items will read (adapters are static): into L2 now, while
      // the o projection streams, instead of from HBM behind the next weight stream later
      tc::named_bar_sync(1, CH_EPI);
      const ChPhase& LP = a.ph[a.lora_ph];
      const int nb = LP.d / 256, gw = c * CH_EPI_WARPS + ((threadIdx.x - 64) >> 5);
      if (lane == 0)
        for (int item = gw; item < a.M * nb; item += gridDim.x * CH_EPI_WARPS) {
          const int t = item / nb, b = item - t * nb;
          const ChTokMeta& mt = meta[t];
          if (mt.slot < 0 || mt.rank <= 0) continue;
#pragma unroll
          for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
            const int n = b * 256 - la.y_col_off[i];
            if (i < la.n_targets && mt.b[i] != nullptr && n >= 0 && n < la.d_out[i]) {
              const int rows = min(256, la.d_out[i] - n);
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(mt.b[i] + (size_t)n * mt.rank),
                           "r"((uint32_t)(rows * mt.rank * 2)) : "memory");
            }
          }
        }
    }
    pdl_wait();
    pdl_trigger();
    const int q = warp & 3;              // TMEM lane quadrant of this warp
    const int r = q * 32 + lane;         // accumulator row (token) of this thread
    const int et = threadIdx.x - 64;     // 0 .. CH_EPI - 1
    // accumulator drains: the first four epilogue warps (one per TMEM lane quadrant)
    const bool qlive = et < 128 && q * 32 < a.bm;   // warp-uniform
    int j = 0;
    for (int p = 0; p < a.n_ph; ++p) {
      const ChPhase& P = a.ph[p];
      if (is_gemm(P.kind)) {
        if (c < P.G) {
          const int acc = j & 1;
          tc::mbar_wait(&tfull[acc], (j >> 1) & 1);
          __syncwarp();
          tc::fence_after_sync();
          if (tr && et == 0) tr[2 * p] = ch_timer();
          const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * CH_BN);
          const int s_ = P.splits, tile = c / s_, piece = c - tile * s_;
          if (P.kind == SLX_CHAIN_GEMM_PIECES) {
            float* dst = P.part + (size_t)(tile * s_ + piece) * a.bm * CH_BN;
            if (qlive) {
              for (int ch = 0; ch < 16; ch += 2) {
                float v0[16], v1[16];
                tc::tmem_ld16x2(tacc + ch * 16, tacc + ch * 16 + 16, v0, v1);
                if (r < a.bm) {
                  float4* p0 = reinterpret_cast<float4*>(dst + ((size_t)ch * a.bm + r) * 16);
                  float4* p1 = reinterpret_cast<float4*>(dst + ((size_t)(ch + 1) * a.bm + r) * 16);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    p0[e] = make_float4(v0[4 * e], v0[4 * e + 1], v0[4 * e + 2], v0[4 * e + 3]);
                    p1[e] = make_float4(v1[4 * e], v1[4 * e + 1], v1[4 * e + 2], v1[4 * e + 3]);
                  }
                }
              }
            }
          } else {   // SiLU * mul of a whole [gate 128 | up 128] tile
            if (qlive) {
              for (int ch = 0; ch < 8; ++ch) {
                float gv[16], uv[16];
                tc::tmem_ld16x2(tacc + ch * 16, tacc + 128 + ch * 16, gv, uv);
                if (r < a.M) {
#pragma unroll
                  for (int e = 0; e < 16; ++e) gv[e] = ch_silu(gv[e]) * uv[e];
                  ch_store16_bf16(P.C + (size_t)r * P.ldc, tile * 128 + ch * 16, P.N / 2, gv);
                }
              }
            }
          }
          tc::fence_before_sync();
          tc::named_bar_sync(1, CH_EPI);
          if (et == 0) tc::mbar_arrive(&tempty[acc]);
          ++j;
        }
      } else {
        if (et == 0) {
          if (p > 0) ch_wait_barrier(a, p - 1);   // (p == 0: the PDL wait above)
          if (tr) tr[2 * p] = ch_timer();
        }
        tc::named_bar_sync(1, CH_EPI);
        const int gw = c * CH_EPI_WARPS + (et >> 5), n_gw = gridDim.x * CH_EPI_WARPS;
        if (P.kind == CH_NORM_A) {
          ch_norm_a(a, P, gw, n_gw, lane, meta);
        } else if (P.kind == CH_NORM_B) {
          ch_norm_b(a, P, gw, n_gw, lane);
        } else {
          ch_reduce(P, a.M, c, et);
        }
      }
      if (p + 1 < a.n_ph) {   // arrive: this CTA's phase-p outputs are written
        tc::named_bar_sync(1, CH_EPI);
        if (et == 0) {
          __threadfence();
          fence_proxy_async_global();
          tc::red_release_gpu_add(a.sync + p, 1u);
          if (tr) tr[2 * p + 1] = ch_timer();
        }
      }
    }
    if (et == 0) {   // departure; the last CTA out re-zeroes the counters
      __threadfence();
      const uint32_t old = atomicAdd(a.sync + CH_DEP, 1u);
      if (old == gridDim.x - 1) {
        for (int b = 0; b < a.n_ph; ++b) a.sync[b] = 0u;
        a.sync[CH_DEP] = 0u;
        __threadfence();
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[63] = ch_timer();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem_base, 2 * CH_BN);
  }
}

size_t ch_smem(int bm, int stages) {
  return 1024 + (size_t)stages * (bm * CH_BK * 2 + 2 * CH_WBOX) + (2 * CH_MAX_STAGES + 4) * 8 + 16 +
         64 * sizeof(ChTokMeta);
}

// Build the kernel arguments; returns SLX_OK or an error status.
int ch_build(const slx_chain_phase* ph, int n, int M, ChArgs* a, int* grid) {
  if (ph == nullptr || n < 1 || n > SLX_CHAIN_MAX_PHASES || M < 1 || M > 64) return SLX_ERR_INVALID;
  *a = ChArgs{};
  a->M = M;
  a->lora_ph = -1;
  a->pf_units = 8;
  a->bm = (M + 15) / 16 * 16;
  const int sms = sm_count();
  int g = 1;
  bool any_gemm = false;
  int np = 0;   // internal phases (a NORM is two)
  for (int p = 0; p < n; ++p) {
    const slx_chain_phase& s = ph[p];
    if (np + 2 > CH_MAX_PH) return SLX_ERR_INVALID;
    ChPhase& P = a->ph[np++];
    P.kind = s.kind;
    if (s.kind == SLX_CHAIN_GEMM_PIECES || s.kind == SLX_CHAIN_GEMM_SILU) {
      any_gemm = true;
      if (!s.A || !s.W || s.N <= 0 || s.K <= 0 || s.K % 8 || s.lda < s.K || s.lda % 8)
        return SLX_ERR_INVALID;
      P.N = s.N;
      P.kblocks = ceil_div(s.K, CH_BK);
      P.n_tiles = ceil_div(s.N, CH_BN);
      P.splits = s.kind == SLX_CHAIN_GEMM_SILU ? 1 : s.splits;
      if (P.splits < 1 || P.splits > 16 || P.kblocks / P.splits < 1) return SLX_ERR_INVALID;
      P.G = P.n_tiles * P.splits;
      if (P.G > sms) return SLX_ERR_UNSUPPORTED;
      g = P.G > g ? P.G : g;
      if (s.kind == SLX_CHAIN_GEMM_PIECES) {
        if (!s.part || s.part_bytes < (size_t)P.G * a->bm * CH_BN * 4) return SLX_ERR_WORKSPACE;
        P.part = s.part;
      } else {
        if (s.N % CH_BN || !s.C || s.ldc < s.N / 2 || s.ldc % 8) return SLX_ERR_INVALID;
        P.C = (bf16*)s.C;
        P.ldc = s.ldc;
      }
      const int w_rows = ceil_div(s.N, 128) * P.kblocks * 128;
      P.wptr = (const char*)s.W;
      if (!make_tmap(&P.tx, s.A, M, s.K, s.lda, a->bm) ||
          !make_tmap(&P.tw, s.W, w_rows, CH_BK, CH_BK, 128))
        return SLX_ERR_CUDA;
    } else if (s.kind == SLX_CHAIN_NORM) {
      if (!s.x || !s.out || !s.norm_w || s.d <= 0 || s.d % 256 || s.d > 256 * CH_MAX_BLK || s.ldx < s.d ||
          s.ldo < s.d || s.ldx % 8 || s.ldo % 8)
        return SLX_ERR_INVALID;
      if (s.has_sk && (!s.sk.part || s.sk.splits < 1 || s.sk.bm != a->bm || s.sk.n_main < s.d))
        return SLX_ERR_INVALID;
      if (s.has_lora) {
        if (!s.has_sk || s.lora.v != nullptr || !delta_valid(&s.lora, true) ||
            s.lora.max_rank > 16)
          return SLX_ERR_UNSUPPORTED;   // v from the pieces, ranks <= 16 (register rows)
        P.lora = delta_args(&s.lora);
        if (a->lora_ph >= 0) return SLX_ERR_UNSUPPORTED;   // one fused delta per chain
        a->lora_ph = np - 1;
      }
      P.x = (bf16*)s.x; P.ldx = s.ldx; P.out = (bf16*)s.out; P.ldo = s.ldo;
      P.nw = (const bf16*)s.norm_w; P.d = s.d; P.eps = s.eps;
      P.has_sk = s.has_sk; P.has_lora = s.has_lora;
      P.sk = split_args(s.has_sk ? &s.sk : nullptr);
      P.kind = CH_NORM_A;
      a->ph[np] = P;
      a->ph[np++].kind = CH_NORM_B;

    } else if (s.kind == SLX_CHAIN_REDUCE) {
      if (!s.has_sk || !s.sk.part || s.sk.bm != a->bm || s.sk.splits < 1 || s.N <= 0 || !s.C ||
          s.ldc % 8 || s.sk.n_main % 16 || s.sk.n_main > s.N || (s.C2 && (s.ldc2 % 4)))
        return SLX_ERR_INVALID;
      P.N = s.N; P.C = (bf16*)s.C; P.ldc = s.ldc; P.C2 = s.C2; P.ldc2 = s.ldc2;
      P.sk = split_args(&s.sk);
      if (!s.C2) P.sk.n_main = s.N;
    } else {
      return SLX_ERR_INVALID;
    }
  }
  a->n_ph = np;
  if (g > sms) return SLX_ERR_UNSUPPORTED;
  for (int p = 0; p < np; ++p)   // a norm's items fit the warps' registers (CH_NI each)
    if (a->ph[p].kind == CH_NORM_A && M * (a->ph[p].d / 256) > CH_NI * g * CH_EPI_WARPS) {
      const int need = ceil_div(M * (a->ph[p].d / 256), CH_NI * CH_EPI_WARPS);
      if (need > sms) return SLX_ERR_UNSUPPORTED;
      g = need;
    }
  const int stage = a->bm * CH_BK * 2 + 2 * CH_WBOX;
  int st = (int)((227 * 1024 - ch_smem(a->bm, 0)) / stage);
  a->stages = st > CH_MAX_STAGES ? CH_MAX_STAGES : st;
  if (a->stages < 2) return SLX_ERR_UNSUPPORTED;
  *grid = g;
  return SLX_OK;
}

}  // namespace
}  // namespace slx

using namespace slx;

extern "C" size_t slx_decode_chain_sync_bytes(void) { return CH_SYNC_BYTES; }

extern "C" int slx_decode_chain_ctas(const slx_chain_phase* phases, int n_phases, int M) {
  ChArgs a;
  int g = 0;
  return ch_build(phases, n_phases, M, &a, &g) == SLX_OK ? g : 0;
}

extern "C" int slx_decode_chain(const slx_chain_phase* phases, int n_phases, int M, void* sync,
                                const slx_l2_prefetch* pf, void* trace, void* stream) {
  if (sync == nullptr) return SLX_ERR_INVALID;
  SLX_CHECK_ALIGN(sync, 16);
  ChArgs a;
  int g = 0;
  const int st = ch_build(phases, n_phases, M, &a, &g);
  if (st != SLX_OK) return st;
  a.sync = (uint32_t*)sync;
  a.ssp = (float*)((char*)sync + CH_SYNC_WORDS * 4);
  a.trace = (unsigned long long*)trace;
  a.pf = pf_args(pf);
  static bool configured = false;
  if (!configured) {
    configure_kernel((const void*)decode_chain_kernel);
    configured = true;
  }
  const int rc = launch_ex(decode_chain_kernel, dim3((unsigned)g), dim3(CH_THREADS), ch_smem(a.bm, a.stages),
                   (cudaStream_t)stream, 1u, a);
  if (rc != SLX_OK) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, decode_chain_kernel);
    fprintf(stderr, "DBG chain launch: %s regs=%d maxthr=%d smem=%zu param=%zu\n",
            cudaGetErrorString(cudaGetLastError()), fa.numRegs, fa.maxThreadsPerBlock,
            ch_smem(a.bm, a.stages), sizeof(ChArgs));
  }
  return rc;
}
