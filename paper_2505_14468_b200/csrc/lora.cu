// K2/K3: multi-LoRA shrink/expand over an adapter-segmented token batch.
//
// plan    : tokens -> (slot, start, count) tiles of <= LORA_TT tokens that share one adapter
//           slot (BGMV: counting sort of the per-token slot; SGMV: the given segments).
// shrink  : v[t, j] = sum_k x[t, k] * A_s[j, k]        (fp32, staged per k-split)
// expand  : y[t, col(n)] += scale_s * sum_j v[t, j] * B_s[n, j]   (scale-and-add fused)
//
// Semantics follow the reference's batch -> adapter association (a batch is one
// function's requests, FlushDecision at /root/reference/pkg/src/slorasim/batching.py:99-105)
// and the unmerged LoRA of PAPER.md:614-621.  The oracle is oracle/llama_lora.py::bgmv/sgmv.
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace slx {

constexpr int LORA_TT = 8;        // tokens per tile (fused decode kernel: 4 CTAs/SM)
constexpr int LORA_MAX_RANK = 64;
constexpr int LORA_MAX_KS = 8;    // k-splits of the shrink
constexpr int PLAN_THREADS = 1024;
constexpr int PLAN_MAX_GROUPS = 2048;
constexpr int LORA_FUSED_MAX_TOK = 256;  // decode-sized batches use the fused cluster kernel

struct LoraTile {
  int slot, start, count, pad;
};

struct LoraWs {  // carved from the caller's workspace
  int* n_tiles;
  int* perm;
  LoraTile* tiles;
  float* v;      // [KS][n_targets][n_tok][max_rank]
  int max_tiles;
};

inline int lora_max_tiles(int n_tok, int n_slots) {
  return ceil_div(n_tok, LORA_TT) + (n_slots < n_tok ? n_slots : n_tok) + 1;
}
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline size_t lora_ws_bytes(int n_tok, int n_slots, int max_rank, int n_targets, LoraWs* out,
                            void* base) {
  const int mt = lora_max_tiles(n_tok, n_slots);
  size_t off = 0;
  const size_t o_n = off;    off = align_up(off + 16, 256);
  const size_t o_perm = off; off = align_up(off + sizeof(int) * (size_t)n_tok, 256);
  const size_t o_tiles = off; off = align_up(off + sizeof(LoraTile) * (size_t)mt, 256);
  const size_t o_v = off;
  off = align_up(off + sizeof(float) * (size_t)LORA_MAX_KS * n_targets * n_tok * max_rank, 256);
  if (out) {
    char* b = (char*)base;
    out->n_tiles = (int*)(b + o_n);
    out->perm = (int*)(b + o_perm);
    out->tiles = (LoraTile*)(b + o_tiles);
    out->v = (float*)(b + o_v);
    out->max_tiles = mt;
  }
  return off;
}

// ---------------------------------------------------------------- plan
// Groups g = 0..G-1 with (slot, start, count) in smem -> tiles of <= LORA_TT tokens.
__device__ void emit_tiles(const int* g_slot, const int* g_start, const int* g_count, int G,
                           LoraTile* tiles, int* n_tiles, int max_tiles) {
  using Scan = cub::BlockScan<int, PLAN_THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int g0 = 0; g0 < G; g0 += PLAN_THREADS) {
    const int g = g0 + threadIdx.x;
    const int nt = (g < G && g_count[g] > 0) ? (g_count[g] + LORA_TT - 1) / LORA_TT : 0;
    int excl, total;
    Scan(tmp).ExclusiveSum(nt, excl, total);
    const int base = carry + excl;
    for (int i = 0; i < nt; ++i) {
      const int k = base + i;
      if (k < max_tiles) {
        const int s0 = g_start[g] + i * LORA_TT;
        const int c = min(LORA_TT, g_count[g] - i * LORA_TT);
        tiles[k] = LoraTile{g_slot[g], s0, c, 0};
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_tiles = min(carry, max_tiles);
}

__global__ void __launch_bounds__(PLAN_THREADS)
plan_tokens_kernel(const int32_t* __restrict__ tok_slot, int n_tok, int n_slots, LoraWs ws) {
  pdl_wait();
  pdl_trigger();
  __shared__ int cnt[PLAN_MAX_GROUPS];
  __shared__ int start[PLAN_MAX_GROUPS];
  __shared__ int slot_id[PLAN_MAX_GROUPS];
  using Scan = cub::BlockScan<int, PLAN_THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  for (int s = threadIdx.x; s < n_slots; s += PLAN_THREADS) { cnt[s] = 0; slot_id[s] = s; }
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tok; t += PLAN_THREADS) {
    const int s = tok_slot[t];
    if (s >= 0 && s < n_slots) atomicAdd(&cnt[s], 1);
  }
  __syncthreads();
  for (int s0 = 0; s0 < n_slots; s0 += PLAN_THREADS) {
    const int s = s0 + threadIdx.x;
    const int c = s < n_slots ? cnt[s] : 0;
    int excl, total;
    Scan(tmp).ExclusiveSum(c, excl, total);
    if (s < n_slots) start[s] = carry + excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  // scatter (order within a slot is irrelevant: every token's arithmetic is independent)
  for (int s = threadIdx.x; s < n_slots; s += PLAN_THREADS) cnt[s] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < n_tok; t += PLAN_THREADS) {
    const int s = tok_slot[t];
    if (s >= 0 && s < n_slots) ws.perm[start[s] + atomicAdd(&cnt[s], 1)] = t;
  }
  __syncthreads();
  emit_tiles(slot_id, start, cnt, n_slots, ws.tiles, ws.n_tiles, ws.max_tiles);
}

__global__ void __launch_bounds__(PLAN_THREADS)
plan_segments_kernel(const int32_t* __restrict__ seg_indptr, const int32_t* __restrict__ seg_slot,
                     int n_seg, int n_tok, int n_slots, LoraWs ws) {
  pdl_wait();
  pdl_trigger();
  __shared__ int cnt[PLAN_MAX_GROUPS];
  __shared__ int start[PLAN_MAX_GROUPS];
  __shared__ int slot_id[PLAN_MAX_GROUPS];
  for (int t = threadIdx.x; t < n_tok; t += PLAN_THREADS) ws.perm[t] = t;
  for (int s = threadIdx.x; s < n_seg; s += PLAN_THREADS) {
    const int lo = max(0, min(seg_indptr[s], n_tok)), hi = max(lo, min(seg_indptr[s + 1], n_tok));
    const int sl = seg_slot[s];
    const bool live = sl >= 0 && sl < n_slots;
    start[s] = lo;
    cnt[s] = live ? hi - lo : 0;
    slot_id[s] = sl;
  }
  __syncthreads();
  emit_tiles(slot_id, start, cnt, n_seg, ws.tiles, ws.n_tiles, ws.max_tiles);
}

// ---------------------------------------------------------------- shrink
struct TargetArgs {
  const uint64_t* a_ptrs[SLX_LORA_MAX_TARGETS];
  const uint64_t* b_ptrs[SLX_LORA_MAX_TARGETS];
  int d_out[SLX_LORA_MAX_TARGETS];
  int col_off[SLX_LORA_MAX_TARGETS];
  int col_blk[SLX_LORA_MAX_TARGETS];
  int col_stride[SLX_LORA_MAX_TARGETS];
};

constexpr int SH_KC = 64;
template <typename T>
__global__ void __launch_bounds__(256)
lora_shrink_kernel(const T* __restrict__ x, int ldx, int n_tok, int d_in, int ks,
                   const int32_t* __restrict__ slot_rank, int max_rank, TargetArgs ta, LoraWs ws) {
  pdl_wait();
  pdl_trigger();
  const int tile_id = blockIdx.x;
  if (tile_id >= *ws.n_tiles) return;
  const LoraTile tile = ws.tiles[tile_id];
  const int tgt = blockIdx.y, kz = blockIdx.z;
  const int rank = min(slot_rank[tile.slot], max_rank);
  const bf16* A = reinterpret_cast<const bf16*>(ta.a_ptrs[tgt][tile.slot]);
  const int kspan = ceil_div(d_in / 8, ks) * 8;
  const int k_lo = kz * kspan, k_hi = min(d_in, k_lo + kspan);
  __shared__ float xs[LORA_TT][SH_KC + 1];
  __shared__ float as[LORA_MAX_RANK][SH_KC + 1];
  __shared__ int toks[LORA_TT];
  if (threadIdx.x < LORA_TT)
    toks[threadIdx.x] = threadIdx.x < tile.count ? ws.perm[tile.start + threadIdx.x] : -1;
  // each thread owns up to 4 (token, j) outputs
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int n_out = tile.count * rank;
  __syncthreads();
  for (int k0 = k_lo; k0 < k_hi; k0 += SH_KC) {
    const int kc = min(SH_KC, k_hi - k0);  // multiple of 8
    // x tile: count rows x kc, vec8 loads
    for (int e = threadIdx.x; e < LORA_TT * (SH_KC / 8); e += blockDim.x) {
      const int i = e / (SH_KC / 8), kk = (e % (SH_KC / 8)) * 8;
      float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (i < tile.count && kk < kc) Vec8<T>::load(x + (size_t)toks[i] * ldx + k0 + kk, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) xs[i][kk + q] = f[q];
    }
    for (int e = threadIdx.x; e < rank * (SH_KC / 8); e += blockDim.x) {
      const int j = e / (SH_KC / 8), kk = (e % (SH_KC / 8)) * 8;
      float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (kk < kc) Vec8<bf16>::load(A + (size_t)j * d_in + k0 + kk, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) as[j][kk + q] = f[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int o = threadIdx.x + q * 256;
      if (o < n_out) {
        const int i = o / rank, j = o % rank;
        float a = acc[q];
        for (int kk = 0; kk < kc; ++kk) a = fmaf(xs[i][kk], as[j][kk], a);
        acc[q] = a;
      }
    }
    __syncthreads();
  }
  float* v = ws.v + (((size_t)kz * gridDim.y + tgt) * n_tok) * max_rank;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int o = threadIdx.x + q * 256;
    if (o < n_out) {
      const int i = o / rank, j = o % rank;
      v[(size_t)(tile.start + i) * max_rank + j] = acc[q];
    }
  }
}

// ---------------------------------------------------------------- expand
template <typename T, int R>
__device__ __forceinline__ void expand_body(T* __restrict__ y, int ldy, const bf16* __restrict__ B,
                                            int rank, int n_lo, int n_hi, int d_out,
                                            const float (*vs)[LORA_MAX_RANK], const int* toks,
                                            int count, int col_off, int col_blk, int col_stride) {
  for (int n = n_lo + threadIdx.x; n < n_hi; n += blockDim.x) {
    float b[R];
    const bf16* br = B + (size_t)n * rank;
#pragma unroll
    for (int j = 0; j < R; j += 8) {
      if (j < rank) {
        Vec8<bf16>::load(br + j, b + j);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) b[j + q] = 0.f;
      }
    }
    const int col = col_off + (n / col_blk) * col_stride + (n % col_blk);
    for (int i = 0; i < count; ++i) {
      float d = 0.f;
#pragma unroll
      for (int j = 0; j < R; ++j) d = fmaf(vs[i][j], b[j], d);
      T* p = y + (size_t)toks[i] * ldy + col;
      *p = from_f32<T>(to_f32(*p) + d);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
lora_expand_kernel(T* __restrict__ y, int ldy, int n_tok, int ks, int n_split,
                   const int32_t* __restrict__ slot_rank, const float* __restrict__ slot_scale,
                   int max_rank, TargetArgs ta, LoraWs ws) {
  pdl_wait();
  pdl_trigger();
  const int tile_id = blockIdx.x;
  if (tile_id >= *ws.n_tiles) return;
  const LoraTile tile = ws.tiles[tile_id];
  const int tgt = blockIdx.y;
  const int rank = min(slot_rank[tile.slot], max_rank);
  const float scale = slot_scale[tile.slot];
  const int d_out = ta.d_out[tgt];
  const int span = ceil_div(ceil_div(d_out, n_split), 8) * 8;
  const int n_lo = blockIdx.z * span, n_hi = min(d_out, n_lo + span);
  if (n_lo >= n_hi) return;
  __shared__ float vs[LORA_TT][LORA_MAX_RANK];
  __shared__ int toks[LORA_TT];
  if (threadIdx.x < LORA_TT)
    toks[threadIdx.x] = threadIdx.x < tile.count ? ws.perm[tile.start + threadIdx.x] : 0;
  for (int e = threadIdx.x; e < LORA_TT * LORA_MAX_RANK; e += blockDim.x) {
    const int i = e / LORA_MAX_RANK, j = e % LORA_MAX_RANK;
    float s = 0.f;
    if (i < tile.count && j < rank) {
      for (int kz = 0; kz < ks; ++kz)
        s += ws.v[((((size_t)kz * gridDim.y + tgt) * n_tok) + tile.start + i) * max_rank + j];
      s *= scale;
    }
    vs[i][j] = s;
  }
  __syncthreads();
  const bf16* B = reinterpret_cast<const bf16*>(ta.b_ptrs[tgt][tile.slot]);
  const int cb = ta.col_blk[tgt], cs = ta.col_stride[tgt], co = ta.col_off[tgt];
  if (rank <= 8)
    expand_body<T, 8>(y, ldy, B, rank, n_lo, n_hi, d_out, vs, toks, tile.count, co, cb, cs);
  else if (rank <= 16)
    expand_body<T, 16>(y, ldy, B, rank, n_lo, n_hi, d_out, vs, toks, tile.count, co, cb, cs);
  else if (rank <= 32)
    expand_body<T, 32>(y, ldy, B, rank, n_lo, n_hi, d_out, vs, toks, tile.count, co, cb, cs);
  else
    expand_body<T, 64>(y, ldy, B, rank, n_lo, n_hi, d_out, vs, toks, tile.count, co, cb, cs);
}


// ---------------------------------------------------------------- fused decode kernel (BGMV)
// One cluster of KS CTAs per (tile, target).  CTA q of the cluster:
//   1. stages x[tile tokens, k-chunk q], A_s[:, k-chunk q] and B_s[n-range q, :] in smem
//      (all loads in flight at once: one HBM round trip),
//   2. computes the partial shrink v_q[i][j] over its k-chunk (warp-per-output, shuffle reduce),
//   3. reduces v = sum_q v_q through DSMEM (fixed order, deterministic) -> smem, x scale,
//   4. expands its n-range: y[t, col(n)] += sum_j v[i][j] B_s[n][j]  (scale-and-add fused).
constexpr int FU_THREADS = 256;
constexpr int FU_MAX_KS = 8;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

template <typename T>
__global__ void __launch_bounds__(FU_THREADS)
lora_fused_kernel(T* __restrict__ y, int ldy, const T* __restrict__ x, int ldx, int n_tok, int d_in,
                  int ks, int kc, int ns, const int32_t* __restrict__ slot_rank,
                  const float* __restrict__ slot_scale, int max_rank, TargetArgs ta, LoraWs ws) {
  extern __shared__ __align__(16) uint8_t fsm[];
  pdl_wait();
  pdl_trigger();
  const int q = (int)tc::cluster_ctarank();
  const int tile_id = blockIdx.x / ks;
  const int tgt = blockIdx.y;
  if (tile_id >= *ws.n_tiles) return;   // uniform over the cluster: no barrier is skipped unevenly
  const LoraTile tile = ws.tiles[tile_id];
  const int cnt = tile.count;
  const int rank = min(slot_rank[tile.slot], max_rank);
  const int R8 = (rank + 7) & ~7;
  const float scale = slot_scale[tile.slot];
  const int d_out = ta.d_out[tgt];
  const int n_lo = min(d_out, q * ns), n_hi = min(d_out, n_lo + ns);
  const int nn = n_hi - n_lo;
  const int k_lo = min(d_in, q * kc), k_hi = min(d_in, k_lo + kc);
  const int kl = k_hi - k_lo;
  const bf16* A = reinterpret_cast<const bf16*>(ta.a_ptrs[tgt][tile.slot]);
  const bf16* B = reinterpret_cast<const bf16*>(ta.b_ptrs[tgt][tile.slot]);
  const int cb = ta.col_blk[tgt], cstr = ta.col_stride[tgt], co = ta.col_off[tgt];
  // an n-range that stays inside one output column block can move y with 16-byte copies
  const int col_lo = co + (n_lo / cb) * cstr + (n_lo % cb);
  const bool y_contig = nn > 0 && (n_lo / cb) == ((n_hi - 1) / cb) && (col_lo % 8) == 0 &&
                        (ldy % 8) == 0 && (nn % 8) == 0;

  // smem: xs [TT][kc] T | ys [TT][ns] T | as [max_rank][kc] bf16 | bs [ns][max_rank] bf16 |
  //       vpart [TT][max_rank] f32 | vfull [TT][max_rank] f32 | toks [TT]
  T* xs = reinterpret_cast<T*>(fsm);
  T* ys = xs + (size_t)LORA_TT * kc;
  bf16* as = reinterpret_cast<bf16*>(ys + (size_t)LORA_TT * ns);
  bf16* bs = as + (size_t)max_rank * kc;
  float* vpart = reinterpret_cast<float*>(bs + (size_t)ns * max_rank);
  float* vfull = vpart + LORA_TT * max_rank;
  int* toks = reinterpret_cast<int*>(vfull + LORA_TT * max_rank);

  if (threadIdx.x < LORA_TT) toks[threadIdx.x] = threadIdx.x < cnt ? ws.perm[tile.start + threadIdx.x] : 0;
  __syncthreads();
  // ---- 1. every load in flight at once (16-byte cp.async): x chunk, y slice, A chunk, B rows
  constexpr int XV = 16 / sizeof(T);
  const int xchunks = kl / XV;
  for (int e = threadIdx.x; e < cnt * xchunks; e += FU_THREADS) {
    const int i = e / xchunks, c = e % xchunks;
    cp_async16(xs + (size_t)i * kc + c * XV, x + (size_t)toks[i] * ldx + k_lo + c * XV);
  }
  if (y_contig) {
    const int ychunks = nn / XV;
    for (int e = threadIdx.x; e < cnt * ychunks; e += FU_THREADS) {
      const int i = e / ychunks, c = e % ychunks;
      cp_async16(ys + (size_t)i * ns + c * XV, y + (size_t)toks[i] * ldy + col_lo + c * XV);
    }
  }
  const int achunks = kl / 8;
  for (int e = threadIdx.x; e < rank * achunks; e += FU_THREADS) {
    const int j = e / achunks, c = e % achunks;
    cp_async16(as + (size_t)j * kc + c * 8, A + (size_t)j * d_in + k_lo + c * 8);
  }
  const int bchunks = nn * rank / 8;   // B rows n_lo..n_hi are contiguous
  for (int e = threadIdx.x; e < bchunks; e += FU_THREADS) {
    const int flat = e * 8;
    const int n = flat / rank, j = flat % rank;
    cp_async16(bs + (size_t)n * max_rank + j, B + (size_t)n_lo * rank + flat);
  }
  cp_async_wait_all();
  __syncthreads();

  // ---- 2. partial shrink over this k-chunk: one warp per (i, j) output
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_out = cnt * rank;
  for (int o = warp; o < n_out; o += FU_THREADS / 32) {
    const int i = o / rank, j = o % rank;
    const T* xr = xs + (size_t)i * kc;
    const bf16* ar = as + (size_t)j * kc;
    float acc = 0.f;
    for (int k = lane * 8; k < kl; k += 32 * 8) {
      float xf[8], af[8];
      Vec8<T>::load(xr + k, xf);
      Vec8<bf16>::load(ar + k, af);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(xf[e], af[e], acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) vpart[i * max_rank + j] = acc;
  }
  tc::cluster_sync();
  // ---- 3. v = sum over the cluster's k-chunks (DSMEM), fixed order, x scale
  const uint32_t vp_base = tc::smem_u32(vpart);
  for (int o = threadIdx.x; o < n_out; o += FU_THREADS) {
    const int i = o / rank, j = o % rank;
    const uint32_t off = vp_base + (uint32_t)((i * max_rank + j) * 4);
    float part[FU_MAX_KS];
#pragma unroll
    for (int s = 0; s < FU_MAX_KS; ++s) part[s] = s < ks ? tc::ld_dsmem(tc::mapa(off, (uint32_t)s)) : 0.f;
    float a = 0.f;
#pragma unroll
    for (int s = 0; s < FU_MAX_KS; ++s) a += part[s];
    vfull[i * max_rank + j] = a * scale;
  }
  // peers may still read our vpart: arrive now, wait before exit
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  // ---- 4. expand + fused add: thread owns 8 consecutive rows n for one token at a time
  const int ngrp = (nn + 7) / 8;
  for (int e = threadIdx.x; e < cnt * ngrp; e += FU_THREADS) {
    const int i = e / ngrp, g8 = e % ngrp;
    const int n0 = g8 * 8;
    const float* vr = vfull + i * max_rank;
    float d[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < R8; j += 8) {
      float vv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) vv[u] = (j + u < rank) ? vr[j + u] : 0.f;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        if (n0 + r >= nn) break;
        float b[8];
        Vec8<bf16>::load(bs + (size_t)(n0 + r) * max_rank + j, b);
#pragma unroll
        for (int u = 0; u < 8; ++u) d[r] = fmaf(vv[u], b[u], d[r]);
      }
    }
    T* yr = y + (size_t)toks[i] * ldy;
    if (y_contig) {
      float yv[8];
      Vec8<T>::load(ys + (size_t)i * ns + n0, yv);
#pragma unroll
      for (int r = 0; r < 8; ++r) yv[r] += d[r];
      Vec8<T>::store(yr + col_lo + n0, yv);
    } else {
      for (int r = 0; r < 8 && n0 + r < nn; ++r) {
        const int n = n_lo + n0 + r;
        const int col = co + (n / cb) * cstr + (n % cb);
        yr[col] = from_f32<T>(to_f32(yr[col]) + d[r]);
      }
    }
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}


// ---------------------------------------------------------------- gathered decode shrink
// Large adapter pools (decode): instead of stacking every slot's A rows into the projection
// GEMM (bytes grow with the pool), the shrink reads only the adapters present in the batch,
// each ONCE per plan tile.
// Work unit = (plan tile, target, 8 rows j0..j0+7 of A; 4 / 2 / 1 rows when d_in is too wide
// for two stages of 8): a slot's rows are contiguous ([rank][d_in]), so a unit is ONE bulk copy
// (TMA engine, 80 KB at d_in 5120).  Persistent
// grid (one CTA per SM), units dealt round robin over a dense table (block scan of the
// (tile, target) unit counts, tile data cached in shared memory: no dead CTAs, no dependent
// global loads per unit).  Two shared-memory stages, each holding a unit's A rows and the
// first SH_XT of its tile's token rows of x, both brought by bulk copies on the stage's
// mbarriers: the adapter pool is static, so thread 0 issues the A rows of the CTA's first two
// units BEFORE griddepcontrol.wait (they stream while the producer of x -- the norm /
// attention -- is still running) and their x rows right after it; a consumed stage is refilled
// (A and x) at once, so unit k+2's bytes are in flight while unit k+1 is computed.  Tiles with
// more than SH_XT tokens stage the rest synchronously.  Each warp dots one A row against the
// staged x rows (16 B per lane per step, conflict-free); per lane the k order
// (lane*8 + 256*c, e inner) is sequential fmaf, then a warp_sum: deterministic and
// independent of the token grouping.
//   v[t, v_col_off[tgt] + j] = x_t . A_{slot(t), tgt}[j]   (j < rank; unscaled)
// Consumers: slx_lora_expand with v_slot_stride = 0, or the fused slx_lora_delta.
constexpr int SH_WARPS = 8;
constexpr int SH_XT = 2;        // token rows of x per stage (at most)
constexpr int SH_STAGES = 2;
constexpr int SH_MAX_PAIRS = 1024;
constexpr int SH_PAIRS_PT = SH_MAX_PAIRS / (SH_WARPS * 32);
constexpr int SH_MAX_TILES = 384;
constexpr size_t SH_DYN_SMEM = 204 * 1024;   // dynamic shared memory (static ~21 KB on top)
struct ShrinkOut {
  int v_off[SLX_LORA_MAX_TARGETS];
  int n_targets;
};
inline size_t shrink_smem_bytes(int d_in, size_t x_elem, int rpu, int xt) {
  return 64 + (size_t)SH_STAGES * ((size_t)rpu * d_in * 2 + (size_t)xt * d_in * x_elem);
}
// A rows per unit (8, or fewer for wide d_in) and token rows of x per stage that fit the
// shared memory (false: d_in too large)
inline bool shrink_geometry(int d_in, size_t x_elem, int* rpu, int* xt) {
  for (int r = SH_WARPS; r >= 1; r >>= 1)
    for (int t = SH_XT; t >= 1; --t)
      if (shrink_smem_bytes(d_in, x_elem, r, t) <= SH_DYN_SMEM) {
        *rpu = r;
        *xt = t;
        return true;
      }
  return false;
}

template <typename T>
__global__ void __launch_bounds__(SH_WARPS * 32, 1)
lora_shrink_v_kernel(float* __restrict__ v, int ldv, const T* __restrict__ x, int ldx, int d_in,
                     const int32_t* __restrict__ slot_rank, int max_rank, TargetArgs ta,
                     ShrinkOut so, LoraWs ws, int rpu, int xt) {
  constexpr int NT = SH_WARPS * 32;
  extern __shared__ __align__(128) unsigned char sh_raw[];
  uint64_t* afull = reinterpret_cast<uint64_t*>(sh_raw);        // [SH_STAGES]
  uint64_t* xfull = afull + SH_STAGES;                            // [SH_STAGES]
  const size_t a_stage = (size_t)rpu * d_in;                      // bf16 elements
  const size_t x_stage = (size_t)xt * d_in;                       // T elements
  bf16* As = reinterpret_cast<bf16*>(sh_raw + 64);                // [SH_STAGES][rpu][d_in]
  T* Xs = reinterpret_cast<T*>(sh_raw + 64 + SH_STAGES * a_stage * 2);   // [SH_STAGES][xt][d_in]
  using Scan = cub::BlockScan<int, NT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int pair_end[SH_MAX_PAIRS];
  __shared__ int tile_rank[SH_MAX_TILES];
  __shared__ int tile_slot[SH_MAX_TILES];
  __shared__ int tile_tok[SH_MAX_TILES][LORA_TT];
  __shared__ int tile_count[SH_MAX_TILES];
  __shared__ int total_units;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NTG = so.n_targets;
  // The stage barriers are initialised first, so the prologue's __syncthreads order the init
  // before any thread's first wait (a wait on an uninitialised mbarrier is undefined).
  if (threadIdx.x == 0) {
    for (int st = 0; st < SH_STAGES; ++st) {
      tc::mbar_init(&afull[st], 1);
      tc::mbar_init(&xfull[st], 1);
    }
    tc::fence_barrier_init();
  }
  // ---- the unit table (plan and adapter pool are >= 2 launches back: before the wait)
  // Two dependent round trips: {tile count, tiles (read speculatively up to the plan's bound)}
  // -> {slot rank, the targets' A pointers, token ids}; a pair's "has A" flag is parked in
  // pair_end until the scan.
  const int nt_plan = *ws.n_tiles;
  const int tmax = min(ws.max_tiles, SH_MAX_TILES);
  for (int tl = threadIdx.x; tl < tmax; tl += NT) {
    const LoraTile tile = ws.tiles[tl];
    const bool ok = tl < nt_plan && tile.count > 0;
    const int r = ok ? min(slot_rank[tile.slot], max_rank) : 0;
#pragma unroll
    for (int tg = 0; tg < SLX_LORA_MAX_TARGETS; ++tg)
      if (tg < NTG && tl * NTG + tg < SH_MAX_PAIRS)
        pair_end[tl * NTG + tg] = ok && ta.a_ptrs[tg][tile.slot] != 0;
    tile_rank[tl] = r;
    tile_slot[tl] = tile.slot;
    tile_count[tl] = ok ? min(tile.count, LORA_TT) : 0;
#pragma unroll
    for (int i = 0; i < LORA_TT; ++i) tile_tok[tl][i] = ok && i < tile.count ? ws.perm[tile.start + i] : 0;
  }
  const int n_tiles = min(nt_plan, tmax);
  const int n_pairs = min(n_tiles * NTG, SH_MAX_PAIRS);
  __syncthreads();
  int cnt[SH_PAIRS_PT];
  int run = 0;
#pragma unroll
  for (int k = 0; k < SH_PAIRS_PT; ++k) {
    const int p = threadIdx.x * SH_PAIRS_PT + k;
    int c = 0;
    if (p < n_pairs) {
      const int r = tile_rank[p / NTG];
      if (r > 0 && pair_end[p]) c = ceil_div(r, rpu);
    }
    run += c;
    cnt[k] = run;
  }
  int excl, tot;
  Scan(scan_tmp).ExclusiveSum(run, excl, tot);
#pragma unroll
  for (int k = 0; k < SH_PAIRS_PT; ++k) pair_end[threadIdx.x * SH_PAIRS_PT + k] = excl + cnt[k];
  if (threadIdx.x == 0) total_units = tot;
  __syncthreads();
  const int U = total_units;
  auto locate = [&](int u, int& pair, int& j0) {   // unit u -> (pair, first row)
    int lo = 0, hi = n_pairs - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pair_end[mid] > u) hi = mid; else lo = mid + 1;
    }
    pair = lo;
    j0 = (u - (lo ? pair_end[lo - 1] : 0)) * rpu;
  };
  auto issue_a = [&](int u, int stage) {   // thread 0: the unit's A rows -> stage
    int pair, j0;
    locate(u, pair, j0);
    const int tl = pair / NTG, tg = pair - tl * NTG;
    const bf16* A = reinterpret_cast<const bf16*>(ta.a_ptrs[tg][tile_slot[tl]]);
    const uint32_t bytes = (uint32_t)min(rpu, tile_rank[tl] - j0) * d_in * 2;
    tc::mbar_arrive_expect_tx(&afull[stage], bytes);
    tc::bulk_g2s(As + stage * a_stage, A + (size_t)j0 * d_in, bytes, &afull[stage],
                 tc::policy_evict_first());
  };
  auto issue_x = [&](int u, int stage) {   // thread 0: the tile's first xt token rows -> stage
    int pair, j0;
    locate(u, pair, j0);
    const int tl = pair / NTG;
    const int nt = min(xt, tile_count[tl]);
    const uint32_t row = (uint32_t)d_in * sizeof(T);
    tc::mbar_arrive_expect_tx(&xfull[stage], row * nt);
    for (int i = 0; i < nt; ++i)
      tc::bulk_g2s(Xs + stage * x_stage + (size_t)i * d_in, x + (size_t)tile_tok[tl][i] * ldx, row,
                   &xfull[stage], tc::policy_evict_normal());
  };
  if (threadIdx.x == 0)   // barriers were initialised before the prologue's block syncs
    for (int k = 0; k < SH_STAGES; ++k)
      if (blockIdx.x + k * gridDim.x < U) issue_a(blockIdx.x + k * gridDim.x, k);
  pdl_wait();   // x comes from the kernel just before us
  pdl_trigger();
  if (threadIdx.x == 0)
    for (int k = 0; k < SH_STAGES; ++k)
      if (blockIdx.x + k * gridDim.x < U) issue_x(blockIdx.x + k * gridDim.x, k);
  constexpr int EPC = 16 / sizeof(T);   // elements per 16-byte copy chunk of x
  const int per = d_in / EPC, nch = d_in >> 3;
  int k = 0;
  for (int u = blockIdx.x; u < U; u += gridDim.x, ++k) {
    const int stage = k % SH_STAGES;
    const uint32_t parity = (uint32_t)((k / SH_STAGES) & 1);
    int pair, j0;
    locate(u, pair, j0);
    const int tl = pair / NTG, tg = pair - tl * NTG;
    const int nrows = min(rpu, tile_rank[tl] - j0), count = tile_count[tl];
    const bool mine = warp < nrows;   // warp-uniform
    const bf16* ar = As + stage * a_stage + (size_t)warp * d_in;
    T* xs = Xs + stage * x_stage;
    tc::mbar_wait(&xfull[stage], parity);
    tc::mbar_wait(&afull[stage], parity);
    for (int i0 = 0; i0 < count; i0 += xt) {
      const int nt = min(xt, count - i0);
      if (i0) {   // tokens beyond the first xt: staged synchronously in the stage's x buffer
        __syncthreads();
        for (int e = threadIdx.x; e < nt * per; e += NT) {
          const int i = e / per, c = e - i * per;
          reinterpret_cast<uint4*>(xs + (size_t)i * d_in)[c] =
              reinterpret_cast<const uint4*>(x + (size_t)tile_tok[tl][i0 + i] * ldx)[c];
        }
        __syncthreads();
      }
      if (!mine) continue;
      for (int i = 0; i < nt; ++i) {
        const T* xr = xs + (size_t)i * d_in;
        float acc = 0.f;
#pragma unroll 4
        for (int ch = lane; ch < nch; ch += 32) {
          float af[8], xf[8];
          Vec8<bf16>::load(ar + ch * 8, af);
          Vec8<T>::load(xr + ch * 8, xf);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc = fmaf(xf[e], af[e], acc);
        }
        const float sum = warp_sum(acc);
        if (lane == 0) v[(size_t)tile_tok[tl][i0 + i] * ldv + so.v_off[tg] + j0 + warp] = sum;
      }
    }
    __syncthreads();   // every warp is done with this stage
    const int un = u + SH_STAGES * gridDim.x;
    if (threadIdx.x == 0 && un < U) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
      issue_a(un, stage);
      issue_x(un, stage);
    }
  }
}

// ---------------------------------------------------------------- decode expand
// y[t, col(n)] += scale * sum_j v[t, off + slot * v_slot_stride + j] * B_slot[n, j] over the
// plan: v from the stacked shrink inside the projection GEMM (stride max_rank) or the gathered
// shrink (stride 0).
// Work unit = (plan tile, target, column block) = 32 KB of B: cpt = 8 / (rank / 8) blocks of
// 256 columns (rank 8: 2048 columns, rank 64: 256), so every unit is the same size and a
// mixed-rank batch balances.  A block's B rows [n0, n0 + 256 * cpt) x rank are contiguous: ONE
// bulk copy (TMA engine) per unit, plus one per token for its v row, on the stage's mbarriers.
// Persistent grid (2 CTAs per SM), units dealt round robin over a dense table (block scan of the
// (tile, target) unit counts, tile data cached in shared memory); two stages per CTA: B is
// static, so the B rows of the CTA's first two units are issued BEFORE griddepcontrol.wait,
// their v rows right after it, and a consumed stage is refilled at once.  Per unit a thread
// owns cpt columns 256 apart: it reads its columns' B rows from shared memory with the 16-byte
// chunks in a per-thread rotated order (conflict-free for power-of-two rank / 8), rotates them
// back in registers, then per token issues the y reads of its columns, runs the sequential
// fmaf chain over j (v * scale first, one rounding of y: bit-identical to the fused
// slx_lora_delta) and stores.
constexpr int EX_THREADS = 256;
constexpr int EX_REGS = LORA_MAX_RANK / 8;   // 16-byte B chunks per thread and unit
constexpr int EX_UNIT_BYTES = EX_THREADS * EX_REGS * 16;   // 32 KB
constexpr int EX_STAGES = 2;
constexpr int EX_MAX_PAIRS = 2048;           // (plan tile, target) pairs per launch
constexpr int EX_PAIRS_PT = EX_MAX_PAIRS / EX_THREADS;
constexpr int EX_MAX_TILES = 384;            // plan tiles per launch (1024 tokens over <= 254 slots)
constexpr size_t EX_STAGE_BYTES = EX_UNIT_BYTES + LORA_TT * LORA_MAX_RANK * 4;
constexpr size_t EX_DYN_SMEM = 64 + EX_STAGES * EX_STAGE_BYTES;

struct ExpandArgs {
  int v_off[SLX_LORA_MAX_TARGETS];
  int v_slot_stride;   // columns between slots' v blocks: max_rank (stacked) or 0 (gathered)
  int n_targets;
};

// One unit for a compile-time R8 = rank / 8 (CPT = EX_REGS / R8 columns per thread).
template <typename T, int R8>
__device__ __forceinline__ void expand_unit(T* __restrict__ y, int ldy, const unsigned char* bs,
                                            const float* vsm, float scale, int n0, int d_out,
                                            int count, const int* toks, int co, int cb, int cstr) {
  constexpr int CPT = EX_REGS / R8;
  constexpr bool POW2 = (R8 & (R8 - 1)) == 0;
  const int t = threadIdx.x;
  // chunk rotation that spreads a quarter-warp's 16-byte reads over all 32 banks
  const int rot = POW2 ? ((t * R8) >> 3) & (R8 - 1) : 0;
  uint4 b[CPT][R8];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const uint4* row = reinterpret_cast<const uint4*>(bs) + (size_t)(c * EX_THREADS + t) * R8;
    uint4 tmp[R8];
#pragma unroll
    for (int q = 0; q < R8; ++q) tmp[q] = row[POW2 ? ((q + rot) & (R8 - 1)) : q];
    // tmp[q] holds chunk (q + rot) mod R8: rotate right by rot (barrel, log2(R8) stages)
    if (POW2) {
#pragma unroll
      for (int sh = 1; sh < R8; sh <<= 1) {
        if (rot & sh) {
          uint4 r2[R8];
#pragma unroll
          for (int q = 0; q < R8; ++q) r2[(q + sh) & (R8 - 1)] = tmp[q];
#pragma unroll
          for (int q = 0; q < R8; ++q) tmp[q] = r2[q];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < R8; ++q) b[c][q] = tmp[q];
  }
  int col[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int n = n0 + c * EX_THREADS + t;
    col[c] = n < d_out ? co + (n / cb) * cstr + (n % cb) : -1;
  }
  for (int i = 0; i < count; ++i) {
    T* yr = y + (size_t)toks[i] * ldy;
    float yv[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) yv[c] = col[c] >= 0 ? to_f32(yr[col[c]]) : 0.f;
    const float* vr = vsm + i * LORA_MAX_RANK;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      float d = 0.f;
#pragma unroll
      for (int q = 0; q < R8; ++q) {
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&b[c][q]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float2 f = __bfloat1622float2(h2[u]);
          d = fmaf(vr[8 * q + 2 * u] * scale, f.x, d);
          d = fmaf(vr[8 * q + 2 * u + 1] * scale, f.y, d);
        }
      }
      if (col[c] >= 0) yr[col[c]] = from_f32<T>(yv[c] + d);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(EX_THREADS, 2)
lora_expand_v_kernel(T* __restrict__ y, int ldy, const float* __restrict__ v, int ldv,
                     const int32_t* __restrict__ slot_rank, const float* __restrict__ slot_scale,
                     int max_rank, TargetArgs ta, ExpandArgs ea, LoraWs ws) {
  extern __shared__ __align__(128) unsigned char ex_raw[];
  uint64_t* bfull = reinterpret_cast<uint64_t*>(ex_raw);   // [EX_STAGES]
  uint64_t* vfull = bfull + EX_STAGES;                       // [EX_STAGES]
  unsigned char* stages = ex_raw + 64;                       // [EX_STAGES][B 32 KB | v 8 x 64 fp32]
  using Scan = cub::BlockScan<int, EX_THREADS>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int pair_end[EX_MAX_PAIRS];   // inclusive prefix of the units per pair
  __shared__ int tile_r8[EX_MAX_TILES];
  __shared__ int tile_slot[EX_MAX_TILES];
  __shared__ int tile_tok[EX_MAX_TILES][LORA_TT];
  __shared__ int tile_count[EX_MAX_TILES];
  __shared__ int total_units;
  const int NTG = ea.n_targets;
  // The stage barriers are initialised first, so the prologue's __syncthreads order the init
  // before any thread's first wait (a wait on an uninitialised mbarrier is undefined).
  if (threadIdx.x == 0) {
    for (int st = 0; st < EX_STAGES; ++st) {
      tc::mbar_init(&bfull[st], 1);
      tc::mbar_init(&vfull[st], 1);
    }
    tc::fence_barrier_init();
  }
  // ---- the unit table (plan and adapter pool are >= 2 launches back: before the wait)
  // Two dependent round trips (as in the shrink): {tile count, tiles} -> {slot rank, the
  // targets' B pointers, token ids}; a pair's "has B" flag is parked in pair_end until the scan.
  const int nt_plan = *ws.n_tiles;
  const int tmax = min(ws.max_tiles, EX_MAX_TILES);
  for (int tl = threadIdx.x; tl < tmax; tl += EX_THREADS) {
    const LoraTile tile = ws.tiles[tl];
    const bool ok = tl < nt_plan && tile.count > 0;
    const int r = ok ? min(slot_rank[tile.slot], max_rank) : 0;
#pragma unroll
    for (int tg = 0; tg < SLX_LORA_MAX_TARGETS; ++tg)
      if (tg < NTG && tl * NTG + tg < EX_MAX_PAIRS)
        pair_end[tl * NTG + tg] = ok && ta.b_ptrs[tg][tile.slot] != 0;
    tile_r8[tl] = (r + 7) >> 3;
    tile_slot[tl] = tile.slot;
    tile_count[tl] = ok ? min(tile.count, LORA_TT) : 0;
#pragma unroll
    for (int i = 0; i < LORA_TT; ++i) tile_tok[tl][i] = ok && i < tile.count ? ws.perm[tile.start + i] : 0;
  }
  const int n_tiles = min(nt_plan, tmax);
  const int n_pairs = min(n_tiles * NTG, EX_MAX_PAIRS);
  __syncthreads();
  int cnt[EX_PAIRS_PT];
  int run = 0;
#pragma unroll
  for (int k = 0; k < EX_PAIRS_PT; ++k) {
    const int p = threadIdx.x * EX_PAIRS_PT + k;
    int c = 0;
    if (p < n_pairs) {
      const int tl = p / NTG, tg = p - tl * NTG;
      const int r8 = tile_r8[tl];
      if (r8 && pair_end[p]) c = ceil_div(ta.d_out[tg], EX_THREADS * (EX_REGS / r8));
    }
    run += c;
    cnt[k] = run;
  }
  int excl, tot;
  Scan(scan_tmp).ExclusiveSum(run, excl, tot);
#pragma unroll
  for (int k = 0; k < EX_PAIRS_PT; ++k) pair_end[threadIdx.x * EX_PAIRS_PT + k] = excl + cnt[k];
  if (threadIdx.x == 0) total_units = tot;
  __syncthreads();
  const int U = total_units;
  auto locate = [&](int u, int& tl, int& tg, int& n0) {
    int lo = 0, hi = n_pairs - 1;   // first pair with pair_end > u
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (pair_end[mid] > u) hi = mid; else lo = mid + 1;
    }
    tl = lo / NTG;
    tg = lo - tl * NTG;
    n0 = (u - (lo ? pair_end[lo - 1] : 0)) * EX_THREADS * (EX_REGS / tile_r8[tl]);
  };
  auto issue_b = [&](int u, int stage) {   // thread 0: the unit's B rows -> stage
    int tl, tg, n0;
    locate(u, tl, tg, n0);
    const int rank = tile_r8[tl] * 8;
    const int cols = min(EX_THREADS * (EX_REGS / tile_r8[tl]), ta.d_out[tg] - n0);
    const bf16* B = reinterpret_cast<const bf16*>(ta.b_ptrs[tg][tile_slot[tl]]);
    const uint32_t bytes = (uint32_t)cols * rank * 2;
    tc::mbar_arrive_expect_tx(&bfull[stage], bytes);
    tc::bulk_g2s(stages + stage * EX_STAGE_BYTES, B + (size_t)n0 * rank, bytes, &bfull[stage],
                 tc::policy_evict_first());
  };
  auto issue_v = [&](int u, int stage) {   // thread 0: the tile's v rows -> stage
    int tl, tg, n0;
    locate(u, tl, tg, n0);
    const int rank = tile_r8[tl] * 8, count = tile_count[tl];
    const int voff = ea.v_off[tg] + tile_slot[tl] * ea.v_slot_stride;
    float* dst = reinterpret_cast<float*>(stages + stage * EX_STAGE_BYTES + EX_UNIT_BYTES);
    tc::mbar_arrive_expect_tx(&vfull[stage], (uint32_t)(count * rank * 4));
    for (int i = 0; i < count; ++i)
      tc::bulk_g2s(dst + i * LORA_MAX_RANK, v + (size_t)tile_tok[tl][i] * ldv + voff,
                   (uint32_t)(rank * 4), &vfull[stage], tc::policy_evict_normal());
  };
  if (threadIdx.x == 0)   // barriers were initialised before the prologue's block syncs
    for (int k = 0; k < EX_STAGES; ++k)
      if (blockIdx.x + k * gridDim.x < U) issue_b(blockIdx.x + k * gridDim.x, k);
  pdl_wait();       // v and y come from the kernels just before us
  pdl_trigger();
  if (threadIdx.x == 0)
    for (int k = 0; k < EX_STAGES; ++k)
      if (blockIdx.x + k * gridDim.x < U) issue_v(blockIdx.x + k * gridDim.x, k);
  int k = 0;
  for (int u = blockIdx.x; u < U; u += gridDim.x, ++k) {
    const int stage = k % EX_STAGES;
    const uint32_t parity = (uint32_t)((k / EX_STAGES) & 1);
    int tl, tg, n0;
    locate(u, tl, tg, n0);
    const int r8 = tile_r8[tl], count = tile_count[tl];
    const float scale = slot_scale[tile_slot[tl]];
    const int d_out = ta.d_out[tg];
    const int cb = ta.col_blk[tg], cstr = ta.col_stride[tg], co = ta.col_off[tg];
    const unsigned char* bs = stages + stage * EX_STAGE_BYTES;
    const float* vsm = reinterpret_cast<const float*>(bs + EX_UNIT_BYTES);
    tc::mbar_wait(&bfull[stage], parity);
    tc::mbar_wait(&vfull[stage], parity);
#define SLX_EXPAND_CASE(r)                                                                    \
  case r:                                                                                     \
    expand_unit<T, r>(y, ldy, bs, vsm, scale, n0, d_out, count, tile_tok[tl], co, cb, cstr);  \
    break;
    switch (r8) {
      SLX_EXPAND_CASE(1) SLX_EXPAND_CASE(2) SLX_EXPAND_CASE(3) SLX_EXPAND_CASE(4)
      SLX_EXPAND_CASE(5) SLX_EXPAND_CASE(6) SLX_EXPAND_CASE(7) SLX_EXPAND_CASE(8)
      default: break;
    }
#undef SLX_EXPAND_CASE
    __syncthreads();   // every thread is done with this stage
    const int un = u + EX_STAGES * gridDim.x;
    if (threadIdx.x == 0 && un < U) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
      issue_b(un, stage);
      issue_v(un, stage);
    }
  }
}

}  // namespace slx

using namespace slx;

extern "C" size_t slx_lora_workspace_bytes(int n_tok, int n_slots, int max_rank, int n_targets) {
  if (n_tok < 0 || n_slots <= 0 || max_rank <= 0 || n_targets <= 0) return 0;
  return lora_ws_bytes(n_tok, n_slots, max_rank, n_targets, nullptr, nullptr);
}

static int carve(void* ws, size_t ws_bytes, int n_tok, int n_slots, int max_rank, int n_targets,
                 LoraWs* out) {
  if (!ws) return SLX_ERR_WORKSPACE;
  SLX_CHECK_ALIGN(ws, 256);
  const size_t need = lora_ws_bytes(n_tok, n_slots, max_rank, n_targets, out, ws);
  return need <= ws_bytes ? SLX_OK : SLX_ERR_WORKSPACE;
}

extern "C" int slx_lora_plan_tokens(const int32_t* tok_slot, int n_tok, int n_slots, void* ws,
                                    size_t ws_bytes, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && n_slots > 0 && n_slots <= PLAN_MAX_GROUPS && (tok_slot || !n_tok));
  LoraWs w;
  // plan only touches the header/perm/tiles region, which does not depend on rank/targets
  int st = carve(ws, ws_bytes, n_tok, n_slots, 1, 1, &w);
  if (st) return st;
  return launch_ex(plan_tokens_kernel, dim3(1), dim3(PLAN_THREADS), 0, (cudaStream_t)stream, 1u,
                   tok_slot, n_tok, n_slots, w);
}

extern "C" int slx_lora_plan_segments(const int32_t* seg_indptr, const int32_t* seg_slot,
                                      int n_seg, int n_tok, int n_slots, void* ws,
                                      size_t ws_bytes, void* stream) {
  SLX_CHECK_ARG(n_seg >= 0 && n_seg <= PLAN_MAX_GROUPS && n_tok >= 0 && n_slots > 0 &&
                (n_seg == 0 || (seg_indptr && seg_slot)));
  LoraWs w;
  int st = carve(ws, ws_bytes, n_tok, n_slots, 1, 1, &w);
  if (st) return st;
  return launch_ex(plan_segments_kernel, dim3(1), dim3(PLAN_THREADS), 0, (cudaStream_t)stream,
                   1u, seg_indptr, seg_slot, n_seg, n_tok, n_slots, w);
}

extern "C" int slx_lora_apply(int dtype, void* y, int ldy, const void* x, int ldx, int n_tok,
                              int d_in, const int32_t* slot_rank, const float* slot_scale,
                              int n_slots, int max_rank, int n_targets,
                              const slx_lora_target* targets, void* ws, size_t ws_bytes,
                              void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d_in > 0 && d_in % 8 == 0 && ldx >= d_in && ldx % 8 == 0 &&
                n_slots > 0 && max_rank > 0 && max_rank <= LORA_MAX_RANK && max_rank % 8 == 0 &&
                n_targets >= 1 && n_targets <= SLX_LORA_MAX_TARGETS && targets && slot_rank &&
                slot_scale && y && x);
  SLX_CHECK_ALIGN(x, 16);
  TargetArgs ta;
  for (int i = 0; i < n_targets; ++i) {
    const slx_lora_target& t = targets[i];
    SLX_CHECK_ARG(t.a_ptrs && t.b_ptrs && t.d_out > 0 && t.d_out % 8 == 0 && t.y_col_offset >= 0 &&
                  t.y_col_block > 0 && t.y_col_stride >= t.y_col_block);
    const long last = (long)t.y_col_offset + (long)((t.d_out - 1) / t.y_col_block) * t.y_col_stride +
                      (t.d_out - 1) % t.y_col_block;
    SLX_CHECK_ARG(last < ldy);
    ta.a_ptrs[i] = t.a_ptrs;
    ta.b_ptrs[i] = t.b_ptrs;
    ta.d_out[i] = t.d_out;
    ta.col_off[i] = t.y_col_offset;
    ta.col_blk[i] = t.y_col_block;
    ta.col_stride[i] = t.y_col_stride;
  }
  LoraWs w;
  int st = carve(ws, ws_bytes, n_tok, n_slots, max_rank, n_targets, &w);
  if (st) return st;
  if (n_tok == 0) return SLX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_tok <= LORA_FUSED_MAX_TOK) {
    int fks = d_in / 512;
    fks = fks < 1 ? 1 : (fks > FU_MAX_KS ? FU_MAX_KS : fks);
    const int kc = ceil_div(ceil_div(d_in, fks), 8) * 8;
    int max_dout = 0;
    for (int i = 0; i < n_targets; ++i) max_dout = targets[i].d_out > max_dout ? targets[i].d_out : max_dout;
    const int ns = ceil_div(ceil_div(max_dout, fks), 8) * 8;
    const size_t tsz = dtype == SLX_DT_BF16 ? 2 : 4;
    const size_t smem = (size_t)LORA_TT * (kc + ns) * tsz + (size_t)max_rank * kc * 2 +
                        (size_t)ns * max_rank * 2 + 2 * LORA_TT * max_rank * 4 + LORA_TT * 4;
    if (smem > 200 * 1024) return SLX_ERR_UNSUPPORTED;
    dim3 gf((unsigned)(w.max_tiles * fks), (unsigned)n_targets);
    if (dtype == SLX_DT_BF16) {
      auto k = lora_fused_kernel<bf16>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SLX_ERR_CUDA;
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      return launch_ex(k, gf, dim3(FU_THREADS), smem, s, (unsigned)fks, (bf16*)y, ldy,
                       (const bf16*)x, ldx, n_tok, d_in, fks, kc, ns, slot_rank, slot_scale, max_rank,
                       ta, w);
    } else if (dtype == SLX_DT_F32) {
      auto k = lora_fused_kernel<float>;
      if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SLX_ERR_CUDA;
      cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      return launch_ex(k, gf, dim3(FU_THREADS), smem, s, (unsigned)fks, (float*)y, ldy,
                       (const float*)x, ldx, n_tok, d_in, fks, kc, ns, slot_rank, slot_scale, max_rank,
                       ta, w);
    }
    return SLX_ERR_INVALID;
  }
  int ks = d_in / 512;
  ks = ks < 1 ? 1 : (ks > LORA_MAX_KS ? LORA_MAX_KS : ks);
  int max_dout = 0;
  for (int i = 0; i < n_targets; ++i) max_dout = targets[i].d_out > max_dout ? targets[i].d_out : max_dout;
  int n_split = ceil_div(max_dout, 512);
  dim3 gs((unsigned)w.max_tiles, (unsigned)n_targets, (unsigned)ks);
  dim3 ge((unsigned)w.max_tiles, (unsigned)n_targets, (unsigned)n_split);
  if (dtype == SLX_DT_BF16) {
    st = launch_ex(lora_shrink_kernel<bf16>, gs, dim3(256), 0, s, 1u, (const bf16*)x, ldx, n_tok,
                   d_in, ks, slot_rank, max_rank, ta, w);
    if (st) return st;
    st = launch_ex(lora_expand_kernel<bf16>, ge, dim3(256), 0, s, 1u, (bf16*)y, ldy, n_tok, ks,
                   n_split, slot_rank, slot_scale, max_rank, ta, w);
  } else if (dtype == SLX_DT_F32) {
    st = launch_ex(lora_shrink_kernel<float>, gs, dim3(256), 0, s, 1u, (const float*)x, ldx, n_tok,
                   d_in, ks, slot_rank, max_rank, ta, w);
    if (st) return st;
    st = launch_ex(lora_expand_kernel<float>, ge, dim3(256), 0, s, 1u, (float*)y, ldy, n_tok, ks,
                   n_split, slot_rank, slot_scale, max_rank, ta, w);
  } else {
    return SLX_ERR_INVALID;
  }
  return st;
}

extern "C" int slx_lora_bgmv(int dtype, void* y, int ldy, const void* x, int ldx,
                             const int32_t* tok_slot, int n_tok, int d_in,
                             const int32_t* slot_rank, const float* slot_scale, int n_slots,
                             int max_rank, int n_targets, const slx_lora_target* targets, void* ws,
                             size_t ws_bytes, void* stream) {
  int st = slx_lora_plan_tokens(tok_slot, n_tok, n_slots, ws, ws_bytes, stream);
  if (st) return st;
  return slx_lora_apply(dtype, y, ldy, x, ldx, n_tok, d_in, slot_rank, slot_scale, n_slots,
                        max_rank, n_targets, targets, ws, ws_bytes, stream);
}

extern "C" int slx_lora_sgmv(int dtype, void* y, int ldy, const void* x, int ldx,
                             const int32_t* seg_indptr, const int32_t* seg_slot, int n_seg,
                             int n_tok, int d_in, const int32_t* slot_rank,
                             const float* slot_scale, int n_slots, int max_rank, int n_targets,
                             const slx_lora_target* targets, void* ws, size_t ws_bytes,
                             void* stream) {
  int st = slx_lora_plan_segments(seg_indptr, seg_slot, n_seg, n_tok, n_slots, ws, ws_bytes,
                                  stream);
  if (st) return st;
  return slx_lora_apply(dtype, y, ldy, x, ldx, n_tok, d_in, slot_rank, slot_scale, n_slots,
                        max_rank, n_targets, targets, ws, ws_bytes, stream);
}

extern "C" int slx_lora_expand(int dtype, void* y, int ldy, const void* v_all, int ldv, int n_tok,
                               const int32_t* slot_rank, const float* slot_scale, int n_slots,
                               int max_rank, int n_targets, const slx_lora_target* targets,
                               const int* v_col_off, int v_slot_stride, void* ws, size_t ws_bytes,
                               void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && n_slots > 0 && max_rank > 0 && max_rank <= LORA_MAX_RANK &&
                max_rank % 8 == 0 && n_targets >= 1 && n_targets <= SLX_LORA_MAX_TARGETS &&
                targets && v_col_off && slot_rank && slot_scale && y && v_all && ldv > 0 &&
                ldv % 4 == 0 && v_slot_stride >= 0 && v_slot_stride % 4 == 0);
  SLX_CHECK_ALIGN(v_all, 16);
  TargetArgs ta{};
  ExpandArgs ea{};
  ea.v_slot_stride = v_slot_stride;
  int max_dout = 0;
  for (int i = 0; i < n_targets; ++i) {
    const slx_lora_target& t = targets[i];
    SLX_CHECK_ARG(t.b_ptrs && t.d_out > 0 && t.d_out % 8 == 0 && t.y_col_block > 0 &&
                  t.y_col_stride >= t.y_col_block && v_col_off[i] >= 0 && v_col_off[i] % 4 == 0 &&
                  v_col_off[i] + (n_slots - 1) * v_slot_stride + max_rank <= ldv);
    ta.a_ptrs[i] = t.a_ptrs;
    ta.b_ptrs[i] = t.b_ptrs;
    ta.d_out[i] = t.d_out;
    ta.col_off[i] = t.y_col_offset;
    ta.col_blk[i] = t.y_col_block;
    ta.col_stride[i] = t.y_col_stride;
    ea.v_off[i] = v_col_off[i];
    max_dout = t.d_out > max_dout ? t.d_out : max_dout;
  }
  LoraWs w;
  int st = carve(ws, ws_bytes, n_tok, n_slots, 1, 1, &w);
  if (st) return st;
  if (n_tok == 0) return SLX_OK;
  if (w.max_tiles * n_targets > EX_MAX_PAIRS || w.max_tiles > EX_MAX_TILES) return SLX_ERR_UNSUPPORTED;
  ea.n_targets = n_targets;
  const int grid = 2 * sm_count();
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == SLX_DT_BF16) {
    if (cudaFuncSetAttribute(lora_expand_v_kernel<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EX_DYN_SMEM) != cudaSuccess)
      return SLX_ERR_CUDA;
    return launch_ex(lora_expand_v_kernel<bf16>, dim3(grid), dim3(EX_THREADS), EX_DYN_SMEM, s, 1u,
                     (bf16*)y, ldy, (const float*)v_all, ldv, slot_rank, slot_scale, max_rank, ta,
                     ea, w);
  }
  if (dtype == SLX_DT_F32) {
    if (cudaFuncSetAttribute(lora_expand_v_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)EX_DYN_SMEM) != cudaSuccess)
      return SLX_ERR_CUDA;
    return launch_ex(lora_expand_v_kernel<float>, dim3(grid), dim3(EX_THREADS), EX_DYN_SMEM, s, 1u,
                     (float*)y, ldy, (const float*)v_all, ldv, slot_rank, slot_scale, max_rank, ta,
                     ea, w);
  }
  return SLX_ERR_INVALID;
}

extern "C" int slx_lora_shrink(int dtype, float* v, int ldv, const void* x, int ldx, int n_tok,
                               int d_in, const int32_t* slot_rank, int n_slots, int max_rank,
                               int n_targets, const slx_lora_target* targets, const int* v_col_off,
                               void* ws, size_t ws_bytes, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d_in > 0 && d_in % 8 == 0 && ldx >= d_in && ldx % 8 == 0 &&
                n_slots > 0 && max_rank > 0 && max_rank <= LORA_MAX_RANK && max_rank % 8 == 0 &&
                n_targets >= 1 && n_targets <= SLX_LORA_MAX_TARGETS && targets && v_col_off &&
                slot_rank && v && x && ldv > 0);
  SLX_CHECK_ALIGN(x, 16);
  TargetArgs ta{};
  ShrinkOut so{};
  for (int i = 0; i < n_targets; ++i) {
    SLX_CHECK_ARG(targets[i].a_ptrs != nullptr && v_col_off[i] >= 0 && v_col_off[i] + max_rank <= ldv);
    ta.a_ptrs[i] = targets[i].a_ptrs;
    so.v_off[i] = v_col_off[i];
  }
  so.n_targets = n_targets;
  LoraWs w;
  int st = carve(ws, ws_bytes, n_tok, n_slots, 1, 1, &w);
  if (st) return st;
  if (n_tok == 0) return SLX_OK;
  if (w.max_tiles * n_targets > SH_MAX_PAIRS || w.max_tiles > SH_MAX_TILES) return SLX_ERR_UNSUPPORTED;
  const dim3 grid((unsigned)sm_count());
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == SLX_DT_BF16) {
    int rpu, xt;
    if (!shrink_geometry(d_in, sizeof(bf16), &rpu, &xt)) return SLX_ERR_UNSUPPORTED;
    const size_t smem = shrink_smem_bytes(d_in, sizeof(bf16), rpu, xt);
    if (cudaFuncSetAttribute(lora_shrink_v_kernel<bf16>,
            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SLX_ERR_CUDA;
    return launch_ex(lora_shrink_v_kernel<bf16>, grid, dim3(SH_WARPS * 32), smem, s, 1u, v, ldv,
                     (const bf16*)x, ldx, d_in, slot_rank, max_rank, ta, so, w, rpu, xt);
  }
  if (dtype == SLX_DT_F32) {
    int rpu, xt;
    if (!shrink_geometry(d_in, sizeof(float), &rpu, &xt)) return SLX_ERR_UNSUPPORTED;
    const size_t smem = shrink_smem_bytes(d_in, sizeof(float), rpu, xt);
    if (cudaFuncSetAttribute(lora_shrink_v_kernel<float>,
            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SLX_ERR_CUDA;
    return launch_ex(lora_shrink_v_kernel<float>, grid, dim3(SH_WARPS * 32), smem, s, 1u, v, ldv,
                     (const float*)x, ldx, d_in, slot_rank, max_rank, ta, so, w, rpu, xt);
  }
  return SLX_ERR_INVALID;
}
