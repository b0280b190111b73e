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

namespace slx {

constexpr int LORA_TT = 16;       // tokens per tile
constexpr int LORA_MAX_RANK = 64;
constexpr int LORA_MAX_KS = 8;    // k-splits of the shrink
constexpr int PLAN_THREADS = 1024;
constexpr int PLAN_MAX_GROUPS = 2048;

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
  SLX_CLEAR_STALE();
  plan_tokens_kernel<<<1, PLAN_THREADS, 0, (cudaStream_t)stream>>>(tok_slot, n_tok, n_slots, w);
  SLX_LAUNCH_CHECK();
  return SLX_OK;
}

extern "C" int slx_lora_plan_segments(const int32_t* seg_indptr, const int32_t* seg_slot,
                                      int n_seg, int n_tok, int n_slots, void* ws,
                                      size_t ws_bytes, void* stream) {
  SLX_CHECK_ARG(n_seg >= 0 && n_seg <= PLAN_MAX_GROUPS && n_tok >= 0 && n_slots > 0 &&
                (n_seg == 0 || (seg_indptr && seg_slot)));
  LoraWs w;
  int st = carve(ws, ws_bytes, n_tok, n_slots, 1, 1, &w);
  if (st) return st;
  SLX_CLEAR_STALE();
  plan_segments_kernel<<<1, PLAN_THREADS, 0, (cudaStream_t)stream>>>(seg_indptr, seg_slot, n_seg,
                                                                     n_tok, n_slots, w);
  SLX_LAUNCH_CHECK();
  return SLX_OK;
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
  int ks = d_in / 512;
  ks = ks < 1 ? 1 : (ks > LORA_MAX_KS ? LORA_MAX_KS : ks);
  int max_dout = 0;
  for (int i = 0; i < n_targets; ++i) max_dout = targets[i].d_out > max_dout ? targets[i].d_out : max_dout;
  int n_split = ceil_div(max_dout, 512);
  dim3 gs((unsigned)w.max_tiles, (unsigned)n_targets, (unsigned)ks);
  dim3 ge((unsigned)w.max_tiles, (unsigned)n_targets, (unsigned)n_split);
  if (dtype == SLX_DT_BF16) {
    SLX_CLEAR_STALE();
    lora_shrink_kernel<bf16><<<gs, 256, 0, s>>>((const bf16*)x, ldx, n_tok, d_in, ks, slot_rank,
                                                max_rank, ta, w);
    SLX_CLEAR_STALE();
    lora_expand_kernel<bf16><<<ge, 256, 0, s>>>((bf16*)y, ldy, n_tok, ks, n_split, slot_rank,
                                                slot_scale, max_rank, ta, w);
  } else if (dtype == SLX_DT_F32) {
    SLX_CLEAR_STALE();
    lora_shrink_kernel<float><<<gs, 256, 0, s>>>((const float*)x, ldx, n_tok, d_in, ks, slot_rank,
                                                 max_rank, ta, w);
    SLX_CLEAR_STALE();
    lora_expand_kernel<float><<<ge, 256, 0, s>>>((float*)y, ldy, n_tok, ks, n_split, slot_rank,
                                                 slot_scale, max_rank, ta, w);
  } else {
    return SLX_ERR_INVALID;
  }
  SLX_LAUNCH_CHECK();
  return SLX_OK;
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
