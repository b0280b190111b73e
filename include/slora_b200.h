/*
 * libslora_b200 — C ABI of the B200-native shared-backbone multi-LoRA hot path.
 *
 * The reference (ServerlessLoRA, /root/reference/pkg = `slorasim`) ships NO native
 * code and no FFI: its forward is the latency law T0 + alpha*(b-1)
 * (pkg/src/slorasim/batching.py:17-21, consumed at pkg/src/slorasim/engine.py:832,888,909)
 * and its pre-load is `usable_at_ms = now + load_ms` (pkg/src/slorasim/engine.py:1040-1053).
 * Each entry point below names the reference interface whose MEANING it replaces; the
 * Python mirror (paper_2505_14468_b200/) binds these with ctypes.
 *
 * Conventions
 *  - every function returns int32 status (SLX_OK = 0, negative = error), never throws,
 *    never allocates device memory (workspaces are passed in), never synchronises, and
 *    enqueues on the caller's stream (`stream` is a cudaStream_t passed as void*).
 *  - activations are row-major with an explicit leading dimension (elements);
 *    dtype SLX_DT_BF16 or SLX_DT_F32 ("fp32 parity mode": fp32 activations, fp32
 *    accumulate, bf16 weights upcast exactly).
 *  - weights are bf16, nn.Linear layout W[out, in] (K-major).  LoRA is PEFT layout:
 *    A [rank, d_in], B [d_out, rank], scale = alpha / rank, unmerged
 *    (PAPER.md:614-621,645-646).
 *  - index arrays are int32 on the device; slot -1 means "no adapter".
 *  - pointers used with 128-bit loads must be 16-byte aligned and row lengths
 *    multiples of 8 elements (SLX_ERR_ALIGN / SLX_ERR_INVALID otherwise).
 */
#ifndef SLORA_B200_H
#define SLORA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SLX_API __attribute__((visibility("default")))
#else
#define SLX_API
#endif

#define SLX_ABI_VERSION 2

enum {
  SLX_OK = 0,
  SLX_ERR_INVALID = -1,     /* bad shape / argument (Python: ValueError) */
  SLX_ERR_ALIGN = -2,       /* pointer or leading dim misaligned (ValueError) */
  SLX_ERR_UNSUPPORTED = -3, /* shape outside the kernel's envelope (ValueError) */
  SLX_ERR_WORKSPACE = -4,   /* workspace too small (ValueError) */
  SLX_ERR_CUDA = -5,        /* CUDA launch/runtime error (RuntimeError) */
  SLX_ERR_NCCL = -6         /* NCCL error (RuntimeError) */
};

enum { SLX_DT_BF16 = 0, SLX_DT_F32 = 1 };

enum {
  SLX_EPI_NONE = 0,     /* C = A W^T */
  SLX_EPI_RESIDUAL = 1, /* C = A W^T + R   (R may alias C) */
  SLX_EPI_SILU_MUL = 2  /* W rows blocked [gate 128 | up 128]*: C[M, N/2] = silu(gate) * up */
};

SLX_API const char* slx_status_string(int status);
SLX_API int slx_abi_version(void);
/* Number of SMs of the current device (cached), for grid sizing in host code. */
SLX_API int slx_device_sm_count(int* out);

/* ------------------------------------------------------------------ K1: backbone GEMM
 * Replaces the prefill/decode "work" of the latency law (batching.py:17-21,
 * engine.py:832 prefill_work_ms, engine.py:888,909 decode gap) for the q/k/v/o,
 * gate/up/down and lm_head projections.
 * C[M,N] = A[M,K] · W[N,K]^T (+ epilogue), bf16 in, fp32 accumulate in TMEM (tcgen05),
 * C dtype c_dtype (bf16 or fp32).  Any N (SiLU: N % 256 == 0), K % 8 == 0,
 * lda/ldc/ldr % 8 == 0.  For few output tiles (decode) the K range is split over CTAs and
 * reduced either across a thread-block cluster in distributed shared memory or, when that
 * covers more SMs, through fp32 partial tiles in `ws` (zero-initialised once, left zeroed;
 * slx_gemm_workspace_bytes; pass NULL to disable).  Both reductions are deterministic.
 */
enum {
  SLX_W_ROWMAJOR = 0, /* W[N, K] row-major (nn.Linear) */
  SLX_W_TILED = 1     /* W packed as [ceil(N/128)][ceil(K/64)][128][64] bf16, zero-padded: every
                         TMA box of the GEMM is one contiguous 16 KB burst (slx_pack_weight) */
};
SLX_API size_t slx_gemm_workspace_bytes(int M, int N, int K, int epilogue);
/* Side output: with C2 != NULL, columns [n_main, N) (e.g. the stacked LoRA A rows appended
 * to a projection's W: the decode shrink) are written in fp32 to C2 [M, ldc2] and get no
 * residual; columns [0, n_main) go to C/R as usual (n_main % 16 == 0; not with SiLU). */
SLX_API int slx_gemm_bf16(const void* A, int lda, const void* W, void* C, int ldc, int c_dtype,
                  const void* R, int ldr, int M, int N, int K, int epilogue, int w_layout,
                  int n_main, void* C2, int ldc2, void* ws, size_t ws_bytes, void* stream);
typedef struct slx_lora_delta slx_lora_delta;   /* defined with the K2/K3 entry points */
typedef struct slx_splitk_in slx_splitk_in;     /* defined with the K4 entry points */

/* L2 prefetch hint: up to two device regions the NEXT kernel on the stream streams first.  A
 * kernel that takes one issues cp.async.bulk.prefetch.L2 of them (split over its CTAs) as soon
 * as its own HBM stream has been issued, so HBM stays busy across the kernel boundary (its
 * epilogue, the next launch and the next prologue) and the next kernel starts from L2. */
typedef struct slx_l2_prefetch {
  const void* ptr[2];
  size_t bytes[2];
} slx_l2_prefetch;
/* Explicit tiling choices (tests / tuning tools; NULL or all-zero = the planner's choice, which
 * is what the product uses).  The library reads no environment variables. */
typedef struct slx_gemm_tuning {
  int tile_kernel;   /* 1: never the stream-K decode kernel (tile kernel, any M) */
  int ctas_per_sm;   /* tile kernel: 1 or 2 */
  int splits;        /* tile kernel: K splits per output tile (1..8) */
  int bn;            /* tile kernel: 128 or 256 weight rows per tile */
  int gsplit;        /* tile kernel: 1 = split-K reduced through global partials, 2 = DSMEM cluster */
  int sk_ctas;       /* stream-K: CTAs (all-SM stream-K partition with this many CTAs) */
  int sk_min_units;  /* stream-K: minimum k-blocks per piece (default 4) */
  int sk_no_cluster; /* stream-K: 1 = reduce uniform splits through global pieces, not DSMEM */
} slx_gemm_tuning;
/* slx_gemm_bf16 + an L2 prefetch hint for the next kernel (pf may be NULL) + explicit tiling
 * (tuning may be NULL). */
SLX_API int slx_gemm_bf16_ex(const void* A, int lda, const void* W, void* C, int ldc, int c_dtype,
                  const void* R, int ldr, int M, int N, int K, int epilogue, int w_layout,
                  int n_main, void* C2, int ldc2, void* ws, size_t ws_bytes,
                  const slx_l2_prefetch* pf, const slx_gemm_tuning* tuning, void* stream);
/* Decode split-K handed to the consumer: W tiled, M <= 128; the N columns are cut in 256-wide
 * tiles and the K range of each tile in `splits` equal pieces, one CTA per piece; every piece
 * is written in fp32 to `part` with no reduction and no epilogue, so the kernel has no tail.
 * Layout (the consumer's contract, e.g. slx_rmsnorm_fused): with bm = M rounded up to 16,
 *   part[((tile * splits + piece) * bm * 256) + ((col % 256) / 16 * bm + m) * 16 + col % 16]
 * and C[m, col] = sum over piece (in order) of the pieces.  part_bytes >= slx_gemm_splitk_bytes. */
SLX_API size_t slx_gemm_splitk_bytes(int M, int N, int splits);
SLX_API int slx_gemm_bf16_splitk(const void* A, int lda, const void* W, int M, int N, int K,
                  int splits, float* part, size_t part_bytes, const slx_l2_prefetch* pf,
                  void* stream);
/* Debug only: following slx_gemm_bf16 launches write 16 u64 globaltimer slots per CTA into
 * the device buffer `buf` (phase timeline: entry, prologue, past PDL wait, first stage landed,
 * last MMA issued, accumulator ready, split-K reduction start, exit, reduction end, segment
 * accumulators ready; unused slots stay as they were).  NULL disables. */
SLX_API int slx_debug_gemm_trace(void* buf);
/* Grouped GEMM (SGMV on tcgen05): CTA tile i = gtiles[i] = {group, m0, m_rows, n0} computes
 * C[m0:m0+m_rows, n0:n0+256] = alpha[group] * A[m0.., :K] . W_group[n0.., :]^T (+ R), where
 * W_group is row-major [w_rows, w_cols] (row stride w_ld) and columns >= w_cols read as 0.
 * Up to 16 groups per call; host arrays w_ptrs/w_rows/w_cols/w_ld/alpha; gtiles on device
 * (slx_gemm_group_tile_bytes() each).  Prefill LoRA: shrink with W = A_adapter (alpha =
 * scale), expand with A = v and W = B_adapter (residual in place).  n_seg > 1 (<= 4): the
 * arrays hold n_groups x n_seg entries (group-major) and output columns [64 s, 64 s + 64) of a
 * tile come from W entry group * n_seg + s (<= 64 rows each; N <= 64 n_seg): e.g. the q, k and
 * v shrinks of one adapter in ONE pass over A. */
SLX_API size_t slx_gemm_group_tile_bytes(void);
SLX_API int slx_gemm_grouped_bf16(const void* A, int lda, int M, int K, int n_groups, int n_seg,
                  const uint64_t* w_ptrs, const int* w_rows, const int* w_cols, const int* w_ld,
                  const float* alpha, void* C, int ldc, int c_dtype, const void* R, int ldr, int N,
                  int epilogue, const void* gtiles, int n_gtiles, void* stream);
/* Prefill backbone GEMM with the LoRA expand folded into its mainloop (grouped tiles
 * {group, m0, m_rows, n0}, 256 columns each): C = A . W^T (+ R) for every tile, and a tile whose
 * group >= 0 accumulates one more K block v[m, t*64 : t*64+64] . B_(group, t)[n - t_bound[t], :]^T,
 * t = the target whose column range [t_bound[t], t_bound[t+1]) holds the tile (t_bound[t] % 256
 * == 0).  v [M, ldv] bf16 is the LoRA shrink with the scale folded in (slx_gemm_grouped_bf16
 * with alpha = scale), zero beyond each adapter's rank; b_ptrs[a * n_targets + t] = B [b_rows[t],
 * ranks[a]] row-major.  <= 16 adapters, <= 3 targets.  No separate expand, no y read-modify-write. */
/* RoPE + KV append fused into the q/k/v projection's epilogue (prefill): with `rope` non-NULL
 * the GEMM output columns [0, H*D) are q, rotated (rotate-half, cos/sin tables fp32
 * [max_pos, D/2] at tok_pos[m]) and stored to C; [H*D, (H+Hkv)*D) are k, rotated and stored to
 * k_cache[tok_seq[m]][kv head][tok_pos[m]][:]; the rest is v, stored to v_cache — the same
 * arithmetic as slx_rope_kv_write on the bf16-rounded projection, without the round trip through
 * C (k and v columns of C are not written).  D = 128, H*D and Hkv*D multiples of 256. */
typedef struct slx_rope_kv {
  const int32_t* tok_pos;
  const int32_t* tok_seq;
  const float* cos_tab;
  const float* sin_tab;
  int max_pos;
  void* k_cache;
  void* v_cache;
  int max_ctx;
  int heads, kv_heads, head_dim;
} slx_rope_kv;
SLX_API int slx_gemm_bf16_lorafold(const void* A, int lda, const void* W, int w_layout, void* C,
                  int ldc, int c_dtype, const void* R, int ldr, int M, int N, int K, int epilogue,
                  const void* gtiles, int n_gtiles, const void* v, int ldv, int n_targets,
                  const int* t_bound, int n_adapters, const uint64_t* b_ptrs, const int* b_rows,
                  const int* ranks, const slx_rope_kv* rope, void* stream);
/* Pack a row-major bf16 W[N, K] (row stride ld) into the SLX_W_TILED layout (device kernel).
 * dst must hold slx_packed_weight_elems(N, K) elements. */
SLX_API size_t slx_packed_weight_elems(int N, int K);
SLX_API int slx_pack_weight(void* dst, const void* src, int N, int K, int ld, void* stream);
/* (Re)write rows [row0, row0 + n_rows) of a packed SLX_W_TILED matrix with K columns from a
 * row-major src [n_rows, K] (row stride ld); src == NULL writes zeros (slot eviction). */
SLX_API int slx_pack_weight_rows(void* dst, const void* src, int n_rows, int K, int ld, int row0,
                  void* stream);
/* fp32-parity GEMM (CUDA cores): A fp32 [M,K], W bf16 [N,K], C/R fp32.  Epilogue NONE or
 * RESIDUAL.  K % 8 == 0. */
SLX_API int slx_gemm_f32(const void* A, int lda, const void* W, void* C, int ldc,
                 const void* R, int ldr, int M, int N, int K, int epilogue, void* stream);

/* ------------------------------------------------------------------ K2/K3: multi-LoRA
 * Replaces the batch → adapter association of the contention-aware batcher's
 * FlushDecision (batching.py:99-105) by a per-token / per-segment adapter slot.
 * One call applies up to SLX_LORA_MAX_TARGETS projections that share the input x:
 *   y[t, col(n)] += scale[s] * sum_j (x[t] . A_s[j]) * B_s[n, j],   s = slot of token t.
 */
#define SLX_LORA_MAX_TARGETS 4
typedef struct slx_lora_target {
  const uint64_t* a_ptrs; /* device [n_slots]: address of A_s [rank_s, d_in] (bf16) */
  const uint64_t* b_ptrs; /* device [n_slots]: address of B_s [d_out, rank_s] (bf16) */
  int d_out;
  int y_col_offset;       /* output column of feature 0 */
  int y_col_block;        /* features per contiguous output block (= d_out when unblocked) */
  int y_col_stride;       /* output-column distance between consecutive blocks */
} slx_lora_target;

/* Workspace for a plan + apply over n_tok tokens (plan is reusable across layers). */
SLX_API size_t slx_lora_workspace_bytes(int n_tok, int n_slots, int max_rank, int n_targets);
/* Plan from a per-token slot (decode, BGMV): stable counting sort of tokens by slot. */
SLX_API int slx_lora_plan_tokens(const int32_t* tok_slot, int n_tok, int n_slots,
                         void* ws, size_t ws_bytes, void* stream);
/* Plan from contiguous segments (prefill, SGMV): tokens [seg_indptr[s], seg_indptr[s+1])
 * use slot seg_slot[s]. seg_indptr: device int32 [n_seg+1]. */
SLX_API int slx_lora_plan_segments(const int32_t* seg_indptr, const int32_t* seg_slot, int n_seg,
                           int n_tok, int n_slots, void* ws, size_t ws_bytes, void* stream);
/* Shrink (x A^T -> v staged fp32) + expand (scale * v B^T added into y) over the plan. */
SLX_API int slx_lora_apply(int dtype, void* y, int ldy, const void* x, int ldx, int n_tok, int d_in,
                   const int32_t* slot_rank, const float* slot_scale, int n_slots, int max_rank,
                   int n_targets, const slx_lora_target* targets,
                   void* ws, size_t ws_bytes, void* stream);
/* Decode expand over the plan in ws (a_ptrs unused): v_all [n_tok, ldv] fp32 holds, for
 * target i, column v_col_off[i] + slot * v_slot_stride + j = x_t . A_slot[j] — the stacked
 * shrink inside the projection GEMM (slx_gemm_bf16 side output, v_slot_stride = max_rank) or
 * the gathered shrink (slx_lora_shrink, v_slot_stride = 0); adds scale * v . B_slot^T into y in
 * place (sequential fmaf in j, one rounding: bit-identical to the fused slx_lora_delta).
 * Persistent, B rows and v rows by TMA bulk copies: ldv, v_col_off[i] and v_slot_stride are
 * multiples of 4 and v_all is 16-byte aligned (else SLX_ERR_INVALID); B tables 16-byte aligned;
 * the plan's tile bound (slx_lora_workspace_bytes' n_tok / n_slots) must satisfy
 * max_tiles <= 384 and max_tiles * n_targets <= 2048, max_tiles = ceil(n_tok / 8) +
 * min(n_slots, n_tok) + 1 (else SLX_ERR_UNSUPPORTED). */
SLX_API int slx_lora_expand(int dtype, void* y, int ldy, const void* v_all, int ldv, int n_tok,
                  const int32_t* slot_rank, const float* slot_scale, int n_slots, int max_rank,
                  int n_targets, const slx_lora_target* targets, const int* v_col_off,
                  int v_slot_stride, void* ws, size_t ws_bytes, void* stream);
/* Gathered shrink (decode with a large adapter pool): over the plan in ws (slx_lora_plan_tokens)
 * v[t, v_col_off[i] + j] = x_t . A_{slot(t), i}[j] for j < rank (fp32, unscaled), reading each
 * adapter present in the batch once per plan tile of <= 8 tokens (a_ptrs of the targets; b_ptrs
 * unused).  Rows of tokens without an adapter are not written.  Consumers: slx_lora_delta with
 * v_slot_stride = 0.  Persistent, A rows and x rows by TMA bulk copies (x 16-byte aligned);
 * max_tiles <= 384 and max_tiles * n_targets <= 1024 (see slx_lora_expand), and two stages of
 * >= 1 A row + 1 x row must fit 204 KB of shared memory (bf16 x: d_in <= 26112), else
 * SLX_ERR_UNSUPPORTED. */
SLX_API int slx_lora_shrink(int dtype, float* v, int ldv, const void* x, int ldx, int n_tok,
                  int d_in, const int32_t* slot_rank, int n_slots, int max_rank, int n_targets,
                  const slx_lora_target* targets, const int* v_col_off, void* ws,
                  size_t ws_bytes, void* stream);
/* Fused decode expand: a consumer kernel adds the LoRA term of the projection it reads while
 * loading it, instead of a separate expand launch + read-modify-write of y.  For output
 * column n of target i of token t (slot s = tok_slot[t] >= 0, rank r = slot_rank[s]):
 *   delta = sum_{j < r} (v[t, v_col_off[i] + s * max_rank + j] * slot_scale[s]) * B_s[n, j]
 * (sequential fmaf in j: bit-identical to slx_lora_expand).  The target's outputs are the row
 * columns [y_col_off[i], y_col_off[i] + d_out[i]).  b_ptrs[i]: device uint64 [n_slots] table of
 * B_s [d_out, r] (bf16; 0 = adapter does not target it).
 * v column of (target i, slot s, rank index j) = v_col_off[i] + s * v_slot_stride + j:
 * v_slot_stride = max_rank for the stacked shrink (every slot's block), 0 for a gathered shrink
 * that writes only the token's own adapter (slx_lora_shrink_gather).
 * Preconditions: ranks are multiples of 8 and <= max_rank (16-byte B rows); v 16-byte aligned. */
typedef struct slx_lora_delta {
  const float* v;            /* fp32 [n_tok, ldv]: the shrink output */
  int ldv;
  const int32_t* tok_slot;   /* [n_tok], -1 = no adapter */
  const int32_t* slot_rank;  /* [n_slots] */
  const float* slot_scale;   /* [n_slots] */
  int max_rank;
  int n_targets;             /* 0 .. SLX_LORA_MAX_TARGETS */
  int v_slot_stride;         /* see above (multiple of 4) */
  const uint64_t* b_ptrs[SLX_LORA_MAX_TARGETS];
  int v_col_off[SLX_LORA_MAX_TARGETS];
  int y_col_off[SLX_LORA_MAX_TARGETS];
  int d_out[SLX_LORA_MAX_TARGETS];
} slx_lora_delta;
/* Convenience: plan_tokens + apply (BGMV) and plan_segments + apply (SGMV). */
SLX_API int slx_lora_bgmv(int dtype, void* y, int ldy, const void* x, int ldx, const int32_t* tok_slot,
                  int n_tok, int d_in, const int32_t* slot_rank, const float* slot_scale,
                  int n_slots, int max_rank, int n_targets, const slx_lora_target* targets,
                  void* ws, size_t ws_bytes, void* stream);
SLX_API int slx_lora_sgmv(int dtype, void* y, int ldy, const void* x, int ldx, const int32_t* seg_indptr,
                  const int32_t* seg_slot, int n_seg, int n_tok, int d_in,
                  const int32_t* slot_rank, const float* slot_scale, int n_slots, int max_rank,
                  int n_targets, const slx_lora_target* targets,
                  void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------ K4: supporting ops
 * KV cache layout per layer: [n_seq_slots][kv_heads][max_ctx][head_dim], dtype = activations.
 * The KV pool honours the ledger's per-request reservation (ledger.py:162-174).
 */
SLX_API int slx_embedding(int dtype, void* out, const void* table, const int32_t* tokens,
                  int n_tok, int d, int vocab, void* stream);
SLX_API int slx_rmsnorm(int dtype, void* out, int ldo, const void* x, int ldx, const void* w,
                int n_tok, int d, float eps, void* stream);
/* Split-K pieces of a projection (slx_gemm_bf16_splitk layout) consumed by the next kernel:
 * columns [0, n_main) are the projection output, columns >= n_main its stacked LoRA shrink rows. */
typedef struct slx_splitk_in {
  const float* part;
  int splits;
  int bm;       /* token rows per piece (M rounded up to 16) */
  int n_main;
} slx_splitk_in;
/* Residual-stream LoRA add + RMSNorm: x[t, :] += delta (slx_lora_delta over the row, rounded
 * to the activation dtype and written back to x), then out = rmsnorm(x) (lora may be NULL). */
SLX_API int slx_rmsnorm_lora(int dtype, void* out, int ldo, void* x, int ldx, const void* w,
                int n_tok, int d, float eps, const slx_lora_delta* lora, void* stream);
/* The residual epilogue of a split-K projection fused in front: x[t, :] = round(x + sum of the
 * pieces) (what slx_gemm_bf16's residual epilogue would have stored), then the LoRA add (its v
 * taken from the pieces' columns >= n_main when lora->v is NULL) and the RMSNorm, as
 * slx_rmsnorm_lora.  d % 2048 == 0 (8-CTA cluster per token).  `pf` (may be NULL): L2 prefetch
 * of the next GEMM's weights, issued at kernel entry (before the PDL wait). */
SLX_API int slx_rmsnorm_fused(int dtype, void* out, int ldo, void* x, int ldx, const void* w,
                int n_tok, int d, float eps, const slx_splitk_in* sk, const slx_lora_delta* lora,
                const slx_l2_prefetch* pf, void* stream);
/* qkv [n_tok, (H + 2 Hkv) D]: rotate q,k in place (rotate-half, cos/sin tables fp32
 * [max_pos, D/2]) and write k, v at (tok_seq[t], tok_pos[t]) of the caches. */
SLX_API int slx_rope_kv_write(int dtype, void* qkv, int ld_qkv, int n_tok, int heads, int kv_heads,
                      int head_dim, const int32_t* tok_pos, const int32_t* tok_seq,
                      const float* cos_tab, const float* sin_tab, int max_pos,
                      void* k_cache, void* v_cache, int max_ctx, void* stream);
/* Causal attention of each token t over cache positions 0..tok_pos[t] of sequence tok_seq[t].
 * q read from qkv (after rope). out [n_tok, H*D]. */
SLX_API int slx_attention(int dtype, void* out, int ldo, const void* qkv, int ld_qkv, int n_tok,
                  int heads, int kv_heads, int head_dim, const int32_t* tok_pos,
                  const int32_t* tok_seq, const void* k_cache, const void* v_cache, int max_ctx,
                  void* stream);
/* Decode step fusion of slx_rope_kv_write + slx_attention when every token is the NEXT
 * position of its own sequence (tok_pos[t] = cached length): RoPE on q and the new key, k/v
 * appended to the pool, attention over cached positions [0, pos) + the new key.  `lora` (may be
 * NULL) fuses the q/k/v LoRA expand: the row values of q (head h), k and v (kv head) get the
 * slx_lora_delta of their qkv-row columns added before RoPE / the append (qkv is not
 * modified).  `pf` (may be NULL): L2 prefetch of the next kernel's first bytes.  `pool_seqs`:
 * sequence slots of the k/v caches ([pool_seqs][kv_heads][max_ctx][head_dim]).
 * bf16 MHA (head_dim 64/128) runs the persistent TMA-pipelined tensor-core kernel; fp32 parity
 * mode and GQA run one CTA per (token, head).  Preconditions: tok_pos[t] < max_ctx; KV rows
 * past tok_pos of a sequence are finite (whole 64-row boxes are multiplied by P = 0 there;
 * the model zero-fills its pool); adapter ranks are multiples of 8. */
SLX_API int slx_rope_attention_decode(int dtype, void* out, int ldo, const void* qkv,
                  int ld_qkv, int n_tok, int heads, int kv_heads, int head_dim,
                  const int32_t* tok_pos, const int32_t* tok_seq, const float* cos_tab,
                  const float* sin_tab, int max_pos, void* k_cache, void* v_cache, int max_ctx,
                  int pool_seqs, const slx_lora_delta* lora, const slx_l2_prefetch* pf,
                  void* stream);
/* Prefill attention (tcgen05 flash attention, head_dim 128, bf16): `tiles` is a device array of
 * n_tiles {int tok0, nq, seq, pos0} (nq <= slx_flash_prefill_tile_queries() queries of one
 * segment each, slx_flash_prefill_tile_bytes() per entry); query t of a tile attends cache
 * positions 0..pos0+t of its sequence (k/v already appended by slx_rope_kv_write, q rotated in
 * qkv [n_tok rows]).  `items` (device, n_items x {int tile_a, tile_b (-1: none), head, 0},
 * slx_flash_prefill_item_bytes() each) is the work list: a persistent CTA per SM runs items
 * c, c + #SMs, ...; pairing a segment's long and short tiles keeps the items' cost equal.  The
 * k/v caches are [pool_seqs][kv_heads][max_ctx][128]. */
SLX_API int slx_flash_prefill_tile_queries(void);   /* max queries per tile (nq) */
SLX_API size_t slx_flash_prefill_tile_bytes(void);
SLX_API size_t slx_flash_prefill_item_bytes(void);
SLX_API int slx_attention_prefill(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok,
                  int heads, int kv_heads, int head_dim, const void* tiles, const void* items,
                  int n_items, const void* k_cache, const void* v_cache, int max_ctx,
                  int pool_seqs, void* stream);
/* gu [n_tok, 2*ffn] in the blocked layout of SLX_EPI_SILU_MUL -> out [n_tok, ffn]. */
SLX_API int slx_silu_mul_blocked(int dtype, void* out, int ldo, const void* gu, int ld_gu, int n_tok,
                         int ffn, void* stream);
/* Row-wise argmax (lowest index on ties) of logits [n_rows, n_cols] (dtype) -> int32. */
SLX_API int slx_argmax(int dtype, int32_t* out, const void* logits, int ld, int n_rows, int n_cols,
               void* stream);

/* ------------------------------------------------------------------ P1: artifact pre-loader
 * Replaces the modelled load `usable_at_ms = now + load_from_container_ms | load_cold_ms`
 * of a PreloadPlan GPU placement (engine.py:1040-1053; ArtifactSpec core.py:56-78).
 */
SLX_API int slx_host_register(void* ptr, size_t bytes);
SLX_API int slx_host_unregister(void* ptr);
/* Chunked pinned-host -> device copy on `stream`; records `done_event` (cudaEvent_t or NULL). */
SLX_API int slx_preload_h2d(void* dst_dev, const void* src_pinned, size_t bytes, size_t chunk_bytes,
                    void* stream, void* done_event);
/* Chunked device -> pinned-host copy on `stream` (demotion of an evicted model to the
 * container tier); records `done_event` (cudaEvent_t or NULL).
 * Replaces the modelled demotion of apply_evictions: the GPU bytes leave at once and the
 * container copy is usable after size / demotion_gbps (offload.py:198-226, engine.py:76). */
SLX_API int slx_offload_d2h(void* dst_pinned, const void* src_dev, size_t bytes, size_t chunk_bytes,
                    void* stream, void* done_event);
/* NCCL communicator owned by the pre-loader (the only collective of the system). */
SLX_API int slx_nccl_unique_id_bytes(void);
SLX_API int slx_nccl_get_unique_id(void* out_id);
SLX_API int slx_nccl_comm_init(void** comm, int nranks, const void* id, int rank);
SLX_API int slx_nccl_comm_destroy(void* comm);
SLX_API int slx_bcast(void* buf, size_t bytes, int root, void* comm, void* stream);
/* Single host read, NVLink fan-out: the root copies chunk i host->device on copy_stream
 * while chunk i-1 is broadcast on comm_stream; non-roots only receive. */
SLX_API int slx_preload_bcast(void* dst_dev, const void* src_pinned, size_t bytes, size_t chunk_bytes,
                      int root, void* comm, void* copy_stream, void* comm_stream);

#ifdef __cplusplus
}
#endif
#endif /* SLORA_B200_H */
