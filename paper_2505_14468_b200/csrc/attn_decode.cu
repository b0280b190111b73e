// K4, decode step: persistent TMA-pipelined RoPE + KV append + attention (bf16, MHA).
//
// One work item = (token t, head h): the token is the NEXT position `pos` of its own sequence.
// Per layer of the 7B decode step the kernel streams 64 tok x 32 heads x 128 cached keys x
// (K + V) = 134 MB of KV cache, so it is HBM-bound and the design goal is to keep every SM's
// copy engine busy.  Two persistent CTAs per SM, each with
//   * one producer thread issuing 1-D bulk copies (TMA) of whole K and V blocks (one contiguous
//     run each in the [seq][head][max_ctx][D] pool) into a 2-stage smem ring, and of the item's
//     "header" (its q/k/v row slices, the cos/sin rows of pos, and the LoRA B rows and v vector
//     of the fused q/k/v expand) into a 2-slot ring — item 0's KV is requested before the PDL
//     wait, and after its last item the producer prefetches the next kernel's first bytes into L2;
//   * eight consumer warps: fused LoRA delta (bit-identical to slx_lora_expand), RoPE, append
//     k/v at pos, then online softmax over the ring's blocks.  Four threads share a key, each
//     reading its quarter of the K row in a per-key rotated chunk order, so the unpadded TMA
//     layout is bank-conflict free.
// The two CTAs of an SM overlap one item's consumer latency chain with the other's copies.
// ops.cu's one-CTA-per-(token, head) kernel stays for fp32 / GQA.
//
// Reference: the decode gap the simulator models as decode_ms_per_token x M
// (/root/reference/pkg/src/slorasim/engine.py:888,909).
#include "common.cuh"
#include "tc_ptx.cuh"

namespace slx {
namespace {

constexpr int AD_CONS = 256;               // consumer threads (8 warps)
constexpr int AD_THREADS = AD_CONS + 32;   // + producer warp
constexpr int AD_RMAX = 16;                // LoRA rank staged by TMA (larger ranks: global loads)
constexpr int AD_STAGES = 2;

template <int D> struct AdCfg { static constexpr int KB = 64; };     // keys per block
template <> struct AdCfg<64> { static constexpr int KB = 128; };

struct AdArgs {
  bf16* out;
  int ldo;
  const bf16* qkv;
  int ld;
  int n_tok, H;
  const int32_t* tok_pos;
  const int32_t* tok_seq;
  const float* cos_tab;
  const float* sin_tab;
  bf16* kc;
  bf16* vc;
  int max_ctx;
  float scale_log2;
  DeltaArgs lora;
  PfArgs pf;
};

// Header (one per item, 2-slot ring).
template <int D>
struct __align__(16) AdHeader {
  bf16 row[3][D];                // q (head h), k, v of the token
  bf16 b[3][D * AD_RMAX];        // B rows [D][rank] of the three column ranges (rank <= AD_RMAX)
  float v[3][AD_RMAX];           // LoRA shrink output of the three targets
  float cs[D];                   // cos[D/2], sin[D/2] of pos
  int ti[3];                     // target index per part (-1: none)
  int rank, staged, pos, seq, slot;
  float lscale;
  int pad;
};

template <int D>
constexpr size_t ad_stage_bytes() { return (size_t)2 * AdCfg<D>::KB * D * 2; }

template <int D>
constexpr size_t ad_smem() {
  return 1024 + (size_t)AD_STAGES * ad_stage_bytes<D>() + 2 * sizeof(AdHeader<D>) +
         (size_t)(D * 2 + 2 * D * 4 + AdCfg<D>::KB * 4 + 64 * 4 + 8 * D * 4 + 3 * D * 4) +
         (size_t)(2 * AD_STAGES + 4) * 8;
}

__device__ __forceinline__ void cons_sync() { tc::named_bar_sync(1, AD_CONS); }

template <int D>
__global__ void __launch_bounds__(AD_THREADS, 2) attn_decode_pipe_kernel(AdArgs a) {
  constexpr int HALF = D / 2;
  constexpr int KB = AdCfg<D>::KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  AdHeader<D>* hdr = reinterpret_cast<AdHeader<D>*>(ring + (size_t)AD_STAGES * ad_stage_bytes<D>());
  bf16* qb = reinterpret_cast<bf16*>(hdr + 2);           // [D] rotated q (bf16)
  float* kn = reinterpret_cast<float*>(qb + D);          // [D] new key
  float* vn = kn + D;                                    // [D] new value
  float* ps = vn + D;                                    // [KB] probabilities
  float* red = ps + KB;                                  // [64]
  float* pv = red + 64;                                  // [8 warps][D] P.V partials
  float* raw = pv + 8 * D;                               // [3][D]
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(raw + 3 * D);
  uint64_t* kv_empty = kv_full + AD_STAGES;
  uint64_t* h_full = kv_empty + AD_STAGES;
  uint64_t* h_empty = h_full + 2;

  const int tid = threadIdx.x;
  const int n_items = a.n_tok * a.H;
  if (tid == 0) {
    for (int s = 0; s < AD_STAGES; ++s) {
      tc::mbar_init(&kv_full[s], 1);
      tc::mbar_init(&kv_empty[s], AD_CONS / 32);   // one arrival per consumer warp
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&h_full[i], 1);
      tc::mbar_init(&h_empty[i], 1);
    }
    tc::fence_barrier_init();
  }
  __syncthreads();

  if (tid >= AD_CONS) {
    // ================================================================ producer (one thread)
    if (tid == AD_CONS) {
      const uint64_t pol_kv = tc::policy_evict_first();    // cache rows are read once
      const uint64_t pol_h = tc::policy_evict_normal();
      int kv_it = 0;
      auto issue_kv = [&](int seq, int h, int blk, int pos) {
        const int s = kv_it % AD_STAGES;
        tc::mbar_wait(&kv_empty[s], ((kv_it / AD_STAGES) & 1) ^ 1);
        const int nk = min(KB, pos - blk * KB);
        const uint32_t bytes = (uint32_t)nk * D * 2;
        const size_t off = (((size_t)seq * a.H + h) * a.max_ctx + (size_t)blk * KB) * D;
        uint8_t* st = ring + (size_t)s * ad_stage_bytes<D>();
        tc::mbar_arrive_expect_tx(&kv_full[s], 2 * bytes);
        tc::bulk_g2s(st, a.kc + off, bytes, &kv_full[s], pol_kv);
        tc::bulk_g2s(st + KB * D * 2, a.vc + off, bytes, &kv_full[s], pol_kv);
        ++kv_it;
      };
      // item 0's cached keys were written >= 2 launches back: start before the PDL wait
      int n_pre = 0;
      if ((int)blockIdx.x < n_items) {
        const int t0 = blockIdx.x / a.H, h0 = blockIdx.x % a.H;
        const int pos0 = a.tok_pos[t0], seq0 = a.tok_seq[t0];
        n_pre = min((pos0 + KB - 1) / KB, AD_STAGES);
        for (int b = 0; b < n_pre; ++b) issue_kv(seq0, h0, b, pos0);
      }
      pdl_wait();
      pdl_trigger();
      int j = 0;
      for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++j) {
        const int t = w / a.H, h = w % a.H;
        const int pos = a.tok_pos[t], seq = a.tok_seq[t];
        const int hb = j & 1;
        // LoRA: slot / rank / target of each part; B rows and v staged when rank <= AD_RMAX
        const DeltaTok dt = delta_tok(a.lora, t);
        int ti[3] = {-1, -1, -1};
        const bf16* bsrc[3] = {nullptr, nullptr, nullptr};
        const float* vsrc[3] = {nullptr, nullptr, nullptr};
        if (dt.slot >= 0 && dt.rank > 0) {
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            const int col = (p == 0 ? h : (p == 1 ? a.H + h : 2 * a.H + h)) * D;
#pragma unroll
            for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
              const int n = col - a.lora.y_col_off[i];
              if (ti[p] < 0 && i < a.lora.n_targets && n >= 0 && n + D <= a.lora.d_out[i]) {
                const bf16* B = reinterpret_cast<const bf16*>(a.lora.b_ptrs[i][dt.slot]);
                if (B != nullptr) {
                  ti[p] = i;
                  bsrc[p] = B + (size_t)n * dt.rank;
                  vsrc[p] = dt.vrow + a.lora.v_col_off[i] + dt.slot * a.lora.max_rank;
                }
              }
            }
          }
        }
        const int staged = dt.rank <= AD_RMAX ? 1 : 0;
        uint32_t bytes = 3 * D * 2 + D * 4;
        for (int p = 0; p < 3; ++p)
          if (ti[p] >= 0 && staged) bytes += (uint32_t)(D * dt.rank * 2 + dt.rank * 4);
        tc::mbar_wait(&h_empty[hb], ((j >> 1) & 1) ^ 1);
        AdHeader<D>* hd = hdr + hb;
        hd->ti[0] = ti[0]; hd->ti[1] = ti[1]; hd->ti[2] = ti[2];
        hd->rank = dt.rank; hd->staged = staged; hd->pos = pos; hd->seq = seq;
        hd->slot = dt.slot; hd->lscale = dt.scale;
        tc::mbar_arrive_expect_tx(&h_full[hb], bytes);   // releases the plain stores above too
        const bf16* rowp = a.qkv + (size_t)t * a.ld;
        tc::bulk_g2s(hd->row[0], rowp + (size_t)h * D, D * 2, &h_full[hb], pol_h);
        tc::bulk_g2s(hd->row[1], rowp + (size_t)(a.H + h) * D, D * 2, &h_full[hb], pol_h);
        tc::bulk_g2s(hd->row[2], rowp + (size_t)(2 * a.H + h) * D, D * 2, &h_full[hb], pol_h);
        tc::bulk_g2s(hd->cs, a.cos_tab + (size_t)pos * HALF, HALF * 4, &h_full[hb], pol_h);
        tc::bulk_g2s(hd->cs + HALF, a.sin_tab + (size_t)pos * HALF, HALF * 4, &h_full[hb], pol_h);
        if (staged) {
          for (int p = 0; p < 3; ++p) {
            if (ti[p] < 0) continue;
            tc::bulk_g2s(hd->b[p], bsrc[p], (uint32_t)(D * dt.rank * 2), &h_full[hb], pol_h);
            tc::bulk_g2s(hd->v[p], vsrc[p], (uint32_t)(dt.rank * 4), &h_full[hb], pol_h);
          }
        }
        for (int b = (j == 0 ? n_pre : 0); b < (pos + KB - 1) / KB; ++b) issue_kv(seq, h, b, pos);
      }
      l2_prefetch_part(a.pf, blockIdx.x, gridDim.x);   // next kernel's first bytes
    } else {
      pdl_wait();
      pdl_trigger();
    }
    __syncwarp();
    return;
  }

  // ================================================================== consumers (8 warps)
  // Each warp runs its own online softmax over its slice of every block (KB / 8 keys), so a
  // block needs no CTA-wide barrier: the warp releases the stage (kv_empty counts 8 arrivals)
  // and the 8 partial (max, sum, acc) states are merged once per item.
  pdl_wait();
  pdl_trigger();
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int KPW = KB / 8;            // keys per warp per block
  constexpr int LPK = 32 / KPW;          // lanes per key in the scores (4 | 2)
  constexpr int CPL = D / LPK / 8;       // 16-byte chunks per lane (4)
  constexpr int DPL = D / 32;            // output dims per lane in P.V (4 | 2)
  const int wkey = lane / LPK, lq = lane % LPK;
  int kv_it = 0, j = 0;
  for (int w = blockIdx.x; w < n_items; w += gridDim.x, ++j) {
    const int t = w / a.H, h = w % a.H;
    const int hb = j & 1;
    tc::mbar_wait(&h_full[hb], (j >> 1) & 1);
    const AdHeader<D>* hd = hdr + hb;
    const int pos = hd->pos, seq = hd->seq, rank = hd->rank;
    // ---- q/k/v of this head with the fused LoRA expand (sequential fmaf: as slx_lora_expand)
    for (int i = tid; i < 3 * D; i += AD_CONS) {
      const int p = i / D, e = i - p * D;
      float v = __bfloat162float(hd->row[p][e]);
      if (hd->ti[p] >= 0) {
        float acc = 0.f;
        if (hd->staged) {
          const bf16* br = hd->b[p] + (size_t)e * rank;
          const float* vv = hd->v[p];
          const float sc = hd->lscale;
          for (int jj = 0; jj < rank; jj += 8) {
            float bf[8];
            Vec8<bf16>::load(br + jj, bf);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = fmaf(vv[jj + u] * sc, bf[u], acc);
          }
        } else {
          const int col = (p == 0 ? h : (p == 1 ? a.H + h : 2 * a.H + h)) * D + e;
          acc = delta_col(a.lora, delta_tok(a.lora, t), col);
        }
        v = __bfloat162float(__float2bfloat16_rn(v + acc));
      }
      raw[i] = v;
    }
    cons_sync();
    // ---- RoPE (rotate-half), new key / value appended at pos
    {
      bf16* kdst = a.kc + (((size_t)seq * a.H + h) * a.max_ctx + pos) * D;
      bf16* vdst = a.vc + (((size_t)seq * a.H + h) * a.max_ctx + pos) * D;
      for (int i = tid; i < HALF; i += AD_CONS) {
        const float c = hd->cs[i], sn = hd->cs[HALF + i];
        const float q1 = raw[i], q2 = raw[i + HALF];
        qb[i] = __float2bfloat16_rn(q1 * c - q2 * sn);
        qb[i + HALF] = __float2bfloat16_rn(q2 * c + q1 * sn);
        const float k1 = raw[D + i], k2 = raw[D + i + HALF];
        const bf16 r1 = __float2bfloat16_rn(k1 * c - k2 * sn), r2 = __float2bfloat16_rn(k2 * c + k1 * sn);
        kn[i] = __bfloat162float(r1);
        kn[i + HALF] = __bfloat162float(r2);
        kdst[i] = r1;
        kdst[i + HALF] = r2;
      }
      for (int i = tid; i < D; i += AD_CONS) {
        const bf16 v = __float2bfloat16_rn(raw[2 * D + i]);
        vn[i] = __bfloat162float(v);
        vdst[i] = v;
      }
    }
    cons_sync();
    if (tid == 0) tc::mbar_arrive(&h_empty[hb]);   // header consumed (pos/seq/cs read above)
    // q slice of this lane (rotation applied per key below) and the new key's score
    float s_new;
    {
      float part = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e)
        part += __bfloat162float(qb[lane * DPL + e]) * kn[lane * DPL + e];
      s_new = warp_sum(part) * a.scale_log2;
    }
    // per-warp online softmax state; warp 0 owns the new key's term
    float m = warp == 0 ? s_new : -INFINITY, l = warp == 0 ? 1.f : 0.f;
    float acc[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] = warp == 0 ? vn[lane * DPL + e] : 0.f;
    const int nb = (pos + KB - 1) / KB;
    for (int b = 0; b < nb; ++b, ++kv_it) {
      const int s = kv_it % AD_STAGES;
      const int nk = min(KB, pos - b * KB);
      tc::mbar_wait(&kv_full[s], (kv_it / AD_STAGES) & 1);
      const bf16* Ks = reinterpret_cast<const bf16*>(ring + (size_t)s * ad_stage_bytes<D>());
      const bf16* Vs = Ks + KB * D;
      const int key = warp * KPW + wkey;
      // scores: LPK lanes per key, each a D/LPK slice read in a key-rotated chunk order
      float sc = 0.f;
      if (key < nk) {
        const bf16* kr = Ks + (size_t)key * D + lq * (D / LPK);
        const bf16* qh = qb + lq * (D / LPK);
        float s4[4] = {0.f, 0.f, 0.f, 0.f};   // independent chains (latency)
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int cc = (c + key) & (CPL - 1);
          float kf[8], qf[8];
          Vec8<bf16>::load(kr + cc * 8, kf);
          Vec8<bf16>::load(qh + cc * 8, qf);
#pragma unroll
          for (int e = 0; e < 8; ++e) s4[e & 3] = fmaf(qf[e], kf[e], s4[e & 3]);
        }
        sc = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      }
#pragma unroll
      for (int o = 1; o < LPK; o <<= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
      sc = key < nk ? sc * a.scale_log2 : -INFINITY;
      const float m_new = fmaxf(m, warp_max(sc));
      const float corr = m_new == -INFINITY ? 1.f : exp2f(m - m_new);
      const float p = key < nk ? exp2f(sc - m_new) : 0.f;
      l = l * corr + warp_sum(lq == 0 ? p : 0.f);
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[e] *= corr;
      // P.V over the warp's keys: lane owns dims [lane*DPL, lane*DPL + DPL)
#pragma unroll
      for (int kk = 0; kk < KPW; ++kk) {
        const float pk = __shfl_sync(0xffffffffu, p, kk * LPK);
        if (warp * KPW + kk < nk) {
          float vf[DPL];
          if (DPL == 4) {
            const uint2 u = *reinterpret_cast<const uint2*>(Vs + (size_t)(warp * KPW + kk) * D + lane * 4);
            const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
            const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
            vf[0] = f0.x; vf[1] = f0.y; vf[2 % DPL] = f1.x; vf[3 % DPL] = f1.y;
          } else {
            const float2 f0 = __bfloat1622float2(
                *reinterpret_cast<const __nv_bfloat162*>(Vs + (size_t)(warp * KPW + kk) * D + lane * 2));
            vf[0] = f0.x; vf[1 % DPL] = f0.y;
          }
#pragma unroll
          for (int e = 0; e < DPL; ++e) acc[e] = fmaf(pk, vf[e], acc[e]);
        }
      }
      m = m_new;
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&kv_empty[s]);   // this warp is done with the stage
    }
    // ---- merge the 8 warp states (fixed order) and write the head's output
    if (lane == 0) {
      red[warp] = m;
      red[8 + warp] = l;
    }
#pragma unroll
    for (int e = 0; e < DPL; ++e) pv[warp * D + lane * DPL + e] = acc[e];
    cons_sync();
    if (tid < D) {
      float mx = red[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) mx = fmaxf(mx, red[q]);
      float o = 0.f, ls = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float f = red[q] == -INFINITY ? 0.f : exp2f(red[q] - mx);
        o = fmaf(pv[q * D + tid], f, o);
        ls = fmaf(red[8 + q], f, ls);
      }
      a.out[(size_t)t * a.ldo + (size_t)h * D + tid] = __float2bfloat16_rn(o / ls);
    }
    cons_sync();   // red / pv / qb / kn / vn / raw reused by the next item
  }
}

}  // namespace

// Host launcher used by slx_rope_attention_decode_pf (ops.cu) for bf16 MHA, D in {64, 128}.
int attn_decode_pipe_launch(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok, int heads,
                            int head_dim, const int32_t* tok_pos, const int32_t* tok_seq,
                            const float* cos_tab, const float* sin_tab, void* k_cache,
                            void* v_cache, int max_ctx, float scale_log2, const DeltaArgs& lora,
                            const PfArgs& pf, cudaStream_t stream) {
  AdArgs a{};
  a.out = (bf16*)out; a.ldo = ldo; a.qkv = (const bf16*)qkv; a.ld = ld_qkv;
  a.n_tok = n_tok; a.H = heads; a.tok_pos = tok_pos; a.tok_seq = tok_seq;
  a.cos_tab = cos_tab; a.sin_tab = sin_tab; a.kc = (bf16*)k_cache; a.vc = (bf16*)v_cache;
  a.max_ctx = max_ctx; a.scale_log2 = scale_log2; a.lora = lora; a.pf = pf;
  const int items = n_tok * heads;
  const int grid = items < 2 * sm_count() ? items : 2 * sm_count();
  auto go = [&](auto kernel, size_t smem) -> int {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SLX_ERR_CUDA;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return launch_ex(kernel, dim3((unsigned)grid), dim3(AD_THREADS), smem, stream, 1u, a);
  };
  if (head_dim == 128) return go(attn_decode_pipe_kernel<128>, ad_smem<128>());
  if (head_dim == 64) return go(attn_decode_pipe_kernel<64>, ad_smem<64>());
  return SLX_ERR_UNSUPPORTED;
}

}  // namespace slx
