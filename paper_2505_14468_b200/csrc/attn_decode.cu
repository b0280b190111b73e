// K4, decode step: persistent TMA-pipelined RoPE + KV append + attention (bf16, MHA).
//
// One work item = (token t, head h): the token is the NEXT position `pos` of its own sequence.
// Per layer of the 7B decode step the kernel streams 64 tok x 32 heads x 128 cached keys x
// (K + V) = 134 MB of KV cache, so it is HBM-bound and the design goal is to keep every SM's
// copy engine busy (the copy ring alone streams at ~7 TB/s).  One persistent CTA per SM:
//   * a producer warp: its 32 lanes resolve the metadata of 32 items at a time (position,
//     sequence, adapter slot / rank / scale, LoRA B rows), then lane 0 issues 1-D bulk copies
//     (TMA) of whole K and V blocks (one contiguous run each in the [seq][head][max_ctx][D]
//     pool) into a 4-stage ring and of each item's header (q/k/v row slices, cos/sin of pos,
//     LoRA v) into a 4-slot ring; item 0's KV is requested before the PDL wait, and after the
//     last item the producer prefetches the next kernel's first bytes into L2;
//   * two consumer groups of 4 warps taking alternate items, so one group's latency chain
//     (fused LoRA delta — bit-identical to slx_lora_expand —, RoPE, k/v append, barriers)
//     overlaps the other's attention.  Within a group each warp runs its own online softmax
//     over its keys of every block (no CTA barrier per block) on the tensor cores (mma.sync
//     m16n8k16 from ldmatrix on the 128B-swizzled 2-D TMA tiles).
// Preconditions (slx_rope_attention_decode in slora_b200.h): adapter ranks are multiples of 8,
// and KV rows past `pos` of a sequence hold finite values (whole 64-row boxes are multiplied by
// P = 0 there; the model zero-fills its pool).
// ops.cu's one-CTA-per-(token, head) kernel stays for fp32 / GQA.
//
// Reference: the decode gap the simulator models as decode_ms_per_token x M
// (/root/reference/pkg/src/slorasim/engine.py:888,909).
#include "common.cuh"
#include "gemm_host.h"
#include "tc_ptx.cuh"

namespace slx {
namespace {

constexpr int AD_GW = 4;                      // warps per consumer group
constexpr int AD_GROUPS = 2;
constexpr int AD_GT = AD_GW * 32;             // threads per group
constexpr int AD_CONS = AD_GROUPS * AD_GT;    // consumer threads
constexpr int AD_THREADS = AD_CONS + 64;      // + header producer warp + KV producer warp
constexpr int AD_STAGES = 4;                  // KV ring
constexpr int AD_HSLOTS = 4;                  // header ring (2 per group)
constexpr int AD_VMAX = 64;                   // LoRA rank staged in the header (v)
constexpr int AD_BST = 16;                    // LoRA rank whose B rows are staged by TMA

struct AdArgs {
  CUtensorMap tmk, tmv;   // K / V pools as 2-D [rows, D] bf16, 64 x 64 boxes, 128B swizzle (MMA)
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
  unsigned long long* trace;   // slx_debug_gemm_trace timeline window (nullptr: off)
};

__device__ __forceinline__ unsigned long long ad_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

struct ItemMeta {
  const bf16* b[3];   // B rows of the three parts' column ranges
  int voff[3];        // v column of the slot block per part
  int ti[3];
  int t, h, pos, seq, slot, rank, valid;
  float scale;
};

// Header (one per item, 4-slot ring).
template <int D>
struct __align__(16) AdHeader {
  bf16 row[3][D];                // q (head h), k, v of the token
  float cs[D];                   // cos[D/2], sin[D/2] of pos
  float v[3][AD_VMAX];           // LoRA shrink output of the three targets (rank <= AD_VMAX)
  bf16 bs[3][D * AD_BST];        // B rows [D][rank] staged by TMA (rank <= AD_BST)
  const bf16* b[3];              // B rows [D][rank] of the three column ranges (nullptr: none)
  int bstaged;
  int kv_base;                   // ring counter of the item's first KV block
  int rank, pos, seq, slot;
  float lscale;
};

// Per-group scratch.
template <int D>
struct __align__(16) AdScratch {
  float raw[3][D];
  float kn[D], vn[D];
  float pv[AD_GW][D];
  float red[2 * AD_GW];
  bf16 qb[D];
};

// shared-memory atomics on a 32-bit word (explicit .shared state space: ATOMS, not generic ATOM)
__device__ __forceinline__ int smem_atom_add(uint32_t addr, int v) {
  int old;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void smem_atom_exch(uint32_t addr, int v) {
  int old;
  asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  (void)old;
}

__device__ __forceinline__ void ad_ldsm_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ad_ldsm_x4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ad_mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t ad_pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int D, int KB>
constexpr size_t ad_stage_bytes() { return (size_t)2 * KB * D * 2; }

template <int D, int KB>
constexpr size_t ad_smem() {
  return 1024 + (size_t)AD_STAGES * ad_stage_bytes<D, KB>() + AD_HSLOTS * sizeof(AdHeader<D>) +
         AD_GROUPS * sizeof(AdScratch<D>) + 32 * sizeof(ItemMeta) +
         (size_t)(2 * AD_STAGES + 2 * AD_HSLOTS) * 8 + 16;
}

__device__ __forceinline__ void group_sync(int g) { tc::named_bar_sync(1 + g, AD_GT); }

// Two packed bf16 (low half = element 0) -> fp32 pair: bf16 is the top half of an fp32.
__device__ __forceinline__ float2 bf2_unpack(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

template <int D, int KB>
__global__ void __launch_bounds__(AD_THREADS, 1) attn_decode_pipe_kernel(const __grid_constant__ AdArgs a) {
  constexpr int HALF = D / 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* ring = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  AdHeader<D>* hdr = reinterpret_cast<AdHeader<D>*>(ring + (size_t)AD_STAGES * ad_stage_bytes<D, KB>());
  AdScratch<D>* scr = reinterpret_cast<AdScratch<D>*>(hdr + AD_HSLOTS);
  ItemMeta* meta = reinterpret_cast<ItemMeta*>(scr + AD_GROUPS);
  uint64_t* kv_full = reinterpret_cast<uint64_t*>(meta + 32);
  uint64_t* kv_empty = kv_full + AD_STAGES;
  uint64_t* h_full = kv_empty + AD_STAGES;
  uint64_t* h_empty = h_full + AD_HSLOTS;
  // KV blocks issued so far (producer lane 0).  The two consumer groups work on different
  // items, so one can reach ring index i while the slot's previous use (i - STAGES, the other
  // group's block) is still pending; an mbarrier parity wait cannot tell phase i from phase
  // i - 2 STAGES.  A consumer therefore waits until block i has been issued (which implies
  // phase i - STAGES completed) before its parity wait.
  // The counter is written and polled with shared-memory atomics (release / acquire through the
  // CTA fences), so the handoff is a synchronised access for the memory model and racecheck.
  int* kv_issued = reinterpret_cast<int*>(h_empty + AD_HSLOTS);

  const int tid = threadIdx.x;
  const int n_items = a.n_tok * a.H;
  if (tid == 0 && a.trace) {
    a.trace[blockIdx.x * 16 + 0] = ad_timer();
    if (blockIdx.x == 0) a.trace[4095] = 5;
  }
  if (tid == 0) {
    for (int s = 0; s < AD_STAGES; ++s) {
      tc::mbar_init(&kv_full[s], 1);
      tc::mbar_init(&kv_empty[s], AD_GW);   // one arrival per warp of the consuming group
    }
    for (int i = 0; i < AD_HSLOTS; ++i) {
      tc::mbar_init(&h_full[i], 1);
      tc::mbar_init(&h_empty[i], 1);
    }
    *kv_issued = 0;
    tc::fence_barrier_init();
  }
  __syncthreads();

  if (tid >= AD_CONS) {
    // ============================================================ producer warps
    // Warp P (tid AD_CONS..+31) resolves the metadata of 32 items at a time (one per lane) and
    // its lane 0 issues the items' headers; warp K's lane 0 issues their KV blocks.  Separate
    // issuers: a header never waits behind ring space for an earlier item's KV (a consumer
    // group would otherwise wait on its next header while the ring drains).
    const bool kvw = tid >= AD_CONS + 32;
    const int pl = tid & 31;
    const uint64_t pol_kv = tc::policy_evict_first();    // cache rows are read once
    const uint64_t pol_h = tc::policy_evict_normal();
    const uint32_t kv_issued_s = tc::smem_u32(kv_issued);
    int kv_it = 0, j = 0, n_pre = 0, kv_base = 0;
    auto issue_kv = [&](int seq, int h, int blk) {
      const int s = kv_it % AD_STAGES;
      tc::mbar_wait(&kv_empty[s], ((kv_it / AD_STAGES) & 1) ^ 1);
      const size_t off = (((size_t)seq * a.H + h) * a.max_ctx + (size_t)blk * KB) * D;
      uint8_t* st = ring + (size_t)s * ad_stage_bytes<D, KB>();
      // whole 64-row boxes (rows past pos are masked), 128B-swizzled
      const int row = (int)(off / D);
      tc::mbar_arrive_expect_tx(&kv_full[s], 2 * KB * D * 2);
#pragma unroll
      for (int hf = 0; hf < D / 64; ++hf) {
        tc::tma_load_2d(st + hf * KB * 128, &a.tmk, &kv_full[s], hf * 64, row, pol_kv);
        tc::tma_load_2d(st + KB * D * 2 + hf * KB * 128, &a.tmv, &kv_full[s], hf * 64, row, pol_kv);
      }
      ++kv_it;
      __threadfence_block();            // the expect-tx above is ordered before the publication
      smem_atom_exch(kv_issued_s, kv_it);
    };
    if (kvw && pl == 0 && (int)blockIdx.x < n_items) {
      // item 0's cached keys were written >= 2 launches back: request them first, before the
      // metadata of the batch (slot / rank / B pointers: dependent loads) is resolved
      const int t0 = blockIdx.x / a.H, h0 = blockIdx.x % a.H;
      const int pos0 = a.tok_pos[t0], seq0 = a.tok_seq[t0];
      n_pre = min((pos0 + KB - 1) / KB, AD_STAGES);
      for (int b = 0; b < n_pre; ++b) issue_kv(seq0, h0, b);
    }
    for (int w0 = blockIdx.x; w0 < n_items; w0 += 32 * gridDim.x) {
      if (!kvw) {
        // ---- metadata of items w0 + i * gridDim.x, lane i (inputs / adapter pool: >= 2 launches old)
        const int w = w0 + pl * (int)gridDim.x;
        ItemMeta mt{};
        mt.valid = w < n_items;
        mt.ti[0] = mt.ti[1] = mt.ti[2] = -1;
        if (mt.valid) {
          const int t = w / a.H, h = w % a.H;
          mt.t = t; mt.h = h;
          mt.pos = a.tok_pos[t];
          mt.seq = a.tok_seq[t];
          const DeltaTok dt = delta_tok(a.lora, t);
          mt.slot = dt.slot; mt.rank = dt.rank; mt.scale = dt.scale;
          if (dt.slot >= 0 && dt.rank > 0) {
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              const int col = (p == 0 ? h : (p == 1 ? a.H + h : 2 * a.H + h)) * D;
#pragma unroll
              for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
                const int n = col - a.lora.y_col_off[i];
                if (mt.ti[p] < 0 && i < a.lora.n_targets && n >= 0 && n + D <= a.lora.d_out[i]) {
                  const bf16* B = reinterpret_cast<const bf16*>(a.lora.b_ptrs[i][dt.slot]);
                  if (B != nullptr) {
                    mt.ti[p] = i;
                    mt.b[p] = B + (size_t)n * dt.rank;
                    mt.voff[p] = a.lora.v_col_off[i] + dt.slot * a.lora.v_slot_stride;
                  }
                }
              }
            }
          }
        }
        meta[pl] = mt;
      }
      tc::named_bar_sync(3, 64);   // meta of this batch visible to both producer warps
      const int nloc = min(32, (n_items - w0 + (int)gridDim.x - 1) / (int)gridDim.x);
      if (w0 == (int)blockIdx.x) {
        pdl_wait();
        pdl_trigger();
        if (!kvw && pl == 0 && a.trace) a.trace[blockIdx.x * 16 + 2] = ad_timer();
      }
      if (pl == 0 && kvw) {
        for (int i = 0; i < nloc; ++i, ++j) {
          const ItemMeta& mt = meta[i];
          for (int b = (j == 0 ? n_pre : 0); b < (mt.pos + KB - 1) / KB; ++b) issue_kv(mt.seq, mt.h, b);
        }
      } else if (pl == 0) {
        for (int i = 0; i < nloc; ++i, ++j) {
          const ItemMeta& mt = meta[i];
          const int hs = j % AD_HSLOTS;
          const bool stage_v = mt.rank <= AD_VMAX;
          const bool stage_b = mt.rank <= AD_BST;
          uint32_t bytes = 3 * D * 2 + D * 4;
          for (int p = 0; p < 3; ++p)
            if (mt.ti[p] >= 0 && stage_v)
              bytes += (uint32_t)(mt.rank * 4) + (stage_b ? (uint32_t)(D * mt.rank * 2) : 0u);
          tc::mbar_wait(&h_empty[hs], ((j / AD_HSLOTS) & 1) ^ 1);
          AdHeader<D>* hd = hdr + hs;
          for (int p = 0; p < 3; ++p) hd->b[p] = (stage_v && mt.ti[p] >= 0) ? mt.b[p] : nullptr;
          hd->kv_base = kv_base;   // ring counter of the item's first KV block (same order)
          kv_base += (mt.pos + KB - 1) / KB;
          hd->bstaged = stage_b ? 1 : 0;
          hd->rank = mt.rank; hd->pos = mt.pos; hd->seq = mt.seq;
          hd->slot = mt.slot; hd->lscale = mt.scale;
          tc::mbar_arrive_expect_tx(&h_full[hs], bytes);   // releases the plain stores above too
          const bf16* rowp = a.qkv + (size_t)mt.t * a.ld;
          tc::bulk_g2s(hd->row[0], rowp + (size_t)mt.h * D, D * 2, &h_full[hs], pol_h);
          tc::bulk_g2s(hd->row[1], rowp + (size_t)(a.H + mt.h) * D, D * 2, &h_full[hs], pol_h);
          tc::bulk_g2s(hd->row[2], rowp + (size_t)(2 * a.H + mt.h) * D, D * 2, &h_full[hs], pol_h);
          tc::bulk_g2s(hd->cs, a.cos_tab + (size_t)mt.pos * HALF, HALF * 4, &h_full[hs], pol_h);
          tc::bulk_g2s(hd->cs + HALF, a.sin_tab + (size_t)mt.pos * HALF, HALF * 4, &h_full[hs], pol_h);
          if (stage_v) {
            const float* vrow = a.lora.v + (size_t)mt.t * a.lora.ldv;
            for (int p = 0; p < 3; ++p)
              if (mt.ti[p] >= 0) {
                tc::bulk_g2s(hd->v[p], vrow + mt.voff[p], (uint32_t)(mt.rank * 4), &h_full[hs], pol_h);
                if (stage_b)
                  tc::bulk_g2s(hd->bs[p], mt.b[p], (uint32_t)(D * mt.rank * 2), &h_full[hs], pol_h);
              }
          }
        }
      } else {
        j += nloc;
      }
      __syncwarp();
      tc::named_bar_sync(3, 64);   // both issuers done with this batch's meta
    }
    if ((int)blockIdx.x >= n_items) {   // no items for this CTA
      pdl_wait();
      pdl_trigger();
    }
    if (!kvw && pl == 0) l2_prefetch_part(a.pf, blockIdx.x, gridDim.x);
    __syncwarp();
    return;
  }

  // ================================================================== consumer groups
  // Group g takes items g, g + 2, ...  Each of its 4 warps runs its own online softmax over
  // KB / 4 keys of every block; the 4 (max, sum, acc) states are merged once per item.
  pdl_wait();
  pdl_trigger();
  const int g = tid / AD_GT, gt = tid % AD_GT;
  const int gw = gt >> 5, lane = tid & 31;
  const uint32_t kv_issued_c = tc::smem_u32(kv_issued);
  AdScratch<D>& sc_ = scr[g];
  constexpr int DPL = D / 32;            // dims per lane of the new key's score
  for (int j = g; (int)blockIdx.x + j * (int)gridDim.x < n_items; j += AD_GROUPS) {
    const int w = blockIdx.x + j * (int)gridDim.x;
    const int t = w / a.H, h = w % a.H;
    const int hs = j % AD_HSLOTS;
    tc::mbar_wait(&h_full[hs], (j / AD_HSLOTS) & 1);
    const AdHeader<D>* hd = hdr + hs;
    const int pos = hd->pos, seq = hd->seq, rank = hd->rank;
    const int nb = (pos + KB - 1) / KB;
    const int kv0 = hd->kv_base;
    // ---- q/k/v of this head with the fused LoRA expand (sequential fmaf: as slx_lora_expand)
    {
      // this thread's (up to NIT) outputs of the 3 x D q/k/v slice, their LoRA dot products
      // interleaved (independent accumulators; each one's fmaf order as slx_lora_expand)
      constexpr int NIT = (3 * D + AD_GT - 1) / AD_GT;
      float acc[NIT];
      const bf16* brs[NIT];
      const float* vvs[NIT];
      bool on[NIT];
      int jr = 0;   // rank of the fused deltas (shared by the item's parts)
#pragma unroll
      for (int k = 0; k < NIT; ++k) {
        const int i = gt + k * AD_GT;
        const int p = i / D, e = i - p * D;
        const bf16* bp = i < 3 * D ? hd->b[p] : nullptr;
        on[k] = bp != nullptr;
        brs[k] = on[k] ? (hd->bstaged ? hd->bs[p] : bp) + (size_t)e * rank : nullptr;
        vvs[k] = hd->v[i < 3 * D ? p : 0];   // scale * v formed in the loop (same rounding)
        acc[k] = 0.f;
        if (on[k]) jr = rank;
      }
      const float lsc = hd->lscale;
      for (int jj = 0; jj < jr; jj += 8) {
#pragma unroll
        for (int k = 0; k < NIT; ++k) {
          if (!on[k]) continue;
          const uint4 u = *reinterpret_cast<const uint4*>(brs[k] + jj);
          float4 v0 = *reinterpret_cast<const float4*>(vvs[k] + jj);
          float4 v1 = *reinterpret_cast<const float4*>(vvs[k] + jj + 4);
          v0.x = __fmul_rn(v0.x, lsc); v0.y = __fmul_rn(v0.y, lsc);
          v0.z = __fmul_rn(v0.z, lsc); v0.w = __fmul_rn(v0.w, lsc);
          v1.x = __fmul_rn(v1.x, lsc); v1.y = __fmul_rn(v1.y, lsc);
          v1.z = __fmul_rn(v1.z, lsc); v1.w = __fmul_rn(v1.w, lsc);
          const float2 b0 = bf2_unpack(u.x), b1 = bf2_unpack(u.y), b2 = bf2_unpack(u.z), b3 = bf2_unpack(u.w);
          float c = acc[k];
          c = fmaf(v0.x, b0.x, c); c = fmaf(v0.y, b0.y, c);
          c = fmaf(v0.z, b1.x, c); c = fmaf(v0.w, b1.y, c);
          c = fmaf(v1.x, b2.x, c); c = fmaf(v1.y, b2.y, c);
          c = fmaf(v1.z, b3.x, c); c = fmaf(v1.w, b3.y, c);
          acc[k] = c;
        }
      }
#pragma unroll
      for (int k = 0; k < NIT; ++k) {
        const int i = gt + k * AD_GT;
        if (i >= 3 * D) continue;
        const int p = i / D, e = i - p * D;
        float v = __bfloat162float(hd->row[p][e]);
        if (on[k]) {
          v = __bfloat162float(__float2bfloat16_rn(v + acc[k]));
        } else if (hd->slot >= 0 && rank > AD_VMAX) {
          const int col = (p == 0 ? h : (p == 1 ? a.H + h : 2 * a.H + h)) * D + e;
          v = __bfloat162float(__float2bfloat16_rn(v + delta_col(a.lora, delta_tok(a.lora, t), col)));
        }
        sc_.raw[p][e] = v;
      }
    }
    group_sync(g);
    // ---- RoPE (rotate-half), new key / value appended at pos
    {
      bf16* kdst = a.kc + (((size_t)seq * a.H + h) * a.max_ctx + pos) * D;
      bf16* vdst = a.vc + (((size_t)seq * a.H + h) * a.max_ctx + pos) * D;
      for (int i = gt; i < HALF; i += AD_GT) {
        const float c = hd->cs[i], sn = hd->cs[HALF + i];
        const float q1 = sc_.raw[0][i], q2 = sc_.raw[0][i + HALF];
        sc_.qb[i] = __float2bfloat16_rn(q1 * c - q2 * sn);
        sc_.qb[i + HALF] = __float2bfloat16_rn(q2 * c + q1 * sn);
        const float k1 = sc_.raw[1][i], k2 = sc_.raw[1][i + HALF];
        const bf16 r1 = __float2bfloat16_rn(k1 * c - k2 * sn), r2 = __float2bfloat16_rn(k2 * c + k1 * sn);
        sc_.kn[i] = __bfloat162float(r1);
        sc_.kn[i + HALF] = __bfloat162float(r2);
        kdst[i] = r1;
        kdst[i + HALF] = r2;
      }
      for (int i = gt; i < D; i += AD_GT) {
        const bf16 v = __float2bfloat16_rn(sc_.raw[2][i]);
        sc_.vn[i] = __bfloat162float(v);
        vdst[i] = v;
      }
    }
    group_sync(g);
    if (gt == 0) tc::mbar_arrive(&h_empty[hs]);   // header consumed
    // the new key's score (every warp, redundantly) and per-warp softmax state
    float s_new;
    {
      float part = 0.f;
#pragma unroll
      for (int e = 0; e < DPL; ++e)
        part += __bfloat162float(sc_.qb[lane * DPL + e]) * sc_.kn[lane * DPL + e];
      s_new = warp_sum(part) * a.scale_log2;
    }
    {
      // Tensor-core scores and P.V (mma.sync m16n8k16, fp32 accumulate) on the 128B-swizzled
      // TMA tiles: warp gw owns keys [16 gw, 16 gw + 16) of every block.  Scores: A = the 16 K
      // rows (ldmatrix), B = q replicated over the 8 columns, so lane (g, c) holds the scores
      // of keys g and g + 8.  P.V: A = P (bf16, rows replicated), B = V via ldmatrix.trans; lane
      // (g, c) accumulates dims 8 nt + 2c, +1 of every n-tile nt.
      const int gq = lane >> 2, cq = lane & 3;
      uint32_t qf[D / 16][2];
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        qf[ks][0] = *reinterpret_cast<const uint32_t*>(sc_.qb + ks * 16 + 2 * cq);
        qf[ks][1] = *reinterpret_cast<const uint32_t*>(sc_.qb + ks * 16 + 2 * cq + 8);
      }
      float o[D / 8][4];
#pragma unroll
      for (int nt = 0; nt < D / 8; ++nt) {
        const float v0 = gw == 0 ? sc_.vn[nt * 8 + 2 * cq] : 0.f;
        const float v1 = gw == 0 ? sc_.vn[nt * 8 + 2 * cq + 1] : 0.f;
        o[nt][0] = v0; o[nt][1] = v1; o[nt][2] = v0; o[nt][3] = v1;
      }
      float m = gw == 0 ? s_new : -INFINITY;
      float l = (gw == 0 && lane == 0) ? 1.f : 0.f;   // lane-partial sums, reduced at the end
      const int mi = lane >> 3;
      const int rr = gw * 16 + (mi & 1) * 8 + (lane & 7);   // this lane's ldmatrix row (key)
      const uint32_t rowoff = (uint32_t)rr * 128;
      const int sw = rr & 7;                                  // 128B swizzle of that row
      for (int b = 0; b < nb; ++b) {
        const int it = kv0 + b, s = it % AD_STAGES;
        const int nk = min(KB, pos - b * KB);
        if (lane == 0)
          while (smem_atom_add(kv_issued_c, 0) <= it) {}
        __syncwarp();
        tc::mbar_wait(&kv_full[s], (it / AD_STAGES) & 1);
        const uint32_t kbase = tc::smem_u32(ring + (size_t)s * ad_stage_bytes<D, KB>());
        const uint32_t vbase = kbase + KB * D * 2;
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const int ch = ((ks & 3) << 1) + (mi >> 1);
          uint32_t af[4];
          ad_ldsm_x4(af, kbase + (uint32_t)((ks >> 2) * KB * 128) + rowoff + (uint32_t)((ch ^ sw) << 4));
          ad_mma16816((ks & 1) ? sb : sa, af, qf[ks][0], qf[ks][1]);
        }
        float s0 = (sa[0] + sb[0]) * a.scale_log2;
        float s1 = (sa[2] + sb[2]) * a.scale_log2;
        if (gw * 16 + gq >= nk) s0 = -INFINITY;
        if (gw * 16 + gq + 8 >= nk) s1 = -INFINITY;
        float mx = fmaxf(s0, s1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float m_new = fmaxf(m, mx);
        const float corr = m_new == -INFINITY ? 1.f : exp2f(m - m_new);
        const float p0 = s0 == -INFINITY ? 0.f : exp2f(s0 - m_new);
        const float p1 = s1 == -INFINITY ? 0.f : exp2f(s1 - m_new);
        l = l * corr + (cq == 0 ? p0 + p1 : 0.f);
        m = m_new;
        const float pa = __shfl_sync(0xffffffffu, p0, 8 * cq);
        const float pb = __shfl_sync(0xffffffffu, p0, 8 * cq + 4);
        const float pc = __shfl_sync(0xffffffffu, p1, 8 * cq);
        const float pd = __shfl_sync(0xffffffffu, p1, 8 * cq + 4);
        uint32_t pf[4];
        pf[0] = ad_pack_bf16(pa, pb);
        pf[1] = pf[0];
        pf[2] = ad_pack_bf16(pc, pd);
        pf[3] = pf[2];
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
          o[nt][0] *= corr; o[nt][1] *= corr; o[nt][2] *= corr; o[nt][3] *= corr;
        }
#pragma unroll
        for (int j = 0; j < D / 16; ++j) {
          const int ch = ((j & 3) << 1) + (mi >> 1);
          uint32_t bf[4];
          ad_ldsm_x4_t(bf, vbase + (uint32_t)((j >> 2) * KB * 128) + rowoff + (uint32_t)((ch ^ sw) << 4));
          ad_mma16816(o[2 * j], pf, bf[0], bf[1]);
          ad_mma16816(o[2 * j + 1], pf, bf[2], bf[3]);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&kv_empty[s]);   // this warp is done with the stage
      }
      l = warp_sum(l);
      if (lane == 0) {
        sc_.red[gw] = m;
        sc_.red[AD_GW + gw] = l;
      }
      if (gq == 0) {
#pragma unroll
        for (int nt = 0; nt < D / 8; ++nt) {
          sc_.pv[gw][nt * 8 + 2 * cq] = o[nt][0];
          sc_.pv[gw][nt * 8 + 2 * cq + 1] = o[nt][1];
        }
      }
    }
    group_sync(g);
    if (gt < D) {
      float mx = sc_.red[0];
#pragma unroll
      for (int q = 1; q < AD_GW; ++q) mx = fmaxf(mx, sc_.red[q]);
      float o = 0.f, ls = 0.f;
#pragma unroll
      for (int q = 0; q < AD_GW; ++q) {
        const float f = sc_.red[q] == -INFINITY ? 0.f : exp2f(sc_.red[q] - mx);
        o = fmaf(sc_.pv[q][gt], f, o);
        ls = fmaf(sc_.red[AD_GW + q], f, ls);
      }
      a.out[(size_t)t * a.ldo + (size_t)h * D + gt] = __float2bfloat16_rn(o / ls);
    }
    group_sync(g);   // scratch reused by the group's next item
  }
  if (gt == 0 && a.trace) a.trace[blockIdx.x * 16 + 7 + g] = ad_timer();
}

}  // namespace

// Host launcher used by slx_rope_attention_decode (ops.cu) for bf16 MHA, D in {64, 128}.
int attn_decode_pipe_launch(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok, int heads,
                            int head_dim, const int32_t* tok_pos, const int32_t* tok_seq,
                            const float* cos_tab, const float* sin_tab, void* k_cache,
                            void* v_cache, int max_ctx, long long n_pool_rows, float scale_log2,
                            const DeltaArgs& lora,
                            const PfArgs& pf, cudaStream_t stream) {
  AdArgs a{};
  a.out = (bf16*)out; a.ldo = ldo; a.qkv = (const bf16*)qkv; a.ld = ld_qkv;
  a.n_tok = n_tok; a.H = heads; a.tok_pos = tok_pos; a.tok_seq = tok_seq;
  a.cos_tab = cos_tab; a.sin_tab = sin_tab; a.kc = (bf16*)k_cache; a.vc = (bf16*)v_cache;
  a.max_ctx = max_ctx; a.scale_log2 = scale_log2; a.lora = lora; a.pf = pf;
  a.trace = next_trace_window(5);
  const int items = n_tok * heads;
  const int grid = items < sm_count() ? items : sm_count();
  auto go = [&](auto kernel, size_t smem) -> int {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SLX_ERR_CUDA;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return launch_ex(kernel, dim3((unsigned)grid), dim3(AD_THREADS), smem, stream, 1u, a);
  };
  const int rows = (int)n_pool_rows;
  if ((head_dim != 128 && head_dim != 64) || n_pool_rows <= 0 || n_pool_rows >= (1LL << 31))
    return SLX_ERR_UNSUPPORTED;
  if (!make_tmap(&a.tmk, k_cache, rows, head_dim, head_dim, 64) ||
      !make_tmap(&a.tmv, v_cache, rows, head_dim, head_dim, 64))
    return SLX_ERR_CUDA;
  if (head_dim == 128) return go(attn_decode_pipe_kernel<128, 64>, ad_smem<128, 64>());
  return go(attn_decode_pipe_kernel<64, 64>, ad_smem<64, 64>());
}

}  // namespace slx
