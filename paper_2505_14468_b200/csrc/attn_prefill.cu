// Prefill attention on the tensor cores: causal flash-attention forward over the KV pool.
//
// CTA = (64-query tile of one prefill segment, head); 4 warps x 16 query rows.  Key/value
// blocks of 64 rows are streamed from the pool ([seq][kv_head][pos][128], written by
// slx_rope_kv_write) into shared memory with cp.async (K double buffered, V single: 68 KB,
// so three CTAs — 12 warps — share an SM; measured 68 -> 64.5 ms on config 3); S = Q K^T and
// O += P V use mma.sync m16n8k16 (bf16 in, fp32 accumulate) with ldmatrix fragments, and the
// softmax is the online exp2 formulation with rows owned by quads of a warp.  Query t of a
// segment starting at cache position p0 attends positions 0..p0+t (prefix + causal).
// (The decode step uses rope_attn_decode_kernel; this kernel serves the mixed prefill batch.)
#include "common.cuh"

namespace slx {

constexpr int FA_BQ = 64, FA_BK = 64, FA_D = 128, FA_THREADS = 128;   // 4 warps x 16 query rows (128-query tiles of 8 warps measured slower)
constexpr int FA_LD = FA_D + 8;   // padded smem row (bf16 elements): conflict-free ldmatrix

struct FaTile {
  int tok0;    // first query token (row of qkv / out)
  int nq;      // queries in this tile (<= FA_BQ)
  int seq;     // KV pool sequence slot
  int pos0;    // cache position of the first query
};

__device__ __forceinline__ uint32_t s_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* s, const void* g, bool pred) {
  const int n = pred ? 16 : 0;   // zero-fill rows past the end
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s_u32(s)), "l"(g), "r"(n)
               : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d,
                                        const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(s_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d,
                                          const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(s_u32(p)));
}
__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__global__ void __launch_bounds__(FA_THREADS, 3)
flash_prefill_kernel(bf16* __restrict__ out, int ldo, const bf16* __restrict__ qkv, int ld, int H,
                     int Hkv, const FaTile* __restrict__ tiles, const bf16* __restrict__ kc,
                     const bf16* __restrict__ vc, int max_ctx, float scale_log2) {
  extern __shared__ __align__(128) uint8_t fsm_raw[];
  bf16* Qs = reinterpret_cast<bf16*>(fsm_raw);             // [FA_BQ][LD]
  bf16* Ks = Qs + FA_BQ * FA_LD;                            // [2][64][LD] (double buffered)
  bf16* Vs = Ks + 2 * FA_BK * FA_LD;                        // [64][LD] (single: 68 KB smem,
                                                            // 3 CTAs per SM)
  pdl_wait();
  pdl_trigger();
  // grid (heads, tiles): all heads of a tile launch together, tiles in table order (the host
  // sorts them longest first, so the last wave holds the short tiles)
  const FaTile tile = tiles[blockIdx.y];
  const int h = blockIdx.x, hk = h / (H / Hkv);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bf16* kbase = kc + ((size_t)tile.seq * Hkv + hk) * max_ctx * FA_D;
  const bf16* vbase = vc + ((size_t)tile.seq * Hkv + hk) * max_ctx * FA_D;
  const int n_keys = tile.pos0 + tile.nq;               // keys visible to the last query
  const int nblk = (n_keys + FA_BK - 1) / FA_BK;

  // Q tile
  for (int e = tid; e < FA_BQ * (FA_D / 8); e += FA_THREADS) {
    const int r = e / (FA_D / 8), c = e % (FA_D / 8);
    cp16(Qs + r * FA_LD + c * 8, qkv + (size_t)(tile.tok0 + min(r, tile.nq - 1)) * ld + h * FA_D + c * 8,
         r < tile.nq);
  }
  auto stage_k = [&](int b, int buf) {
    const int k0 = b * FA_BK;
    for (int e = tid; e < FA_BK * (FA_D / 8); e += FA_THREADS) {
      const int r = e / (FA_D / 8), c = e % (FA_D / 8);
      const size_t off = (size_t)min(k0 + r, n_keys - 1) * FA_D + c * 8;
      cp16(Ks + (buf * FA_BK + r) * FA_LD + c * 8, kbase + off, k0 + r < n_keys);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto stage_v = [&](int b) {
    const int k0 = b * FA_BK;
    for (int e = tid; e < FA_BK * (FA_D / 8); e += FA_THREADS) {
      const int r = e / (FA_D / 8), c = e % (FA_D / 8);
      const size_t off = (size_t)min(k0 + r, n_keys - 1) * FA_D + c * 8;
      cp16(Vs + r * FA_LD + c * 8, vbase + off, k0 + r < n_keys);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  stage_k(0, 0);
  stage_v(0);

  // per thread: 2 query rows (lane/4 and lane/4+8 of the warp's 16), quad-shared
  const int qr0 = warp * 16 + (lane >> 2);
  const int q_pos0 = tile.pos0 + qr0, q_pos1 = q_pos0 + 8;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[FA_D / 8][4];
#pragma unroll
  for (int j = 0; j < FA_D / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  uint32_t qf[FA_D / 16][4];

  for (int b = 0; b < nblk; ++b) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");   // K(b), V(b) (and Q) landed
    __syncthreads();
    if (b + 1 < nblk) stage_k(b + 1, (b + 1) & 1);         // overlaps S = Q K^T and softmax
    if (b == 0) {
#pragma unroll
      for (int kk = 0; kk < FA_D / 16; ++kk) {
        const bf16* p = Qs + (warp * 16 + (lane & 15)) * FA_LD + kk * 16 + (lane >> 4) * 8;
        ldsm_x4(qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3], p);
      }
    }
    const bf16* K = Ks + (b & 1) * FA_BK * FA_LD;
    const bf16* V = Vs;
    // S = Q K^T for this warp's 16 rows x 64 keys
    float sacc[FA_BK / 8][4];
#pragma unroll
    for (int j = 0; j < FA_BK / 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < FA_D / 16; ++kk) {
#pragma unroll
      for (int j = 0; j < FA_BK / 16; ++j) {   // two 8-key n-tiles per ldmatrix.x4
        uint32_t b0, b1, b2, b3;
        const bf16* p = K + (j * 16 + (lane & 7) + ((lane >> 4) << 3)) * FA_LD + kk * 16 +
                        ((lane >> 3) & 1) * 8;
        ldsm_x4(b0, b1, b2, b3, p);
        mma16816(sacc[2 * j], qf[kk], b0, b1);
        mma16816(sacc[2 * j + 1], qf[kk], b2, b3);
      }
    }
    // scale, causal mask, online softmax (rows q_pos0, q_pos1)
    const int k0 = b * FA_BK;
    float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < FA_BK / 8; ++j) {
      const int kc0 = k0 + j * 8 + (lane & 3) * 2;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kpos = kc0 + e;
        float s0 = sacc[j][e] * scale_log2, s1 = sacc[j][2 + e] * scale_log2;
        if (kpos > q_pos0 || kpos >= n_keys) s0 = -INFINITY;
        if (kpos > q_pos1 || kpos >= n_keys) s1 = -INFINITY;
        sacc[j][e] = s0;
        sacc[j][2 + e] = s1;
        bm0 = fmaxf(bm0, s0);
        bm1 = fmaxf(bm1, s1);
      }
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, off));
      bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, off));
    }
    const float mn0 = fmaxf(m0, bm0), mn1 = fmaxf(m1, bm1);
    // fully masked rows so far keep -inf max: use 0 as the reference to avoid inf - inf
    const float ref0 = mn0 == -INFINITY ? 0.f : mn0, ref1 = mn1 == -INFINITY ? 0.f : mn1;
    const float c0 = exp2f(m0 - ref0), c1 = exp2f(m1 - ref1);
    float rs0 = 0.f, rs1 = 0.f;
    uint32_t pf[FA_BK / 16][4];
#pragma unroll
    for (int j = 0; j < FA_BK / 8; ++j) {
      const float p00 = exp2f(sacc[j][0] - ref0), p01 = exp2f(sacc[j][1] - ref0);
      const float p10 = exp2f(sacc[j][2] - ref1), p11 = exp2f(sacc[j][3] - ref1);
      rs0 += p00 + p01;
      rs1 += p10 + p11;
      // accumulator layout of an m16n8 tile == A-fragment layout of the k16 step j/2
      pf[j >> 1][(j & 1) * 2 + 0] = pack_bf16(p00, p01);
      pf[j >> 1][(j & 1) * 2 + 1] = pack_bf16(p10, p11);
    }
#pragma unroll
    for (int off = 1; off <= 2; off <<= 1) {
      rs0 += __shfl_xor_sync(0xffffffffu, rs0, off);
      rs1 += __shfl_xor_sync(0xffffffffu, rs1, off);
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
    m0 = mn0;
    m1 = mn1;
#pragma unroll
    for (int j = 0; j < FA_D / 8; ++j) {
      o[j][0] *= c0; o[j][1] *= c0;
      o[j][2] *= c1; o[j][3] *= c1;
    }
    // O += P V : A = P (16 x 64 keys), B = V (keys x D) via ldmatrix.trans
#pragma unroll
    for (int kk = 0; kk < FA_BK / 16; ++kk) {
      uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int j = 0; j < FA_D / 16; ++j) {    // two 8-dim n-tiles per ldmatrix.x4.trans
        uint32_t b0, b1, b2, b3;
        const bf16* p = V + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * FA_LD + j * 16 +
                        (lane >> 4) * 8;
        ldsm_x4_t(b0, b1, b2, b3, p);
        mma16816(o[2 * j], a, b0, b1);
        mma16816(o[2 * j + 1], a, b2, b3);
      }
    }
    __syncthreads();   // every warp is done with V(b) (and K(b), refilled next iteration)
    if (b + 1 < nblk) stage_v(b + 1);
  }
  // normalise and store
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int r0 = qr0, r1 = qr0 + 8;
#pragma unroll
  for (int j = 0; j < FA_D / 8; ++j) {
    const int d = j * 8 + (lane & 3) * 2;
    if (r0 < tile.nq)
      *reinterpret_cast<uint32_t*>(out + (size_t)(tile.tok0 + r0) * ldo + h * FA_D + d) =
          pack_bf16(o[j][0] * inv0, o[j][1] * inv0);
    if (r1 < tile.nq)
      *reinterpret_cast<uint32_t*>(out + (size_t)(tile.tok0 + r1) * ldo + h * FA_D + d) =
          pack_bf16(o[j][2] * inv1, o[j][3] * inv1);
  }
}

}  // namespace slx

using namespace slx;

extern "C" size_t slx_flash_prefill_tile_bytes(void) { return sizeof(FaTile); }
extern "C" int slx_flash_prefill_tile_queries(void) { return FA_BQ; }

extern "C" int slx_attention_prefill(void* out, int ldo, const void* qkv, int ld_qkv, int heads,
                                     int kv_heads, int head_dim, const void* tiles, int n_tiles,
                                     const void* k_cache, const void* v_cache, int max_ctx,
                                     void* stream) {
  SLX_CHECK_ARG(out && qkv && tiles && k_cache && v_cache && heads > 0 && kv_heads > 0 &&
                heads % kv_heads == 0 && n_tiles >= 0 && max_ctx > 0 &&
                ld_qkv >= (heads + 2 * kv_heads) * head_dim && ldo >= heads * head_dim &&
                ld_qkv % 8 == 0 && ldo % 2 == 0);
  if (head_dim != FA_D) return SLX_ERR_UNSUPPORTED;
  SLX_CHECK_ALIGN(qkv, 16);
  SLX_CHECK_ALIGN(k_cache, 16);
  SLX_CHECK_ALIGN(v_cache, 16);
  if (n_tiles == 0) return SLX_OK;
  const size_t smem = (size_t)(FA_BQ + 3 * FA_BK) * FA_LD * sizeof(bf16);
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(flash_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return SLX_ERR_CUDA;
    configured = true;
  }
  const float scale = 1.4426950408889634f / sqrtf((float)head_dim);
  return launch_ex(flash_prefill_kernel, dim3((unsigned)heads, (unsigned)n_tiles),
                   dim3(FA_THREADS), smem, (cudaStream_t)stream, 1u, (bf16*)out, ldo,
                   (const bf16*)qkv, ld_qkv, heads, kv_heads, (const FaTile*)tiles,
                   (const bf16*)k_cache, (const bf16*)v_cache, max_ctx, scale);
}
