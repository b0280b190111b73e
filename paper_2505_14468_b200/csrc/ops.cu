// K4 supporting ops of the multi-LoRA Llama forward: embedding, RMSNorm, RoPE + KV write,
// causal attention over the KV pool, blocked SiLU*mul, argmax, and the fp32-parity SIMT GEMM.
// All templated on the activation type (bf16 throughput mode / fp32 parity mode); weights
// are always bf16 and accumulation is always fp32.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "gemm_host.h"

namespace slx {

int attn_decode_pipe_launch(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok, int heads,
                            int head_dim, const int32_t* tok_pos, const int32_t* tok_seq,
                            const float* cos_tab, const float* sin_tab, void* k_cache,
                            void* v_cache, int max_ctx, long long n_pool_rows, float scale_log2,
                            const DeltaArgs& lora,
                            const PfArgs& pf, cudaStream_t stream);   // attn_decode.cu

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embedding_kernel(T* __restrict__ out, const bf16* __restrict__ table,
                                 const int32_t* __restrict__ tokens, int d, int vocab) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  int tok = tokens[t];
  tok = tok < 0 ? 0 : (tok >= vocab ? vocab - 1 : tok);
  const bf16* src = table + (size_t)tok * d;
  T* dst = out + (size_t)t * d;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8];
    Vec8<bf16>::load(src + i, f);
    Vec8<T>::store(dst + i, f);
  }
}

// ------------------------------------------------------------------ RMSNorm
// out = x * (1 / sqrt(mean(x^2) + eps)) * w     (oracle/llama_lora.py::rmsnorm)
template <typename T>
__global__ void rmsnorm_kernel(T* __restrict__ out, int ldo, const T* __restrict__ x, int ldx,
                               const bf16* __restrict__ w, int d, float eps) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const T* xr = x + (size_t)t * ldx;
  float ss = 0.f;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8];
    Vec8<T>::load(xr + i, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  T* orow = out + (size_t)t * ldo;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8], g[8];
    Vec8<T>::load(xr + i, f);
    Vec8<bf16>::load(w + i, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (f[j] * inv) * g[j];
    Vec8<T>::store(orow + i, f);
  }
}

// Four 8-column chunks per thread (d / 32 threads: 160 for d = 5120), the row kept in
// registers between the sum of squares and the scaling: one read of x, one write of out, and
// small CTAs so an SM keeps ~12 rows (~120 KB) of loads in flight — the prefill norms are
// HBM-bound (16384 x 5120 bf16 rows in and out per config-3 layer).
constexpr int RN_CH = 4;
template <typename T>
__global__ void __launch_bounds__(256) rmsnorm_row_kernel(T* __restrict__ out, int ldo,
                                                          const T* __restrict__ x, int ldx,
                                                          const bf16* __restrict__ w, int d,
                                                          float eps) {
  __shared__ float red[33];
  const int t = blockIdx.x;
  const int nt = blockDim.x;
  pdl_wait();
  pdl_trigger();
  float f[RN_CH][8];
#pragma unroll
  for (int c = 0; c < RN_CH; ++c) Vec8<T>::load(x + (size_t)t * ldx + (c * nt + threadIdx.x) * 8, f[c]);
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < RN_CH; ++c)
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[c][j] * f[c][j];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (nt >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[32] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[32] / (float)d + eps);
#pragma unroll
  for (int c = 0; c < RN_CH; ++c) {
    const int i0 = (c * nt + threadIdx.x) * 8;
    float g[8];
    Vec8<bf16>::load(w + i0, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[c][j] = (f[c][j] * inv) * g[j];
    Vec8<T>::store(out + (size_t)t * ldo + i0, f[c]);
  }
}

// x[t] += LoRA delta (rounded to T, written back), then out = rmsnorm(x).  The o-projection
// expand of the decode step fused into the post-attention norm (slx_rmsnorm_lora).
template <typename T>
__global__ void __launch_bounds__(512) rmsnorm_lora_kernel(T* __restrict__ out, int ldo, T* __restrict__ x, int ldx,
                                    const bf16* __restrict__ w, int d, float eps, DeltaArgs lora) {
  const int t = blockIdx.x;   // the slot table / adapter pool are >= 2 launches old (PDL)
  T* xr = x + (size_t)t * ldx;
  const DeltaTok dt = delta_tok(lora, t);
  float ss = 0.f;
  const int i0 = threadIdx.x * 8;
  if (d == (int)blockDim.x * 8 && dt.slot >= 0 && dt.rank <= 16) {
    // one 8-column group per thread: B rows fetched in registers before the PDL wait
    DeltaRow<2> dr[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) delta_prefetch<2>(lora, dt, i0 + j, dr[j]);
    pdl_wait();
    pdl_trigger();
    __shared__ float vs[DELTA_VS];
    float f[8];
    Vec8<T>::load(xr + i0, f);
    delta_stage_v(lora, dt, vs, threadIdx.x, blockDim.x);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_finish<2>(dt, dr[j], vs)));
    Vec8<T>::store(xr + i0, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  } else {
    pdl_wait();
    pdl_trigger();
    for (int i = i0; i < d; i += blockDim.x * 8) {
      float f[8];
      Vec8<T>::load(xr + i, f);
      if (dt.slot >= 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_col(lora, dt, i + j)));
        Vec8<T>::store(xr + i, f);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
    }
  }
  __shared__ float red[32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();   // also orders this CTA's x write-back before the re-read below
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  T* orow = out + (size_t)t * ldo;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8], g[8];
    Vec8<T>::load(xr + i, f);
    Vec8<bf16>::load(w + i, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (f[j] * inv) * g[j];
    Vec8<T>::store(orow + i, f);
  }
}

constexpr int AD_LORA_FAST_RANK = 16;
// Cluster variant: one 8-CTA cluster per token, each CTA d/8 columns (8 per thread), the
// sum of squares reduced over the cluster through DSMEM in a fixed rank order.  Spreads the
// o-projection B rows (d x rank per token) over 8 SMs instead of one.
constexpr int RNL_CL = 8;
template <typename T>
__global__ void __launch_bounds__(128) rmsnorm_lora_cluster_kernel(T* __restrict__ out, int ldo,
                                                                   T* __restrict__ x, int ldx,
                                                                   const bf16* __restrict__ w,
                                                                   int d, float eps, DeltaArgs lora,
                                                                   SplitArgs sk, PfArgs pf,
                                                                   unsigned long long* trace) {
  __shared__ float vs[DELTA_VS];
  __shared__ float red[8];
  auto stamp = [&](int i) {
    if (trace && threadIdx.x == 0 && blockIdx.x % RNL_CL == 0) {   // cluster rank 0 per token
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)::"memory");
      trace[(blockIdx.x / RNL_CL % 256) * 16 + i] = tt;
      if (blockIdx.x == 0 && i == 0) trace[4095] = 6;
    }
  };
  stamp(0);
  // the next GEMM's weights beyond what the previous kernel prefetched (constant: before the
  // wait), so HBM keeps streaming while this latency-bound kernel runs
  if (threadIdx.x == 0) l2_prefetch_part(pf, blockIdx.x, gridDim.x);
  const int t = blockIdx.x / RNL_CL, cr = blockIdx.x % RNL_CL;
  const int i0 = cr * (d / RNL_CL) + threadIdx.x * 8;
  T* xr = x + (size_t)t * ldx;
  const DeltaTok dt = delta_tok(lora, t);   // slot tables / adapter pool: >= 2 launches old
  const bool fast = dt.slot >= 0 && dt.rank <= 16;
  DeltaRow<2> dr[8];
  if (fast) {
#pragma unroll
    for (int j = 0; j < 8; ++j) delta_prefetch<2>(lora, dt, i0 + j, dr[j]);
  }
  pdl_wait();
  pdl_trigger();
  stamp(2);
  float f[8];
  Vec8<T>::load(xr + i0, f);
  if (sk.part != nullptr) {   // the projection's residual epilogue: round(x + sum of pieces)
    float ps[8];
    split_sum8(sk, t, i0, ps);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + ps[j]));
    if (dt.slot < 0) Vec8<T>::store(xr + i0, f);
  }
  if (fast) {
    if (lora.v == nullptr) {   // LoRA v from the pieces' stacked columns
      for (int e = threadIdx.x; e < lora.n_targets * 64; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        int off = 0;
#pragma unroll
        for (int q = 0; q < SLX_LORA_MAX_TARGETS; ++q)
          if (q == i) off = lora.v_col_off[q];
        if (j < dt.rank) vs[e] = split_sum1(sk, t, sk.n_main + off + dt.slot * lora.v_slot_stride + j) * dt.scale;
      }
    } else {
      delta_stage_v(lora, dt, vs, threadIdx.x, blockDim.x);
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_finish<2>(dt, dr[j], vs)));
    Vec8<T>::store(xr + i0, f);
  } else if (dt.slot >= 0 && lora.v != nullptr) {
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_col(lora, dt, i0 + j)));
    Vec8<T>::store(xr + i0, f);
  } else if (dt.slot >= 0 && sk.part != nullptr) {
    Vec8<T>::store(xr + i0, f);   // rank > 16 with v in the pieces: not fused (host rejects)
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float c = 0.f;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) c += red[q];
    red[4] = c;   // this CTA's partial
  }
  stamp(3);
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  stamp(4);
  float tot = 0.f;
  {
    const uint32_t a_local = static_cast<uint32_t>(__cvta_generic_to_shared(&red[4]));
#pragma unroll
    for (int r = 0; r < RNL_CL; ++r) {   // fixed rank order: deterministic
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a_local), "r"(r));
      float v;
      asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
      tot += v;
    }
  }
  const float inv = 1.0f / sqrtf(tot / (float)d + eps);
  float g[8];
  Vec8<bf16>::load(w + i0, g);
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = (f[j] * inv) * g[j];
  Vec8<T>::store(out + (size_t)t * ldo + i0, f);
  // keep red[4] alive until every peer has read it
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  stamp(7);
}

// One CTA per token (d / 8 threads, 8 columns each): the same fused residual-pieces + LoRA +
// RMSNorm without a cluster, so it launches as one small wave and its CTAs can start early
// under PDL.  The LoRA B rows are loaded after the pieces (register budget at 512+ threads).
template <typename T>
__global__ void __launch_bounds__(640) rmsnorm_fused_tok_kernel(T* __restrict__ out, int ldo,
                                                                 T* __restrict__ x, int ldx,
                                                                 const bf16* __restrict__ w, int d,
                                                                 float eps, DeltaArgs lora,
                                                                 SplitArgs sk, PfArgs pf,
                                                                 unsigned long long* trace) {
  __shared__ float vs[DELTA_VS];
  __shared__ float red[33];
  auto stamp = [&](int i) {
    if (trace && threadIdx.x == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)::"memory");
      trace[(blockIdx.x % 256) * 16 + i] = tt;
      if (blockIdx.x == 0 && i == 0) trace[4095] = 6;
    }
  };
  stamp(0);
  if (threadIdx.x == 0) l2_prefetch_part(pf, blockIdx.x, gridDim.x);   // next GEMM, pre-wait
  const int t = blockIdx.x;
  const int i0 = threadIdx.x * 8;
  T* xr = x + (size_t)t * ldx;
  const DeltaTok dt = delta_tok(lora, t);   // slot tables: >= 2 launches old
  pdl_wait();
  pdl_trigger();
  stamp(2);
  float f[8];
  Vec8<T>::load(xr + i0, f);
  if (sk.part != nullptr) {
    float ps[8];
    split_sum8(sk, t, i0, ps);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + ps[j]));
  }
  if (dt.slot >= 0 && dt.rank <= AD_LORA_FAST_RANK) {
    if (lora.v == nullptr) {
      for (int e = threadIdx.x; e < lora.n_targets * 64; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        int off = 0;
#pragma unroll
        for (int q = 0; q < SLX_LORA_MAX_TARGETS; ++q)
          if (q == i) off = lora.v_col_off[q];
        if (j < dt.rank) vs[e] = split_sum1(sk, t, sk.n_main + off + dt.slot * lora.v_slot_stride + j) * dt.scale;
      }
    } else {
      delta_stage_v(lora, dt, vs, threadIdx.x, blockDim.x);
    }
    DeltaRow<2> dr[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) delta_prefetch<2>(lora, dt, i0 + j, dr[j]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_finish<2>(dt, dr[j], vs)));
  } else if (dt.slot >= 0 && lora.v != nullptr) {
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = to_f32(from_f32<T>(f[j] + delta_col(lora, dt, i0 + j)));
  }
  if (sk.part != nullptr || dt.slot >= 0) Vec8<T>::store(xr + i0, f);
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;   // fixed order
    v = warp_sum(v);
    if (threadIdx.x == 0) red[32] = v;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[32] / (float)d + eps);
  float g[8];
  Vec8<bf16>::load(w + i0, g);
#pragma unroll
  for (int j = 0; j < 8; ++j) f[j] = (f[j] * inv) * g[j];
  Vec8<T>::store(out + (size_t)t * ldo + i0, f);
  stamp(7);
}

// ------------------------------------------------------------------ RoPE + KV write
// One CTA per token; thread i handles rotation pair (i, i + D/2) of every head.
template <typename T>
__global__ void rope_kv_kernel(T* __restrict__ qkv, int ld, int H, int Hkv, int D,
                               const int32_t* __restrict__ tok_pos,
                               const int32_t* __restrict__ tok_seq,
                               const float* __restrict__ cos_tab, const float* __restrict__ sin_tab,
                               T* __restrict__ kc, T* __restrict__ vc, int max_ctx) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int pos = tok_pos[t];
  const int seq = tok_seq[t];
  const int half = D >> 1;
  T* row = qkv + (size_t)t * ld;
  const float* cr = cos_tab + (size_t)pos * half;
  const float* sr = sin_tab + (size_t)pos * half;
  const int n_rot = (H + Hkv) * half;
  for (int idx = threadIdx.x; idx < n_rot; idx += blockDim.x) {
    const int h = idx / half, i = idx % half;
    T* base = row + h * D;  // q heads then k heads are contiguous
    const float c = cr[i], s = sr[i];
    const float x1 = to_f32(base[i]), x2 = to_f32(base[i + half]);
    const float r1 = x1 * c - x2 * s;
    const float r2 = x2 * c + x1 * s;
    base[i] = from_f32<T>(r1);
    base[i + half] = from_f32<T>(r2);
    if (h >= H) {
      const int hk = h - H;
      T* dst = kc + (((size_t)seq * Hkv + hk) * max_ctx + pos) * D;
      dst[i] = from_f32<T>(r1);
      dst[i + half] = from_f32<T>(r2);
    }
  }
  const T* vsrc = row + (H + Hkv) * D;
  for (int idx = threadIdx.x; idx < Hkv * D; idx += blockDim.x) {
    const int hk = idx / D, i = idx % D;
    vc[(((size_t)seq * Hkv + hk) * max_ctx + pos) * D + i] = vsrc[idx];
  }
}

// Vectorised variant (head_dim % 16 == 0, 16-byte aligned rows): each thread rotates 8 pairs
// with 16-byte loads / stores, same arithmetic and rounding as rope_kv_kernel.
template <typename T>
__global__ void __launch_bounds__(128) rope_kv_vec_kernel(T* __restrict__ qkv, int ld, int H, int Hkv, int D,
                                   const int32_t* __restrict__ tok_pos,
                                   const int32_t* __restrict__ tok_seq,
                                   const float* __restrict__ cos_tab,
                                   const float* __restrict__ sin_tab, T* __restrict__ kc,
                                   T* __restrict__ vc, int max_ctx) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  const int pos = tok_pos[t];
  const int seq = tok_seq[t];
  const int half = D >> 1, hv = half >> 3;
  T* row = qkv + (size_t)t * ld;
  const float* cr = cos_tab + (size_t)pos * half;
  const float* sr = sin_tab + (size_t)pos * half;
  const int n_rot = (H + Hkv) * hv;
  for (int idx = threadIdx.x; idx < n_rot; idx += blockDim.x) {
    const int h = idx / hv, i = (idx - h * hv) * 8;
    T* base = row + h * D;
    float x1[8], x2[8], c[8], sn[8], r1[8], r2[8];
    Vec8<T>::load(base + i, x1);
    Vec8<T>::load(base + i + half, x2);
    Vec8<float>::load(cr + i, c);
    Vec8<float>::load(sr + i, sn);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      r1[j] = x1[j] * c[j] - x2[j] * sn[j];
      r2[j] = x2[j] * c[j] + x1[j] * sn[j];
    }
    Vec8<T>::store(base + i, r1);
    Vec8<T>::store(base + i + half, r2);
    if (h >= H) {
      T* dst = kc + (((size_t)seq * Hkv + (h - H)) * max_ctx + pos) * D;
      Vec8<T>::store(dst + i, r1);
      Vec8<T>::store(dst + i + half, r2);
    }
  }
  const T* vsrc = row + (H + Hkv) * D;
  const int dv = D >> 3;
  for (int idx = threadIdx.x; idx < Hkv * dv; idx += blockDim.x) {
    const int hk = idx / dv, i = (idx - hk * dv) * 8;
    float v[8];
    Vec8<T>::load(vsrc + hk * D + i, v);
    Vec8<T>::store(vc + (((size_t)seq * Hkv + hk) * max_ctx + pos) * D + i, v);
  }
}

// ------------------------------------------------------------------ attention over the KV pool
// One CTA of 4 warps per (token, head); warp w streams key chunks c = w, w+4, ... of 32 keys.
// Lane j of a chunk loads key row j0+j with 16-byte loads (the whole chunk's K in flight at
// once), computes its score, the warp does an online-softmax update (exp2, fp32), then the
// chunk's V rows are loaded (lane owns D/32 output dims) and accumulated.  Warps are merged
// through shared memory at the end.  Causal: token t attends positions 0..tok_pos[t].
constexpr int ATT_WARPS = 4;

// PL consecutive elements -> floats with one vector load (8 B for 4 x bf16, 16 B for 4 x f32).
template <typename T, int PL> __device__ __forceinline__ void load_pl(const T* p, float* f);
template <> __device__ __forceinline__ void load_pl<bf16, 4>(const bf16* p, float* f) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
template <> __device__ __forceinline__ void load_pl<bf16, 2>(const bf16* p, float* f) {
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
  f[0] = a.x; f[1] = a.y;
}
template <> __device__ __forceinline__ void load_pl<float, 4>(const float* p, float* f) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
}
template <> __device__ __forceinline__ void load_pl<float, 2>(const float* p, float* f) {
  const float2 a = *reinterpret_cast<const float2*>(p);
  f[0] = a.x; f[1] = a.y;
}

template <typename T, int D>
__global__ void __launch_bounds__(ATT_WARPS * 32)
attention_kernel(T* __restrict__ out, int ldo, const T* __restrict__ qkv, int ld, int H, int Hkv,
                 const int32_t* __restrict__ tok_pos, const int32_t* __restrict__ tok_seq,
                 const T* __restrict__ kc, const T* __restrict__ vc, int max_ctx, float scale_log2) {
  pdl_wait();
  pdl_trigger();
  constexpr int PL = D / 32;   // output dims per lane
  __shared__ float qs[D];
  __shared__ float m_s[ATT_WARPS], l_s[ATT_WARPS];
  __shared__ float acc_s[ATT_WARPS][D];
  const int t = blockIdx.x / H, h = blockIdx.x % H;
  const int hk = h / (H / Hkv);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_keys = tok_pos[t] + 1;
  const int seq = tok_seq[t];
  for (int i = threadIdx.x; i < D; i += blockDim.x)
    qs[i] = to_f32(qkv[(size_t)t * ld + h * D + i]) * scale_log2;
  __syncthreads();
  const T* kbase = kc + ((size_t)seq * Hkv + hk) * max_ctx * D;
  const T* vbase = vc + ((size_t)seq * Hkv + hk) * max_ctx * D;
  float m = -INFINITY, l = 0.f;
  float acc[PL];
#pragma unroll
  for (int i = 0; i < PL; ++i) acc[i] = 0.f;
  for (int j0 = warp * 32; j0 < n_keys; j0 += ATT_WARPS * 32) {
    const int nk = min(32, n_keys - j0);
    // ---- scores: lane = key
    float sc = -INFINITY;
    if (lane < nk) {
      const T* kr = kbase + (size_t)(j0 + lane) * D;
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < D; i += 8) {
        float f[8];
        Vec8<T>::load(kr + i, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot = fmaf(qs[i + e], f[e], dot);
      }
      sc = dot;
    }
    const float m_new = fmaxf(m, warp_max(sc));
    const float corr = exp2f(m - m_new);
    const float p = lane < nk ? exp2f(sc - m_new) : 0.f;
    l = l * corr + warp_sum(p);
#pragma unroll
    for (int i = 0; i < PL; ++i) acc[i] *= corr;
    m = m_new;
    // ---- P.V: lane owns dims [lane*PL, lane*PL + PL); 16 rows' loads in flight at a time
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      float vv[16][PL];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int jj = half * 16 + u;
        if (jj < nk) load_pl<T, PL>(vbase + (size_t)(j0 + jj) * D + lane * PL, vv[u]);
        else {
#pragma unroll
          for (int i = 0; i < PL; ++i) vv[u][i] = 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float pj = __shfl_sync(0xffffffffu, p, half * 16 + u);
#pragma unroll
        for (int i = 0; i < PL; ++i) acc[i] = fmaf(pj, vv[u][i], acc[i]);
      }
    }
  }
  if (lane == 0) { m_s[warp] = m; l_s[warp] = l; }
#pragma unroll
  for (int i = 0; i < PL; ++i) acc_s[warp][lane * PL + i] = acc[i];
  __syncthreads();
  if (warp == 0) {
    float mg = -INFINITY;
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) mg = fmaxf(mg, m_s[w]);
    float lg = 0.f, cw[ATT_WARPS];
#pragma unroll
    for (int w = 0; w < ATT_WARPS; ++w) {
      cw[w] = (l_s[w] > 0.f) ? exp2f(m_s[w] - mg) : 0.f;
      lg += l_s[w] * cw[w];
    }
    const float inv = 1.0f / lg;
#pragma unroll
    for (int i = 0; i < PL; ++i) {
      float o = 0.f;
#pragma unroll
      for (int w = 0; w < ATT_WARPS; ++w) o += acc_s[w][lane * PL + i] * cw[w];
      out[(size_t)t * ldo + h * D + lane * PL + i] = from_f32<T>(o * inv);
    }
  }
}

template <typename T, int D>
constexpr size_t att_smem() { return 0; }

// ------------------------------------------------------------------ fused decode attention
// Decode (one new token per sequence): CTA (token t, head h) applies RoPE to q and to the new
// key in registers, appends k/v at tok_pos[t] to the KV pool (the group-leader head of a GQA
// group writes), then attends over the cached positions [0, pos) — staged KB keys at a time
// in shared memory with one burst of 16-byte cp.async per block — plus the new key/value.
// Replaces rope_kv_write + attention for the decode step (one launch instead of two).
template <typename T> struct DecCfg { static constexpr int KB = 128; };
template <> struct DecCfg<float> { static constexpr int KB = 64; };

template <typename T, int D>
constexpr size_t dec_smem() {
  return (size_t)2 * DecCfg<T>::KB * (D + 16 / sizeof(T)) * sizeof(T) +
         (size_t)(3 * D + DecCfg<T>::KB + 2 * 128 + 8 + 3 * D + DELTA_VS) * 4;
}

template <typename T, int D>
__global__ void __launch_bounds__(128)
rope_attn_decode_kernel(T* __restrict__ out, int ldo, const T* __restrict__ qkv, int ld, int H,
                        int Hkv, const int32_t* __restrict__ tok_pos,
                        const int32_t* __restrict__ tok_seq, const float* __restrict__ cos_tab,
                        const float* __restrict__ sin_tab, T* __restrict__ kc, T* __restrict__ vc,
                        int max_ctx, float scale_log2, DeltaArgs lora, PfArgs pf, int pf_from) {
  constexpr int KB = DecCfg<T>::KB;
  constexpr int VEC = 16 / sizeof(T);
  constexpr int DP = D + VEC;          // padded smem row
  constexpr int CH = D / VEC;          // 16-byte chunks per row
  constexpr int NT = 128;
  constexpr int KP = NT / D;           // key partitions in P.V (1 for D=128, 2 for D=64)
  constexpr int PER = (3 * D + NT - 1) / NT;   // q/k/v row columns per thread
  extern __shared__ __align__(16) uint8_t dsm[];
  T* Ks = reinterpret_cast<T*>(dsm);                   // [KB][DP]
  T* Vs = Ks + KB * DP;                                 // [KB][DP]
  float* qs = reinterpret_cast<float*>(Vs + KB * DP);   // [D] rotated, scaled q
  float* kn = qs + D;                                    // [D] new key (rounded to T)
  float* vn = kn + D;                                    // [D] new value
  float* ps = vn + D;                                    // [KB]
  float* red = ps + KB;                                  // [2*128] partials / reductions
  float* misc = red + 2 * 128;                           // [8]
  float* raw = misc + 8;                                 // [3][D] q, k, v row (+ LoRA delta)
  float* vs = raw + 3 * D;                               // [DELTA_VS] scale * LoRA v

  const int tid = threadIdx.x;
  const int t = blockIdx.x / H, h = blockIdx.x % H;
  const int group = H / Hkv, hk = h / group;
  // step inputs (token positions / sequences / adapter slots), the adapter pool and the cached
  // keys and values before `pos` were all written two or more launches back (PDL invariant,
  // common.cuh): fetch them before waiting on the projection GEMM.
  const int pos = tok_pos[t], seq = tok_seq[t];
  const DeltaTok dt = delta_tok(lora, t);
  const T* kbase = kc + ((size_t)seq * Hkv + hk) * max_ctx * D;
  const T* vbase = vc + ((size_t)seq * Hkv + hk) * max_ctx * D;
  auto load_block = [&](int k0, int nk) {
    for (int e = tid; e < nk * CH; e += NT) {
      const int r = e / CH, c = e % CH;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(Ks + r * DP + c * VEC))),
                   "l"(kbase + (size_t)(k0 + r) * D + c * VEC) : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(Vs + r * DP + c * VEC))),
                   "l"(vbase + (size_t)(k0 + r) * D + c * VEC) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int n_cached = pos;
  if (n_cached > 0) load_block(0, min(KB, n_cached));
  // the last wave prefetches the next kernel's first bytes into L2 (HBM busy across the boundary)
  if (tid == 0 && (int)blockIdx.x >= pf_from)
    l2_prefetch_part(pf, blockIdx.x - pf_from, gridDim.x - pf_from);
  const bool fast = dt.slot >= 0 && dt.rank <= 16;
  DeltaRow<2> dr[PER];
  auto col_of = [&](int i) {
    const int part = i / D, e = i - part * D;
    return (part == 0 ? h : (part == 1 ? H + hk : H + Hkv + hk)) * D + e;
  };
  if (fast) {
#pragma unroll
    for (int p = 0; p < PER; ++p)
      if (tid + p * NT < 3 * D) delta_prefetch<2>(lora, dt, col_of(tid + p * NT), dr[p]);
  }
  pdl_wait();
  pdl_trigger();

  const int half = D / 2;
  const T* row = qkv + (size_t)t * ld;
  const float* cr = cos_tab + (size_t)pos * half;
  const float* sr = sin_tab + (size_t)pos * half;
  T* kdst = kc + (((size_t)seq * Hkv + hk) * max_ctx + pos) * D;
  T* vdst = vc + (((size_t)seq * Hkv + hk) * max_ctx + pos) * D;
  // the projection outputs of this head, with the fused LoRA expand added and rounded to T
  // exactly as slx_lora_expand would have stored them in qkv
  float rv[PER];
#pragma unroll
  for (int p = 0; p < PER; ++p) rv[p] = tid + p * NT < 3 * D ? to_f32(row[col_of(tid + p * NT)]) : 0.f;
  if (fast) {
    delta_stage_v(lora, dt, vs, tid, NT);
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int i = tid + p * NT;
    if (i < 3 * D) {
      float v = rv[p];
      if (dt.slot >= 0)
        v = to_f32(from_f32<T>(v + (fast ? delta_finish<2>(dt, dr[p], vs) : delta_col(lora, dt, col_of(i)))));
      raw[i] = v;
    }
  }
  __syncthreads();
  for (int i = tid; i < half; i += NT) {
    const float c = cr[i], sn = sr[i];
    const float q1 = raw[i], q2 = raw[i + half];
    // q is rounded to T exactly as the unfused path stores it before attention reads it back
    qs[i] = to_f32(from_f32<T>(q1 * c - q2 * sn)) * scale_log2;
    qs[i + half] = to_f32(from_f32<T>(q2 * c + q1 * sn)) * scale_log2;
    const float k1 = raw[D + i], k2 = raw[D + i + half];
    const T r1 = from_f32<T>(k1 * c - k2 * sn), r2 = from_f32<T>(k2 * c + k1 * sn);
    kn[i] = to_f32(r1);
    kn[i + half] = to_f32(r2);
    if (h % group == 0) {
      kdst[i] = r1;
      kdst[i + half] = r2;
    }
  }
  for (int i = tid; i < D; i += NT) {
    const T v = from_f32<T>(raw[2 * D + i]);
    vn[i] = to_f32(v);
    if (h % group == 0) vdst[i] = v;
  }
  __syncthreads();

  // the new key first: its score seeds the running max
  float s_new = 0.f;
  {
    float part = 0.f;
    for (int i = tid; i < D; i += NT) part += qs[i] * kn[i];
    part = warp_sum(part);
    if ((tid & 31) == 0) red[tid >> 5] = part;
    __syncthreads();
    s_new = red[0] + red[1] + red[2] + red[3];
    __syncthreads();
  }
  float m = s_new, l = 1.f;
  const int dd = tid % D, kp = tid / D;   // P.V: dim dd over key partition kp
  float acc = kp == 0 ? vn[dd] : 0.f;     // p_new = exp2(s_new - m) = 1
  for (int k0 = 0; k0 < n_cached; k0 += KB) {
    const int nk = min(KB, n_cached - k0);
    if (k0 > 0) load_block(k0, nk);   // block 0 was issued before the PDL wait
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    // scores: thread = key (KB <= 128 threads)
    float sc = -INFINITY;
    if (tid < nk) {
      const T* kr = Ks + tid * DP;
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < D; i += 8) {
        float f[8];
        Vec8<T>::load(kr + i, f);
#pragma unroll
        for (int e = 0; e < 8; ++e) dot = fmaf(qs[i + e], f[e], dot);
      }
      sc = dot;
    }
    float bm = warp_max(sc);
    if ((tid & 31) == 0) red[tid >> 5] = bm;
    __syncthreads();
    bm = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float m_new = fmaxf(m, bm);
    const float corr = exp2f(m - m_new);
    const float p = tid < nk ? exp2f(sc - m_new) : 0.f;
    if (tid < KB) ps[tid] = p;
    float bs = warp_sum(p);
    __syncthreads();   // ps visible; red[0..3] consumed
    if ((tid & 31) == 0) red[4 + (tid >> 5)] = bs;
    // P.V over this block
    float a = 0.f;
    for (int j = kp; j < nk; j += KP) a = fmaf(ps[j], to_f32(Vs[j * DP + dd]), a);
    __syncthreads();
    l = l * corr + (red[4] + red[5] + red[6] + red[7]);
    acc = acc * corr + a;
    m = m_new;
    __syncthreads();   // Ks/Vs/ps reused by the next block
  }
  if (KP > 1) {
    red[tid] = acc;
    __syncthreads();
    if (tid < D) {
      float o = 0.f;
      for (int q = 0; q < KP; ++q) o += red[q * D + tid];
      out[(size_t)t * ldo + h * D + tid] = from_f32<T>(o / l);
    }
  } else {
    out[(size_t)t * ldo + h * D + tid] = from_f32<T>(acc / l);
  }
}

// ------------------------------------------------------------------ SiLU * mul (blocked gate/up)
template <typename T>
__global__ void silu_mul_kernel(T* __restrict__ out, int ldo, const T* __restrict__ gu, int ld_gu,
                                int ffn) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.y;
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i >= ffn) return;
  const int blk = i >> 7, off = i & 127;
  const T* g = gu + (size_t)t * ld_gu + blk * 256 + off;
  float a[8], b[8];
  Vec8<T>::load(g, a);
  Vec8<T>::load(g + 128, b);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (a[j] / (1.0f + expf(-a[j]))) * b[j];
  Vec8<T>::store(out + (size_t)t * ldo + i, a);
}

// ------------------------------------------------------------------ argmax
template <typename T>
__global__ void argmax_kernel(int32_t* __restrict__ out, const T* __restrict__ x, int ld, int n) {
  pdl_wait();
  pdl_trigger();
  const T* row = x + (size_t)blockIdx.x * ld;
  float best = -FLT_MAX;
  int bi = 0x7fffffff;
  if (sizeof(T) == 4 && n % 4 == 0 && ld % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0) {   // fp32 logits: 16-byte loads
    const float4* r4 = reinterpret_cast<const float4*>(row);
    for (int i = threadIdx.x; i < n / 4; i += blockDim.x) {
      const float4 v = r4[i];   // indices 4i .. 4i+3 in order: strict > keeps the first max
      if (v.x > best) { best = v.x; bi = 4 * i; }
      if (v.y > best) { best = v.y; bi = 4 * i + 1; }
      if (v.z > best) { best = v.z; bi = 4 * i + 2; }
      if (v.w > best) { best = v.w; bi = 4 * i + 3; }
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const float v = to_f32(row[i]);
      if (v > best) { best = v; bi = i; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sv[w] = best; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (sv[k] > best || (sv[k] == best && si[k] < bi)) { best = sv[k]; bi = si[k]; }
    out[blockIdx.x] = bi;
  }
}

// ------------------------------------------------------------------ fp32-parity SIMT GEMM
// C[M,N] = A[M,K] (fp32) . W[N,K]^T (bf16) [+ R].  64x64 tile, BK 16, 4x4 per thread.
constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;
__global__ void __launch_bounds__(256)
gemm_f32_kernel(const float* __restrict__ A, int lda, const bf16* __restrict__ W,
                float* __restrict__ C, int ldc, const float* __restrict__ R, int ldr,
                int M, int N, int K) {
  pdl_wait();
  pdl_trigger();
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Ws[SG_BK][SG_BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  float acc[4][4] = {};
  // loader mapping: 256 threads x 4 elements = 64 rows x 16 k
  const int lr = threadIdx.x / 4, lk = (threadIdx.x % 4) * 4;
  for (int k0 = 0; k0 < K; k0 += SG_BK) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = k0 + lk + e;
      const int am = m0 + lr, wn = n0 + lr;
      As[lk + e][lr] = (am < M && k < K) ? A[(size_t)am * lda + k] : 0.f;
      Ws[lk + e][lr] = (wn < N && k < K) ? __bfloat162float(W[(size_t)wn * K + k]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (R) v += R[(size_t)m * ldr + n];
      C[(size_t)m * ldc + n] = v;
    }
  }
}

}  // namespace slx

using namespace slx;

template <typename T, int D>
static int att_attr() {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(attention_kernel<T, D>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done = true;
  }
  return 0;
}

// ================================================================== C ABI
#define DISPATCH_DT(dtype, ...)                      \
  do {                                               \
    if ((dtype) == SLX_DT_BF16) {                    \
      using T = bf16;                                \
      __VA_ARGS__;                                   \
    } else if ((dtype) == SLX_DT_F32) {              \
      using T = float;                               \
      __VA_ARGS__;                                   \
    } else {                                         \
      return SLX_ERR_INVALID;                        \
    }                                                \
  } while (0)

extern "C" int slx_embedding(int dtype, void* out, const void* table, const int32_t* tokens,
                             int n_tok, int d, int vocab, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d > 0 && d % 8 == 0 && vocab > 0 && out && table && tokens);
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(table, 16);
  if (n_tok == 0) return SLX_OK;
  int st = SLX_OK;
  DISPATCH_DT(dtype, st = launch_ex(embedding_kernel<T>, dim3(n_tok), dim3(128), 0, (cudaStream_t)stream, 1u, (T*)out, (const bf16*)table, tokens, d, vocab));
  return st;
}

extern "C" int slx_rmsnorm(int dtype, void* out, int ldo, const void* x, int ldx, const void* w,
                           int n_tok, int d, float eps, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d > 0 && d % 8 == 0 && ldo % 8 == 0 && ldx % 8 == 0 && ldo >= d &&
                ldx >= d && out && x && w);
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(x, 16);
  SLX_CHECK_ALIGN(w, 16);
  if (n_tok == 0) return SLX_OK;
  int st = SLX_OK;
  if (d % (RN_CH * 8 * 32) == 0 && d / (RN_CH * 8) <= 256) {   // the row in registers
    DISPATCH_DT(dtype, st = launch_ex(rmsnorm_row_kernel<T>, dim3(n_tok), dim3(d / (RN_CH * 8)), 0, (cudaStream_t)stream, 1u, (T*)out, ldo, (const T*)x, ldx, (const bf16*)w, d, eps));
    return st;
  }
  int threads = d >= 4096 ? 512 : (d >= 1024 ? 128 : 32);
  DISPATCH_DT(dtype, st = launch_ex(rmsnorm_kernel<T>, dim3(n_tok), dim3(threads), 0, (cudaStream_t)stream, 1u, (T*)out, ldo, (const T*)x, ldx, (const bf16*)w, d, eps));
  return st;
}

extern "C" int slx_rmsnorm_lora(int dtype, void* out, int ldo, void* x, int ldx, const void* w,
                                int n_tok, int d, float eps, const slx_lora_delta* lora,
                                void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d > 0 && d % 8 == 0 && ldo % 8 == 0 && ldx % 8 == 0 && ldo >= d &&
                ldx >= d && out && x && w && delta_valid(lora));
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(x, 16);
  SLX_CHECK_ALIGN(w, 16);
  if (n_tok == 0) return SLX_OK;
  const DeltaArgs la = delta_args(lora);
  int st = SLX_OK;
  if (d % (RNL_CL * 8 * 32) == 0 && d / (RNL_CL * 8) <= 128) {
    const int thr = d / (RNL_CL * 8);
    DISPATCH_DT(dtype, st = launch_ex(rmsnorm_lora_cluster_kernel<T>, dim3(n_tok * RNL_CL), dim3(thr), 0, (cudaStream_t)stream, (unsigned)RNL_CL, (T*)out, ldo, (T*)x, ldx, (const bf16*)w, d, eps, la, SplitArgs{}, PfArgs{}, next_trace_window(6)));
    return st;
  }
  int threads = d >= 4096 ? 512 : (d >= 1024 ? 128 : 32);
  DISPATCH_DT(dtype, st = launch_ex(rmsnorm_lora_kernel<T>, dim3(n_tok), dim3(threads), 0, (cudaStream_t)stream, 1u, (T*)out, ldo, (T*)x, ldx, (const bf16*)w, d, eps, la));
  return st;
}

extern "C" int slx_rmsnorm_fused(int dtype, void* out, int ldo, void* x, int ldx, const void* w,
                                 int n_tok, int d, float eps, const slx_splitk_in* sk,
                                 const slx_lora_delta* lora, const slx_l2_prefetch* pf,
                                 void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && d > 0 && ldo % 8 == 0 && ldx % 8 == 0 && ldo >= d && ldx >= d &&
                out && x && w && delta_valid(lora, sk != nullptr));
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(x, 16);
  SLX_CHECK_ALIGN(w, 16);
  if (sk != nullptr) {
    SLX_CHECK_ARG(sk->part && sk->splits >= 1 && sk->splits <= 16 && sk->bm >= n_tok &&
                  sk->bm % 16 == 0 && sk->n_main >= d);
    SLX_CHECK_ALIGN(sk->part, 16);
    if (lora && lora->n_targets > 0 && lora->v == nullptr && lora->max_rank > 16)
      return SLX_ERR_UNSUPPORTED;
  }
  if (n_tok == 0) return SLX_OK;
  const DeltaArgs la = delta_args(lora);
  const SplitArgs sa = split_args(sk);
  const PfArgs pa = pf_args(pf);
  int st = SLX_OK;
  // the 8-CTA cluster kernel (measured faster in the decode graph); a d the cluster split cannot
  // take: one CTA per token
  const bool cl_ok = d % (RNL_CL * 8 * 32) == 0 && d / (RNL_CL * 8) <= 128;
  if (!cl_ok && d % 256 == 0 && d / 8 <= 640 && (!sk || sk->splits <= 8)) {
    DISPATCH_DT(dtype, st = launch_ex(rmsnorm_fused_tok_kernel<T>, dim3(n_tok), dim3(d / 8), 0, (cudaStream_t)stream, 1u, (T*)out, ldo, (T*)x, ldx, (const bf16*)w, d, eps, la, sa, pa, next_trace_window(6)));
    return st;
  }
  if (d % (RNL_CL * 8 * 32) != 0 || d / (RNL_CL * 8) > 128) return SLX_ERR_UNSUPPORTED;
  const int thr = d / (RNL_CL * 8);
  DISPATCH_DT(dtype, st = launch_ex(rmsnorm_lora_cluster_kernel<T>, dim3(n_tok * RNL_CL), dim3(thr), 0, (cudaStream_t)stream, (unsigned)RNL_CL, (T*)out, ldo, (T*)x, ldx, (const bf16*)w, d, eps, la, sa, pa, next_trace_window(6)));
  return st;
}

extern "C" int slx_rope_kv_write(int dtype, void* qkv, int ld_qkv, int n_tok, int heads,
                                 int kv_heads, int head_dim, const int32_t* tok_pos,
                                 const int32_t* tok_seq, const float* cos_tab,
                                 const float* sin_tab, int max_pos, void* k_cache, void* v_cache,
                                 int max_ctx, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && heads > 0 && kv_heads > 0 && heads % kv_heads == 0 &&
                head_dim % 2 == 0 && ld_qkv >= (heads + 2 * kv_heads) * head_dim && max_pos > 0 &&
                max_ctx > 0 && qkv && tok_pos && tok_seq && cos_tab && sin_tab && k_cache &&
                v_cache);
  if (n_tok == 0) return SLX_OK;
  int st = SLX_OK;
  // bf16 only: the fp32 parity mode keeps the scalar kernel's exact FMA contraction
  const bool vec = dtype == SLX_DT_BF16 && head_dim % 16 == 0 && ld_qkv % 8 == 0 &&
                   ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(k_cache) |
                     reinterpret_cast<uintptr_t>(v_cache) | reinterpret_cast<uintptr_t>(cos_tab) |
                     reinterpret_cast<uintptr_t>(sin_tab)) & 31) == 0;
  if (vec)
    return launch_ex(rope_kv_vec_kernel<bf16>, dim3(n_tok), dim3(128), 0, (cudaStream_t)stream, 1u,
                     (bf16*)qkv, ld_qkv, heads, kv_heads, head_dim, tok_pos, tok_seq, cos_tab,
                     sin_tab, (bf16*)k_cache, (bf16*)v_cache, max_ctx);
  DISPATCH_DT(dtype, st = launch_ex(rope_kv_kernel<T>, dim3(n_tok), dim3(256), 0, (cudaStream_t)stream, 1u, (T*)qkv, ld_qkv, heads, kv_heads, head_dim, tok_pos, tok_seq, cos_tab,
                         sin_tab, (T*)k_cache, (T*)v_cache, max_ctx));
  return st;
}

extern "C" int slx_attention(int dtype, void* out, int ldo, const void* qkv, int ld_qkv, int n_tok,
                             int heads, int kv_heads, int head_dim, const int32_t* tok_pos,
                             const int32_t* tok_seq, const void* k_cache, const void* v_cache,
                             int max_ctx, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && heads > 0 && kv_heads > 0 && heads % kv_heads == 0 &&
                ld_qkv >= (heads + 2 * kv_heads) * head_dim && ldo >= heads * head_dim && out &&
                qkv && tok_pos && tok_seq && k_cache && v_cache);
  SLX_CHECK_ARG(ldo % 8 == 0 && ld_qkv % 8 == 0);
  SLX_CHECK_ALIGN(k_cache, 16);
  SLX_CHECK_ALIGN(v_cache, 16);
  if (head_dim != 64 && head_dim != 128) return SLX_ERR_UNSUPPORTED;
  if (n_tok == 0) return SLX_OK;
  const float scale = 1.4426950408889634f / sqrtf((float)head_dim);   // log2(e)/sqrt(D)
  const dim3 grid((unsigned)n_tok * heads);
  cudaStream_t s = (cudaStream_t)stream;
  int st = SLX_OK;
  if (head_dim == 64) {
    DISPATCH_DT(dtype, st = att_attr<T, 64>() ? SLX_ERR_CUDA : launch_ex(attention_kernel<T, 64>, dim3(grid), dim3(ATT_WARPS * 32), 0, s, 1u, (T*)out, ldo, (const T*)qkv, ld_qkv, heads, kv_heads, tok_pos, tok_seq,
                           (const T*)k_cache, (const T*)v_cache, max_ctx, scale));
  } else {
    DISPATCH_DT(dtype, st = att_attr<T, 128>() ? SLX_ERR_CUDA : launch_ex(attention_kernel<T, 128>, dim3(grid), dim3(ATT_WARPS * 32), 0, s, 1u, (T*)out, ldo, (const T*)qkv, ld_qkv, heads, kv_heads, tok_pos, tok_seq,
                           (const T*)k_cache, (const T*)v_cache, max_ctx, scale));
  }
  return st;
}

extern "C" int slx_silu_mul_blocked(int dtype, void* out, int ldo, const void* gu, int ld_gu,
                                    int n_tok, int ffn, void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && ffn > 0 && ffn % 128 == 0 && ld_gu >= 2 * ffn && ldo >= ffn &&
                ldo % 8 == 0 && ld_gu % 8 == 0 && out && gu);
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(gu, 16);
  if (n_tok == 0) return SLX_OK;
  dim3 grid((unsigned)ceil_div(ffn / 8, 128), (unsigned)n_tok);
  int st = SLX_OK;
  DISPATCH_DT(dtype, st = launch_ex(silu_mul_kernel<T>, dim3(grid), dim3(128), 0, (cudaStream_t)stream, 1u, (T*)out, ldo, (const T*)gu, ld_gu, ffn));
  return st;
}

extern "C" int slx_argmax(int dtype, int32_t* out, const void* logits, int ld, int n_rows,
                          int n_cols, void* stream) {
  SLX_CHECK_ARG(n_rows >= 0 && n_cols > 0 && ld >= n_cols && out && logits);
  if (n_rows == 0) return SLX_OK;
  int st = SLX_OK;
  DISPATCH_DT(dtype, st = launch_ex(argmax_kernel<T>, dim3(n_rows), dim3(512), 0, (cudaStream_t)stream, 1u, out, (const T*)logits, ld, n_cols));
  return st;
}

extern "C" int slx_gemm_f32(const void* A, int lda, const void* W, void* C, int ldc, const void* R,
                            int ldr, int M, int N, int K, int epilogue, void* stream) {
  SLX_CHECK_ARG(M >= 0 && N > 0 && K > 0 && lda >= K && ldc >= N && A && W && C);
  if (epilogue == SLX_EPI_RESIDUAL) {
    SLX_CHECK_ARG(R != nullptr && ldr >= N);
  } else if (epilogue != SLX_EPI_NONE) {
    return SLX_ERR_UNSUPPORTED;
  }
  if (M == 0) return SLX_OK;
  dim3 grid((unsigned)ceil_div(N, SG_BN), (unsigned)ceil_div(M, SG_BM));
  return launch_ex(gemm_f32_kernel, grid, dim3(256), 0, (cudaStream_t)stream, 1u,
                   (const float*)A, lda, (const bf16*)W, (float*)C, ldc,
                   epilogue == SLX_EPI_RESIDUAL ? (const float*)R : nullptr, ldr, M, N, K);
}

template <typename T, int D>
static int launch_rope_attn(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok, int heads,
                            int kv_heads, const int32_t* tok_pos, const int32_t* tok_seq,
                            const float* cos_tab, const float* sin_tab, void* k_cache,
                            void* v_cache, int max_ctx, float scale, const DeltaArgs& lora,
                            const PfArgs& pf, cudaStream_t s) {
  auto k = rope_attn_decode_kernel<T, D>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dec_smem<T, D>()) !=
        cudaSuccess)
      return SLX_ERR_CUDA;
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    configured = true;
  }
  return launch_ex(k, dim3((unsigned)n_tok * heads), dim3(128), dec_smem<T, D>(), s, 1u, (T*)out,
                   ldo, (const T*)qkv, ld_qkv, heads, kv_heads, tok_pos, tok_seq, cos_tab, sin_tab,
                   (T*)k_cache, (T*)v_cache, max_ctx, scale, lora, pf,
                   max(0, n_tok * heads - 3 * sm_count()));
}

extern "C" int slx_rope_attention_decode(int dtype, void* out, int ldo, const void* qkv,
                                            int ld_qkv, int n_tok, int heads, int kv_heads,
                                            int head_dim, const int32_t* tok_pos,
                                            const int32_t* tok_seq, const float* cos_tab,
                                            const float* sin_tab, int max_pos, void* k_cache,
                                            void* v_cache, int max_ctx, int pool_seqs,
                                            const slx_lora_delta* lora, const slx_l2_prefetch* pf,
                                            void* stream) {
  SLX_CHECK_ARG(n_tok >= 0 && heads > 0 && kv_heads > 0 && heads % kv_heads == 0 &&
                ld_qkv >= (heads + 2 * kv_heads) * head_dim && ldo >= heads * head_dim && out &&
                qkv && tok_pos && tok_seq && cos_tab && sin_tab && k_cache && v_cache &&
                max_pos > 0 && max_ctx > 0 && pool_seqs >= 0);
  SLX_CHECK_ARG(ldo % 8 == 0 && ld_qkv % 8 == 0 && delta_valid(lora));
  SLX_CHECK_ALIGN(k_cache, 16);
  SLX_CHECK_ALIGN(v_cache, 16);
  if (head_dim != 64 && head_dim != 128) return SLX_ERR_UNSUPPORTED;
  if (n_tok == 0) return SLX_OK;
  const float scale = 1.4426950408889634f / sqrtf((float)head_dim);
  const DeltaArgs la = delta_args(lora);
  const PfArgs pa = pf_args(pf);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == SLX_DT_BF16 && heads == kv_heads && pool_seqs > 0 && ld_qkv % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(qkv) & 15) == 0)
    return attn_decode_pipe_launch(out, ldo, qkv, ld_qkv, n_tok, heads, head_dim, tok_pos, tok_seq,
                                   cos_tab, sin_tab, k_cache, v_cache, max_ctx,
                                   (long long)pool_seqs * kv_heads * max_ctx, scale, la, pa, s);
  if (dtype == SLX_DT_BF16)
    return head_dim == 64 ? launch_rope_attn<bf16, 64>(out, ldo, qkv, ld_qkv, n_tok, heads, kv_heads, tok_pos, tok_seq, cos_tab, sin_tab, k_cache, v_cache, max_ctx, scale, la, pa, s)
                          : launch_rope_attn<bf16, 128>(out, ldo, qkv, ld_qkv, n_tok, heads, kv_heads, tok_pos, tok_seq, cos_tab, sin_tab, k_cache, v_cache, max_ctx, scale, la, pa, s);
  if (dtype == SLX_DT_F32)
    return head_dim == 64 ? launch_rope_attn<float, 64>(out, ldo, qkv, ld_qkv, n_tok, heads, kv_heads, tok_pos, tok_seq, cos_tab, sin_tab, k_cache, v_cache, max_ctx, scale, la, pa, s)
                          : launch_rope_attn<float, 128>(out, ldo, qkv, ld_qkv, n_tok, heads, kv_heads, tok_pos, tok_seq, cos_tab, sin_tab, k_cache, v_cache, max_ctx, scale, la, pa, s);
  return SLX_ERR_INVALID;
}
