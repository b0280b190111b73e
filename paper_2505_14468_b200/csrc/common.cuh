// Shared device/host helpers for libslora_b200 (sm_100a only).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/slora_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libslora_b200 targets sm_100a only"
#endif

namespace slx {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------- host-side status plumbing
#define SLX_CHECK_ARG(cond)                      \
  do {                                           \
    if (!(cond)) return SLX_ERR_INVALID;         \
  } while (0)
#define SLX_CHECK_ALIGN(ptr, n)                                          \
  do {                                                                   \
    if ((reinterpret_cast<uintptr_t>(ptr) % (n)) != 0) return SLX_ERR_ALIGN; \
  } while (0)
// Clear a stale (non-sticky) error left by an earlier unrelated runtime call so that the
// check after our launch reports only our launch.
#define SLX_CLEAR_STALE() (void)cudaGetLastError()
#define SLX_LAUNCH_CHECK()                                   \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return SLX_ERR_CUDA;              \
  } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------- conversions
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f32<bf16>(float v) { return __float2bfloat16_rn(v); }

// 8 consecutive elements <-> 8 floats. bf16: one 16 B load; float: two 16 B loads.
template <typename T> struct Vec8;
template <> struct Vec8<bf16> {
  __device__ __forceinline__ static void load(const bf16* p, float* f) {
    uint4 u = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ __forceinline__ static void store(bf16* p, const float* f) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = u;
  }
};
template <> struct Vec8<float> {
  __device__ __forceinline__ static void load(const float* p, float* f) {
    float4 a = *reinterpret_cast<const float4*>(p);
    float4 b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
  __device__ __forceinline__ static void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
};

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Cached per-device attributes (read once; no other global mutable state).
int sm_count();

}  // namespace slx

// ---------------------------------------------------------------- fused LoRA expand (slx_lora_delta)
namespace slx {
struct DeltaArgs {
  const float* v;
  int ldv;
  const int32_t* tok_slot;
  const int32_t* slot_rank;
  const float* slot_scale;
  int max_rank, n_targets;
  int v_slot_stride;   // v column of (target i, slot s, j) = v_col_off[i] + s * v_slot_stride + j
  const uint64_t* b_ptrs[SLX_LORA_MAX_TARGETS];
  int v_col_off[SLX_LORA_MAX_TARGETS], y_col_off[SLX_LORA_MAX_TARGETS], d_out[SLX_LORA_MAX_TARGETS];
};
inline DeltaArgs delta_args(const slx_lora_delta* d) {
  DeltaArgs a{};
  if (d == nullptr) return a;
  a.v = d->v; a.ldv = d->ldv; a.tok_slot = d->tok_slot; a.slot_rank = d->slot_rank;
  a.slot_scale = d->slot_scale; a.max_rank = d->max_rank; a.n_targets = d->n_targets;
  a.v_slot_stride = d->v_slot_stride;
  for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
    a.b_ptrs[i] = i < d->n_targets ? d->b_ptrs[i] : nullptr;
    a.v_col_off[i] = d->v_col_off[i]; a.y_col_off[i] = d->y_col_off[i]; a.d_out[i] = d->d_out[i];
  }
  return a;
}
inline bool delta_valid(const slx_lora_delta* d, bool v_optional = false) {
  if (d == nullptr) return true;
  if (d->n_targets < 0 || d->n_targets > SLX_LORA_MAX_TARGETS) return false;
  if (d->n_targets == 0) return true;
  if ((!d->v && !v_optional) || !d->tok_slot || !d->slot_rank || !d->slot_scale || d->max_rank <= 0 || (d->v && d->ldv <= 0))
    return false;
  // 16-byte v / B vectors: ldv, offsets, max_rank multiples of 4 / 8; v 16-byte aligned
  if (d->ldv % 4 || d->max_rank % 8 || (reinterpret_cast<uintptr_t>(d->v) & 15)) return false;
  if (d->v_slot_stride < 0 || d->v_slot_stride % 4) return false;
  for (int i = 0; i < d->n_targets; ++i)
    if (!d->b_ptrs[i] || d->d_out[i] <= 0 || d->y_col_off[i] < 0 || d->v_col_off[i] < 0 ||
        d->v_col_off[i] % 4)
      return false;
  return true;
}
// Per-token view: slot, rank, scale resolved once.
struct DeltaTok {
  int slot, rank;
  float scale;
  const float* vrow;
};
__device__ __forceinline__ DeltaTok delta_tok(const DeltaArgs& d, int t) {
  DeltaTok k{-1, 0, 0.f, nullptr};
  if (d.n_targets == 0) return k;
  k.slot = d.tok_slot[t];
  if (k.slot >= 0) {
    k.rank = min(d.slot_rank[k.slot], d.max_rank);
    k.scale = d.slot_scale[k.slot];
    k.vrow = d.v ? d.v + (size_t)t * d.ldv : nullptr;
  }
  return k;
}
// LoRA delta of row column `col` (0 when no target covers it / no adapter).
__device__ __forceinline__ float delta_dot(const DeltaTok& k, const uint64_t* b_tab, int v_off, int n,
                                           int v_slot_stride) {
  const bf16* B = reinterpret_cast<const bf16*>(b_tab[k.slot]);
  if (B == nullptr) return 0.f;
  const float* vr = k.vrow + v_off + k.slot * v_slot_stride;
  const bf16* br = B + (size_t)n * k.rank;   // rank % 8 == 0 (pool invariant): 16 B rows
  float acc = 0.f;
  for (int j = 0; j < k.rank; j += 8) {
    float b[8];
    Vec8<bf16>::load(br + j, b);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fmaf(vr[j + u] * k.scale, b[u], acc);
  }
  return acc;
}
// Register-resident fast path (rank <= 8 * RV): the B row of output column `col` is fetched
// before the PDL wait (adapters are static); after it, the CTA stages scale * v of every target
// once in shared memory (delta_stage_v) and each thread finishes its columns from there.
template <int RV>
struct DeltaRow {
  uint4 b[RV];
  int ti;   // target index (-1: no delta)
};
template <int RV>
__device__ __forceinline__ void delta_prefetch(const DeltaArgs& d, const DeltaTok& k, int col,
                                               DeltaRow<RV>& r) {
  r.ti = -1;
  if (k.slot < 0 || k.rank == 0) return;
#pragma unroll
  for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {
    const int n = col - d.y_col_off[i];
    if (r.ti < 0 && i < d.n_targets && n >= 0 && n < d.d_out[i]) {
      const bf16* B = reinterpret_cast<const bf16*>(__ldg(&d.b_ptrs[i][k.slot]));
      if (B != nullptr) {
        r.ti = i;
        const uint4* src = reinterpret_cast<const uint4*>(B + (size_t)n * k.rank);
#pragma unroll
        for (int j = 0; j < RV; ++j) r.b[j] = j * 8 < k.rank ? __ldg(src + j) : make_uint4(0, 0, 0, 0);
      }
    }
  }
}
constexpr int DELTA_VS = SLX_LORA_MAX_TARGETS * 64;   // staged floats (rank <= 64)
// vs[i * 64 + j] = v[t, v_col_off[i] + slot * v_slot_stride + j] * scale  (j < rank), cooperative.
__device__ __forceinline__ void delta_stage_v(const DeltaArgs& d, const DeltaTok& k, float* vs,
                                              int tid, int nthreads) {
  if (k.slot < 0 || k.rank == 0) return;
  for (int e = tid; e < d.n_targets * 64; e += nthreads) {
    const int i = e >> 6, j = e & 63;
    int off = 0;
#pragma unroll
    for (int q = 0; q < SLX_LORA_MAX_TARGETS; ++q)
      if (q == i) off = d.v_col_off[q];
    if (j < k.rank) vs[e] = k.vrow[off + k.slot * d.v_slot_stride + j] * k.scale;
  }
}
// delta = sum_j vs[j] * B[j], sequential fmaf (bit-identical to delta_col)
template <int RV>
__device__ __forceinline__ float delta_finish(const DeltaTok& k, const DeltaRow<RV>& r, const float* vs) {
  if (r.ti < 0) return 0.f;
  const float* v = vs + r.ti * 64;
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < RV; ++j) {
    if (j * 8 < k.rank) {
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&r.b[j]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 f = __bfloat1622float2(h2[u]);
        acc = fmaf(v[8 * j + 2 * u], f.x, acc);
        acc = fmaf(v[8 * j + 2 * u + 1], f.y, acc);
      }
    }
  }
  return acc;
}

__device__ __forceinline__ float delta_col(const DeltaArgs& d, const DeltaTok& k, int col) {
  if (k.slot < 0 || k.rank == 0) return 0.f;
  float res = 0.f;
  bool hit = false;
#pragma unroll
  for (int i = 0; i < SLX_LORA_MAX_TARGETS; ++i) {   // static indices: params stay in the cbank
    const int n = col - d.y_col_off[i];
    if (!hit && i < d.n_targets && n >= 0 && n < d.d_out[i]) {
      hit = true;
      res = delta_dot(k, d.b_ptrs[i], d.v_col_off[i], n, d.v_slot_stride);
    }
  }
  return res;
}
}  // namespace slx

// ---------------------------------------------------------------- L2 prefetch (slx_l2_prefetch)
namespace slx {
struct PfArgs {
  const char* ptr[2];
  unsigned long long bytes[2];
};
inline PfArgs pf_args(const slx_l2_prefetch* p) {
  PfArgs a{};
  if (p == nullptr) return a;
  for (int i = 0; i < 2; ++i) {
    a.ptr[i] = static_cast<const char*>(p->ptr[i]);
    a.bytes[i] = p->ptr[i] ? (p->bytes[i] & ~15ull) : 0;
  }
  return a;
}
// Part `part` of `parts` of both regions, as bulk L2 prefetches of <= 64 KB (one thread).
__device__ __forceinline__ void l2_prefetch_part(const PfArgs& pf, int part, int parts) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const unsigned long long n = pf.bytes[r];
    if (n == 0) continue;
    const unsigned long long per = ((n + parts - 1) / parts + 15) & ~15ull;
    unsigned long long lo = per * part, hi = lo + per;
    hi = hi > n ? n : hi;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    for (unsigned long long o = lo; o < hi; o += 65536) {
      const unsigned sz = (unsigned)((hi - o) < 65536 ? (hi - o) : 65536);
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(pf.ptr[r] + o),
                   "r"(sz), "l"(pol)
                   : "memory");
    }
  }
}
}  // namespace slx

// ---------------------------------------------------------------- split-K pieces (slx_splitk_in)
namespace slx {
struct SplitArgs {
  const float* part;
  int splits, bm, n_main;
};
inline SplitArgs split_args(const slx_splitk_in* s) {
  SplitArgs a{};
  if (s) { a.part = s->part; a.splits = s->splits; a.bm = s->bm; a.n_main = s->n_main; }
  return a;
}
// sum over the pieces (in order) of columns [col, col + 8) of row m (col % 8 == 0)
__device__ __forceinline__ void split_sum8(const SplitArgs& sa, int m, int col, float* out) {
  const size_t piece = (size_t)sa.bm * 256;
  const float* p = sa.part + (size_t)(col >> 8) * sa.splits * piece +
                   ((size_t)((col & 255) >> 4) * sa.bm + m) * 16 + (col & 15);
#pragma unroll
  for (int e = 0; e < 8; ++e) out[e] = 0.f;
  for (int i0 = 0; i0 < sa.splits; i0 += 8) {   // pieces in order, 8 loads in flight
    float4 q[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i0 + i < sa.splits) {
        q[i][0] = __ldcg(reinterpret_cast<const float4*>(p + (i0 + i) * piece));
        q[i][1] = __ldcg(reinterpret_cast<const float4*>(p + (i0 + i) * piece) + 1);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i0 + i < sa.splits) {
        out[0] += q[i][0].x; out[1] += q[i][0].y; out[2] += q[i][0].z; out[3] += q[i][0].w;
        out[4] += q[i][1].x; out[5] += q[i][1].y; out[6] += q[i][1].z; out[7] += q[i][1].w;
      }
    }
  }
}
__device__ __forceinline__ float split_sum1(const SplitArgs& sa, int m, int col) {
  const size_t piece = (size_t)sa.bm * 256;
  const float* p = sa.part + (size_t)(col >> 8) * sa.splits * piece +
                   ((size_t)((col & 255) >> 4) * sa.bm + m) * 16 + (col & 15);
  float s = 0.f;
  for (int i0 = 0; i0 < sa.splits; i0 += 8) {   // 8 loads in flight, summed in piece order
    float q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = i0 + i < sa.splits ? __ldcg(p + (i0 + i) * piece) : 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i0 + i < sa.splits) s += q[i];
  }
  return s;
}
}  // namespace slx

// ---------------------------------------------------------------- launch plumbing (PDL + clusters)
namespace slx {

// Programmatic dependent launch: every kernel of the library calls pdl_wait() before it
// touches global memory produced or consumed by earlier kernels on the stream, and
// pdl_trigger() only AFTER its own pdl_wait(), so the next kernel's prologue (barrier init,
// TMEM alloc, weight prefetch) overlaps this kernel's body.  Invariant this buys: when a
// kernel of the library starts, every library kernel two or more launches back on the
// stream has completed, so data they produced (e.g. the step's LoRA plan) may be read
// before this kernel's own pdl_wait().  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}


template <typename... KArgs, typename... Args>
inline int launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[2];
  unsigned n = 0;
  attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster_x > 1) {
    attrs[n].id = cudaLaunchAttributeClusterDimension;
    attrs[n].val.clusterDim.x = cluster_x;
    attrs[n].val.clusterDim.y = 1;
    attrs[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attrs;
  cfg.numAttrs = n;
  (void)cudaGetLastError();
  if (cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) != cudaSuccess) return SLX_ERR_CUDA;
  return cudaGetLastError() == cudaSuccess ? SLX_OK : SLX_ERR_CUDA;
}

}  // namespace slx
