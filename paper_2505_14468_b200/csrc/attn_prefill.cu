// Prefill attention on the 5th-gen tensor cores: causal flash attention over the KV pool with
// tcgen05.mma (TMEM accumulators) fed by TMA, warp-specialised, persistent, two query tiles
// per CTA in ping-pong.
//
// Work: a tile is <= 128 queries of one prefill segment; an item is (tile a, tile b, head) with
// tile b the segment's tile just before tile a (its keys a prefix of a's), so both tiles stream
// the SAME K/V blocks (b stops two 64-key blocks earlier).  Items are ordered longest first and
// CTA c runs items c, c + G, ... (G = #SMs).
//
// Per tile t in {a, b} (128 query rows = the 128 TMEM lanes, head_dim 128, key blocks of 64):
//   S_j = Q_t . K_j^T     tcgen05.mma M128 N64 K16 x8 (K-major, 128B-swizzled TMA boxes) into one
//                         of the tile's two TMEM S buffers (64 columns each)
//   P_j = exp2(S_j * scale - m)   softmax warpgroup t: thread r owns query row r (tcgen05.ld of
//                         its lane), causal mask, online max with LAZY rescale (the running max
//                         used for P and O/l only moves when a row's max grows by > 2^8), P
//                         written to shared memory as the next MMA's K-major A operand
//   O_t += P_j . V_j      tcgen05.mma M128 N128 K16 x4, V_j as an MN-major B operand
// Two softmax warpgroups (one per tile) give every SM sub-partition two softmax warps, so one
// warp's exp2 / max / pack chain overlaps the other's, and each tile has its own MMA issuer
// (P.V(j), then S(j+2)) — the tensor core computes one tile's scores while the other tile's
// softmax runs; scores run two blocks ahead of the softmax.  Roles (352
// threads): warp 0 lane 0 TMA producer (Q_a, Q_b once per item, K and V through 4-stage rings
// shared by both tiles; one P buffer per tile), warps 1 / 2 lane 0 the MMA issuers of tiles a / b
// (one issuer would convoy the tiles), warps 3-6 softmax + epilogue of tile a, warps 7-10 of
// tile b (warp w reads TMEM lanes 32 (w % 4) ..).  TMEM: tile t at 256 t: S0 [0, 64), S1 [64, 128), O [128, 256).
// Query i of a tile starting at cache position p0 attends positions 0..p0+i (prefix + causal),
// k/v already appended by slx_rope_kv_write.
#include "common.cuh"
#include "gemm_host.h"
#include "tc_ptx.cuh"

namespace slx {
namespace {

constexpr int FT_BQ = 128, FT_BK = 64, FT_D = 128;
constexpr int FT_KST = 4, FT_VST = 4;
constexpr int FT_PBUF = 1;                            // P buffers per tile
constexpr int FT_THREADS = 352;
constexpr int FT_Q_BYTES = FT_BQ * FT_D * 2;          // 32 KB: two [128][64] boxes
constexpr int FT_KV_BYTES = FT_BK * FT_D * 2;         // 16 KB: two [64][64] boxes
constexpr int FT_P_BYTES = FT_BQ * FT_BK * 2;         // 16 KB: [128][64]
constexpr int FT_OFF_K = 2 * FT_Q_BYTES;
constexpr int FT_OFF_V = FT_OFF_K + FT_KST * FT_KV_BYTES;
constexpr int FT_OFF_P = FT_OFF_V + FT_VST * FT_KV_BYTES;     // [tile][FT_PBUF][16 KB]
constexpr int FT_OFF_BAR = FT_OFF_P + 2 * FT_PBUF * FT_P_BYTES;
// per tile: q_full, q_empty, s_full[2], s_free[2], p_full[2], p_empty[2], o_empty = 11
constexpr int FT_TBAR = 11;
constexpr int FT_NBAR = 2 * FT_KST + 2 * FT_VST + 2 * FT_TBAR + 1;
constexpr size_t FT_SMEM = 1024 + FT_OFF_BAR + FT_NBAR * 8 + 16;
constexpr uint32_t FT_TMEM_COLS = 512;
constexpr float FT_RESCALE_LOG2 = 8.0f;   // lazy rescale threshold (P <= 2^8 stays exact in fp32/bf16)

struct FtTile {
  int tok0, nq, seq, pos0;
};
struct FtItem {
  int ta, tb, h, pad;
};

struct FtArgs {
  bf16* out;
  int ldo;
  const FtTile* tiles;
  const FtItem* items;
  int n_items;
  int H, Hkv, max_ctx;
  float scale_log2;
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// (d0, d1) = (a0, a1) * (b, b) + (c, c) as one FFMA2
__device__ __forceinline__ void fma2s(float& d0, float& d1, float a0, float a1, float b, float c) {
  uint64_t d, av, bv, cv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(cv) : "f"(c));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(av), "l"(bv), "l"(cv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(d));
}
// (s0, s1) += (a0, a1) as one FADD2
__device__ __forceinline__ void add2(float& s0, float& s1, float a0, float a1) {
  uint64_t d, sv, av;
  asm("mov.b64 %0, {%1, %2};" : "=l"(sv) : "f"(s0), "f"(s1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(av) : "f"(a0), "f"(a1));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(sv), "l"(av));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(s0), "=f"(s1) : "l"(d));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])),
      "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])),
      "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// MN-major (V as the B operand: N = head dim contiguous) 128B-swizzled descriptor: 64-element
// MN atoms `lbo` bytes apart, 8-row K groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ int n_blocks(const FtTile& t) { return (t.pos0 + t.nq + FT_BK - 1) / FT_BK; }

__global__ void __launch_bounds__(FT_THREADS, 1)
flash_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                const __grid_constant__ CUtensorMap tv, const FtArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + FT_OFF_BAR);
  uint64_t* k_full = bar;
  uint64_t* k_empty = k_full + FT_KST;
  uint64_t* v_full = k_empty + FT_KST;
  uint64_t* v_empty = v_full + FT_VST;
  uint64_t* tb0 = v_empty + FT_VST;   // per-tile barriers: tb0 + FT_TBAR * t
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tb0 + 2 * FT_TBAR);
  auto q_full = [&](int t) { return tb0 + FT_TBAR * t; };
  auto q_empty = [&](int t) { return tb0 + FT_TBAR * t + 1; };
  auto s_full = [&](int t, int b) { return tb0 + FT_TBAR * t + 2 + b; };
  auto s_free = [&](int t, int b) { return tb0 + FT_TBAR * t + 4 + b; };
  auto p_full = [&](int t, int b) { return tb0 + FT_TBAR * t + 6 + b; };
  auto p_empty = [&](int t, int b) { return tb0 + FT_TBAR * t + 8 + b; };
  auto o_empty = [&](int t) { return tb0 + FT_TBAR * t + 10; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    tc::tma_prefetch_desc(&tq);
    tc::tma_prefetch_desc(&tk);
    tc::tma_prefetch_desc(&tv);
    // K / V stages are released by both tiles' MMA warps (every block, used or not)
    for (int s = 0; s < FT_KST; ++s) { tc::mbar_init(&k_full[s], 1); tc::mbar_init(&k_empty[s], 2); }
    for (int s = 0; s < FT_VST; ++s) { tc::mbar_init(&v_full[s], 1); tc::mbar_init(&v_empty[s], 2); }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(q_full(t), 1);
      tc::mbar_init(q_empty(t), 1);
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(s_full(t, b), 1);
        tc::mbar_init(s_free(t, b), 4);
        tc::mbar_init(p_full(t, b), 4);
        tc::mbar_init(p_empty(t, b), 1);
      }
      tc::mbar_init(o_empty(t), 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, FT_TMEM_COLS);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();   // q (rotated) and the appended k/v come from the previous kernels
  pdl_trigger();
  const int group = a.H / a.Hkv;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_q = tc::policy_evict_first();
      const uint64_t pol_kv = tc::policy_evict_last();   // re-read by the segment's other tiles
      int qi[2] = {0, 0}, ki = 0, vi = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
        const FtItem item = a.items[it];
        const FtTile ta = a.tiles[item.ta];
        const int row0 = (ta.seq * a.Hkv + item.h / group) * a.max_ctx;
        for (int t = 0; t < 2; ++t) {
          const int ti = t == 0 ? item.ta : item.tb;
          if (ti < 0) continue;
          const int tok0 = a.tiles[ti].tok0;
          tc::mbar_wait(q_empty(t), (qi[t] & 1) ^ 1);
          uint8_t* qd = sm + t * FT_Q_BYTES;
          tc::mbar_arrive_expect_tx(q_full(t), FT_Q_BYTES);
          tc::tma_load_2d(qd, &tq, q_full(t), item.h * FT_D, tok0, pol_q);
          tc::tma_load_2d(qd + FT_Q_BYTES / 2, &tq, q_full(t), item.h * FT_D + 64, tok0, pol_q);
          ++qi[t];
        }
        const int nb = n_blocks(ta);
        for (int j = 0; j < nb; ++j) {
          const int ks = ki % FT_KST;
          tc::mbar_wait(&k_empty[ks], ((ki / FT_KST) & 1) ^ 1);
          uint8_t* kd = sm + FT_OFF_K + ks * FT_KV_BYTES;
          tc::mbar_arrive_expect_tx(&k_full[ks], FT_KV_BYTES);
          tc::tma_load_2d(kd, &tk, &k_full[ks], 0, row0 + j * FT_BK, pol_kv);
          tc::tma_load_2d(kd + FT_KV_BYTES / 2, &tk, &k_full[ks], 64, row0 + j * FT_BK, pol_kv);
          ++ki;
          const int vs = vi % FT_VST;
          tc::mbar_wait(&v_empty[vs], ((vi / FT_VST) & 1) ^ 1);
          uint8_t* vd = sm + FT_OFF_V + vs * FT_KV_BYTES;
          tc::mbar_arrive_expect_tx(&v_full[vs], FT_KV_BYTES);
          tc::tma_load_2d(vd, &tv, &v_full[vs], 0, row0 + j * FT_BK, pol_kv);
          tc::tma_load_2d(vd + FT_KV_BYTES / 2, &tv, &v_full[vs], 64, row0 + j * FT_BK, pol_kv);
          ++vi;
        }
      }
    }
    __syncwarp();
  } else if (warp <= 2) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuers
      // warp 1 issues tile a's MMAs, warp 2 tile b's: each tile's S / P.V pipeline advances at
      // its own softmax's pace (one issuer would convoy them).  Both walk every K / V block of
      // the item and release it (count-2 barriers); the full-barrier waits keep a warp from
      // releasing a stage's next use before the other released this one.
      const int t = warp - 1;
      const uint32_t id_s = tc::idesc_bf16_f32(FT_BQ, FT_BK);
      const uint32_t id_o = tc::idesc_bf16_f32(FT_BQ, FT_D) | (1u << 16);   // B (V) MN-major
      const uint32_t sq = tc::smem_u32(sm + t * FT_Q_BYTES);
      int qi = 0, si = 0, pi = 0, oi = 0, ki = 0, vi = 0;
      for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
        const FtItem item = a.items[it];
        const int nb = n_blocks(a.tiles[item.ta]);
        const int ti = t == 0 ? item.ta : item.tb;
        const int mine = ti >= 0 ? n_blocks(a.tiles[ti]) : 0;
        if (mine > 0) tc::mbar_wait(q_full(t), qi & 1);
        // scores of block jj (this tile), or just the release of K_jj
        auto issue_s = [&](int jj) {
          const int ks = ki % FT_KST;
          tc::mbar_wait(&k_full[ks], (ki / FT_KST) & 1);
          if (jj < mine) {
            const uint32_t kb = tc::smem_u32(sm + FT_OFF_K + ks * FT_KV_BYTES);
            const int sb = si & 1;
            tc::mbar_wait(s_free(t, sb), ((si >> 1) & 1) ^ 1);
            tc::fence_after_sync();
#pragma unroll
            for (int ks16 = 0; ks16 < FT_D / 16; ++ks16) {
              const uint32_t off = (uint32_t)((ks16 >> 2) * (FT_Q_BYTES / 2) + (ks16 & 3) * 32);
              const uint32_t offk = (uint32_t)((ks16 >> 2) * (FT_KV_BYTES / 2) + (ks16 & 3) * 32);
              tc::mma_bf16_ss(tmem + 256 * t + sb * FT_BK, tc::smem_desc_sw128(sq + off),
                              tc::smem_desc_sw128(kb + offk), id_s, ks16 > 0 ? 1u : 0u);
            }
            tc::mma_commit(s_full(t, sb));
            ++si;
            if (jj == mine - 1) {
              tc::mma_commit(q_empty(t));
              ++qi;
            }
          }
          tc::mma_commit(&k_empty[ks]);
          ++ki;
        };
        // scores run two blocks ahead of the softmax (two S buffers)
        int sj = 0;
        for (; sj < 2 && sj < nb; ++sj) issue_s(sj);
        for (int j = 0; j < nb; ++j) {
          const int vs = vi % FT_VST;
          tc::mbar_wait(&v_full[vs], (vi / FT_VST) & 1);
          if (j < mine) {   // O += P(j) . V(j)
            const int pb = pi % FT_PBUF;
            tc::mbar_wait(p_full(t, pb), (pi / FT_PBUF) & 1);
            if (j == 0) {
              tc::mbar_wait(o_empty(t), (oi & 1) ^ 1);   // the previous tile's epilogue read O
              ++oi;
            }
            tc::fence_after_sync();
            const uint32_t va = tc::smem_u32(sm + FT_OFF_V + vs * FT_KV_BYTES);
            const uint32_t pa = tc::smem_u32(sm + FT_OFF_P + (FT_PBUF * t + pb) * FT_P_BYTES);
#pragma unroll
            for (int kk = 0; kk < FT_BK / 16; ++kk)
              tc::mma_bf16_ss(tmem + 256 * t + 128, tc::smem_desc_sw128(pa + kk * 32),
                              desc_mn_sw128(va + kk * 2048, FT_KV_BYTES / 2), id_o,
                              (j > 0 || kk > 0) ? 1u : 0u);
            tc::mma_commit(p_empty(t, pb));
            ++pi;
          }
          tc::mma_commit(&v_empty[vs]);
          ++vi;
          if (sj < nb) issue_s(sj++);
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int t = (warp - 3) >> 2;                       // tile slot of this warpgroup
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;                        // query row = TMEM lane
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t tbase = tmem + 256 * t;
    const float sl2 = a.scale_log2;
    int si = 0, pi = 0;
    for (int it = blockIdx.x; it < a.n_items; it += gridDim.x) {
      const FtItem item = a.items[it];
      const int ti = t == 0 ? item.ta : item.tb;
      if (ti < 0) continue;
      const FtTile tl = a.tiles[ti];
      const int nb = n_blocks(tl);
      const int n_keys = tl.pos0 + tl.nq;
      const int lim = min(tl.pos0 + r, n_keys - 1);   // last visible key of this row
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j) {
        const int sb = si & 1;
        tc::mbar_wait(s_full(t, sb), (si >> 1) & 1);
        tc::fence_after_sync();
        float s[FT_BK];
        tmem_ld32(tbase + lane_off + sb * FT_BK, s);
        tmem_ld32(tbase + lane_off + sb * FT_BK + 32, s + 32);
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(s_free(t, sb));
        ++si;
        const int k0 = j * FT_BK;
        if (k0 + FT_BK - 1 > lim) {   // only blocks on the diagonal (or past the end) mask keys
#pragma unroll
          for (int c = 0; c < FT_BK; ++c)
            if (k0 + c > lim) s[c] = -INFINITY;
        }
        float mq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // four independent 3-input max chains
          mq[q] = fmaxf(s[16 * q], s[16 * q + 1]);
#pragma unroll
          for (int c = 16 * q + 2; c < 16 * q + 16; c += 2) mq[q] = max3f(mq[q], s[c], s[c + 1]);
        }
        const float mx = max3f(fmaxf(mq[0], mq[1]), mq[2], mq[3]);
        const float m_new = fmaxf(m_used, mx);
        if (j == 0) {
          m_used = m_new;
        } else {
          const bool need = (m_new - m_used) * sl2 > FT_RESCALE_LOG2;
          if (__any_sync(0xffffffffu, need)) {
            // O holds P_0..P_{j-1} . V: wait for the last PV before rescaling it in TMEM
            const int lp = pi - 1;
            tc::mbar_wait(p_empty(t, lp % FT_PBUF), (lp / FT_PBUF) & 1);
            tc::fence_after_sync();
            const float corr = need ? ex2_approx((m_used - m_new) * sl2) : 1.f;
            if (need) {
              m_used = m_new;
              l *= corr;
            }
#pragma unroll 1
            for (int c0 = 0; c0 < FT_D; c0 += 32) {
              float o[32];
              tmem_ld32(tbase + lane_off + 128 + c0, o);
#pragma unroll
              for (int e = 0; e < 32; ++e) o[e] *= corr;
              tmem_st32(tbase + lane_off + 128 + c0, o);
            }
          }
        }
        const float msl = m_used * sl2;
        uint32_t pk[FT_BK / 2];
        float ls0 = 0.f, ls1 = 0.f;
#pragma unroll
        for (int c = 0; c < FT_BK; c += 2) {
          float x0, x1;
          fma2s(x0, x1, s[c], s[c + 1], sl2, -msl);
          const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
          add2(ls0, ls1, p0, p1);
          pk[c / 2] = pack2(p0, p1);
        }
        l += ls0 + ls1;
        const int pb = pi % FT_PBUF;
        if (pi >= FT_PBUF)   // the P.V that last read this buffer has completed
          tc::mbar_wait(p_empty(t, pb), ((pi - FT_PBUF) / FT_PBUF) & 1);
        uint8_t* prow = sm + FT_OFF_P + (FT_PBUF * t + pb) * FT_P_BYTES + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(p_full(t, pb));
        ++pi;
      }
      // epilogue: O / l of this row -> bf16 out
      const int lp = pi - 1;
      tc::mbar_wait(p_empty(t, lp % FT_PBUF), (lp / FT_PBUF) & 1);
      tc::fence_after_sync();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16* orow = a.out + (size_t)(tl.tok0 + r) * a.ldo + (size_t)item.h * FT_D;
#pragma unroll 1
      for (int c0 = 0; c0 < FT_D; c0 += 32) {
        float o[32];
        tmem_ld32(tbase + lane_off + 128 + c0, o);
        if (r < tl.nq) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(orow + c0 + 8 * q) =
                make_uint4(pack2(o[8 * q] * inv, o[8 * q + 1] * inv),
                           pack2(o[8 * q + 2] * inv, o[8 * q + 3] * inv),
                           pack2(o[8 * q + 4] * inv, o[8 * q + 5] * inv),
                           pack2(o[8 * q + 6] * inv, o[8 * q + 7] * inv));
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(o_empty(t));
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, FT_TMEM_COLS);
  }
}

}  // namespace
}  // namespace slx

using namespace slx;

extern "C" size_t slx_flash_prefill_tile_bytes(void) { return sizeof(FtTile); }
extern "C" size_t slx_flash_prefill_item_bytes(void) { return sizeof(FtItem); }
extern "C" int slx_flash_prefill_tile_queries(void) { return FT_BQ; }

extern "C" int slx_attention_prefill(void* out, int ldo, const void* qkv, int ld_qkv, int n_tok,
                                     int heads, int kv_heads, int head_dim, const void* tiles,
                                     const void* items, int n_items, const void* k_cache,
                                     const void* v_cache, int max_ctx, int pool_seqs,
                                     void* stream) {
  SLX_CHECK_ARG(out && qkv && tiles && items && k_cache && v_cache && heads > 0 && kv_heads > 0 &&
                heads % kv_heads == 0 && n_items >= 0 && n_tok > 0 && max_ctx > 0 &&
                pool_seqs > 0 && ld_qkv >= (heads + 2 * kv_heads) * head_dim &&
                ldo >= heads * head_dim && ld_qkv % 8 == 0 && ldo % 8 == 0);
  if (head_dim != FT_D) return SLX_ERR_UNSUPPORTED;
  SLX_CHECK_ALIGN(qkv, 16);
  SLX_CHECK_ALIGN(out, 16);
  SLX_CHECK_ALIGN(k_cache, 16);
  SLX_CHECK_ALIGN(v_cache, 16);
  if (n_items == 0) return SLX_OK;
  const long long rows = (long long)pool_seqs * kv_heads * max_ctx;
  if (rows >= (1ll << 31)) return SLX_ERR_UNSUPPORTED;
  CUtensorMap mq, mk, mv;
  if (!make_tmap(&mq, qkv, n_tok, heads * head_dim, ld_qkv, FT_BQ) ||
      !make_tmap(&mk, k_cache, (int)rows, FT_D, FT_D, FT_BK) ||
      !make_tmap(&mv, v_cache, (int)rows, FT_D, FT_D, FT_BK))
    return SLX_ERR_CUDA;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(flash_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)FT_SMEM) != cudaSuccess)
      return SLX_ERR_CUDA;
    configured = true;
  }
  FtArgs a{};
  a.out = (bf16*)out; a.ldo = ldo; a.tiles = (const FtTile*)tiles; a.items = (const FtItem*)items;
  a.n_items = n_items; a.H = heads; a.Hkv = kv_heads; a.max_ctx = max_ctx;
  a.scale_log2 = 1.4426950408889634f / sqrtf((float)head_dim);
  const int grid = n_items < sm_count() ? n_items : sm_count();
  return launch_ex(flash_tc_kernel, dim3((unsigned)grid), dim3(FT_THREADS), FT_SMEM,
                   (cudaStream_t)stream, 1u, mq, mk, mv, a);
}
