// K3 (head_dim 128): backward as two tcgen05 kernels that keep their re-used operand in TMEM.
//
// Measured on B200 (tools/mma_rate.cu): a cta_group::1 SS-mode MMA with N=64 is bound by the
// 128 B/clk shared-memory operand path (48 instead of 32 cycles), while TS-mode MMAs (A from
// TMEM) run at the tensor floor for every N.  A fused backward must re-read the key/value
// tile from shared memory for every query tile and pays fp32 atomics for dQ; splitting it
// gives each kernel enough TMEM to hold the operand it re-uses:
//
//   dkdv kernel  one CTA per (128-key tile, head, subsequence), loop over 64-query tiles:
//                K, V rows are placed in TMEM once (A operands), then per tile
//                  S^T = K Q^T, dP^T = V dO^T          (TS, N = 64)
//                  P^T = exp2(S^T c - lse2), dS^T = P^T (dP^T - delta)   (8 compute warps)
//                  dV += P^T dO, dK += dS^T Q  (TS: P^T and dS^T written back to TMEM
//                  over the consumed S^T / dP^T columns)
//                TMEM: K 64 | V 64 | S^T/P^T 64 | dP^T/dS^T 64 | dV 128 | dK 128.
//   dq kernel    one CTA per (128-query tile, head, subsequence), loop over 64-key tiles:
//                Q, dO rows in TMEM; per tile S = Q K^T, dP = dO V^T (TS, N = 64, double
//                buffered), dS = P (dP - delta) written back to TMEM as bf16, dQ += dS K
//                (TS).  TMEM: Q 64 | dO 64 | S x2 128 | dP x2 128 | dQ 128.
//   No atomics: every gradient element has one owner CTA.
#include "osp_common.cuh"
#include "osp_internal.h"

namespace osp {
namespace {

constexpr int kThreads = 512;
constexpr int D = 128;

struct SplitArgs {
  const float* lse2;   // (n_seq, heads, seq_pad) log2-domain lse, +inf pads
  const float* delta;  // (n_seq, heads, seq_pad)
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  const __nv_bfloat16* dout;
  int64_t q_stride, k_stride, v_stride, do_stride;
  __nv_bfloat16* dq;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t dq_stride, dk_stride, dv_stride;
  const uint32_t* valid_bits;
  int words_per_seq;
  int seq_len, seq_pad, heads;
  float scale, scale_log2;
};

__device__ __forceinline__ void bulk_load_s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Copy one 128-d bf16 row (global, 16B aligned) into 64 TMEM columns of this thread's lane,
// the kind::f16 A-operand layout (column c = elements 2c, 2c+1).  Rows past the end -> 0.
__device__ __forceinline__ void row_to_tmem(uint32_t taddr, const __nv_bfloat16* row, bool ok) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t r[32];
    if (ok) {
      const uint4* src = reinterpret_cast<const uint4*>(row + h * 64);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = __ldg(src + i);
        r[4 * i + 0] = v.x;
        r[4 * i + 1] = v.y;
        r[4 * i + 2] = v.z;
        r[4 * i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = 0u;
    }
    tmem_st32(taddr + h * 32, r);
  }
}

// ============================================================================ dK / dV kernel
struct DkdvLayout {
  static constexpr int kStages = 4;
  static constexpr int kQ = 0;                          // stages x (64 q x 128 d) = 16 KB
  static constexpr int kDO = kQ + kStages * 16384;
  static constexpr int kStat = kDO + kStages * 16384;   // stages x (lse2[64], delta[64])
  static constexpr int kBar = kStat + kStages * 512;
  static constexpr int kSmem = kBar + 256;
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmDO,
                         const SplitArgs a) {
  using Ly = DkdvLayout;
  constexpr int NS = Ly::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_qf = bars + 0;       // [NS] Q, dO, stats landed
  uint64_t* bar_qe = bars + NS;      // [NS] stage free
  uint64_t* bar_kv = bars + 2 * NS;  // K, V rows in TMEM (256 arrivals)
  uint64_t* bar_s = bar_kv + 1;      // S^T ready
  uint64_t* bar_dp = bar_kv + 2;     // dP^T ready
  uint64_t* bar_p = bar_kv + 3;      // P^T in TMEM (256)
  uint64_t* bar_ds = bar_kv + 4;     // dS^T written into TMEM over dP^T (256)
  uint64_t* bar_fin = bar_kv + 5;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_kv + 6);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int seq = blockIdx.z;
  const int kv0 = blockIdx.x * 128;
  const int n_q = (a.seq_len + 63) / 64;

  if ((smem_u32(sm) & 1023) != 0) __trap();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(bar_qf + i, 1);
      mbar_init(bar_qe + i, 1);
    }
    mbar_init(bar_kv, 256);
    mbar_init(bar_s, 1);
    mbar_init(bar_dp, 1);
    mbar_init(bar_p, 256);
    mbar_init(bar_ds, 256);
    mbar_init(bar_fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tK = tmem, tV = tmem + 64, tS = tmem + 128, tDP = tmem + 192, tDV = tmem + 256,
                 tDK = tmem + 384;
  const int64_t sh = static_cast<int64_t>(seq) * a.heads + head;

  if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------------ TMA producer
      tma_prefetch(&tmQ);
      tma_prefetch(&tmDO);
      const float* lse2_g = a.lse2 + sh * a.seq_pad;
      const float* delta_g = a.delta + sh * a.seq_pad;
      for (int i = 0; i < n_q; ++i) {
        const int st = i % NS;
        mbar_wait(bar_qe + st, ((i / NS) & 1) ^ 1);
        mbar_expect_tx(bar_qf + st, 2 * 16384 + 512);
        for (int s = 0; s < 2; ++s) {
          tma_load_3d(sm + Ly::kQ + st * 16384 + s * 8192, &tmQ, bar_qf + st, head * D + s * 64,
                      i * 64, seq);
          tma_load_3d(sm + Ly::kDO + st * 16384 + s * 8192, &tmDO, bar_qf + st, head * D + s * 64,
                      i * 64, seq);
        }
        bulk_load_s(sm + Ly::kStat + st * 512, lse2_g + i * 64, 256, bar_qf + st);
        bulk_load_s(sm + Ly::kStat + st * 512 + 256, delta_g + i * 64, 256, bar_qf + st);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // -------------------------------------------------------------------- MMA issuer
    constexpr uint32_t kIdS = idesc_bf16(128, 64, 0, 0);    // S^T, dP^T (TS)
    constexpr uint32_t kIdKV = idesc_bf16(128, 128, 0, 1);  // dV (TS), dK (SS)
    const uint32_t tm = __shfl_sync(0xFFFFFFFFu, tmem, 0);
    const uint32_t mK = tm, mV = tm + 64, mS = tm + 128, mDP = tm + 192, mDV = tm + 256, mDK = tm + 384;
    const uint32_t q_base0 = smem_u32(sm + Ly::kQ);
    const uint32_t do_base0 = smem_u32(sm + Ly::kDO);
    if (elect_one()) {
      auto issue_s = [&](int i) {
        const uint32_t qb = q_base0 + (i % NS) * 16384;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(mS, mK + kk * 8, sdesc_sw128(qb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), kIdS,
                 kk > 0);
        tc_commit(bar_s);
      };
      auto issue_dp = [&](int i) {
        const uint32_t db = do_base0 + (i % NS) * 16384;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(mDP, mV + kk * 8, sdesc_sw128(db + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), kIdS,
                 kk > 0);
        tc_commit(bar_dp);
      };
      mbar_wait(bar_kv, 0);
      mbar_wait(bar_qf + 0, 0);
      tc_fence_after();
      issue_s(0);
      issue_dp(0);
      for (int i = 0; i < n_q; ++i) {
        const int st = i % NS;
        const int b = i & 1;
        const uint32_t qb = q_base0 + st * 16384;
        const uint32_t db = do_base0 + st * 16384;
        mbar_wait(bar_p, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(mDV, mS + kk * 8, sdesc_sw128(db + kk * 2048, 8192, 1024), kIdKV,
                 (i > 0 || kk > 0) ? 1u : 0u);
        if (i + 1 < n_q) {
          mbar_wait(bar_qf + (i + 1) % NS, ((i + 1) / NS) & 1);
          tc_fence_after();
          issue_s(i + 1);
        }
        // dK += dS^T Q with dS^T read from TMEM (written over the consumed dP^T columns)
        mbar_wait(bar_ds, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(mDK, mDP + kk * 8, sdesc_sw128(qb + kk * 2048, 8192, 1024), kIdKV,
                 (i > 0 || kk > 0) ? 1u : 0u);
        tc_commit(bar_qe + st);
        if (i + 1 < n_q) issue_dp(i + 1);
      }
      tc_commit(bar_fin);
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    // -------------------------------------------------------------------- compute warps:
    // thread = key row; warpgroup `half` owns query columns [32*half, 32*half+32)
    const int half = (warp - 4) >> 2;
    const int wq = warp & 3;
    const uint32_t la = static_cast<uint32_t>(wq * 32) << 16;
    const int krow = wq * 32 + lane;
    const int kglob = kv0 + krow;
    const bool in_range = kglob < a.seq_len;
    bool kvalid = in_range;
    if (kvalid && a.valid_bits) {
      const uint32_t* vb = a.valid_bits + static_cast<int64_t>(seq) * a.words_per_seq;
      kvalid = (__ldg(vb + (kglob >> 5)) >> (kglob & 31)) & 1u;
    }
    // K (warpgroup 0) / V (warpgroup 1) rows -> TMEM A operands
    if (half == 0)
      row_to_tmem(tK + la, a.k + (static_cast<int64_t>(seq) * a.seq_len + kglob) * a.k_stride +
                               static_cast<int64_t>(head) * D, in_range);
    else
      row_to_tmem(tV + la, a.v + (static_cast<int64_t>(seq) * a.seq_len + kglob) * a.v_stride +
                               static_cast<int64_t>(head) * D, in_range);
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(bar_kv);
    const float c = a.scale_log2;
    for (int i = 0; i < n_q; ++i) {
      const int st = i % NS;
      const float* lse_s = reinterpret_cast<const float*>(sm + Ly::kStat + st * 512) + half * 32;
      const float* del_s = lse_s + 64;
      mbar_wait(bar_qf + st, (i / NS) & 1);
      mbar_wait(bar_s, i & 1);
      tc_fence_after();
      float p[32];
      {
        uint32_t s0[32];
        tmem_ld32(tS + la + half * 32, s0);
        tmem_wait_ld(s0);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 l0 = *reinterpret_cast<const float4*>(lse_s + j4 * 4);
          p[j4 * 4 + 0] = ex2(fmaf(__uint_as_float(s0[j4 * 4 + 0]), c, -l0.x));
          p[j4 * 4 + 1] = ex2(fmaf(__uint_as_float(s0[j4 * 4 + 1]), c, -l0.y));
          p[j4 * 4 + 2] = ex2(fmaf(__uint_as_float(s0[j4 * 4 + 2]), c, -l0.z));
          p[j4 * 4 + 3] = ex2(fmaf(__uint_as_float(s0[j4 * 4 + 3]), c, -l0.w));
        }
      }
      if (!kvalid) {
#pragma unroll
        for (int j = 0; j < 32; ++j) p[j] = 0.f;
      }
      {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(p[2 * j], p[2 * j + 1]);
        tmem_st16(tS + la + half * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p);

      mbar_wait(bar_dp, i & 1);
      tc_fence_after();
      {
        uint32_t dp[32];
        tmem_ld32(tDP + la + half * 32, dp);
        tmem_wait_ld(dp);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 d2 = *reinterpret_cast<const float2*>(del_s + 2 * j);
          pk[j] = pack_bf16(p[2 * j] * (__uint_as_float(dp[2 * j]) - d2.x),
                            p[2 * j + 1] * (__uint_as_float(dp[2 * j + 1]) - d2.y));
        }
        // both warpgroups must finish reading dP^T before either overwrites it with dS^T
        named_bar_sync(1, 256);
        tmem_st16(tDP + la + half * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_ds);
    }
    // ------------------------------------------------------------------ epilogue: dV | dK
    mbar_wait(bar_fin, 0);
    tc_fence_after();
    const uint32_t base = (half == 0 ? tDV : tDK) + la;
    const float mul = half == 0 ? 1.f : a.scale;
    __nv_bfloat16* dst = (half == 0 ? a.dv : a.dk) +
                         (static_cast<int64_t>(seq) * a.seq_len + kglob) *
                             (half == 0 ? a.dv_stride : a.dk_stride) +
                         static_cast<int64_t>(head) * D;
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(base + cc * 32, o);
      tmem_wait_ld(o);
      if (in_range) {
        uint4 pk[4];
        uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pw[j] = pack_bf16(__uint_as_float(o[2 * j]) * mul, __uint_as_float(o[2 * j + 1]) * mul);
        uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
        for (int j = 0; j < 4; ++j) d4[j] = pk[j];
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================================ dQ kernel
struct DqLayout {
  static constexpr int kStages = 4;
  static constexpr int kK = 0;                      // stages x (64 keys x 128 d) = 16 KB
  static constexpr int kV = kK + kStages * 16384;
  static constexpr int kBar = kV + kStages * 16384;
  static constexpr int kSmem = kBar + 256;
};

__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       const SplitArgs a) {
  using Ly = DqLayout;
  constexpr int NS = Ly::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_kf = bars + 0;        // [NS] K_j, V_j landed
  uint64_t* bar_ke = bars + NS;       // [NS] stage free
  uint64_t* bar_qd = bars + 2 * NS;   // Q, dO rows in TMEM (256)
  uint64_t* bar_s = bar_qd + 1;       // [2] S_j ready
  uint64_t* bar_dp = bar_qd + 3;      // [2] dP_j ready
  uint64_t* bar_ds = bar_qd + 5;      // [2] dS_j in TMEM (256)
  uint64_t* bar_fin = bar_qd + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_qd + 9);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int seq = blockIdx.z;
  const int q0 = blockIdx.x * 128;
  const int n_kv = (a.seq_len + 63) / 64;

  if ((smem_u32(sm) & 1023) != 0) __trap();
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(bar_kf + i, 1);
      mbar_init(bar_ke + i, 1);
    }
    mbar_init(bar_qd, 256);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_s + i, 1);
      mbar_init(bar_dp + i, 1);
      mbar_init(bar_ds + i, 256);
    }
    mbar_init(bar_fin, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tQ = tmem, tDO = tmem + 64, tS = tmem + 128, tDP = tmem + 256, tDQ = tmem + 384;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NS;
        mbar_wait(bar_ke + st, ((j / NS) & 1) ^ 1);
        mbar_expect_tx(bar_kf + st, 2 * 16384);
        for (int s = 0; s < 2; ++s) {
          tma_load_3d(sm + Ly::kK + st * 16384 + s * 8192, &tmK, bar_kf + st, head * D + s * 64,
                      j * 64, seq);
          tma_load_3d(sm + Ly::kV + st * 16384 + s * 8192, &tmV, bar_kf + st, head * D + s * 64,
                      j * 64, seq);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    constexpr uint32_t kIdS = idesc_bf16(128, 64, 0, 0);   // S, dP (TS)
    constexpr uint32_t kIdQ = idesc_bf16(128, 128, 0, 1);  // dQ (TS, B = K MN-major)
    const uint32_t tm = __shfl_sync(0xFFFFFFFFu, tmem, 0);
    const uint32_t mQ = tm, mDO = tm + 64, mS = tm + 128, mDP = tm + 256, mDQ = tm + 384;
    const uint32_t k_base0 = smem_u32(sm + Ly::kK);
    const uint32_t v_base0 = smem_u32(sm + Ly::kV);
    if (elect_one()) {
      auto issue_sdp = [&](int j) {
        const int st = j % NS;
        const int b = j & 1;
        const uint32_t kb = k_base0 + st * 16384, vb = v_base0 + st * 16384;
        mbar_wait(bar_kf + st, (j / NS) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(mS + b * 64, mQ + kk * 8, sdesc_sw128(kb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024),
                 kIdS, kk > 0);
        tc_commit(bar_s + b);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(mDP + b * 64, mDO + kk * 8,
                 sdesc_sw128(vb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), kIdS, kk > 0);
        tc_commit(bar_dp + b);
      };
      mbar_wait(bar_qd, 0);
      tc_fence_after();
      issue_sdp(0);
      if (n_kv > 1) issue_sdp(1);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j % NS;
        const int b = j & 1;
        const uint32_t kb = k_base0 + st * 16384;
        mbar_wait(bar_ds + b, (j >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ts(mDQ, mS + b * 64 + kk * 8, sdesc_sw128(kb + kk * 2048, 8192, 1024), kIdQ,
                 (j > 0 || kk > 0) ? 1u : 0u);
        tc_commit(bar_ke + st);
        if (j + 2 < n_kv) issue_sdp(j + 2);
      }
      tc_commit(bar_fin);
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    // -------------------------------------------------------------------- compute warps:
    // thread = query row; warpgroup `half` owns key columns [32*half, 32*half+32) of a tile
    const int half = (warp - 4) >> 2;
    const int wq = warp & 3;
    const uint32_t la = static_cast<uint32_t>(wq * 32) << 16;
    const int qrow = wq * 32 + lane;
    const int qg = q0 + qrow;
    const bool in_range = qg < a.seq_len;
    const int64_t sh = static_cast<int64_t>(seq) * a.heads + head;
    if (half == 0)
      row_to_tmem(tQ + la, a.q + (static_cast<int64_t>(seq) * a.seq_len + qg) * a.q_stride +
                               static_cast<int64_t>(head) * D, in_range);
    else
      row_to_tmem(tDO + la, a.dout + (static_cast<int64_t>(seq) * a.seq_len + qg) * a.do_stride +
                                static_cast<int64_t>(head) * D, in_range);
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(bar_qd);
    const float lse2 = __ldg(a.lse2 + sh * a.seq_pad + qg);     // +inf for pads / dead rows
    const float dlt = __ldg(a.delta + sh * a.seq_pad + qg);
    const float c = a.scale_log2;
    const uint32_t* vb = a.valid_bits ? a.valid_bits + static_cast<int64_t>(seq) * a.words_per_seq : nullptr;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      // key validity of this warpgroup's 32 columns: one bit word
      const int kc0 = j * 64 + half * 32;
      uint32_t kmask = 0xFFFFFFFFu;
      if (vb) kmask = (kc0 >> 5) < a.words_per_seq ? __ldg(vb + (kc0 >> 5)) : 0u;
      const int rem = a.seq_len - kc0;
      if (rem < 32) kmask &= rem <= 0 ? 0u : ((1u << rem) - 1u);
      mbar_wait(bar_s + b, (j >> 1) & 1);
      mbar_wait(bar_dp + b, (j >> 1) & 1);
      tc_fence_after();
      uint32_t s0[32], dp[32];
      tmem_ld32(tS + b * 64 + la + half * 32, s0);
      tmem_ld32(tDP + b * 64 + la + half * 32, dp);
      tmem_wait_ld(s0);
      tmem_wait_ld(dp);
      uint32_t pk[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        float p0 = ex2(fmaf(__uint_as_float(s0[2 * jj]), c, -lse2));
        float p1 = ex2(fmaf(__uint_as_float(s0[2 * jj + 1]), c, -lse2));
        p0 = ((kmask >> (2 * jj)) & 1u) ? p0 : 0.f;
        p1 = ((kmask >> (2 * jj + 1)) & 1u) ? p1 : 0.f;
        pk[jj] = pack_bf16(p0 * (__uint_as_float(dp[2 * jj]) - dlt),
                           p1 * (__uint_as_float(dp[2 * jj + 1]) - dlt));
      }
      tmem_st16(tS + b * 64 + la + half * 16, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_ds + b);
    }
    // ------------------------------------------------------------------ epilogue: dQ (each
    // warpgroup drains half of the 128 columns)
    mbar_wait(bar_fin, 0);
    tc_fence_after();
    __nv_bfloat16* dst = a.dq + (static_cast<int64_t>(seq) * a.seq_len + qg) * a.dq_stride +
                         static_cast<int64_t>(head) * D + half * 64;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      uint32_t o[32];
      tmem_ld32(tDQ + la + half * 64 + cc * 32, o);
      tmem_wait_ld(o);
      if (in_range) {
        uint4 pk4[4];
        uint32_t* pw = reinterpret_cast<uint32_t*>(pk4);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj)
          pw[jj] = pack_bf16(__uint_as_float(o[2 * jj]) * a.scale, __uint_as_float(o[2 * jj + 1]) * a.scale);
        uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) d4[jj] = pk4[jj];
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

int launch_attn_bwd_split(const void* q, const void* k, const void* v, const void* dout,
                          const float* lse2, const float* delta, void* dq, void* dk, void* dv,
                          const AttnShape& s, int64_t qs, int64_t ks, int64_t vs, int64_t dos,
                          int64_t dqs, int64_t dks, int64_t dvs, const uint32_t* bits, float scale,
                          int64_t seq_pad, cudaStream_t stream) {
  if (s.head_dim != D) {
    set_error("split backward is specialised for head_dim 128");
    return kUnsupported;
  }
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(dout) | reinterpret_cast<uintptr_t>(dq) |
       reinterpret_cast<uintptr_t>(dk) | reinterpret_cast<uintptr_t>(dv)) & 15 ||
      ((qs | ks | vs | dos | dqs | dks | dvs) * 2) % 16) {
    set_error("attention backward needs 16-byte aligned bases and row strides");
    return kValue;
  }
  CUtensorMap mq, mdo, mk, mv;
  const int64_t cols = s.heads * D;
  int rc;
  if ((rc = make_tmap_bf16_3d(&mq, q, cols, s.seq_len, s.n_seq, qs, 64)) != kOk) return rc;
  if ((rc = make_tmap_bf16_3d(&mdo, dout, cols, s.seq_len, s.n_seq, dos, 64)) != kOk) return rc;
  if ((rc = make_tmap_bf16_3d(&mk, k, cols, s.seq_len, s.n_seq, ks, 64)) != kOk) return rc;
  if ((rc = make_tmap_bf16_3d(&mv, v, cols, s.seq_len, s.n_seq, vs, 64)) != kOk) return rc;
  SplitArgs a;
  a.lse2 = lse2;
  a.delta = delta;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.q_stride = qs;
  a.k_stride = ks;
  a.v_stride = vs;
  a.do_stride = dos;
  a.dq = static_cast<__nv_bfloat16*>(dq);
  a.dk = static_cast<__nv_bfloat16*>(dk);
  a.dv = static_cast<__nv_bfloat16*>(dv);
  a.dq_stride = dqs;
  a.dk_stride = dks;
  a.dv_stride = dvs;
  a.valid_bits = bits;
  a.words_per_seq = static_cast<int>((s.seq_len + 31) / 32);
  a.seq_len = static_cast<int>(s.seq_len);
  a.seq_pad = static_cast<int>(seq_pad);
  a.heads = static_cast<int>(s.heads);
  a.scale = scale;
  a.scale_log2 = scale * 1.4426950408889634f;
  static bool attr = false;
  if (!attr) {
    rc = check_cuda(cudaFuncSetAttribute(attn_bwd_dkdv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DkdvLayout::kSmem),
                    "cudaFuncSetAttribute(dkdv)");
    if (rc != kOk) return rc;
    rc = check_cuda(cudaFuncSetAttribute(attn_bwd_dq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DqLayout::kSmem),
                    "cudaFuncSetAttribute(dq)");
    if (rc != kOk) return rc;
    attr = true;
  }
  const unsigned tiles = static_cast<unsigned>(seq_pad / 128);
  dim3 grid(tiles, static_cast<unsigned>(s.heads), static_cast<unsigned>(s.n_seq));
  attn_bwd_dkdv_kernel<<<grid, kThreads, DkdvLayout::kSmem, stream>>>(mq, mdo, a);
  rc = check_cuda(cudaGetLastError(), "attn_bwd_dkdv_kernel launch");
  if (rc != kOk) return rc;
  attn_bwd_dq_kernel<<<grid, kThreads, DqLayout::kSmem, stream>>>(mk, mv, a);
  return check_cuda(cudaGetLastError(), "attn_bwd_dq_kernel launch");
}

}  // namespace osp
