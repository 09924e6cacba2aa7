// K3: backward of the per-subsequence attention (no reference counterpart: the reference
// attention.py has no backward; semantics follow the forward's exact-zero rules, so masked
// keys, pad queries and key-less rows get zero gradient).
//
// Three launches:
//   1. prep     : delta[q] = sum_c dO[q,c] O[q,c] (fp32), lse2 = lse*log2(e) (+inf kept),
//                 both padded to a multiple of 128 queries (+inf / 0), dq accumulator zeroed.
//   2. main     : one CTA per (128-key tile, head, subsequence) streams all 128-query tiles.
//                 Transposed scores so a thread owns a key row:
//                   S^T = K Q^T, dP^T = V dO^T            (SS MMAs into TMEM)
//                   P^T = exp2(S^T*c - lse2), dS^T = P^T (dP^T - delta)   (compute warps)
//                   dV += P^T dO   (P^T read from TMEM),  dK += dS^T Q,  dQ_i = dS K
//                 dV/dK accumulate in TMEM across the whole loop.  dQ_i is drained from TMEM by
//                 four writer warps: d = 64 (attn_bwd_kernel) adds it with fp32 vector atomics
//                 into the workspace; d = 128 (attn_bwd_v2_kernel, 64-query tiles) stages each
//                 tile in shared memory and adds it with ONE cp.reduce.async.bulk (32 KB) into
//                 the L2-resident accumulator.
//                 TMEM (d = 64): [0,128) S^T/P^T, [128,256) dP^T then dQ_i, [256,256+D) dV,
//                 [256+D, 256+2D) dK; the d = 128 layout is described at attn_bwd_v2_kernel.
//   3. finalize : dq = bf16(scale * dq_acc).
#include "osp_common.cuh"
#include "osp_internal.h"

#include <cstdlib>

// Experiment switches (BwdArgs::flags) are compiled in only with -DOSP_BWD_EXPERIMENTS=1, so the
// production kernels carry no never-taken branches.
#ifndef OSP_BWD_EXPERIMENTS
#define OSP_BWD_EXPERIMENTS 0
#endif

// K into TMEM copied from the TMA-landed K tile by both compute warpgroups, with the K / V TMA
// issued at barrier init (1); or K rows read from global by warpgroup 0 after setup (0, rounds 1-2).
#ifndef OSP_BWD_EARLY_K
#define OSP_BWD_EARLY_K 1
#endif
// dK / dV epilogue through a shared-memory stage with whole-row coalesced stores (1), or one
// row per thread straight from registers (0, rounds 1-2).
#ifndef OSP_BWD_STAGED_EPI
#define OSP_BWD_STAGED_EPI 1
#endif
// Phase timing (-DOSP_BWD_TIMING=1 builds only): clock64 sums of the v2 kernel's MMA issuer waits
// and per-CTA prologue / loop / epilogue cycles, read back with osp_debug_counters_bwd().
#ifndef OSP_BWD_TIMING
#define OSP_BWD_TIMING 0
#endif

// Ring depths of the d = 128 kernel: Q / dO stages and dQ staging buffers (shared memory allows
// 2 + 2 or 3 + 1)
#ifndef OSP_BWD_QSTAGES
#define OSP_BWD_QSTAGES 2
#endif
#ifndef OSP_BWD_XBUFS
#define OSP_BWD_XBUFS 2
#endif
// Q (+ lse2 / delta) and dO of a stage complete on separate barriers, so S^T_{i+1} (which needs only
// Q) is not held back by the dO half of the stage
#ifndef OSP_BWD_SPLITQ
#define OSP_BWD_SPLITQ 1
#endif

namespace osp {
__device__ unsigned long long g_bwd_counters[64];
namespace {

constexpr int kBwdThreads = 384;
constexpr int kBwdV2Threads = 512;
constexpr float kLog2e = 1.4426950408889634f;

template <int D>
struct BwdLayout {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kK = 0;
  static constexpr int kV = kK + kTile;
  static constexpr int kQ = kV + kTile;            // 2 stages
  static constexpr int kDO = kQ + 2 * kTile;       // 2 stages
  static constexpr int kDS = kDO + 2 * kTile;      // 128 keys x 128 queries bf16 = 32 KB
  static constexpr int kStat = kDS + 32768;        // 2 stages x (lse2[128], delta[128]) fp32
  static constexpr int kBar = kStat + 2 * 1024;
  static constexpr int kSmem = kBar + 256;
};

struct BwdArgs {
  const float* lse2;    // (n_seq, heads, Lp)
  const float* delta;   // (n_seq, heads, Lp)
  float* dq_acc;        // (n_seq, L, heads, D)
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  int64_t dk_stride, dv_stride;
  const uint32_t* valid_bits;
  int words_per_seq;
  int seq_len, seq_pad, heads, n_q;  // seq_len = capacity (row stride of a sequence)
  const int* seq_lens;               // per-sequence valid length (<= seq_len) or null
  const int* row_index;              // gather mode (D = 128): (n_seq, seq_len) token rows or -1
  int n_rows;
  float scale, scale_log2;
  const __nv_bfloat16* k_rows;  // K (for the TMEM copy of the key tile)
  int64_t k_row_stride;
  int flags;  // debug experiments (OSP_BWD_FLAGS): 1 = skip dQ reductions, 2 = skip compute math,
            // 32 = per-thread vector atomics instead of the bulk reduction, 64 = no Q/dO reloads
};

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Copy one 128-d bf16 row (global, 16B aligned) into 64 TMEM columns of this thread's lane in
// the kind::f16 A-operand layout (column c = elements 2c, 2c+1); rows past the end -> 0.
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

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                    const BwdArgs a) {
  using Ly = BwdLayout<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_kv = bars + 0;
  uint64_t* bar_qf = bars + 1;    // [2] Q, dO, lse2, delta of a stage landed
  uint64_t* bar_qe = bars + 3;    // [2] stage free
  uint64_t* bar_s = bars + 5;     // S^T ready
  uint64_t* bar_dp = bars + 6;    // dP^T ready
  uint64_t* bar_p = bars + 7;     // P^T written (128 arrivals)
  uint64_t* bar_ds = bars + 8;    // dS^T written (128 arrivals)
  uint64_t* bar_dsf = bars + 9;   // dS smem free again
  uint64_t* bar_dq = bars + 10;   // dQ_i ready in TMEM
  uint64_t* bar_dqf = bars + 11;  // dQ_i drained (128 arrivals)
  uint64_t* bar_fin = bars + 12;  // dK, dV final
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int seq = blockIdx.z;
  const int kv0 = blockIdx.x * 128;
  const int len = a.seq_lens ? __ldg(a.seq_lens + seq) : a.seq_len;
  if (kv0 >= len) {  // whole key tile past the sequence: dk, dv rows 0
    const int r1 = min(kv0 + 128, a.seq_len);
    const int64_t hoff = static_cast<int64_t>(head) * D;
    zero_rows_bf16(a.dv + static_cast<int64_t>(seq) * a.seq_len * a.dv_stride + hoff, a.dv_stride, kv0, r1, D);
    zero_rows_bf16(a.dk + static_cast<int64_t>(seq) * a.seq_len * a.dk_stride + hoff, a.dk_stride, kv0, r1, D);
    return;
  }
  const int n_q = (len + 127) / 128;

  if ((smem_u32(sm) & 1023) != 0) __trap();

  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_qf + i, 1);
      mbar_init(bar_qe + i, 1);
    }
    mbar_init(bar_s, 1);
    mbar_init(bar_dp, 1);
    mbar_init(bar_p, 128);
    mbar_init(bar_ds, 128);
    mbar_init(bar_dsf, 1);
    mbar_init(bar_dq, 1);
    mbar_init(bar_dqf, 128);
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
  const uint32_t tA = tmem, tB = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D;

  const float* lse2_g = a.lse2 + (static_cast<int64_t>(seq) * a.heads + head) * a.seq_pad;
  const float* delta_g = a.delta + (static_cast<int64_t>(seq) * a.heads + head) * a.seq_pad;

  if (warp < 4) {
    regs_dec<56>();
  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ TMA producer
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmDO);
      mbar_expect_tx(bar_kv, 2 * Ly::kTile);
#pragma unroll
      for (int s = 0; s < D / 64; ++s) {
        tma_load_3d(sm + Ly::kK + s * 16384, &tmK, bar_kv, head * D + s * 64, kv0, seq);
        tma_load_3d(sm + Ly::kV + s * 16384, &tmV, bar_kv, head * D + s * 64, kv0, seq);
      }
      for (int i = 0; i < n_q; ++i) {
        const int st = i & 1;
        mbar_wait(bar_qe + st, ((i >> 1) & 1) ^ 1);
        mbar_expect_tx(bar_qf + st, 2 * Ly::kTile + 1024);
#pragma unroll
        for (int s = 0; s < D / 64; ++s) {
          tma_load_3d(sm + Ly::kQ + st * Ly::kTile + s * 16384, &tmQ, bar_qf + st,
                      head * D + s * 64, i * 128, seq);
          tma_load_3d(sm + Ly::kDO + st * Ly::kTile + s * 16384, &tmDO, bar_qf + st,
                      head * D + s * 64, i * 128, seq);
        }
        bulk_load(sm + Ly::kStat + st * 1024, lse2_g + i * 128, 512, bar_qf + st);
        bulk_load(sm + Ly::kStat + st * 1024 + 512, delta_g + i * 128, 512, bar_qf + st);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t kIdSS = idesc_bf16(128, 128, 0, 0);   // S^T, dP^T
      constexpr uint32_t kIdKmn = idesc_bf16(128, D, 0, 1);    // dV (TS), dK
      constexpr uint32_t kIdMNmn = idesc_bf16(128, D, 1, 1);   // dQ
      const uint32_t k_base = smem_u32(sm + Ly::kK);
      const uint32_t v_base = smem_u32(sm + Ly::kV);
      const uint32_t ds_base = smem_u32(sm + Ly::kDS);
      mbar_wait(bar_kv, 0);
      for (int i = 0; i < n_q; ++i) {
        const int st = i & 1;
        const uint32_t q_base = smem_u32(sm + Ly::kQ + st * Ly::kTile);
        const uint32_t do_base = smem_u32(sm + Ly::kDO + st * Ly::kTile);
        mbar_wait(bar_qf + st, (i >> 1) & 1);
        tc_fence_after();
        // S^T = K Q^T  -> tA
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tA, sdesc_sw128(k_base + off, 16, 1024), sdesc_sw128(q_base + off, 16, 1024), kIdSS,
                 kk > 0);
        }
        tc_commit(bar_s);
        // dP^T = V dO^T -> tB (after the previous dQ was drained)
        if (i > 0) {
          mbar_wait(bar_dqf, (i - 1) & 1);
          tc_fence_after();
        }
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tB, sdesc_sw128(v_base + off, 16, 1024), sdesc_sw128(do_base + off, 16, 1024), kIdSS,
                 kk > 0);
        }
        tc_commit(bar_dp);
        // dV += P^T dO   (A = P^T from TMEM)
        mbar_wait(bar_p, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tDV, tA + kk * 8, sdesc_sw128(do_base + kk * 2048, 16384, 1024), kIdKmn,
                 (i > 0 || kk > 0) ? 1u : 0u);
        // dK += dS^T Q   (A = dS^T, K-major in smem)
        mbar_wait(bar_ds, i & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tDK, sdesc_sw128(ds_base + off, 16, 1024), sdesc_sw128(q_base + kk * 2048, 16384, 1024),
                 kIdKmn, (i > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(bar_qe + st);
        // dQ_i = dS K  -> tB   (A = dS, M(query)-major view of the same smem buffer)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ss(tB, sdesc_sw128(ds_base + kk * 2048, 16384, 1024),
                 sdesc_sw128(k_base + kk * 2048, 16384, 1024), kIdMNmn, kk > 0);
        tc_commit(bar_dq);
        tc_commit(bar_dsf);
      }
      tc_commit(bar_fin);
    }
  }
  } else if (warp < 8) {
    regs_inc<232>();
    // -------------------------------------------------------------- compute warps (key rows)
    const int wq = warp & 3;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const int krow = wq * 32 + lane;  // key row within the tile
    const int kglob = kv0 + krow;
    bool kvalid = kglob < len;
    if (kvalid && a.valid_bits) {
      const uint32_t* vb = a.valid_bits + static_cast<int64_t>(seq) * a.words_per_seq;
      kvalid = (__ldg(vb + (kglob >> 5)) >> (kglob & 31)) & 1u;
    }
    const float c = a.scale_log2;
    uint8_t* ds_row0 = sm + Ly::kDS + krow * 128;
    for (int i = 0; i < n_q; ++i) {
      const int st = i & 1;
      const float* lse_s = reinterpret_cast<const float*>(sm + Ly::kStat + st * 1024);
      const float* del_s = lse_s + 128;
      mbar_wait(bar_qf + st, (i >> 1) & 1);  // lse2 / delta of this stage landed
      mbar_wait(bar_s, i & 1);
      tc_fence_after();
      float p[128];
      {
        uint32_t s[4][32];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) tmem_ld32(tA + lane_addr + cc * 32, s[cc]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) tmem_wait_ld(s[cc]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 l4 = *reinterpret_cast<const float4*>(lse_s + cc * 32 + i4 * 4);
            p[cc * 32 + i4 * 4 + 0] = ex2(fmaf(__uint_as_float(s[cc][i4 * 4 + 0]), c, -l4.x));
            p[cc * 32 + i4 * 4 + 1] = ex2(fmaf(__uint_as_float(s[cc][i4 * 4 + 1]), c, -l4.y));
            p[cc * 32 + i4 * 4 + 2] = ex2(fmaf(__uint_as_float(s[cc][i4 * 4 + 2]), c, -l4.z));
            p[cc * 32 + i4 * 4 + 3] = ex2(fmaf(__uint_as_float(s[cc][i4 * 4 + 3]), c, -l4.w));
          }
        }
      }
      if (!kvalid) {
#pragma unroll
        for (int j = 0; j < 128; ++j) p[j] = 0.f;
      }
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(p[cc * 32 + 2 * j], p[cc * 32 + 2 * j + 1]);
        tmem_st16(tA + lane_addr + cc * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p);

      mbar_wait(bar_dp, i & 1);
      tc_fence_after();
      if (i > 0) mbar_wait(bar_dsf, (i - 1) & 1);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t dp[32];
        tmem_ld32(tB + lane_addr + cc * 32, dp);
        tmem_wait_ld(dp);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float d0 = del_s[cc * 32 + 2 * j], d1 = del_s[cc * 32 + 2 * j + 1];
          const float ds0 = p[cc * 32 + 2 * j] * (__uint_as_float(dp[2 * j]) - d0);
          const float ds1 = p[cc * 32 + 2 * j + 1] * (__uint_as_float(dp[2 * j + 1]) - d1);
          pk[j] = pack_bf16(ds0, ds1);
        }
        // queries cc*32 .. cc*32+31 = 4 16-byte chunks of sub-tile cc/2, chunk base (cc&1)*4
        uint8_t* sub = ds_row0 + (cc >> 1) * 16384;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int logical = (cc & 1) * 4 + ch;
          const int phys = logical ^ (krow & 7);
          *reinterpret_cast<uint4*>(sub + phys * 16) =
              make_uint4(pk[ch * 4 + 0], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar_ds);
    }
    // ---------------------------------------------------------------- dK / dV epilogue
    mbar_wait(bar_fin, 0);
    tc_fence_after();
    const bool row_ok = kglob < a.seq_len;  // rows in [len, cap) hold exact zeros
    __nv_bfloat16* dvrow = a.dv + (static_cast<int64_t>(seq) * a.seq_len + kglob) * a.dv_stride +
                           static_cast<int64_t>(head) * D;
    __nv_bfloat16* dkrow = a.dk + (static_cast<int64_t>(seq) * a.seq_len + kglob) * a.dk_stride +
                           static_cast<int64_t>(head) * D;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t base = (which == 0 ? tDV : tDK) + lane_addr;
      const float mul = which == 0 ? 1.f : a.scale;
      __nv_bfloat16* row = which == 0 ? dvrow : dkrow;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(base + cc * 32, o);
        tmem_wait_ld(o);
        if (row_ok) {
          uint4 pk[4];
          uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            pw[j] = pack_bf16(__uint_as_float(o[2 * j]) * mul, __uint_as_float(o[2 * j + 1]) * mul);
          uint4* dst = reinterpret_cast<uint4*>(row + cc * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) dst[j] = pk[j];
        }
      }
    }
  } else {
    regs_dec<152>();
    // -------------------------------------------------------------- dQ writer warps
    const int wq = warp & 3;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const int qrow = wq * 32 + lane;
    for (int i = 0; i < n_q; ++i) {
      mbar_wait(bar_dq, i & 1);
      tc_fence_after();
      const int qg = i * 128 + qrow;
      float* dst = a.dq_acc + ((static_cast<int64_t>(seq) * a.seq_len + qg) * a.heads + head) * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t v[32];
        tmem_ld32(tB + lane_addr + cc * 32, v);
        tmem_wait_ld(v);
        if (cc == D / 32 - 1) {
          tc_fence_before();
          mbar_arrive(bar_dqf);
        }
        if (qg < len && !((OSP_BWD_EXPERIMENTS ? a.flags : 0) & 1)) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            red_add_v4(dst + cc * 32 + j * 4, __uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                       __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        }
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

// ---------------------------------------------------------------------------------------------
// Main kernel for head_dim 128.  One CTA per (128-key tile, head, subsequence) streams 64-query
// tiles.  Shared-memory operand bandwidth (128 B/clk/SM for tcgen05 SS mode, measured with
// tools/mma_rate.cu) is the binding resource, so operands that can live in TMEM do:
//   TMEM: [0,64) K (A operand of S^T, copied once), [64,128) S^T then P^T (query half h
//         packed at [64 + 32h, 80 + 32h)),
//         [128,192) dP^T then dS^T (half h at +32h), [192,256) dQ^T, [256,384) dV, [384,512) dK.
//   S^T = K Q^T (TS), dP^T = V dO^T (SS), dV += P^T dO (TS), dK += dS^T Q (TS),
//   dQ^T_i = K^T dS_i^T (SS, dS^T also staged in smem as the B operand).
//   dQ^T is drained by four writer warps (thread = d): tcgen05.ld into registers, staged in
//   shared memory in the accumulator's (q/4, d, q%4) fp32 layout, and added into the
//   (seq*head, q/4, d, q%4) L2 accumulator by ONE cp.reduce.async.bulk of 32 KB per tile.
//   Eight compute warps (thread = key row) split each tile's 64 query columns.
//   MMA order: S_0, dP_0, then per i: dV_i, S_{i+1}, dK_i, dQ^T_i, dP_{i+1}.
struct BwdV2Layout {
  static constexpr int kK = 0;                    // 128 keys x 128 d  (2 x 16 KB)
  static constexpr int kV = 32768;
  static constexpr int kStages = OSP_BWD_QSTAGES;  // Q / dO ring depth
  static constexpr int kQ = 65536;                // stages x (64 q x 128 d = 2 x 8 KB)
  static constexpr int kDO = kQ + kStages * 16384;
  static constexpr int kDS = kDO + kStages * 16384;   // 2 x (128 keys x 64 q) bf16
  static constexpr int kStat = kDS + 2 * 16384;       // 3 x (lse2[64], delta[64])
  static constexpr int kBar = kStat + kStages * 512;
  static constexpr int kSmem = kBar + 256;
  // dQ^T staging for the asynchronous bulk reduction: one 64-query tile in the accumulator's
  // (q/4, d, q%4) layout = 32 KB
  static constexpr int kXBufs = OSP_BWD_XBUFS;
  static constexpr int kX = kSmem;
  static constexpr int kSmemX = kX + kXBufs * 32768;
};
static_assert(BwdV2Layout::kSmemX + 1024 <= 232448, "bwd v2 smem with staging");

__device__ __forceinline__ void red_add_v4_plain(float* addr, const uint32_t* v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}

__global__ void __launch_bounds__(kBwdV2Threads, 1)
    attn_bwd_v2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                       const BwdArgs a) {
  constexpr int D = 128;
  using Ly = BwdV2Layout;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_kv = bars + 0;
  uint64_t* bar_qf = bars + 1;    // [3]
  uint64_t* bar_qe = bars + 4;    // [3]
  uint64_t* bar_s = bars + 7;
  uint64_t* bar_dp = bars + 8;
  uint64_t* bar_p = bars + 9;     // 128 arrivals
  uint64_t* bar_ds = bars + 10;   // [2] 128 arrivals
  uint64_t* bar_dsf = bars + 12;  // [2]
  uint64_t* bar_dq = bars + 14;   // [2]
  uint64_t* bar_dqf = bars + 16;  // [2] 128 arrivals
  uint64_t* bar_fin = bars + 18;
  uint64_t* bar_kt = bars + 19;   // K rows in TMEM (256 arrivals)
  uint64_t* bar_df = OSP_BWD_SPLITQ ? bars + 21 : bar_qf;  // [3] dO of a stage landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int seq = blockIdx.z;
  const int kv0 = blockIdx.x * 128;
  const int len = a.seq_lens ? __ldg(a.seq_lens + seq) : a.seq_len;
  if (kv0 >= len) {  // whole key tile past the sequence: dk, dv rows 0
    if (a.row_index) return;  // gather mode: such rows have no destination
    const int r1 = min(kv0 + 128, a.seq_len);
    const int64_t hoff = static_cast<int64_t>(head) * D;
    zero_rows_bf16(a.dv + static_cast<int64_t>(seq) * a.seq_len * a.dv_stride + hoff, a.dv_stride, kv0, r1, D);
    zero_rows_bf16(a.dk + static_cast<int64_t>(seq) * a.seq_len * a.dk_stride + hoff, a.dk_stride, kv0, r1, D);
    return;
  }
  const int n_q = (len + 63) / 64;
#if OSP_BWD_TIMING
  const long long t_entry = clock64();
  long long t_first = 0, t_fin = 0;
#endif

  if ((smem_u32(sm) & 1023) != 0) __trap();
  if (threadIdx.x == 0) {
    mbar_init(bar_kv, 1);
    for (int i = 0; i < Ly::kStages; ++i) {
      mbar_init(bar_qf + i, 1);
      if (OSP_BWD_SPLITQ) mbar_init(bar_df + i, 1);
      mbar_init(bar_qe + i, 1);
    }
    mbar_init(bar_s, 1);
    mbar_init(bar_dp, 1);
    mbar_init(bar_p, 256);
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_ds + i, 256);
      mbar_init(bar_dsf + i, 1);
      mbar_init(bar_dq + i, 1);
      mbar_init(bar_dqf + i, 128);
    }
    mbar_init(bar_fin, 1);
    mbar_init(bar_kt, 256);
    fence_barrier_init();
#if OSP_BWD_EARLY_K
    if (!a.row_index) {  // K / V tiles in flight before the TMEM allocation and the block barrier
      mbar_expect_tx(bar_kv, 65536);
      for (int s2 = 0; s2 < 2; ++s2) {
        tma_load_3d(sm + Ly::kK + s2 * 16384, &tmK, bar_kv, head * D + s2 * 64, kv0, seq);
        tma_load_3d(sm + Ly::kV + s2 * 16384, &tmV, bar_kv, head * D + s2 * 64, kv0, seq);
      }
    }
#endif
  }
  if (warp == 2) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tK = tmem, tS = tmem + 64, tDP = tmem + 128, tDQ = tmem + 192, tDV = tmem + 256,
                 tDK = tmem + 384;
  const int64_t sh = static_cast<int64_t>(seq) * a.heads + head;

  // register budget (setmaxnreg, total < 64K): control warps 64, compute 176, writers 88
  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0 && a.row_index) {
      // -------------------------------------------------------------- TMA producer, gather mode:
      // tile::gather4 of 4 token rows per lane and 64 columns (K, V once; Q, dO per query tile)
      const int* ridx = a.row_index + static_cast<int64_t>(seq) * a.seq_len;
      auto rows4 = [&](int row0) {
        const int4 r = *reinterpret_cast<const int4*>(ridx + row0);
        const int oob = a.n_rows;
        return make_int4(r.x < 0 ? oob : r.x, r.y < 0 ? oob : r.y, r.z < 0 ? oob : r.z, r.w < 0 ? oob : r.w);
      };
      if (lane == 0) {
        tma_prefetch(&tmQ);
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
        tma_prefetch(&tmDO);
        mbar_expect_tx(bar_kv, 65536);
      }
      __syncwarp();
      {
        const int4 r = rows4(kv0 + 4 * lane);
        for (int s = 0; s < 2; ++s) {
          tma_gather4(sm + Ly::kK + s * 16384 + lane * 512, &tmK, bar_kv, head * D + s * 64, r.x, r.y, r.z, r.w);
          tma_gather4(sm + Ly::kV + s * 16384 + lane * 512, &tmV, bar_kv, head * D + s * 64, r.x, r.y, r.z, r.w);
        }
      }
      const float* lse2_g = a.lse2 + sh * a.seq_pad;
      const float* delta_g = a.delta + sh * a.seq_pad;
      const int half_lane = lane & 15;  // lanes 0-15 fetch Q rows, 16-31 dO rows
      const CUtensorMap* mapq = lane < 16 ? &tmQ : &tmDO;
      const int base_off = lane < 16 ? Ly::kQ : Ly::kDO;
      for (int i = 0; i < n_q; ++i) {
        const int st = i % Ly::kStages;
        mbar_wait(bar_qe + st, ((i / Ly::kStages) & 1) ^ 1);
        if (lane == 0) {
          if (OSP_BWD_SPLITQ) {
            mbar_expect_tx(bar_qf + st, 16384 + 512);
            mbar_expect_tx(bar_df + st, 16384);
          } else {
            mbar_expect_tx(bar_qf + st, 2 * 16384 + 512);
          }
          bulk_load(sm + Ly::kStat + st * 512, lse2_g + i * 64, 256, bar_qf + st);
          bulk_load(sm + Ly::kStat + st * 512 + 256, delta_g + i * 64, 256, bar_qf + st);
        }
        __syncwarp();
        const int4 r = rows4(i * 64 + 4 * half_lane);
        for (int s = 0; s < 2; ++s)
          tma_gather4(sm + base_off + st * 16384 + s * 8192 + half_lane * 512, mapq,
                      lane < 16 ? bar_qf + st : bar_df + st,
                      head * D + s * 64, r.x, r.y, r.z, r.w);
      }
    } else if (warp == 0) {
      if (elect_one()) {
      // ---------------------------------------------------------------- TMA producer
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      tma_prefetch(&tmDO);
      if (!OSP_BWD_EARLY_K) {
        mbar_expect_tx(bar_kv, 65536);
        for (int s = 0; s < 2; ++s) {
          tma_load_3d(sm + Ly::kK + s * 16384, &tmK, bar_kv, head * D + s * 64, kv0, seq);
          tma_load_3d(sm + Ly::kV + s * 16384, &tmV, bar_kv, head * D + s * 64, kv0, seq);
        }
      }
      const float* lse2_g = a.lse2 + sh * a.seq_pad;
      const float* delta_g = a.delta + sh * a.seq_pad;
      for (int i = 0; i < n_q; ++i) {
        const int st = i % Ly::kStages;
        mbar_wait(bar_qe + st, ((i / Ly::kStages) & 1) ^ 1);
        if (((OSP_BWD_EXPERIMENTS ? a.flags : 0) & 64) && i >= 2) {  // experiment 64: no Q/dO reloads (stale tiles, timing only)
          mbar_arrive(bar_qf + st);
          if (OSP_BWD_SPLITQ) mbar_arrive(bar_df + st);
          continue;
        }
        if (OSP_BWD_SPLITQ) {
          // Q and its row statistics first (S^T_i needs them), dO after on its own barrier
          mbar_expect_tx(bar_qf + st, 16384 + 512);
          for (int s = 0; s < 2; ++s)
            tma_load_3d(sm + Ly::kQ + st * 16384 + s * 8192, &tmQ, bar_qf + st, head * D + s * 64,
                        i * 64, seq);
          bulk_load(sm + Ly::kStat + st * 512, lse2_g + i * 64, 256, bar_qf + st);
          bulk_load(sm + Ly::kStat + st * 512 + 256, delta_g + i * 64, 256, bar_qf + st);
          mbar_expect_tx(bar_df + st, 16384);
          for (int s = 0; s < 2; ++s)
            tma_load_3d(sm + Ly::kDO + st * 16384 + s * 8192, &tmDO, bar_df + st, head * D + s * 64,
                        i * 64, seq);
        } else {
          mbar_expect_tx(bar_qf + st, 2 * 16384 + 512);
          for (int s = 0; s < 2; ++s) {
            tma_load_3d(sm + Ly::kQ + st * 16384 + s * 8192, &tmQ, bar_qf + st, head * D + s * 64,
                        i * 64, seq);
            tma_load_3d(sm + Ly::kDO + st * 16384 + s * 8192, &tmDO, bar_qf + st, head * D + s * 64,
                        i * 64, seq);
          }
          bulk_load(sm + Ly::kStat + st * 512, lse2_g + i * 64, 256, bar_qf + st);
          bulk_load(sm + Ly::kStat + st * 512 + 256, delta_g + i * 64, 256, bar_qf + st);
        }
      }
      }
      __syncwarp();
    } else if (warp == 1) {
      // ---------------------------------------------------------------- MMA issuer (one elected lane runs
      // the whole loop; operands are derived from warp-uniform values, so they live in
      // uniform registers and no per-GEMM reconvergence is needed)
      constexpr uint32_t kIdS = idesc_bf16(128, 64, 0, 0);     // S^T, dP^T
      constexpr uint32_t kIdKV = idesc_bf16(128, 128, 0, 1);   // dV (TS), dK
      constexpr uint32_t kIdQ = idesc_bf16(128, 64, 1, 1);     // dQ^T
      const uint32_t tm = __shfl_sync(0xFFFFFFFFu, tmem, 0);
      const uint32_t mK = tm, mS = tm + 64, mDP = tm + 128, mDQ = tm + 192, mDV = tm + 256, mDK = tm + 384;
      const uint32_t k_base = smem_u32(sm + Ly::kK);
      const uint32_t v_base = smem_u32(sm + Ly::kV);
      const uint32_t ds_base = smem_u32(sm + Ly::kDS);
      const uint32_t q_base0 = smem_u32(sm + Ly::kQ);
      const uint32_t do_base0 = smem_u32(sm + Ly::kDO);
      auto issue_s = [&](int i) {
        const uint32_t qb = q_base0 + (i % Ly::kStages) * 16384;
        {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ts(mS, mK + kk * 8, sdesc_sw128(qb + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), kIdS,
                   kk > 0);
          tc_commit(bar_s);
        }
      };
      auto issue_dp = [&](int i) {
        const uint32_t db = do_base0 + (i % Ly::kStages) * 16384;
        if (OSP_BWD_SPLITQ) {
          mbar_wait(bar_df + i % Ly::kStages, (i / Ly::kStages) & 1);
          tc_fence_after();
        }
        {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(mDP, sdesc_sw128(v_base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                   sdesc_sw128(db + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), kIdS, kk > 0);
          tc_commit(bar_dp);
        }
      };
      if (elect_one()) {
      mbar_wait(bar_kv, 0);
      mbar_wait(bar_kt, 0);
      mbar_wait(bar_qf + 0, 0);
      tc_fence_after();
#if OSP_BWD_TIMING
      t_first = clock64();
#endif
      issue_s(0);
      issue_dp(0);
      for (int i = 0; i < n_q; ++i) {
        const int st = i % Ly::kStages;
        const int b = i & 1;
        const uint32_t qb = q_base0 + st * 16384;
        const uint32_t db = do_base0 + st * 16384;
        // dV += P^T dO
#if OSP_BWD_TIMING
        long long t0 = clock64();
#define OSP_BT(k) do { const long long _t = clock64(); atomicAdd(&g_bwd_counters[k], static_cast<unsigned long long>(_t - t0)); t0 = _t; } while (0)
#else
#define OSP_BT(k) do { } while (0)
#endif
        mbar_wait(bar_p, i & 1);
        OSP_BT(0);
        tc_fence_after();
        {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(mDV, mS + (kk >> 1) * 32 + (kk & 1) * 8, sdesc_sw128(db + kk * 2048, 8192, 1024),
                   kIdKV, (i > 0 || kk > 0) ? 1u : 0u);
        }
        // S_{i+1} (tS is free once dV_i has been issued: tcgen05 ops execute in order)
        if (i + 1 < n_q) {
#if OSP_BWD_TIMING
          t0 = clock64();
#endif
          mbar_wait(bar_qf + (i + 1) % Ly::kStages, ((i + 1) / Ly::kStages) & 1);
          OSP_BT(1);
          tc_fence_after();
          issue_s(i + 1);
        }
        // dK += dS^T Q
#if OSP_BWD_TIMING
        t0 = clock64();
#endif
        mbar_wait(bar_ds + b, (i >> 1) & 1);
        OSP_BT(2);
        tc_fence_after();
        const uint32_t dsb = ds_base + b * 16384;
        {
          // dK += dS^T Q with dS^T read from TMEM (TS; written over the consumed dP^T columns)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts(mDK, mDP + (kk >> 1) * 32 + (kk & 1) * 8, sdesc_sw128(qb + kk * 2048, 8192, 1024), kIdKV,
                   (i > 0 || kk > 0) ? 1u : 0u);
          tc_commit(bar_qe + st);
        }
        // dQ^T_i = K^T dS_i^T (single TMEM buffer; the writers drain it right after it lands)
        if (i >= 1) {
#if OSP_BWD_TIMING
          t0 = clock64();
#endif
          mbar_wait(bar_dqf, (i - 1) & 1);
          OSP_BT(3);
          tc_fence_after();
        }
        {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            mma_ss(mDQ, sdesc_sw128(k_base + kk * 2048, 16384, 1024),
                   sdesc_sw128(dsb + kk * 2048, 8192, 1024), kIdQ, kk > 0);
          tc_commit(bar_dq);
          tc_commit(bar_dsf + b);
        }
        if (i + 1 < n_q) issue_dp(i + 1);
#if OSP_BWD_TIMING
        atomicAdd(&g_bwd_counters[7], 1ull);
#endif
      }
      tc_commit(bar_fin);
#if OSP_BWD_TIMING
      t_fin = clock64();
#endif
      }
      __syncwarp();
    }
  } else if (warp < 12) {
    regs_inc<176>();
    // ------------------------------------------------------------------ compute warps: thread =
    // key row, the two warpgroups split the 64 query columns of a tile (32 each)
    const int half = (warp - 4) >> 2;
    const int wq = warp & 3;
    const uint32_t la = static_cast<uint32_t>(wq * 32) << 16;
    const int krow = wq * 32 + lane;
    const int kglob = kv0 + krow;
    bool kvalid = kglob < len;
    if (kvalid && a.valid_bits) {
      const uint32_t* vb = a.valid_bits + static_cast<int64_t>(seq) * a.words_per_seq;
      kvalid = (__ldg(vb + (kglob >> 5)) >> (kglob & 31)) & 1u;
    }
#if OSP_BWD_EARLY_K
    {
      // K into TMEM from the TMA-landed K tile (128B-swizzled: 16-byte chunk c of row r at
      // c ^ (r & 7)); warpgroup h copies columns [64h, 64h + 64) of its key row
      mbar_wait(bar_kv, 0);
      const uint8_t* src = sm + Ly::kK + half * 16384 + krow * 128;
      uint32_t r[32];
#pragma unroll
      for (int c2 = 0; c2 < 8; ++c2) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + ((c2 ^ (krow & 7)) * 16));
        r[4 * c2 + 0] = v.x;
        r[4 * c2 + 1] = v.y;
        r[4 * c2 + 2] = v.z;
        r[4 * c2 + 3] = v.w;
      }
      tmem_st32(tK + la + half * 32, r);
    }
#else
    if (half == 0)
      row_to_tmem(tK + la,
                  a.k_rows + (a.row_index ? (kglob < len ? static_cast<int64_t>(a.row_index[static_cast<int64_t>(seq) * a.seq_len + kglob]) : 0)
                                          : static_cast<int64_t>(seq) * a.seq_len + kglob) * a.k_row_stride +
                      static_cast<int64_t>(head) * D,
                  kglob < len);
#endif
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(bar_kt);
    const float c = a.scale_log2;
    for (int i = 0; i < n_q; ++i) {
      const int st = i % Ly::kStages;
      const int b = i & 1;
      const float* lse_s = reinterpret_cast<const float*>(sm + Ly::kStat + st * 512) + half * 32;
      const float* del_s = lse_s + 64;
      mbar_wait(bar_qf + st, (i / Ly::kStages) & 1);
      // lse2 / delta of this tile's 32 query columns into registers now: shared memory is busy
      // feeding SS-mode MMAs, so these loads must not sit on the softmax critical path
      float lse_r[32], del_r[32];
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        const float4 l4 = *reinterpret_cast<const float4*>(lse_s + j4 * 4);
        const float4 d4 = *reinterpret_cast<const float4*>(del_s + j4 * 4);
        lse_r[j4 * 4 + 0] = l4.x;
        lse_r[j4 * 4 + 1] = l4.y;
        lse_r[j4 * 4 + 2] = l4.z;
        lse_r[j4 * 4 + 3] = l4.w;
        del_r[j4 * 4 + 0] = d4.x;
        del_r[j4 * 4 + 1] = d4.y;
        del_r[j4 * 4 + 2] = d4.z;
        del_r[j4 * 4 + 3] = d4.w;
      }
      mbar_wait(bar_s, i & 1);
      tc_fence_after();
      if ((OSP_BWD_EXPERIMENTS ? a.flags : 0) & 2) {  // experiment: synchronisation skeleton only
        tc_fence_before();
        mbar_arrive(bar_p);
        mbar_wait(bar_dp, i & 1);
        if (i >= 2) mbar_wait(bar_dsf + b, ((i - 2) >> 1) & 1);
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(bar_ds + b);
        continue;
      }
      float p[32];
      {
        uint32_t s0[32];
        tmem_ld32(tS + la + half * 32, s0);
        tmem_wait_ld(s0);
#pragma unroll
        for (int j = 0; j < 32; ++j) p[j] = ex2(fmaf(__uint_as_float(s0[j]), c, -lse_r[j]));
      }
      if (!kvalid) {
#pragma unroll
        for (int j = 0; j < 32; ++j) p[j] = 0.f;
      }
      {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(p[2 * j], p[2 * j + 1]);
        // P^T of query half h goes to columns [32h, 32h + 16): inside the S^T columns this
        // warpgroup itself read, never over the other warpgroup's, which may still be loading
        // them (placing half 1 at [16, 32) raced with half 0's S^T load)
        tmem_st16(tS + la + half * 32, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(bar_p);

      mbar_wait(bar_dp, i & 1);
      tc_fence_after();
      if (i >= 2) mbar_wait(bar_dsf + b, ((i - 2) >> 1) & 1);
      uint8_t* row = sm + Ly::kDS + b * 16384 + krow * 128;
      {
        uint32_t dp[32];
        tmem_ld32(tDP + la + half * 32, dp);
        tmem_wait_ld(dp);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float ds0 = p[2 * j] * (__uint_as_float(dp[2 * j]) - del_r[2 * j]);
          const float ds1 = p[2 * j + 1] * (__uint_as_float(dp[2 * j + 1]) - del_r[2 * j + 1]);
          pk[j] = pack_bf16(ds0, ds1);
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int phys = (half * 4 + ch) ^ (krow & 7);
          *reinterpret_cast<uint4*>(row + phys * 16) =
              make_uint4(pk[ch * 4 + 0], pk[ch * 4 + 1], pk[ch * 4 + 2], pk[ch * 4 + 3]);
        }
        // dS^T of query half h goes to columns [32h, 32h + 16): inside the dP^T columns this
        // warpgroup itself read, so neither warpgroup waits for the other
        tmem_st16(tDP + la + half * 32, pk);
      }
      tmem_wait_st();
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(bar_ds + b);
    }
    // ------------------------------------------------------------------ dK / dV epilogue
    // (warpgroup 0 drains dV, warpgroup 1 drains dK)
    mbar_wait(bar_fin, 0);
    tc_fence_after();
    // rows in [len, cap) hold exact zeros; in gather mode they have no destination
    const int64_t out_row =
        a.row_index ? (kglob < len ? a.row_index[static_cast<int64_t>(seq) * a.seq_len + kglob] : -1)
                    : (kglob < a.seq_len ? static_cast<int64_t>(seq) * a.seq_len + kglob : -1);
    const bool row_ok = out_row >= 0;
#if OSP_BWD_STAGED_EPI
    {
      // Staged through the K (dV) / V (dK) buffers, free once bar_fin has fired: the warp's 32
      // rows go to its quarter with 16-byte chunks XOR-swizzled by row, then out two whole
      // 256-byte rows per store instruction instead of 16 bytes of 32 different rows.
      const int which = half;
      const uint32_t base = (which == 0 ? tDV : tDK) + la;
      const float mul = which == 0 ? 1.f : a.scale;
      uint8_t* stg = sm + (which == 0 ? Ly::kK : Ly::kV) + wq * 8192;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(base + cc * 32, o);
        tmem_wait_ld(o);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 pk;
          pk.x = pack_bf16(__uint_as_float(o[8 * i + 0]) * mul, __uint_as_float(o[8 * i + 1]) * mul);
          pk.y = pack_bf16(__uint_as_float(o[8 * i + 2]) * mul, __uint_as_float(o[8 * i + 3]) * mul);
          pk.z = pack_bf16(__uint_as_float(o[8 * i + 4]) * mul, __uint_as_float(o[8 * i + 5]) * mul);
          pk.w = pack_bf16(__uint_as_float(o[8 * i + 6]) * mul, __uint_as_float(o[8 * i + 7]) * mul);
          *reinterpret_cast<uint4*>(stg + lane * 256 + (((cc * 4 + i) ^ (lane & 15)) * 16)) = pk;
        }
      }
      __syncwarp();
      __nv_bfloat16* out = (which == 0 ? a.dv : a.dk) + static_cast<int64_t>(head) * D;
      const int64_t ostride = which == 0 ? a.dv_stride : a.dk_stride;
      const int ch = lane & 15;
#pragma unroll 4
      for (int rr = 0; rr < 16; ++rr) {
        const int r = 2 * rr + (lane >> 4);
        const long long dst_row = __shfl_sync(0xFFFFFFFFu, static_cast<long long>(out_row), r);
        const uint4 v = *reinterpret_cast<const uint4*>(stg + r * 256 + ((ch ^ (r & 15)) * 16));
        if (dst_row >= 0) *reinterpret_cast<uint4*>(out + dst_row * ostride + ch * 8) = v;
      }
    }
#else
    {
      const int which = half;
      const uint32_t base = (which == 0 ? tDV : tDK) + la;
      const float mul = which == 0 ? 1.f : a.scale;
      __nv_bfloat16* dst = (which == 0 ? a.dv : a.dk) + (row_ok ? out_row : 0) * (which == 0 ? a.dv_stride : a.dk_stride) +
                           static_cast<int64_t>(head) * D;
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        uint32_t o[32];
        tmem_ld32(base + cc * 32, o);
        tmem_wait_ld(o);
        if (row_ok) {
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
#endif
  } else {
    regs_dec<88>();
    // ------------------------------------------------------------------ dQ^T writer warps (thread = d)
    const int wq = warp & 3;
    const uint32_t la = static_cast<uint32_t>(wq * 32) << 16;
    const int dcol = wq * 32 + lane;
    float* acc = a.dq_acc + sh * static_cast<int64_t>(a.seq_pad) * D;
    const bool leader = warp == 12 && lane == 0;
    for (int i = 0; i < n_q; ++i) {
      mbar_wait(bar_dq, i & 1);
      tc_fence_after();
      uint32_t v0[32], v1[32];
      tmem_ld32(tDQ + la, v0);
      tmem_ld32(tDQ + la + 32, v1);
      tmem_wait_ld(v0);
      tmem_wait_ld(v1);
      tc_fence_before();
      mbar_arrive(bar_dqf);
      if ((OSP_BWD_EXPERIMENTS ? a.flags : 0) & 1) continue;
      if ((OSP_BWD_EXPERIMENTS ? a.flags : 0) & 32) {  // experiment 32: per-thread vector atomics (the previous scheme)
        float* base = acc + (static_cast<int64_t>(i) * 16 * D + dcol) * 4;  // q/4 block = i*16
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) red_add_v4_plain(base + j4 * D * 4, v0 + j4 * 4);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) red_add_v4_plain(base + (8 + j4) * D * 4, v1 + j4 * 4);
        continue;
      }
      // Stage the tile in smem and hand it to one asynchronous bulk L2 reduction, so the writers
      // never queue behind reductions: the staging buffer is reused once the previous tile's
      // bulk reduction has read it (one tile of slack).
      const int xb = i % Ly::kXBufs;
      if (i >= Ly::kXBufs) {
        if (leader) bulk_wait_read<Ly::kXBufs - 1>();
        named_bar_sync(5, 128);
      }
      float* xs = reinterpret_cast<float*>(sm + Ly::kX + xb * 32768) + dcol * 4;
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        *reinterpret_cast<uint4*>(xs + j4 * D * 4) = make_uint4(v0[4 * j4], v0[4 * j4 + 1], v0[4 * j4 + 2], v0[4 * j4 + 3]);
        *reinterpret_cast<uint4*>(xs + (8 + j4) * D * 4) = make_uint4(v1[4 * j4], v1[4 * j4 + 1], v1[4 * j4 + 2], v1[4 * j4 + 3]);
      }
      fence_proxy_async_smem();
      named_bar_sync(5, 128);
      if (leader) {
        bulk_reduce_add_f32(acc + static_cast<int64_t>(i) * 16 * D * 4, sm + Ly::kX + xb * 32768, 32768);
        tma_store_commit();
      }
    }
    if (leader) tma_store_wait_all();
  }

  tc_fence_before();
  __syncthreads();
#if OSP_BWD_TIMING
  // per CTA, on the MMA issuer's lane: entry -> first S^T issue (prologue), the query-tile loop,
  // last issue -> every warp done (epilogue: dK/dV drain, the last dQ reductions)
  if (t_first != 0) {
    atomicAdd(&g_bwd_counters[8], static_cast<unsigned long long>(t_first - t_entry));
    atomicAdd(&g_bwd_counters[9], static_cast<unsigned long long>(t_fin - t_first));
    atomicAdd(&g_bwd_counters[10], static_cast<unsigned long long>(clock64() - t_fin));
    atomicAdd(&g_bwd_counters[11], 1ull);
  }
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dq = bf16(scale * acc) from the v2 (seq*head, q/4, d, q%4) accumulator.  A thread takes 4
// consecutive d of one q/4 block: one 64-byte read, four 8-byte row writes (a warp covers a whole
// 128-d head slice, so both sides are contiguous).
__global__ void dq_finalize_v2_kernel(const float* __restrict__ acc, __nv_bfloat16* dq, int64_t dq_stride,
                                      int64_t n_seq, int heads, int seq_len, int seq_pad, float scale,
                                      const int* __restrict__ row_index) {
  constexpr int D = 128;
  const int64_t nqb = seq_pad / 4;
  const int64_t total = n_seq * heads * nqb * (D / 4);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int d0 = static_cast<int>(i % (D / 4)) * 4;
    const int64_t r = i / (D / 4);
    const int64_t qb = r % nqb;
    const int64_t sh = r / nqb;
    const int h = static_cast<int>(sh % heads);
    const int64_t s = sh / heads;
    const float4* src = reinterpret_cast<const float4*>(acc) + r * D + d0;  // [d0..d0+3][q%4]
    const float4 a0 = src[0], a1 = src[1], a2 = src[2], a3 = src[3];
    const float col[4][4] = {{a0.x, a1.x, a2.x, a3.x}, {a0.y, a1.y, a2.y, a3.y},
                             {a0.z, a1.z, a2.z, a3.z}, {a0.w, a1.w, a2.w, a3.w}};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = qb * 4 + j;
      if (q >= seq_len) break;
      const int64_t row = row_index ? row_index[s * seq_len + q] : s * seq_len + q;
      if (row < 0) continue;
      const __nv_bfloat162 lo = __floats2bfloat162_rn(col[j][0] * scale, col[j][1] * scale);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(col[j][2] * scale, col[j][3] * scale);
      uint2 pk;
      pk.x = *reinterpret_cast<const uint32_t*>(&lo);
      pk.y = *reinterpret_cast<const uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(dq + row * dq_stride + static_cast<int64_t>(h) * D + d0) = pk;
    }
  }
}

// delta and log2-domain lse per (seq, head, query), padded to seq_pad.  D/8 lanes per row, each
// with one 16-byte load of O and of dO (a row's head slice is one contiguous 2*D-byte segment).
// Scatter mode (out_index): O and dO rows are read through the forward's output table and the
// dO head slice is also written to the contiguous operand image do_image (n_seq, seq_len, heads*D),
// zeros past the sequence length -- the gather of dO rides on this pass, which reads them anyway.
template <int D>
__global__ void bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, int64_t o_stride,
                                const __nv_bfloat16* __restrict__ dout, int64_t do_stride,
                                const float* __restrict__ lse, float* lse2, float* delta, int64_t n_seq,
                                int heads, int seq_len, int seq_pad, const int* __restrict__ seq_lens,
                                const int* __restrict__ row_index, const int* __restrict__ out_index,
                                __nv_bfloat16* __restrict__ do_image) {
  constexpr int G = D / 8;             // lanes per row
  constexpr int R = 32 / G;            // rows per warp
  const int64_t total = n_seq * heads * static_cast<int64_t>(seq_pad);
  const int lane = threadIdx.x & 31;
  const int sub = lane / G, gl = lane % G;
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int* tab = row_index ? row_index : out_index;
  for (int64_t wb = warp0 * R; wb < total; wb += nwarps * R) {
    const int64_t w = wb + sub;
    const bool in = w < total;
    // 32-bit index arithmetic (64-bit division is a long software sequence); total < 2^31 is
    // checked by the launcher
    const uint32_t w32 = in ? static_cast<uint32_t>(w) : 0u;
    const int q = static_cast<int>(w32 % static_cast<uint32_t>(seq_pad));
    const uint32_t sh32 = w32 / static_cast<uint32_t>(seq_pad);
    const int64_t sh = sh32;
    const int h = static_cast<int>(sh32 % static_cast<uint32_t>(heads));
    const int64_t s = sh32 / static_cast<uint32_t>(heads);
    const int len = seq_lens ? __ldg(seq_lens + s) : seq_len;
    float acc = 0.f;
    uint4 dv = make_uint4(0u, 0u, 0u, 0u);
    if (in && q < len) {
      const int64_t row = tab ? __ldg(tab + s * seq_len + q) : s * seq_len + q;
      if (row >= 0) {
        const uint4 ov = *reinterpret_cast<const uint4*>(o + row * o_stride + static_cast<int64_t>(h) * D + gl * 8);
        dv = *reinterpret_cast<const uint4*>(dout + row * do_stride + static_cast<int64_t>(h) * D + gl * 8);
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
        const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 of = __bfloat1622float2(o2[j]);
          const float2 df = __bfloat1622float2(d2[j]);
          acc += of.x * df.x + of.y * df.y;
        }
      }
    }
    if (do_image && in && q < seq_len)
      *reinterpret_cast<uint4*>(do_image + (s * seq_len + q) * (static_cast<int64_t>(heads) * D) +
                                static_cast<int64_t>(h) * D + gl * 8) = dv;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, off);
    if (in && gl == 0) {
      delta[w] = acc;
      lse2[w] = q < len ? lse[sh * seq_len + q] * kLog2e : INFINITY;
    }
  }
}

template <int D>
__global__ void dq_finalize_kernel(const float* __restrict__ acc, __nv_bfloat16* dq, int64_t dq_stride,
                                   int64_t rows, int heads, float scale) {
  const int64_t per_row = static_cast<int64_t>(heads) * D / 4;
  const int64_t total = rows * per_row;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, c4 = i - r * per_row;
    const float4 v = reinterpret_cast<const float4*>(acc)[i];
    uint2 pk;
    pk.x = pack_bf16(v.x * scale, v.y * scale);
    pk.y = pack_bf16(v.z * scale, v.w * scale);
    *reinterpret_cast<uint2*>(dq + r * dq_stride + c4 * 4) = pk;
  }
}

struct BwdWs {
  float* dq_acc;
  float* lse2;
  float* delta;
};

BwdWs carve(void* ws, const AttnShape& s) {
  const int64_t seq_pad = (s.seq_len + 127) / 128 * 128;
  BwdWs w;
  uint8_t* p = static_cast<uint8_t*>(ws);
  w.dq_acc = reinterpret_cast<float*>(p);
  p += ((s.n_seq * seq_pad * s.heads * s.head_dim * 4 + 255) / 256) * 256;
  w.lse2 = reinterpret_cast<float*>(p);
  p += ((s.n_seq * s.heads * seq_pad * 4 + 255) / 256) * 256;
  w.delta = reinterpret_cast<float*>(p);
  return w;
}

unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

template <int D>
int launch_bwd_t(const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, void* dq, void* dk, void* dv, const AttnShape& s, int64_t qs,
                 int64_t ks, int64_t vs, int64_t os, int64_t dos, int64_t dqs, int64_t dks,
                 int64_t dvs, const uint32_t* bits, float scale, void* workspace, cudaStream_t stream) {
  const int64_t seq_pad = (s.seq_len + 127) / 128 * 128;
  BwdWs w = carve(workspace, s);
  if ((os % 8) || (dos % 8) || (reinterpret_cast<uintptr_t>(o) & 15) || (reinterpret_cast<uintptr_t>(dout) & 15)) {
    set_error("o / dout need 16-byte aligned bases and row strides");
    return kValue;
  }
  int rc = check_cuda(cudaMemsetAsync(w.dq_acc, 0, s.n_seq * seq_pad * s.heads * D * 4, stream),
                      "memset dq_acc");
  if (rc != kOk) return rc;
  if (s.n_seq * s.heads * seq_pad >= (int64_t(1) << 31)) {
    set_error("attention backward: n_seq * heads * padded length must stay below 2^31");
    return kValue;
  }
  {
    const int64_t rows = s.n_seq * s.heads * seq_pad;
    bwd_prep_kernel<D><<<grid_for(rows * 32 / (32 / (D / 8)), 256), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(o), os, static_cast<const __nv_bfloat16*>(dout), dos, lse,
        w.lse2, w.delta, s.n_seq, static_cast<int>(s.heads), static_cast<int>(s.seq_len),
        static_cast<int>(seq_pad), s.seq_lens, s.row_index, s.out_index,
        static_cast<__nv_bfloat16*>(s.out_index ? s.do_image : nullptr));
    rc = check_cuda(cudaGetLastError(), "bwd_prep launch");
    if (rc != kOk) return rc;
  }
  if (s.out_index) {  // scatter mode: the main kernel reads the contiguous dO image
    dout = s.do_image;
    dos = s.heads * D;
  }
  CUtensorMap mq, mk, mv, mdo;
  const int64_t cols = s.heads * D;
  const int qbox = D == 128 ? 64 : 128;
  if (s.row_index) {
    if (D != 128 || s.seq_len % 4) {
      set_error("gather-mode backward needs head_dim 128 and a row-index capacity multiple of 4");
      return kUnsupported;
    }
    if ((rc = make_tmap_bf16_2d(&mq, q, cols, s.n_rows, qs, 1)) != kOk) return rc;
    if ((rc = make_tmap_bf16_2d(&mk, k, cols, s.n_rows, ks, 1)) != kOk) return rc;
    if ((rc = make_tmap_bf16_2d(&mv, v, cols, s.n_rows, vs, 1)) != kOk) return rc;
    if ((rc = make_tmap_bf16_2d(&mdo, dout, cols, s.n_rows, dos, 1)) != kOk) return rc;
  } else {
    if ((rc = make_tmap_bf16_3d(&mq, q, cols, s.seq_len, s.n_seq, qs, qbox)) != kOk) return rc;
    if ((rc = make_tmap_bf16_3d(&mk, k, cols, s.seq_len, s.n_seq, ks, 128)) != kOk) return rc;
    if ((rc = make_tmap_bf16_3d(&mv, v, cols, s.seq_len, s.n_seq, vs, 128)) != kOk) return rc;
    if ((rc = make_tmap_bf16_3d(&mdo, dout, cols, s.seq_len, s.n_seq, dos, qbox)) != kOk) return rc;
  }
  if ((dks * 2) % 16 || (dvs * 2) % 16 || (reinterpret_cast<uintptr_t>(dk) & 15) ||
      (reinterpret_cast<uintptr_t>(dv) & 15) || (dqs * 2) % 8 || (reinterpret_cast<uintptr_t>(dq) & 7)) {
    set_error("gradient outputs need 16-byte aligned bases/row strides");
    return kValue;
  }
  BwdArgs a;
  a.lse2 = w.lse2;
  a.delta = w.delta;
  a.dq_acc = w.dq_acc;
  a.dk = static_cast<__nv_bfloat16*>(dk);
  a.dv = static_cast<__nv_bfloat16*>(dv);
  a.dk_stride = dks;
  a.dv_stride = dvs;
  a.valid_bits = bits;
  a.words_per_seq = static_cast<int>((s.seq_len + 31) / 32);
  a.seq_len = static_cast<int>(s.seq_len);
  a.seq_lens = s.seq_lens;
  a.row_index = s.row_index;
  a.n_rows = static_cast<int>(s.n_rows);
  a.seq_pad = static_cast<int>(seq_pad);
  a.heads = static_cast<int>(s.heads);
  a.n_q = static_cast<int>(seq_pad / 128);
  a.scale = scale;
  a.scale_log2 = scale * kLog2e;
  a.k_rows = static_cast<const __nv_bfloat16*>(k);
  a.k_row_stride = ks;
  static const int bwd_flags = env_int("OSP_BWD_FLAGS", 0);
  a.flags = bwd_flags;
  static std::atomic<uint64_t> attr_done_v1{0}, attr_done_v2{0};
  if constexpr (D == 128)
    rc = set_smem_attr(reinterpret_cast<const void*>(attn_bwd_v2_kernel), BwdV2Layout::kSmemX, attr_done_v2,
                       "cudaFuncSetAttribute(attn_bwd_v2)");
  else
    rc = set_smem_attr(reinterpret_cast<const void*>(attn_bwd_kernel<D>), BwdLayout<D>::kSmem, attr_done_v1,
                       "cudaFuncSetAttribute(attn_bwd)");
  if (rc != kOk) return rc;
  dim3 grid(static_cast<unsigned>(seq_pad / 128), static_cast<unsigned>(s.heads),
            static_cast<unsigned>(s.n_seq));
  if constexpr (D == 128) {
    attn_bwd_v2_kernel<<<grid, kBwdV2Threads, BwdV2Layout::kSmemX, stream>>>(mq, mk, mv, mdo, a);
    rc = check_cuda(cudaGetLastError(), "attn_bwd_v2_kernel launch");
    if (rc != kOk) return rc;
    dq_finalize_v2_kernel<<<grid_for(s.n_seq * s.heads * seq_pad / 4 * (D / 4), 256), 256, 0, stream>>>(
        w.dq_acc, static_cast<__nv_bfloat16*>(dq), dqs, s.n_seq, static_cast<int>(s.heads),
        static_cast<int>(s.seq_len), static_cast<int>(seq_pad), scale, s.row_index);
    return check_cuda(cudaGetLastError(), "dq_finalize_v2 launch");
  }
  attn_bwd_kernel<D><<<grid, kBwdThreads, BwdLayout<D>::kSmem, stream>>>(mq, mk, mv, mdo, a);
  rc = check_cuda(cudaGetLastError(), "attn_bwd_kernel launch");
  if (rc != kOk) return rc;
  const int64_t rows = s.n_seq * s.seq_len;
  dq_finalize_kernel<D><<<grid_for(rows * s.heads * D / 4, 256), 256, 0, stream>>>(
      w.dq_acc, static_cast<__nv_bfloat16*>(dq), dqs, rows, static_cast<int>(s.heads), scale);
  return check_cuda(cudaGetLastError(), "dq_finalize launch");
}

}  // namespace

size_t attn_bwd_workspace_bytes(const AttnShape& s) {
  const int64_t seq_pad = (s.seq_len + 127) / 128 * 128;
  const int64_t a = ((s.n_seq * seq_pad * s.heads * s.head_dim * 4 + 255) / 256) * 256;
  const int64_t b = ((s.n_seq * s.heads * seq_pad * 4 + 255) / 256) * 256;
  return static_cast<size_t>(a + 2 * b);
}

int debug_counters_bwd(unsigned long long* host, int n, int reset) {
  if (n > 64) n = 64;
  int rc = check_cuda(cudaMemcpyFromSymbol(host, g_bwd_counters, n * sizeof(unsigned long long)),
                      "cudaMemcpyFromSymbol");
  if (rc != kOk || !reset) return rc;
  static const unsigned long long zeros[64] = {};
  return check_cuda(cudaMemcpyToSymbol(g_bwd_counters, zeros, sizeof(zeros)), "cudaMemcpyToSymbol");
}

int launch_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                    const float* lse, void* dq, void* dk, void* dv, const AttnShape& s,
                    int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                    int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                    const uint32_t* valid_bits, int zero_invalid_queries, float scale,
                    void* workspace, size_t workspace_bytes, cudaStream_t stream) {
  (void)zero_invalid_queries;  // encoded in lse (+inf rows) by the forward
  (void)workspace_bytes;
  if (s.head_dim == 128)
    return launch_bwd_t<128>(q, k, v, o, dout, lse, dq, dk, dv, s, q_stride, k_stride, v_stride,
                             o_stride, do_stride, dq_stride, dk_stride, dv_stride, valid_bits, scale,
                             workspace, stream);
  if (s.head_dim == 64)
    return launch_bwd_t<64>(q, k, v, o, dout, lse, dq, dk, dv, s, q_stride, k_stride, v_stride,
                            o_stride, do_stride, dq_stride, dk_stride, dv_stride, valid_bits, scale,
                            workspace, stream);
  set_error("attention kernels support head_dim 64 or 128");
  return kUnsupported;
}

}  // namespace osp
