// K2: per-subsequence attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Replaces the reference's dense_attention hot loop (attention.py:47-67) as called
// per subsequence by skiparse_attention (attention.py:126): out = softmax(q k^T * scale +
// key mask) v, with the reference's exact-zero rules (attention.py:35-44): masked keys weigh
// 0, a row with no valid key outputs 0; optionally pad-query rows output 0
// (attention.py:127-130).
//
// One CTA owns two 128-row query tiles of one (subsequence, head) and streams 128-key tiles.
//   warp 0      TMA producer (Q once, K/V double-buffered, 128B-swizzled boxes of 64 cols)
//   warp 1      MMA issuer   (single thread; S_t = Q_t K^T into TMEM, O_t += P_t V with P
//                             read straight from TMEM)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O0 | O1)
//   warps 4-7   softmax for query tile 0, warps 8-11 for tile 1: one thread per row,
//               online softmax in the log2 domain, lazy O rescaling (only when the running
//               max grows by > 2^8), P written back into the S columns as packed bf16.
//               Per tile: load S, exact row max, (rare) O rescale, then the exp phase -- only
//               scale, exp2 (MUFU or, for 1/8 of the columns, an FMA-pipe polynomial), bf16 pack
//               and the TMEM store -- then P is handed to the MMA and the row sum is added.  The
//               two warpgroups' exp phases run concurrently (OSP_FWD_PINGPONG=1 serialises them
//               on named barriers; measured 3-8% slower).
// MMA order per key tile j: QK0_j, PV1_{j-1}, QK1_j, PV0_j, so one tile's softmax overlaps
// the other tile's tensor-core work.
#include "osp_common.cuh"
#include "osp_internal.h"

#include <cstdlib>
#include <type_traits>

namespace osp {
namespace {

constexpr int kFwdThreads = 384;
constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
// every kPolyEvery-th packed column pair of a full tile uses the polynomial exp2 (0 = never)
#ifndef OSP_FWD_POLY
#define OSP_FWD_POLY 8
#endif
constexpr int kPolyEvery = OSP_FWD_POLY;
// on tiles without masked keys the last kPolyChunks of the four 32-key chunks take the polynomial
// exp2, computed before the warpgroup's MUFU turn (0-2)
#ifndef OSP_FWD_POLY_CHUNKS
#define OSP_FWD_POLY_CHUNKS 0
#endif
constexpr int kPolyChunks = OSP_FWD_POLY_CHUNKS;
// bf16 P by truncation (one PRMT per pair on the ALU pipe) instead of F2FP round-to-nearest; the
// row sum l then adds the truncated values, so O / l stays an exactly normalised combination
#ifndef OSP_FWD_TRUNC
#define OSP_FWD_TRUNC 0
#endif
// hand P over in two 64-key halves (PV issued as two K = 64 halves, the first under the second
// half's exps) instead of one
#ifndef OSP_FWD_SPLITPV
#define OSP_FWD_SPLITPV 0
#endif
// serialise the two softmax warpgroups' exp phases (1) or let them overlap (0)
#ifndef OSP_FWD_PINGPONG
#define OSP_FWD_PINGPONG 0
#endif

// V tiles get a deeper ring than K: V_j is released only by PV_{j} of the second query tile, late
// in the key loop, so with two stages its reload has about one key tile of lead
#ifndef OSP_FWD_VSTAGES
#define OSP_FWD_VSTAGES 2
#endif
constexpr int kFwdVStages = OSP_FWD_VSTAGES;

template <int D>
struct FwdLayout {
  static constexpr int kSub = D / 64;
  static constexpr int kTile = kBM * D * 2;
  static constexpr int kQ = 0;
  static constexpr int kK = kQ + 2 * kTile;
  static constexpr int kV = kK + 2 * kTile;
  static constexpr int kBar = kV + kFwdVStages * kTile;
  static constexpr int kSmem = kBar + 256 + 1024;
};

struct FwdArgs {
  __nv_bfloat16* o;
  int64_t o_stride;
  float* lse;
  const uint32_t* valid_bits;
  int words_per_seq;
  int seq_len;              // capacity (row stride of a sequence)
  const int* seq_lens;      // per-sequence valid length (<= seq_len) or null
  const int* row_index;     // gather mode: (n_seq, seq_len) token rows of q/k/v/o (-1 = none)
  int n_rows;               // gather mode: rows of the q/k/v/o tensors
  const int* out_index;     // scatter mode: (n_seq, seq_len) destination rows of o (-1 = none)
  const int* zero_rows;     // scatter mode: destination rows with no source (zero-filled)
  int n_zero;
  int heads;
  float scale_log2;
  int zero_invalid_q;
  int flags;  // debug experiments (OSP_FWD_FLAGS): 1 = no exp, 2 = softmax skeleton only,
             // 4 = no exp-phase ping-pong, 8 = no K/V reloads, 16 = no P store, 32 = no row sum
};

__device__ __forceinline__ bool bit_at(const uint32_t* bits, int words, int i) {
  int w = i >> 5;
  return w < words && ((__ldg(bits + w) >> (i & 31)) & 1u);
}

// Q tiles requested by thread 0 right after the barrier init (1), or by the producer after the
// block barrier (0, rounds 1-2).
#ifndef OSP_FWD_EARLY_Q
#define OSP_FWD_EARLY_Q 1
#endif
// Epilogue through a shared-memory stage with whole-row coalesced stores (1) or one row per
// thread straight from registers (0, rounds 1-2).
#ifndef OSP_FWD_STAGED_EPI
#define OSP_FWD_STAGED_EPI 1
#endif
// Phase timing (-DOSP_FWD_TIMING=1 builds only): per-phase clock64 sums of the first softmax
// warp of each warpgroup and of the MMA issuer, and per-CTA prologue / loop / epilogue cycles,
// read back with osp_debug_counters().
#ifndef OSP_FWD_TIMING
#define OSP_FWD_TIMING 0
#endif
__device__ unsigned long long g_fwd_counters[64];

// Experiment switches (FwdArgs::flags) are compiled in only with -DOSP_FWD_EXPERIMENTS=1: the
// softmax loop sits at its register budget, and even never-taken runtime branches cost time.
#ifndef OSP_FWD_EXPERIMENTS
#define OSP_FWD_EXPERIMENTS 0
#endif

template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const FwdArgs a) {
  using Ly = FwdLayout<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_q = bars + 0;
  uint64_t* bar_kf = bars + 2;
  uint64_t* bar_ke = bars + 4;
  uint64_t* bar_s = bars + 6;
  uint64_t* bar_p = bars + 8;
  uint64_t* bar_o = bars + 10;
  uint64_t* bar_pb = bars + 12;  // second P half (OSP_FWD_SPLITPV)
  uint64_t* bar_vf = bars + 14;  // [kFwdVStages]
  uint64_t* bar_ve = bars + 14 + kFwdVStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14 + 2 * kFwdVStages);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int flags = OSP_FWD_EXPERIMENTS ? a.flags : 0;
  const int head = blockIdx.y;
  const int seq = blockIdx.z;
  const int q_row0 = blockIdx.x * 2 * kBM;
  // variable-length sequences: rows >= len are neither keys nor queries (compacted layouts)
  const int len = a.seq_lens ? __ldg(a.seq_lens + seq) : a.seq_len;
  if (a.n_zero && warp == 3) {
    // scatter mode: this CTA's share of the destination rows no sequence row lands on (disjoint
    // from every stored row), head slice `head`; 16 lanes x 16 B per 128-d row
    const int64_t n_cta = static_cast<int64_t>(gridDim.x) * gridDim.z;
    const int64_t b = blockIdx.x + static_cast<int64_t>(gridDim.x) * blockIdx.z;
    const int64_t r0 = b * a.n_zero / n_cta, r1 = (b + 1) * a.n_zero / n_cta;
    constexpr int kLanesPerRow = D / 8;
    constexpr int kRowsPerIter = 32 / kLanesPerRow;
    for (int64_t r = r0 + lane / kLanesPerRow; r < r1; r += kRowsPerIter) {
      const int64_t row = __ldg(a.zero_rows + r);
      *reinterpret_cast<uint4*>(a.o + row * a.o_stride + static_cast<int64_t>(head) * D +
                                (lane % kLanesPerRow) * 8) = make_uint4(0u, 0u, 0u, 0u);
    }
  }
  if (q_row0 >= len) {  // whole CTA past the sequence: o rows 0, lse +inf
    const int r1 = min(q_row0 + 2 * kBM, a.seq_len);
    if (!a.row_index && !a.out_index)  // gather / scatter mode: rows past the length have no destination
      zero_rows_bf16(a.o + static_cast<int64_t>(seq) * a.seq_len * a.o_stride + static_cast<int64_t>(head) * D,
                     a.o_stride, q_row0, r1, D);
    for (int r = q_row0 + static_cast<int>(threadIdx.x); r < r1; r += blockDim.x)
      a.lse[(static_cast<int64_t>(seq) * a.heads + head) * a.seq_len + r] = INFINITY;
    return;
  }
  const int n_kv = (len + kBN - 1) / kBN;
#if OSP_FWD_TIMING
  const long long t_entry = clock64();
  long long t_first = 0, t_fin = 0;
#endif

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_q + i, 1);
      mbar_init(bar_kf + i, 1);
      mbar_init(bar_ke + i, 1);

      mbar_init(bar_s + i, 1);
      mbar_init(bar_p + i, 128);
      mbar_init(bar_pb + i, 128);
      mbar_init(bar_o + i, 1);
    }
    for (int i = 0; i < kFwdVStages; ++i) {
      mbar_init(bar_vf + i, 1);
      mbar_init(bar_ve + i, 1);
    }
    fence_barrier_init();
#if OSP_FWD_EARLY_Q
    if (!a.row_index) {  // the Q tiles in flight before the TMEM allocation and the block barrier
      for (int t = 0; t < 2; ++t) {
        mbar_expect_tx(bar_q + t, Ly::kTile);
#pragma unroll
        for (int s = 0; s < Ly::kSub; ++s)
          tma_load_3d(sm + Ly::kQ + t * Ly::kTile + s * 16384, &tmQ, bar_q + t, head * D + s * 64,
                      q_row0 + t * kBM, seq);
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

  if (warp < 4) {
    regs_dec<56>();
  if (warp == 0 && a.row_index) {
    // -------------------------------------------------------------- TMA producer, gather mode:
    // each lane fetches 4 token rows of a 128-row tile with one tile::gather4 per 64 columns
    const int* ridx = a.row_index + static_cast<int64_t>(seq) * a.seq_len;
    auto gather_tile = [&](uint8_t* dst, const CUtensorMap* m, uint64_t* bar, int row0) {
      const int4 r = *reinterpret_cast<const int4*>(ridx + row0 + 4 * lane);
      const int oob = a.n_rows;  // out-of-range rows are zero-filled by the TMA
      const int r0 = r.x < 0 ? oob : r.x, r1 = r.y < 0 ? oob : r.y, r2 = r.z < 0 ? oob : r.z,
                r3 = r.w < 0 ? oob : r.w;
#pragma unroll
      for (int s = 0; s < Ly::kSub; ++s)
        tma_gather4(dst + s * 16384 + lane * 512, m, bar, head * D + s * 64, r0, r1, r2, r3);
    };
    if (lane == 0) {
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      mbar_expect_tx(bar_q + 0, Ly::kTile);
      mbar_expect_tx(bar_q + 1, Ly::kTile);
    }
    __syncwarp();
    for (int t = 0; t < 2; ++t) gather_tile(sm + Ly::kQ + t * Ly::kTile, &tmQ, bar_q + t, q_row0 + t * kBM);
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      mbar_wait(bar_ke + st, ph ^ 1);
      if (lane == 0) mbar_expect_tx(bar_kf + st, Ly::kTile);
      __syncwarp();
      gather_tile(sm + Ly::kK + st * Ly::kTile, &tmK, bar_kf + st, j * kBN);
      const int vs = j % kFwdVStages;
      mbar_wait(bar_ve + vs, ((j / kFwdVStages) & 1) ^ 1);
      if (lane == 0) mbar_expect_tx(bar_vf + vs, Ly::kTile);
      __syncwarp();
      gather_tile(sm + Ly::kV + vs * Ly::kTile, &tmV, bar_vf + vs, j * kBN);
    }
  } else if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------ TMA producer
      tma_prefetch(&tmQ);
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
      for (int t = 0; t < 2 && !OSP_FWD_EARLY_Q; ++t) {
        mbar_expect_tx(bar_q + t, Ly::kTile);
#pragma unroll
        for (int s = 0; s < Ly::kSub; ++s)
          tma_load_3d(sm + Ly::kQ + t * Ly::kTile + s * 16384, &tmQ, bar_q + t, head * D + s * 64,
                      q_row0 + t * kBM, seq);
      }
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        if ((flags & 8) && j >= 2) {  // experiment 8: no K/V reloads (stale tiles, timing only)
          mbar_wait(bar_ke + st, ph ^ 1);
          mbar_arrive(bar_kf + st);
          mbar_wait(bar_ve + j % kFwdVStages, ((j / kFwdVStages) & 1) ^ 1);
          mbar_arrive(bar_vf + j % kFwdVStages);
          continue;
        }
        mbar_wait(bar_ke + st, ph ^ 1);
        mbar_expect_tx(bar_kf + st, Ly::kTile);
#pragma unroll
        for (int s = 0; s < Ly::kSub; ++s)
          tma_load_3d(sm + Ly::kK + st * Ly::kTile + s * 16384, &tmK, bar_kf + st,
                      head * D + s * 64, j * kBN, seq);
        const int vs = j % kFwdVStages;
        mbar_wait(bar_ve + vs, ((j / kFwdVStages) & 1) ^ 1);
        mbar_expect_tx(bar_vf + vs, Ly::kTile);
#pragma unroll
        for (int s = 0; s < Ly::kSub; ++s)
          tma_load_3d(sm + Ly::kV + vs * Ly::kTile + s * 16384, &tmV, bar_vf + vs,
                      head * D + s * 64, j * kBN, seq);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (whole warp
    // runs the control flow; one elected lane issues, so operands stay warp-uniform)
    constexpr uint32_t kIdQK = idesc_bf16(kBM, kBN, 0, 0);
    constexpr uint32_t kIdPV = idesc_bf16(kBM, D, 0, 1);
    const uint32_t tm_ = __shfl_sync(0xFFFFFFFFu, tmem, 0);
    const uint32_t q_base = smem_u32(sm + Ly::kQ);
    const uint32_t k_base = smem_u32(sm + Ly::kK);
    const uint32_t v_base = smem_u32(sm + Ly::kV);
    // The bases go through an opaque move at every use, so the compiler re-derives the ~40
    // descriptor / TMEM addresses with a few adds instead of hoisting them out of the key loop
    // into registers the 64-register control-warp budget cannot hold (they spilled to local
    // memory and every MMA group reloaded them).
    auto opaque = [](uint32_t v) {
      asm volatile("mov.b32 %0, %0;" : "+r"(v));
      return v;
    };
    auto qk = [&](int t, int st, uint64_t* bar_a, uint64_t* bar_b) {
      const uint32_t qa = opaque(q_base) + t * Ly::kTile;
      const uint32_t kb = opaque(k_base) + st * Ly::kTile;
      const uint32_t tm = opaque(tm_);
      {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tm + t * 128, sdesc_sw128(qa + off, 16, 1024), sdesc_sw128(kb + off, 16, 1024),
                 kIdQK, kk > 0);
        }
        tc_commit(bar_a);
        if (bar_b) tc_commit(bar_b);
      }
    };
    // O_t += P_t V over keys [16*k0, 16*k1) of the tile
    auto pv_part = [&](int t, int st, bool acc, int k0, int k1) {
      const uint32_t vb = opaque(v_base) + st * Ly::kTile;
      const uint32_t tm = opaque(tm_);
#pragma unroll
      for (int kk = k0; kk < k1; ++kk)
        mma_ts(tm + 256 + t * 128, tm + t * 128 + kk * 8, sdesc_sw128(vb + kk * 2048, 16384, 1024),
               kIdPV, (acc || kk > 0) ? 1u : 0u);
    };
    // waits for P_t (both halves, or the two halves one after the other) and issues PV_t
    auto pv = [&](int t, int st, bool acc, uint32_t ph, uint64_t* bar_a, uint64_t* bar_b, uint64_t* bar_c) {
      mbar_wait(bar_p + t, ph);
      tc_fence_after();
      if (OSP_FWD_SPLITPV) {
        pv_part(t, st, acc, 0, kBN / 32);
        mbar_wait(bar_pb + t, ph);
        tc_fence_after();
        pv_part(t, st, true, kBN / 32, kBN / 16);
      } else {
        pv_part(t, st, acc, 0, kBN / 16);
      }
      if (bar_a) tc_commit(bar_a);
      if (bar_b) tc_commit(bar_b);
      if (bar_c) tc_commit(bar_c);
    };
    if (elect_one()) {
    mbar_wait(bar_q + 0, 0);
    mbar_wait(bar_q + 1, 0);
    tc_fence_after();
#if OSP_FWD_TIMING
    t_first = clock64();
    unsigned long long mt[4] = {0, 0, 0, 0};
    long long m0 = clock64();
#define OSP_MT(k) do { const long long _t = clock64(); mt[k] += _t - m0; m0 = _t; } while (0)
#else
#define OSP_MT(k) do { } while (0)
#endif
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      const uint32_t ph = (j >> 1) & 1;
#if OSP_FWD_TIMING
      m0 = clock64();
#endif
      mbar_wait(bar_kf + st, ph);
      OSP_MT(0);
      tc_fence_after();
      qk(0, st, bar_s + 0, nullptr);
      if (j > 0) {
#if OSP_FWD_TIMING
        m0 = clock64();
#endif
        pv(1, (j - 1) % kFwdVStages, j - 1 > 0, (j - 1) & 1, bar_ve + (j - 1) % kFwdVStages, nullptr, nullptr);
        OSP_MT(1);
      }
      qk(1, st, bar_s + 1, bar_ke + st);
#if OSP_FWD_TIMING
      m0 = clock64();
#endif
      mbar_wait(bar_vf + j % kFwdVStages, (j / kFwdVStages) & 1);
      OSP_MT(2);
      pv(0, j % kFwdVStages, j > 0, j & 1, nullptr, nullptr, nullptr);
      OSP_MT(3);
    }
#if OSP_FWD_TIMING
    for (int k = 0; k < 4; ++k) atomicAdd(&g_fwd_counters[16 + k], mt[k]);
    atomicAdd(&g_fwd_counters[20], static_cast<unsigned long long>(n_kv));
#endif
    const int last = n_kv - 1;
    pv(1, last % kFwdVStages, last > 0, last & 1, bar_ve + last % kFwdVStages, bar_o + 0, bar_o + 1);
#if OSP_FWD_TIMING
    t_fin = clock64();
#endif
    }
    __syncwarp();
  }
  } else {
    regs_inc<224>();
    // -------------------------------------------------------------- softmax / epilogue
    const int t = (warp - 4) >> 2;
    const int wq = warp & 3;
    const uint32_t lane_addr = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t tS = tmem + lane_addr + t * 128;
    const uint32_t tO = tmem + lane_addr + 256 + t * 128;
    const int q_row = q_row0 + t * kBM + wq * 32 + lane;
    const uint32_t* vbits =
        a.valid_bits ? a.valid_bits + static_cast<int64_t>(seq) * a.words_per_seq : nullptr;
    const float c = a.scale_log2;
    // The two softmax warpgroups share the SM's MUFU (16 ex2/clk).  Their exp phases are
    // serialised in tile order (named barriers 2 and 3, ping-pong) so each tile's softmax
    // finishes within the window the other tile's MMAs cover, instead of both running at half
    // speed.  Warpgroup 1 opens the first turn for warpgroup 0.
    const uint32_t my_turn = 2 + t, next_turn = 3 - t;
    const bool pingpong = OSP_FWD_PINGPONG && !(flags & 4);  // experiment 4: no exp-phase serialisation
    if (t == 1 && pingpong) asm volatile("bar.arrive %0, 256;" ::"r"(2u) : "memory");

    float m_used = -INFINITY;
    float l = 0.f;
    // key-mask words of tile j (validity bits and the subsequence tail), fetched one tile ahead
    auto mask_words = [&](int j, uint32_t (&w)[4]) {
      const int kv0 = j * kBN;
      const int nvalid = min(kBN, len - kv0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t m = vbits ? ((kv0 >> 5) + i < a.words_per_seq ? __ldg(vbits + (kv0 >> 5) + i) : 0u)
                           : 0xFFFFFFFFu;
        const int lo = i * 32;
        if (nvalid <= lo) m = 0u;
        else if (nvalid < lo + 32) m &= (1u << (nvalid - lo)) - 1u;
        w[i] = m;
      }
    };
    uint32_t w_next[4];
    mask_words(0, w_next);
#if OSP_FWD_TIMING
    unsigned long long sp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long s0t = clock64();
#define OSP_ST(k) do { const long long _t = clock64(); sp[k] += _t - s0t; s0t = _t; } while (0)
#else
#define OSP_ST(k) do { } while (0)
#endif
    for (int j = 0; j < n_kv; ++j) {
#if OSP_FWD_TIMING
      s0t = clock64();
#endif
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = w_next[i];
      if (j + 1 < n_kv) mask_words(j + 1, w_next);
      mbar_wait(bar_s + t, j & 1);
      OSP_ST(0);
      tc_fence_after();
      if (flags & 2) {
        tc_fence_before();
        mbar_arrive(bar_p + t);
        mbar_arrive(bar_pb + t);
        continue;
      }
      uint32_t s[4][32];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tmem_ld32(tS + cc * 32, s[cc]);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) tmem_wait_ld(s[cc]);
      OSP_ST(1);
      if ((w[0] & w[1] & w[2] & w[3]) != 0xFFFFFFFFu) {
#pragma unroll
        for (int cc = 0; cc < 4; ++cc)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (!((w[cc] >> i) & 1u)) s[cc][i] = __float_as_uint(-INFINITY);
      }
      // Rescale O (in TMEM) and l to a new running max.  PV_{j-1} of this tile is complete:
      // S_j was committed after it and tcgen05 operations execute in order.
      auto rescale = [&](float m_new) {
        const float m_upd = fmaxf(m_new, m_used);
        const float alpha = (m_used == -INFINITY) ? 0.f : ex2((m_used - m_upd) * c);
        if (j > 0) {
#pragma unroll
          for (int cc = 0; cc < D / 32; ++cc) {
            uint32_t o[32];
            tmem_ld32(tO + cc * 32, o);
            tmem_wait_ld(o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(tO + cc * 32, o);
          }
        }
        l *= alpha;
        m_used = m_upd;
      };
      auto row_max = [&]() {
        float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          mx0 = fmaxf(mx0, __uint_as_float(s[0][i]));
          mx1 = fmaxf(mx1, __uint_as_float(s[1][i]));
          mx2 = fmaxf(mx2, __uint_as_float(s[2][i]));
          mx3 = fmaxf(mx3, __uint_as_float(s[3][i]));
        }
        return fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      };
      auto needs_rescale = [&](float m_new) {
        return (m_new > m_used) && (m_used == -INFINITY || (m_new - m_used) * c > kRescaleThreshold);
      };
      // The exp phase is the serialised resource (the two warpgroups take turns on the SM's
      // MUFU), so it holds only what must run in it: scale (FFMA2), exp2, bf16 pack, P -> TMEM.
      // The row max runs before the turn and the row sum after P is handed over, both while the
      // other warpgroup exponentiates.  On tiles without masked keys every kPolyEvery-th column
      // pair takes the FMA-pipe polynomial instead of MUFU.EX2.  p overwrites s in place (fp32)
      // for the row sum.
      const float2 c2 = make_float2(c, c);
      float2 nms2;  // -(running max) * c, set once the max for this tile is final
      // One 32-key chunk: scale, exp2 (MUFU, or with POLY the FMA-pipe polynomial), bf16 pack,
      // P -> TMEM; p overwrites s in place (fp32) for the row sum.  MIX: inside a MUFU chunk every
      // kPolyEvery-th pair still takes the polynomial (tiles without masked keys only).
      auto chunk = [&](int cc, auto poly_tag, auto mix_tag, bool pass_turn) {
        constexpr bool kAllPoly = decltype(poly_tag)::value;
        constexpr bool kMix = decltype(mix_tag)::value;
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = __ffma2_rn(
              make_float2(__uint_as_float(s[cc][2 * i]), __uint_as_float(s[cc][2 * i + 1])), c2, nms2);
          float2 p;
          if (flags & 1) {  // experiment 1: no exp2 at all (timing only)
            p = x;
          } else if (kAllPoly || (kMix && kPolyEvery > 0 && (i % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1)) {
            p = exp2_poly2(x);
          } else {
            p.x = ex2(x.x);
            p.y = ex2(x.y);
          }
          s[cc][2 * i] = __float_as_uint(p.x);
          s[cc][2 * i + 1] = __float_as_uint(p.y);
          pk[i] = OSP_FWD_TRUNC ? pack_bf16_trunc(p.x, p.y) : pack_bf16(p.x, p.y);
        }
        if (pass_turn && pingpong && !(t == 1 && j == n_kv - 1))
          asm volatile("bar.arrive %0, 256;" ::"r"(next_turn) : "memory");
        if (!(flags & 16)) tmem_st16(tS + cc * 16, pk);  // experiment 16: no P store (timing only)
        if (OSP_FWD_SPLITPV && cc == 1) {  // keys 0-63 of P ready: PV's first half may run
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar_p + t);
        }
      };
      // Exact running max before the exps (off the MUFU turn).  The rescale of O, when the max
      // grew by more than 2^kRescaleThreshold, is legal here: PV_{j-1} of this tile is complete.
      const float m_new = fmaxf(m_used, row_max());
      if (__any_sync(0xFFFFFFFFu, needs_rescale(m_new))) rescale(m_new);
      {
        const float ms = (m_used == -INFINITY) ? 0.f : m_used * c;
        nms2 = make_float2(-ms, -ms);
      }
      using T_ = std::true_type;
      using F_ = std::false_type;
      if ((w[0] & w[1] & w[2] & w[3]) == 0xFFFFFFFFu) {
        // the last kPolyChunks chunks run on the FMA pipe BEFORE the MUFU turn, i.e. while the
        // other warpgroup holds the MUFU; the rest on MUFU during this warpgroup's turn
#pragma unroll
        for (int cc = 4 - kPolyChunks; cc < 4; ++cc) chunk(cc, T_{}, F_{}, false);
        if (pingpong) named_bar_sync(my_turn, 256);
        OSP_ST(2);
#pragma unroll
        for (int cc = 0; cc < 4 - kPolyChunks; ++cc) chunk(cc, F_{}, T_{}, cc == 3 - kPolyChunks);
      } else {
        // masked keys need exact zeros: MUFU everywhere
        if (pingpong) named_bar_sync(my_turn, 256);
        OSP_ST(2);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) chunk(cc, F_{}, F_{}, cc == 3);
      }
      OSP_ST(3);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(OSP_FWD_SPLITPV ? bar_pb + t : bar_p + t);
      OSP_ST(4);
      if (!(flags & 32)) {  // experiment 32: no row sum (timing only)
        float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0, a3 = a0;
        if (OSP_FWD_TRUNC) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int i = 0; i < 32; ++i) s[cc][i] &= 0xFFFF0000u;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          a0 = __fadd2_rn(a0, make_float2(__uint_as_float(s[0][2 * i]), __uint_as_float(s[0][2 * i + 1])));
          a1 = __fadd2_rn(a1, make_float2(__uint_as_float(s[1][2 * i]), __uint_as_float(s[1][2 * i + 1])));
          a2 = __fadd2_rn(a2, make_float2(__uint_as_float(s[2][2 * i]), __uint_as_float(s[2][2 * i + 1])));
          a3 = __fadd2_rn(a3, make_float2(__uint_as_float(s[3][2 * i]), __uint_as_float(s[3][2 * i + 1])));
        }
        const float2 t2 = __fadd2_rn(__fadd2_rn(a0, a1), __fadd2_rn(a2, a3));
        l += t2.x + t2.y;
      }
      OSP_ST(5);
    }
#if OSP_FWD_TIMING
    if (lane == 0 && wq == 0) {
      for (int k = 0; k < 6; ++k) atomicAdd(&g_fwd_counters[t * 8 + k], sp[k]);
      atomicAdd(&g_fwd_counters[t * 8 + 7], static_cast<unsigned long long>(n_kv));
    }
#endif

    // ---------------------------------------------------------------- epilogue
    mbar_wait(bar_o + t, 0);
    tc_fence_after();
    const bool row_ok = q_row < len;
    const bool in_cap = q_row < a.seq_len;  // rows in [len, cap) are written as 0 / +inf
    bool q_valid = true;
    if (a.zero_invalid_q && vbits && row_ok) q_valid = bit_at(vbits, a.words_per_seq, q_row);
    const bool live = row_ok && q_valid && l > 0.f;
    const float inv_l = live ? 1.f / l : 0.f;
    const int* tab = a.row_index ? a.row_index : a.out_index;
    const int64_t out_row =
        tab ? (row_ok ? __ldg(tab + static_cast<int64_t>(seq) * a.seq_len + q_row) : -1)
            : static_cast<int64_t>(seq) * a.seq_len + q_row;
    const bool write_o = tab ? out_row >= 0 : in_cap;
#if OSP_FWD_STAGED_EPI
    // The warp's 32 rows are staged in its quarter of this tile's Q buffer (free: bar_o follows
    // the last MMA, and tcgen05 ops complete in order), 16-byte chunks XOR-swizzled by row so
    // both passes are bank-conflict free, then stored two whole 256-byte rows per instruction
    // instead of one 16-byte piece of 32 different rows.
    constexpr int kCh = D / 8;               // 16-byte chunks per row
    constexpr int kRowsPerIns = 32 / kCh;    // rows per coalesced warp store
    uint8_t* stg = sm + Ly::kQ + t * Ly::kTile + wq * (32 * D * 2);
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(tO + cc * 32, o);
      tmem_wait_ld(o);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 pk;
        pk.x = pack_bf16(__uint_as_float(o[8 * i + 0]) * inv_l, __uint_as_float(o[8 * i + 1]) * inv_l);
        pk.y = pack_bf16(__uint_as_float(o[8 * i + 2]) * inv_l, __uint_as_float(o[8 * i + 3]) * inv_l);
        pk.z = pack_bf16(__uint_as_float(o[8 * i + 4]) * inv_l, __uint_as_float(o[8 * i + 5]) * inv_l);
        pk.w = pack_bf16(__uint_as_float(o[8 * i + 6]) * inv_l, __uint_as_float(o[8 * i + 7]) * inv_l);
        *reinterpret_cast<uint4*>(stg + lane * (D * 2) + (((cc * 4 + i) ^ (lane & (kCh - 1))) * 16)) = pk;
      }
    }
    __syncwarp();
    {
      const int ch = lane % kCh;
#pragma unroll 4
      for (int rr = 0; rr < 32 / kRowsPerIns; ++rr) {
        const int r = kRowsPerIns * rr + lane / kCh;
        const long long dst_row = __shfl_sync(0xFFFFFFFFu, static_cast<long long>(out_row), r);
        const bool w = __shfl_sync(0xFFFFFFFFu, write_o ? 1 : 0, r) != 0;
        const uint4 v = *reinterpret_cast<const uint4*>(stg + r * (D * 2) + ((ch ^ (r & (kCh - 1))) * 16));
        if (w)
          *reinterpret_cast<uint4*>(a.o + dst_row * a.o_stride + static_cast<int64_t>(head) * D + ch * 8) = v;
      }
    }
#else
    __nv_bfloat16* orow = a.o + out_row * a.o_stride + static_cast<int64_t>(head) * D;
#pragma unroll
    for (int cc = 0; cc < D / 32; ++cc) {
      uint32_t o[32];
      tmem_ld32(tO + cc * 32, o);
      tmem_wait_ld(o);
      if (write_o) {
        uint4 pk[4];
        uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          pw[i] = pack_bf16(__uint_as_float(o[2 * i]) * inv_l, __uint_as_float(o[2 * i + 1]) * inv_l);
        uint4* dst = reinterpret_cast<uint4*>(orow + cc * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = pk[i];
      }
    }
#endif
    if (in_cap) {
      const float ms = (m_used == -INFINITY) ? 0.f : m_used * c;
      a.lse[(static_cast<int64_t>(seq) * a.heads + head) * a.seq_len + q_row] =
          live ? (ms + __log2f(l)) * kLn2 : INFINITY;
    }
  }

  tc_fence_before();
  __syncthreads();
#if OSP_FWD_TIMING
  // per CTA, on the MMA issuer's lane: entry -> Q landed (prologue), the key loop, last PV issued
  // -> every warp done (epilogue)
  if (t_first != 0) {
    atomicAdd(&g_fwd_counters[24], static_cast<unsigned long long>(t_first - t_entry));
    atomicAdd(&g_fwd_counters[25], static_cast<unsigned long long>(t_fin - t_first));
    atomicAdd(&g_fwd_counters[26], static_cast<unsigned long long>(clock64() - t_fin));
    atomicAdd(&g_fwd_counters[27], 1ull);
  }
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
int launch_fwd_t(const void* q, const void* k, const void* v, void* o, float* lse,
                 const AttnShape& s, int64_t qs, int64_t ks, int64_t vs, int64_t os,
                 const uint32_t* bits, int zero_invalid_q, float scale, cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  const int64_t cols = s.heads * D;
  int st;
  if (s.row_index) {
    if (s.seq_len % 4) {
      set_error("gather mode needs the row-index capacity to be a multiple of 4");
      return kValue;
    }
    if ((st = make_tmap_bf16_2d(&mq, q, cols, s.n_rows, qs, 1)) != kOk) return st;
    if ((st = make_tmap_bf16_2d(&mk, k, cols, s.n_rows, ks, 1)) != kOk) return st;
    if ((st = make_tmap_bf16_2d(&mv, v, cols, s.n_rows, vs, 1)) != kOk) return st;
  } else {
    if ((st = make_tmap_bf16_3d(&mq, q, cols, s.seq_len, s.n_seq, qs, kBM)) != kOk) return st;
    if ((st = make_tmap_bf16_3d(&mk, k, cols, s.seq_len, s.n_seq, ks, kBN)) != kOk) return st;
    if ((st = make_tmap_bf16_3d(&mv, v, cols, s.seq_len, s.n_seq, vs, kBN)) != kOk) return st;
  }
  FwdArgs a;
  a.o = static_cast<__nv_bfloat16*>(o);
  a.o_stride = os;
  a.lse = lse;
  a.valid_bits = bits;
  a.words_per_seq = static_cast<int>((s.seq_len + 31) / 32);
  a.seq_len = static_cast<int>(s.seq_len);
  a.heads = static_cast<int>(s.heads);
  a.seq_lens = s.seq_lens;
  a.row_index = s.row_index;
  a.n_rows = static_cast<int>(s.n_rows);
  a.out_index = s.out_index;
  a.zero_rows = s.zero_rows;
  a.n_zero = static_cast<int>(s.n_zero);
  a.scale_log2 = scale * 1.4426950408889634f;
  a.zero_invalid_q = zero_invalid_q;
  static const int fwd_flags = env_int("OSP_FWD_FLAGS", 0);
  a.flags = fwd_flags;
  const int n_qt = static_cast<int>((s.seq_len + kBM - 1) / kBM);
  dim3 grid((n_qt + 1) / 2, static_cast<unsigned>(s.heads), static_cast<unsigned>(s.n_seq));
  static std::atomic<uint64_t> attr_done{0};
  st = set_smem_attr(reinterpret_cast<const void*>(attn_fwd_kernel<D>), FwdLayout<D>::kSmem, attr_done,
                     "cudaFuncSetAttribute(attn_fwd)");
  if (st != kOk) return st;
  attn_fwd_kernel<D><<<grid, kFwdThreads, FwdLayout<D>::kSmem, stream>>>(mq, mk, mv, a);
  return check_cuda(cudaGetLastError(), "attn_fwd_kernel launch");
}

}  // namespace

int debug_counters(unsigned long long* host, int n, int reset) {
  if (n > 64) n = 64;
  int rc = check_cuda(cudaMemcpyFromSymbol(host, g_fwd_counters, n * sizeof(unsigned long long)),
                      "cudaMemcpyFromSymbol");
  if (rc != kOk || !reset) return rc;
  static const unsigned long long zeros[64] = {};
  return check_cuda(cudaMemcpyToSymbol(g_fwd_counters, zeros, sizeof(zeros)), "cudaMemcpyToSymbol");
}

int launch_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                    const AttnShape& s, int64_t q_stride, int64_t k_stride, int64_t v_stride,
                    int64_t o_stride, const uint32_t* valid_bits, int zero_invalid_queries,
                    float scale, cudaStream_t stream) {
  if (s.head_dim == 128)
    return launch_fwd_t<128>(q, k, v, o, lse, s, q_stride, k_stride, v_stride, o_stride,
                             valid_bits, zero_invalid_queries, scale, stream);
  if (s.head_dim == 64)
    return launch_fwd_t<64>(q, k, v, o, lse, s, q_stride, k_stride, v_stride, o_stride,
                            valid_bits, zero_invalid_queries, scale, stream);
  set_error("attention kernels support head_dim 64 or 128");
  return kUnsupported;
}

}  // namespace osp
