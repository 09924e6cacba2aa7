// K6: QKV projection with the QK-RMSNorm + 3-D RoPE prologue of the attention (SURVEY.md sec. 8f
// row 2) on sm_100a -- one tcgen05 GEMM whose epilogue writes the attention-ready q | k | v in the
// pattern layout.
//
//   out[r, :] = x[r, :] @ W          x: (rows, C) bf16 in the pattern layout (rows = k^2*B*L)
//                                    W: given as W^T (3C, C) bf16, K-major
//   q, k columns ([0, 2C)), per 128-wide head:
//     norm 1 (per head):   v *= rsqrt(mean_head(v^2) + eps) * gamma[c]
//     norm 2 (per token over all C channels, Wan-style): the epilogue writes bf16 v and adds the
//                          row's sum of squares into `sumsq`; qk_norm_rope_kernel then scales and
//                          rotates in place
//     rope:                pairs (2i, 2i+1) of each head rotated by pos_axis(i) * freq(i); the
//                          64 pairs split over (t, h, w) as (d - 4*(d/6), 2*(d/6), 2*(d/6)) / 2;
//                          positions are the token's padded-grid coordinates, recovered in closed
//                          form from its pattern-layout row (skiparse.py:68-114 inverted).
// The reference's projection (attention.py:20-32) is this GEMM with norm 0 and rope off.
//
// Kernel: persistent, clusters of two CTAs on vertically adjacent 128 x 256 output tiles.  Default
// (OSP_PROJ_PAIR=1): a CTA pair running tcgen05.mma.cta_group::2 (M=256 across both CTAs' TMEM,
// N=256 with each CTA holding a 128-row half of the 256 x 64 weight slice), issued by the leader
// CTA; each CTA's TMA lands its operands in its own smem and completes on the leader's barrier;
// 6-stage ring of 32 KB per CTA.  Alternative (OSP_PROJ_PAIR=0): two independent M=128 CTAs with
// the weight slice TMA-multicast into both, 4 stages of 48 KB.  Either way, two 256-column TMEM
// accumulators let the epilogue of tile i overlap the main loop of tile i+1, and tiles are visited
// in bands of OSP_PROJ_BAND (default 12) column tiles swept over all row pairs (OSP_PROJ_ORDER=0:
// bands of row pairs swept over all column tiles).
#include "osp_common.cuh"
#include "osp_internal.h"

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <type_traits>

namespace osp {
namespace {

constexpr int kPBM = 128, kPBN = 256, kPBK = 64, kPStages = 4;
constexpr int kPThreads = 256;

// Epilogue rows staged in shared memory and stored as whole coalesced rows (1), or one row per
// thread straight from registers (0, rounds 1-2).
// L2 policy: the W band's TMA loads evict-last, output stores streaming (1), or default (0).
#ifndef OSP_PROJ_L2HINT
#define OSP_PROJ_L2HINT 1
#endif
// Staged epilogue rows leave through TMA stores (1) or coalesced st.global (0).
#ifndef OSP_PROJ_TMA_STORE
#define OSP_PROJ_TMA_STORE 1
#endif
#ifndef OSP_PROJ_STAGED_EPI
#define OSP_PROJ_STAGED_EPI 1
#endif
constexpr int kPStage = OSP_PROJ_STAGED_EPI ? 4 * 32 * 256 : 0;  // 4 epilogue warps x 32 rows x 256 B

struct ProjLayout {
  static constexpr int kA = 0;                                   // stages x 16 KB
  static constexpr int kB = kPStages * kPBM * kPBK * 2;          // stages x 32 KB
  static constexpr int kBar = kB + kPStages * kPBN * kPBK * 2;
  static constexpr int kStg = kBar + 1024;
  static constexpr int kSmem = kStg + kPStage;
};

// CTA-pair variant: per stage each CTA holds its 128 x rows and its 128-row half of the W slice
constexpr int kP2Stages = 6;
struct Proj2Layout {
  static constexpr int kA = 0;                                   // stages x 16 KB
  static constexpr int kB = kP2Stages * kPBM * kPBK * 2;         // stages x 16 KB (W half)
  static constexpr int kBar = kB + kP2Stages * (kPBN / 2) * kPBK * 2;
  static constexpr int kStg = kBar + 1024;
  static constexpr int kSmem = kStg + kPStage;
};
static_assert(Proj2Layout::kSmem <= 232448 && ProjLayout::kSmem <= 232448, "K6 shared memory");

struct ProjArgs {
  __nv_bfloat16* out;
  int64_t out_stride;
  int rows, chan, n_cols, n_pairs_m, n_tiles_n, k_steps;
  int band;                 // rasterisation: tile pairs per band (all column tiles per band)
  int* work_counter;        // pair kernel: units handed out in global order by an atomic counter
                            // (null: each cluster takes units cluster + k * n_clusters)
  int col_bands;            // 1: bands of `band` column tiles over all row pairs instead
  int norm;                 // 0 none, 1 per head, 2 per token (two-phase)
  const float* gamma_q;     // (C) or null
  const float* gamma_k;
  float eps;
  float* sumsq;             // (rows, 2) for norm 2
  const float2* rope;       // (T + H + W, 32) cos/sin, or null
  int pattern;              // 0 original, 1 TSA, 2 GSA
  int B, T, H, W, k, L;     // padded grid, batch, subsequence length
  int row_offset;           // global pattern-layout row of local row 0 (SSP shards)
  int d_t, d_h;             // pairs on the t and h axes (the rest on w)
};

// Padded-grid (t, h, w) of pattern-layout row `r` (inverse of skiparse.py:68-114).
__device__ __forceinline__ void row_coords(const ProjArgs& a, int r, int& t, int& h, int& w) {
  r += a.row_offset;
  if (a.pattern == 0) {
    const int pos = r % (a.T * a.H * a.W);
    w = pos % a.W;
    h = (pos / a.W) % a.H;
    t = pos / (a.W * a.H);
    return;
  }
  const int s = r / a.L, pos = r % a.L;
  const int pq = s / a.B;
  const int p = pq / a.k, q = pq % a.k;
  if (a.pattern == 1) {
    const int hk = a.H / a.k, wk = a.W / a.k;
    const int ww = pos % wk, hh = (pos / wk) % hk;
    t = pos / (wk * hk);
    h = hh * a.k + p;
    w = ww * a.k + q;
  } else {
    const int k2 = a.k * a.k;
    const int hk2 = a.H / k2, wk2 = a.W / k2;
    const int q2 = pos % a.k;
    const int x = pos / a.k;
    const int wg = x % wk2;
    const int y = x / wk2;
    const int p2 = y % a.k;
    const int txh = y / a.k;
    const int hg = txh % hk2;
    t = txh / hk2;
    h = hg * k2 + p * a.k + p2;
    w = wg * k2 + q * a.k + q2;
  }
}

// Normalise (norm 1) and rotate one 128-channel head held by this thread.
__device__ __forceinline__ void head_epilogue(float (&v)[128], const ProjArgs& a, const float* gamma,
                                              int c0, int t, int h, int w, bool rope) {
  if (a.norm == 1) {
    float ss0 = 0.f, ss1 = 0.f;
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      ss0 = fmaf(v[i], v[i], ss0);
      ss1 = fmaf(v[i + 1], v[i + 1], ss1);
    }
    const float r = rsqrtf((ss0 + ss1) * (1.f / 128.f) + a.eps);
#pragma unroll
    for (int i = 0; i < 128; ++i) v[i] *= r * (gamma ? __ldg(gamma + (c0 + i)) : 1.f);
  }
  if (rope) {
    const float2* rt = a.rope + static_cast<int64_t>(t) * 32;
    const float2* rh = a.rope + static_cast<int64_t>(a.T + h) * 32;
    const float2* rw = a.rope + static_cast<int64_t>(a.T + a.H + w) * 32;
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const float2 cs = i < a.d_t ? __ldg(rt + i) : (i < a.d_t + a.d_h ? __ldg(rh + (i - a.d_t))
                                                                         : __ldg(rw + (i - a.d_t - a.d_h)));
      const float x0 = v[2 * i], x1 = v[2 * i + 1];
      v[2 * i] = x0 * cs.x - x1 * cs.y;
      v[2 * i + 1] = x0 * cs.y + x1 * cs.x;
    }
  }
}

// kPair = false: each CTA of the cluster runs M=128 MMAs on its own tile, the W slice being
// TMA-multicast into both.  kPair = true: the cluster is a CTA pair running cta_group::2 MMAs
// (M=256 over both CTAs' TMEM, N=256 with each CTA holding a 128-row half of the W slice), issued
// by the leader CTA; each CTA's TMA lands its operands in its own smem and signals the leader.
// kQuad (with kPair): clusters of two such pairs on vertically adjacent row pairs and the same
// column tile; each CTA loads a quarter of the W slice and multicasts it to its counterpart in the
// other pair, so the W slice crosses L2 -> SM once per 512 rows (as cuBLAS's 2x1 clusters do).
template <bool kPair, bool kQuad = false>
__global__ void __launch_bounds__(kPThreads, 1)
    qkv_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmO, const ProjArgs a) {
  using Ly = std::conditional_t<kPair, Proj2Layout, ProjLayout>;
  constexpr int kStages = kPair ? kP2Stages : kPStages;
  constexpr int kBRows = kPair ? kPBN / 2 : kPBN;   // W rows per CTA per stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::kBar);
  uint64_t* bar_full = bars;                  // [stages] TMA -> MMA (pair: the leader's counts)
  uint64_t* bar_empty = bars + kStages;       // [stages] MMA -> TMA
  uint64_t* bar_acc = bars + 2 * kStages;     // [2] MMA -> epilogue
  uint64_t* bar_accf = bars + 2 * kStages + 2;  // [2] epilogue -> MMA (128, pair: 256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  // dynamic schedule (pair kernel): a 4-slot ring of unit ids per CTA, filled by the leader's
  // producer (atomic counter) for both CTAs; bar_uf: id written (1 arrival), bar_ue (leader only):
  // slot consumed by the leader's MMA issuer and 4 epilogue warps and the peer's producer and 4
  // epilogue warps (10 arrivals)
  uint64_t* bar_uf = bars + 2 * kStages + 5;
  uint64_t* bar_ue = bars + 2 * kStages + 9;
  int* unit_ring = reinterpret_cast<int*>(bars + 2 * kStages + 13);
  const bool dyn = kPair && a.work_counter != nullptr;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  constexpr int kCtas = kQuad ? 4 : 2;             // CTAs per cluster
  const uint32_t lead = crank & ~1u;               // this CTA's pair leader (MMA issuer)
  const int cluster = blockIdx.x / kCtas, n_clusters = gridDim.x / kCtas;
  // a unit = kCtas vertically adjacent 128-row tiles x one 256-column tile
  const int n_row_units = kQuad ? (a.n_pairs_m + 1) / 2 : a.n_pairs_m;
  const int n_units = n_row_units * a.n_tiles_n;
  auto tile_mn = [&](int id, int& tm, int& tn) {
    if (a.col_bands) {  // bands of a.band column tiles swept over all row pairs (W band L2-resident)
      const int band_units = a.band * n_row_units;
      const int band = id / band_units;
      const int rem = id % band_units;
      const int cols_in_band = min(a.band, a.n_tiles_n - band * a.band);
      tn = band * a.band + rem % cols_in_band;
      tm = kCtas * (rem / cols_in_band) + static_cast<int>(crank);
      return;
    }
    const int band_units = a.band * a.n_tiles_n;
    const int band = id / band_units;
    const int rem = id % band_units;
    const int pairs_in_band = min(a.band, n_row_units - band * a.band);
    tm = kCtas * (band * a.band + rem % pairs_in_band) + static_cast<int>(crank);
    tn = rem / pairs_in_band;
  };

  // Unit enumeration shared by the three roles.  Static: id = cluster + k * n_clusters.  Dynamic
  // (pair): units in global order from an atomic counter, so the clusters work on neighbouring
  // units at any moment however their speeds drift (the W band and the x rows in flight stay
  // L2-resident, as with a non-persistent launch).  role 0: the leader's producer (draws the id
  // and publishes it to both CTAs), 1: the leader's MMA issuer, 2: an epilogue warp (whole warp),
  // 3: the peer's producer.  f(id) is called per unit; returns when the units are exhausted.
  auto for_each_unit = [&](int role, auto&& f) {
    if (!dyn) {
      for (int id = cluster; id < n_units; id += n_clusters) f(id);
      return;
    }
    for (int q = 0;; ++q) {
      const int slot = q & 3;
      const uint32_t ph = (q >> 2) & 1;
      int id;
      if (role == 0) {
        mbar_wait(bar_ue + slot, ph ^ 1);
        id = atomicAdd(a.work_counter, 1);
        if (id >= n_units) id = -1;
        unit_ring[slot] = id;
        for (uint32_t r = 1; r < kCtas; ++r)
          st_cluster_u32(mapa_u32(smem_u32(unit_ring + slot), r), static_cast<uint32_t>(id));
        mbar_arrive(bar_uf + slot);
        for (uint32_t r = 1; r < kCtas; ++r) mbar_arrive_cluster(mapa_u32(smem_u32(bar_uf + slot), r));
      } else {
        mbar_wait(bar_uf + slot, ph);
        fence_acq_rel_cluster();
        id = *reinterpret_cast<volatile int*>(unit_ring + slot);
        if (role == 2) __syncwarp();
        if (role != 2 || lane == 0) {
          if (crank == 0) mbar_arrive(bar_ue + slot);
          else mbar_arrive_cluster(mapa_u32(smem_u32(bar_ue + slot), 0));
        }
      }
      if (id < 0) return;
      f(id);
    }
  };

  if ((smem_u32(sm) & 1023) != 0) __trap();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar_full + i, 1);
      // multicast: both CTAs' MMAs read the W half; quad: both pairs' MMAs read my W quarter
      mbar_init(bar_empty + i, kPair ? (kQuad ? 2 : 1) : 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar_acc + i, 1);
      mbar_init(bar_accf + i, kPair ? 256 : 128);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(bar_uf + i, 1);
      // consumers: the pair leaders' MMA issuers, 4 epilogue warps per CTA, the other producers
      mbar_init(bar_ue + i, kCtas / 2 + 4 * kCtas + (kCtas - 1));
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (kPair) {
      tmem_alloc_pair(tmem_slot, 512);
    } else {
      tmem_alloc(tmem_slot, 512);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      const uint64_t pol_w = l2_policy_evict_last();
      (void)pol_w;
      int it = 0;
      for_each_unit(crank == 0 ? 0 : 3, [&](int id) {
        int tm, tn;
        tile_mn(id, tm, tn);
        for (int ks = 0; ks < a.k_steps; ++ks, ++it) {
          const int st = it % kStages;
          mbar_wait(bar_empty + st, ((it / kStages) & 1) ^ 1);
          if constexpr (kQuad) {
            // my pair leader counts both CTAs' A tiles and W halves; my W half arrives as two
            // quarters, mine and the one my counterpart in the other pair multicasts
            const uint32_t leader_full = mapa_u32(smem_u32(bar_full + st), lead);
            if ((crank & 1) == 0) mbar_expect_tx(bar_full + st, 2 * (kPBM + kBRows) * kPBK * 2);
            tma_load_3d_pair(sm + Ly::kA + st * kPBM * kPBK * 2, &tmA, leader_full, ks * kPBK, tm * kPBM, 0);
            const uint32_t half = crank & 1, pair = crank >> 1;
            tma_load_3d_pair_multicast(sm + Ly::kB + st * kBRows * kPBK * 2 + pair * (kBRows / 2) * kPBK * 2, &tmB,
                                       leader_full, ks * kPBK,
                                       tn * kPBN + static_cast<int>(half) * kBRows + static_cast<int>(pair) * (kBRows / 2),
                                       0, static_cast<uint16_t>((1u << half) | (1u << (2 + half))), pol_w);
          } else if constexpr (kPair) {
            // both CTAs' A and W halves complete on the leader's full barrier
            const uint32_t leader_full = mapa_u32(smem_u32(bar_full + st), 0);
            if (crank == 0) mbar_expect_tx(bar_full + st, 2 * (kPBM + kBRows) * kPBK * 2);
            if (OSP_PROJ_L2HINT) {
              // the band's W slice is reused by every row pair of the band: keep it in L2
              tma_load_3d_pair(sm + Ly::kA + st * kPBM * kPBK * 2, &tmA, leader_full, ks * kPBK, tm * kPBM, 0);
              tma_load_3d_pair_hint(sm + Ly::kB + st * kBRows * kPBK * 2, &tmB, leader_full, ks * kPBK,
                                    tn * kPBN + static_cast<int>(crank) * kBRows, 0, pol_w);
            } else {
              tma_load_3d_pair(sm + Ly::kA + st * kPBM * kPBK * 2, &tmA, leader_full, ks * kPBK, tm * kPBM, 0);
              tma_load_3d_pair(sm + Ly::kB + st * kBRows * kPBK * 2, &tmB, leader_full, ks * kPBK,
                               tn * kPBN + static_cast<int>(crank) * kBRows, 0);
            }
          } else {
            mbar_expect_tx(bar_full + st, (kPBM + kPBN) * kPBK * 2);
            tma_load_3d(sm + Ly::kA + st * kPBM * kPBK * 2, &tmA, bar_full + st, ks * kPBK, tm * kPBM, 0);
            // my half of the shared W slice, delivered to both CTAs
            tma_load_3d_multicast(sm + Ly::kB + st * kPBN * kPBK * 2 + crank * (kPBN / 2) * kPBK * 2, &tmB,
                                  bar_full + st, ks * kPBK, tn * kPBN + static_cast<int>(crank) * (kPBN / 2), 0,
                                  0x3);
          }
        }
      });
    }
    __syncwarp();
  } else if (warp == 1 && (!kPair || (crank & 1) == 0)) {
    constexpr uint32_t kId = idesc_bf16(kPair ? 2 * kPBM : kPBM, kPBN, 0, 0);
    if (elect_one()) {
      int it = 0, lt = 0;
      for_each_unit(1, [&](int) {
        const int buf = lt & 1;
        if (lt >= 2) mbar_wait(bar_accf + buf, ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * kPBN;
        for (int ks = 0; ks < a.k_steps; ++ks, ++it) {
          const int st = it % kStages;
          mbar_wait(bar_full + st, (it / kStages) & 1);
          tc_fence_after();
          const uint32_t ab = smem_u32(sm + Ly::kA + st * kPBM * kPBK * 2);
          const uint32_t bb = smem_u32(sm + Ly::kB + st * kBRows * kPBK * 2);
#pragma unroll
          for (int kk = 0; kk < kPBK / 16; ++kk) {
            if constexpr (kPair)
              mma_ss_pair(acc, sdesc_sw128(ab + kk * 32, 16, 1024), sdesc_sw128(bb + kk * 32, 16, 1024), kId,
                          (ks > 0 || kk > 0) ? 1u : 0u);
            else
              mma_ss(acc, sdesc_sw128(ab + kk * 32, 16, 1024), sdesc_sw128(bb + kk * 32, 16, 1024), kId,
                     (ks > 0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (kQuad)
            tc_commit_pair(bar_empty + st, 0xF);  // every CTA's W quarter fed both pairs
          else if constexpr (kPair)
            tc_commit_pair(bar_empty + st, 0x3);
          else
            tc_commit_multicast(bar_empty + st, 0x3);
        }
        if constexpr (kPair)
          tc_commit_pair(bar_acc + buf, static_cast<uint16_t>(0x3u << lead));
        else
          tc_commit(bar_acc + buf);
        ++lt;
      });
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue (thread = row)
    const int wq = warp & 3;
    const uint32_t la = static_cast<uint32_t>(wq * 32) << 16;
    int lt = 0;
    for_each_unit(2, [&](int id) {
      int tm, tn;
      tile_mn(id, tm, tn);
      const int buf = lt & 1;
      mbar_wait(bar_acc + buf, (lt >> 1) & 1);
      tc_fence_after();
      const int row = tm * kPBM + wq * 32 + lane;
      const bool row_ok = row < a.rows;
      int t = 0, h = 0, w = 0;
      if (a.rope) row_coords(a, row_ok ? row : 0, t, h, w);
      for (int hc = 0; hc < kPBN / 128; ++hc) {
        float v[128];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          uint32_t r[32];
          tmem_ld32(tmem + la + buf * kPBN + hc * 128 + cc * 32, r);
          tmem_wait_ld(r);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[cc * 32 + i] = __uint_as_float(r[i]);
        }
        if (hc == kPBN / 128 - 1) {
          tc_fence_before();
          if (kPair && (crank & 1) != 0)
            mbar_arrive_cluster(mapa_u32(smem_u32(bar_accf + buf), lead));
          else
            mbar_arrive(bar_accf + buf);
        }
        const int c0 = tn * kPBN + hc * 128;          // first output column of this head
        if (c0 >= a.n_cols) continue;                 // partial last column tile (3C % 256 == 128)
        const bool is_q = c0 < a.chan, is_k = !is_q && c0 < 2 * a.chan;
        if (is_q || is_k) {
          if (a.norm == 2 && row_ok) {
            float ss = 0.f;
#pragma unroll
            for (int i = 0; i < 128; ++i) {
              const float b = __bfloat162float(__float2bfloat16(v[i]));
              ss = fmaf(b, b, ss);
            }
            atomicAdd(a.sumsq + static_cast<int64_t>(row) * 2 + (is_q ? 0 : 1), ss);
          } else {
            head_epilogue(v, a, is_q ? a.gamma_q : a.gamma_k, is_q ? c0 : c0 - a.chan, t, h, w,
                          a.rope != nullptr);
          }
        }
#if OSP_PROJ_STAGED_EPI && OSP_PROJ_TMA_STORE
        {
          // the warp's 32 rows x 128 columns go to its 8 KB stage as two 128B-swizzled boxes of
          // 32 rows x 64 columns, which one lane then hands to two TMA stores (rows past the
          // matrix are clipped by the tensor map); the stage is rewritten only after the
          // previous stores have read it
          uint8_t* stg = sm + Ly::kStg + wq * 8192;
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            *reinterpret_cast<uint4*>(stg + (j >> 3) * 4096 + lane * 128 + (((j & 7) ^ (lane & 7)) * 16)) =
                make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                           pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int row0 = tm * kPBM + wq * 32;
            tma_store_3d(&tmO, stg, c0, row0, 0);
            tma_store_3d(&tmO, stg + 4096, c0 + 64, row0, 0);
            tma_store_commit();
          }
        }
#elif OSP_PROJ_STAGED_EPI
        {
          // the warp's 32 rows x 128 columns go through its 8 KB stage (16-byte chunks
          // XOR-swizzled by row: both passes bank-conflict free), then out two whole 256-byte
          // rows per store instruction
          uint8_t* stg = sm + Ly::kStg + wq * 8192;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            *reinterpret_cast<uint4*>(stg + lane * 256 + ((j ^ (lane & 15)) * 16)) =
                make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                           pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
          __syncwarp();
          const int ch = lane & 15;
          const int row0 = tm * kPBM + wq * 32;
#pragma unroll 4
          for (int rr = 0; rr < 16; ++rr) {
            const int r = 2 * rr + (lane >> 4);
            if (row0 + r < a.rows) {
              uint4* dst = reinterpret_cast<uint4*>(a.out + static_cast<int64_t>(row0 + r) * a.out_stride + c0 + ch * 8);
              const uint4 v4 = *reinterpret_cast<const uint4*>(stg + r * 256 + ((ch ^ (r & 15)) * 16));
              if (OSP_PROJ_L2HINT) __stcs(dst, v4);   // streamed out: do not displace the W band
              else *dst = v4;
            }
          }
          __syncwarp();
        }
#else
        if (row_ok) {
          uint4* dst = reinterpret_cast<uint4*>(a.out + static_cast<int64_t>(row) * a.out_stride + c0);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            dst[j] = make_uint4(pack_bf16(v[8 * j], v[8 * j + 1]), pack_bf16(v[8 * j + 2], v[8 * j + 3]),
                                pack_bf16(v[8 * j + 4], v[8 * j + 5]), pack_bf16(v[8 * j + 6], v[8 * j + 7]));
        }
#endif
      }
      ++lt;
    });
    if (OSP_PROJ_STAGED_EPI && OSP_PROJ_TMA_STORE && lane == 0) tma_store_wait_all();
  }
  tc_fence_before();
  cluster_sync();  // the peer may still multicast into / arrive on this CTA until it is done
  if (warp == 2) {
    tc_fence_after();
    if constexpr (kPair)
      tmem_dealloc_pair(tmem, 512);
    else
      tmem_dealloc(tmem, 512);
  }
}

// Second phase of norm 2: q, k rows scaled by rsqrt(mean over C + eps) * gamma, then RoPE.
// One warp per (row, q|k), each lane owns 4 heads' worth of channel pairs in turn.
__global__ void __launch_bounds__(256) qk_norm_rope_kernel(ProjArgs a) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= static_cast<int64_t>(a.rows) * 2) return;
  const int row = static_cast<int>(gw >> 1);
  const int which = static_cast<int>(gw & 1);
  const float r = rsqrtf(a.sumsq[static_cast<int64_t>(row) * 2 + which] / a.chan + a.eps);
  const float* gamma = which == 0 ? a.gamma_q : a.gamma_k;
  int t = 0, h = 0, w = 0;
  if (a.rope) row_coords(a, row, t, h, w);
  __nv_bfloat162* base = reinterpret_cast<__nv_bfloat162*>(a.out + static_cast<int64_t>(row) * a.out_stride +
                                                           static_cast<int64_t>(which) * a.chan);
  for (int pidx = lane; pidx < a.chan / 2; pidx += 32) {
    const int c = 2 * pidx;
    const float2 x = __bfloat1622float2(base[pidx]);
    float x0 = x.x * r * (gamma ? __ldg(gamma + c) : 1.f);
    float x1 = x.y * r * (gamma ? __ldg(gamma + c + 1) : 1.f);
    if (a.rope) {
      const int i = pidx & 63;  // pair within the head
      const float2 cs = i < a.d_t ? a.rope[static_cast<int64_t>(t) * 32 + i]
                                  : (i < a.d_t + a.d_h ? a.rope[static_cast<int64_t>(a.T + h) * 32 + (i - a.d_t)]
                                                       : a.rope[static_cast<int64_t>(a.T + a.H + w) * 32 +
                                                                (i - a.d_t - a.d_h)]);
      const float y0 = x0 * cs.x - x1 * cs.y;
      const float y1 = x0 * cs.y + x1 * cs.x;
      x0 = y0;
      x1 = y1;
    }
    base[pidx] = __floats2bfloat162_rn(x0, x1);
  }
}


// Backward of the q/k epilogue: g, the gradient of the normalised and
// rotated q | k, becomes the gradient of the pre-norm GEMM output, IN PLACE.  One warp per
// (row, q|k): transpose of the RoPE pair rotation, dg = gamma * g (with a norm), then the RMSNorm
// backward dy = r*dg - y*r^3*mean(dg*y) over the head (norm 1) or the whole row (norm 2), with
// y the pre-norm output and r = rsqrt(mean(y^2) + eps).  fp32 math, bf16 in and out.
__global__ void __launch_bounds__(256) qk_norm_rope_bwd_kernel(ProjArgs a, __nv_bfloat16* g, int64_t g_stride,
                                                               const __nv_bfloat16* y, int64_t y_stride) {
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= static_cast<int64_t>(a.rows) * 2) return;
  const int row = static_cast<int>(gw >> 1);
  const int which = static_cast<int>(gw & 1);
  const float* gamma = which == 0 ? a.gamma_q : a.gamma_k;
  int t = 0, h = 0, w = 0;
  if (a.rope) row_coords(a, row, t, h, w);
  __nv_bfloat162* gp = reinterpret_cast<__nv_bfloat162*>(g + static_cast<int64_t>(row) * g_stride +
                                                         static_cast<int64_t>(which) * a.chan);
  const __nv_bfloat162* yp = y ? reinterpret_cast<const __nv_bfloat162*>(
                                     y + static_cast<int64_t>(row) * y_stride + static_cast<int64_t>(which) * a.chan)
                               : nullptr;
  // unrotated (and gamma-scaled) gradient of pair pidx
  auto dg_pair = [&](int pidx) {
    float2 d = __bfloat1622float2(gp[pidx]);
    if (a.rope) {
      const int i = pidx & 63;
      const float2 cs = i < a.d_t ? a.rope[static_cast<int64_t>(t) * 32 + i]
                                  : (i < a.d_t + a.d_h ? a.rope[static_cast<int64_t>(a.T + h) * 32 + (i - a.d_t)]
                                                       : a.rope[static_cast<int64_t>(a.T + a.H + w) * 32 +
                                                                (i - a.d_t - a.d_h)]);
      d = make_float2(d.x * cs.x + d.y * cs.y, -d.x * cs.y + d.y * cs.x);
    }
    if (a.norm && gamma) {
      const int c = 2 * pidx;
      d.x *= __ldg(gamma + c);
      d.y *= __ldg(gamma + c + 1);
    }
    return d;
  };
  auto warp_sum = [](float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
  };
  const int n_pairs = a.chan / 2;
  if (a.norm == 0) {
    for (int pidx = lane; pidx < n_pairs; pidx += 32) {
      const float2 d = dg_pair(pidx);
      gp[pidx] = __floats2bfloat162_rn(d.x, d.y);
    }
    return;
  }
  // norm 1: groups of 64 pairs (one head), lanes take pairs lane and lane + 32 of the group;
  // norm 2: one group spanning the row
  const int group_pairs = a.norm == 1 ? 64 : n_pairs;
  for (int p0 = 0; p0 < n_pairs; p0 += group_pairs) {
    float ss = 0.f, sd = 0.f;
    for (int pidx = p0 + lane; pidx < p0 + group_pairs; pidx += 32) {
      const float2 d = dg_pair(pidx);
      const float2 v = __bfloat1622float2(yp[pidx]);
      ss = fmaf(v.x, v.x, fmaf(v.y, v.y, ss));
      sd = fmaf(d.x, v.x, fmaf(d.y, v.y, sd));
    }
    ss = warp_sum(ss);
    sd = warp_sum(sd);
    const float n = 2.f * group_pairs;
    const float r = rsqrtf(ss / n + a.eps);
    const float coef = r * r * r * (sd / n);
    for (int pidx = p0 + lane; pidx < p0 + group_pairs; pidx += 32) {
      const float2 d = dg_pair(pidx);
      const float2 v = __bfloat1622float2(yp[pidx]);
      gp[pidx] = __floats2bfloat162_rn(r * d.x - v.x * coef, r * d.y - v.y * coef);
    }
  }
}

}  // namespace

int launch_qkv_project(const void* x, const void* w_t, void* out, int64_t rows, int64_t chan,
                       int64_t out_stride, int norm, const float* gamma_q, const float* gamma_k,
                       float eps, float* sumsq, const float* rope_table, int64_t t, int64_t h,
                       int64_t w, int64_t k, int pattern, int64_t batch, int64_t row_offset,
                       cudaStream_t stream) {
  if (chan % 128 != 0 || chan < 128) {
    set_error("qkv projection: chan must be a positive multiple of 128 (head_dim 128)");
    return kUnsupported;
  }
  if (norm < 0 || norm > 2 || (norm == 2 && !sumsq)) {
    set_error("qkv projection: norm must be 0, 1 or 2 (2 needs a sumsq workspace)");
    return kValue;
  }
  const int64_t n = 3 * chan;
  if (out_stride < n || (out_stride * 2) % 16) {
    set_error("qkv projection: out row stride must be >= 3*chan and 16-byte aligned");
    return kValue;
  }
  if (rows == 0) return kOk;
  ProjArgs a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.out_stride = out_stride;
  a.rows = static_cast<int>(rows);
  a.chan = static_cast<int>(chan);
  a.n_cols = static_cast<int>(n);
  a.n_pairs_m = static_cast<int>((rows + 2 * kPBM - 1) / (2 * kPBM));
  a.n_tiles_n = static_cast<int>((n + kPBN - 1) / kPBN);
  a.k_steps = static_cast<int>(chan / kPBK);
  a.norm = norm;
  a.gamma_q = gamma_q;
  a.gamma_k = gamma_k;
  a.eps = eps;
  a.sumsq = sumsq;
  a.rope = reinterpret_cast<const float2*>(rope_table);
  a.pattern = pattern;
  a.B = static_cast<int>(batch);
  a.T = static_cast<int>(t);
  a.H = static_cast<int>(h);
  a.W = static_cast<int>(w);
  a.k = static_cast<int>(k);
  a.row_offset = static_cast<int>(row_offset);
  const int64_t k2 = k * k;
  a.L = pattern == 0 ? static_cast<int>(t * h * w) : static_cast<int>(t * h * w / k2);
  a.d_t = (128 - 4 * (128 / 6)) / 2;
  a.d_h = (2 * (128 / 6)) / 2;
  if (rope_table) {
    if (pattern < 0 || pattern > 2 || k < 1 || (pattern == 1 && (h % k || w % k)) ||
        (pattern == 2 && (h % k2 || w % k2)) || row_offset < 0 ||
        (rows + row_offset) > (pattern == 0 ? batch * t * h * w : batch * t * h * w)) {
      set_error("qkv projection: rope needs a pattern layout consistent with the grid");
      return kPattern;
    }
  }
  int rc;
  CUtensorMap ma, mb;
  if ((rc = make_tmap_bf16_3d(&ma, x, chan, rows, 1, chan, kPBM)) != kOk) return rc;
  // W half per CTA; quad clusters load it as two multicast quarters
  static const bool quad_map = env_int("OSP_PROJ_QUAD", 0) != 0 && env_int("OSP_PROJ_PAIR", 1) != 0 &&
                               env_int("OSP_PROJ_DYN", 1) != 0;
  if ((rc = make_tmap_bf16_3d(&mb, w_t, chan, n, 1, chan, quad_map ? kPBN / 4 : kPBN / 2)) != kOk) return rc;
  CUtensorMap mo;
  if ((rc = make_tmap_bf16_3d(&mo, out, n, rows, 1, out_stride, 32)) != kOk) return rc;  // epilogue boxes
  static std::atomic<uint64_t> attr_done_1{0}, attr_done_2{0}, attr_done_4{0};
  rc = set_smem_attr(reinterpret_cast<const void*>(qkv_gemm_kernel<false>), ProjLayout::kSmem, attr_done_1,
                     "cudaFuncSetAttribute(qkv_gemm)");
  if (rc != kOk) return rc;
  rc = set_smem_attr(reinterpret_cast<const void*>(qkv_gemm_kernel<true>), Proj2Layout::kSmem, attr_done_2,
                     "cudaFuncSetAttribute(qkv_gemm pair)");
  if (rc != kOk) return rc;
  rc = set_smem_attr(reinterpret_cast<const void*>(qkv_gemm_kernel<true, true>), Proj2Layout::kSmem, attr_done_4,
                     "cudaFuncSetAttribute(qkv_gemm quad)");
  if (rc != kOk) return rc;
  // bands of 12 (measured best at cfg3, tools/bench_proj.py); column bands (the band's W slice
  // stays L2-resident while x streams): at cfg3 8.9 GB of DRAM reads per launch instead of 13.5
  // with row bands, 2-3% faster (profiles/r02_proj_order.txt)
  static const int band = env_int("OSP_PROJ_BAND", 12);
  static const int col_bands = env_int("OSP_PROJ_ORDER", 1);
  static const bool pair = env_int("OSP_PROJ_PAIR", 1) != 0;
  // two pairs per cluster sharing the W slice (needs the dynamic schedule)
  static const bool quad_env = env_int("OSP_PROJ_QUAD", 0) != 0;
  a.band = band < 1 ? 12 : band;
  a.col_bands = col_bands;
  if (norm == 2) {
    rc = check_cuda(cudaMemsetAsync(sumsq, 0, rows * 2 * sizeof(float), stream), "memset sumsq");
    if (rc != kOk) return rc;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool quad = pair && quad_env && env_int("OSP_PROJ_DYN", 1) != 0;
  const int ctas = quad ? 4 : 2;
  const int n_units = (quad ? (a.n_pairs_m + 1) / 2 : a.n_pairs_m) * a.n_tiles_n;
  // dynamic unit schedule (pair kernel): a work counter zeroed on the stream before the launch;
  // launches rotate through 64 counters per device, so concurrent launches on other streams do
  // not share one
  static const bool dynamic = env_int("OSP_PROJ_DYN", 1) != 0;
  a.work_counter = nullptr;
  if (pair && dynamic) {
    static std::mutex mu;
    static int* counters[64] = {};
    static std::atomic<unsigned> seq{0};
    if (dev < 0 || dev >= 64) {
      set_error("qkv projection: device index out of range");
      return kValue;
    }
    {
      std::lock_guard<std::mutex> lock(mu);
      if (!counters[dev]) {
        void* p = nullptr;
        if ((rc = check_cuda(cudaMalloc(&p, 64 * sizeof(int)), "cudaMalloc(work counters)")) != kOk) return rc;
        counters[dev] = static_cast<int*>(p);
      }
    }
    a.work_counter = counters[dev] + (seq.fetch_add(1) % 64);
    if ((rc = check_cuda(cudaMemsetAsync(a.work_counter, 0, sizeof(int), stream), "memset work counter")) != kOk)
      return rc;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas * min(n_units, sms / ctas));
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = pair ? Proj2Layout::kSmem : ProjLayout::kSmem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  rc = check_cuda(quad   ? cudaLaunchKernelEx(&cfg, qkv_gemm_kernel<true, true>, ma, mb, mo, a)
                  : pair ? cudaLaunchKernelEx(&cfg, qkv_gemm_kernel<true>, ma, mb, mo, a)
                         : cudaLaunchKernelEx(&cfg, qkv_gemm_kernel<false>, ma, mb, mo, a),
                  "qkv_gemm launch");
  if (rc != kOk || norm != 2) return rc;
  const int64_t warps = rows * 2;
  qk_norm_rope_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, stream>>>(a);
  return check_cuda(cudaGetLastError(), "qk_norm_rope launch");
}

int launch_qk_norm_rope_bwd(void* g, int64_t g_stride, const void* y, int64_t y_stride, int64_t rows,
                            int64_t chan, int norm, const float* gamma_q, const float* gamma_k, float eps,
                            const float* rope_table, int64_t t, int64_t h, int64_t w, int64_t k, int pattern,
                            int64_t batch, int64_t row_offset, cudaStream_t stream) {
  if (chan % 128 != 0 || chan < 128) {
    set_error("qk norm/rope backward: chan must be a positive multiple of 128 (head_dim 128)");
    return kUnsupported;
  }
  if (norm < 0 || norm > 2 || (norm != 0 && !y)) {
    set_error("qk norm/rope backward: norm must be 0, 1 or 2 (1 and 2 need the pre-norm output y)");
    return kValue;
  }
  if (g_stride < 2 * chan || (norm && y_stride < 2 * chan) || (g_stride * 2) % 4 || (y_stride * 2) % 4) {
    set_error("qk norm/rope backward: row strides must cover q|k and keep bf16 pairs aligned");
    return kValue;
  }
  if (rows == 0) return kOk;
  ProjArgs a{};
  a.rows = static_cast<int>(rows);
  a.chan = static_cast<int>(chan);
  a.norm = norm;
  a.gamma_q = gamma_q;
  a.gamma_k = gamma_k;
  a.eps = eps;
  a.rope = reinterpret_cast<const float2*>(rope_table);
  a.pattern = pattern;
  a.B = static_cast<int>(batch);
  a.T = static_cast<int>(t);
  a.H = static_cast<int>(h);
  a.W = static_cast<int>(w);
  a.k = static_cast<int>(k);
  a.row_offset = static_cast<int>(row_offset);
  const int64_t k2 = k * k;
  a.L = pattern == 0 ? static_cast<int>(t * h * w) : static_cast<int>(t * h * w / k2);
  a.d_t = (128 - 4 * (128 / 6)) / 2;
  a.d_h = (2 * (128 / 6)) / 2;
  if (rope_table && (pattern < 0 || pattern > 2 || k < 1 || (pattern == 1 && (h % k || w % k)) ||
                     (pattern == 2 && (h % k2 || w % k2)) || row_offset < 0 ||
                     rows + row_offset > batch * t * h * w)) {
    set_error("qk norm/rope backward: rope needs a pattern layout consistent with the grid");
    return kPattern;
  }
  const int64_t warps = rows * 2;
  qk_norm_rope_bwd_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, stream>>>(
      a, static_cast<__nv_bfloat16*>(g), g_stride, static_cast<const __nv_bfloat16*>(y), y_stride);
  return check_cuda(cudaGetLastError(), "qk_norm_rope_bwd launch");
}

}  // namespace osp
