// Self-test kernel for the tcgen05 building blocks used by K2/K3: one CTA computes
// S = A B^T (SS MMA, both operands K-major SW128 via TMA) and O = bf16(S) V (TS MMA, P read
// from TMEM, V MN-major SW128), exporting S and O in fp32.  Exposed through
// osp_debug_mma() so GPU tests can localise a descriptor/layout bug to one instruction form.
#include "osp_common.cuh"
#include "osp_internal.h"

namespace osp {
namespace {

template <int D>
__global__ void __launch_bounds__(128, 1)
    debug_mma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmV, float* s_out, float* o_out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~static_cast<uintptr_t>(1023));
  constexpr int kTile = 128 * D * 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 3 * kTile);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(bars + i, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    mbar_expect_tx(bars + 0, 3 * kTile);
    for (int s = 0; s < D / 64; ++s) {
      tma_load_3d(sm + s * 16384, &tmA, bars + 0, s * 64, 0, 0);
      tma_load_3d(sm + kTile + s * 16384, &tmB, bars + 0, s * 64, 0, 0);
      tma_load_3d(sm + 2 * kTile + s * 16384, &tmV, bars + 0, s * 64, 0, 0);
    }
    mbar_wait(bars + 0, 0);
    tc_fence_after();
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + kTile);
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
      mma_ss(tmem, sdesc_sw128(a0 + off, 16, 1024), sdesc_sw128(b0 + off, 16, 1024),
             idesc_bf16(128, 128, 0, 0), kk > 0);
    }
    tc_commit(bars + 1);
  }
  __syncwarp();
  mbar_wait(bars + 1, 0);
  tc_fence_after();
  const uint32_t lane_addr = static_cast<uint32_t>(warp * 32) << 16;
  const int row = warp * 32 + lane;
  for (int cc = 0; cc < 4; ++cc) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_addr + cc * 32, r);
    tmem_wait_ld(r);
    for (int i = 0; i < 32; ++i) s_out[row * 128 + cc * 32 + i] = __uint_as_float(r[i]);
    uint32_t pk[16];
    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    tmem_st16(tmem + lane_addr + 128 + cc * 16, pk);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t v0 = smem_u32(sm + 2 * kTile);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)
      mma_ts(tmem + 256, tmem + 128 + kk * 8, sdesc_sw128(v0 + kk * 2048, 16384, 1024),
             idesc_bf16(128, D, 0, 1), kk > 0);
    tc_commit(bars + 2);
  }
  __syncwarp();
  mbar_wait(bars + 2, 0);
  tc_fence_after();
  for (int cc = 0; cc < D / 32; ++cc) {
    uint32_t r[32];
    tmem_ld32(tmem + lane_addr + 256 + cc * 32, r);
    tmem_wait_ld(r);
    for (int i = 0; i < 32; ++i) o_out[row * D + cc * 32 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D>
int run(const void* a, const void* b, const void* v, float* s_out, float* o_out,
        cudaStream_t stream) {
  CUtensorMap ma, mb, mv;
  int st;
  if ((st = make_tmap_bf16_3d(&ma, a, D, 128, 1, D, 128)) != kOk) return st;
  if ((st = make_tmap_bf16_3d(&mb, b, D, 128, 1, D, 128)) != kOk) return st;
  if ((st = make_tmap_bf16_3d(&mv, v, D, 128, 1, D, 128)) != kOk) return st;
  const int smem = 3 * 128 * D * 2 + 64 + 1024;
  int rc = check_cuda(cudaFuncSetAttribute(debug_mma_kernel<D>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                      "cudaFuncSetAttribute(debug_mma)");
  if (rc != kOk) return rc;
  debug_mma_kernel<D><<<1, 128, smem, stream>>>(ma, mb, mv, s_out, o_out);
  return check_cuda(cudaGetLastError(), "debug_mma_kernel launch");
}

}  // namespace

int launch_debug_mma(const void* a, const void* b, const void* v, float* s_out, float* o_out,
                     int d, cudaStream_t stream) {
  if (d == 128) return run<128>(a, b, v, s_out, o_out, stream);
  if (d == 64) return run<64>(a, b, v, s_out, o_out, stream);
  set_error("debug_mma supports d in {64, 128}");
  return kUnsupported;
}

}  // namespace osp
