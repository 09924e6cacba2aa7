// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM with W warps (W/4 per lane quadrant).
#include <cstdio>
#include <cstdlib>

#include "../paper_2605_28691_b200/csrc/osp_common.cuh"

using namespace osp;

template <bool ST, bool BATCH = false>
__global__ void __launch_bounds__(512, 1) tmem_kernel(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t col0 = (warp >> 2) * 128;  // warps in the same quadrant use different columns
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (!ST && BATCH) {  // four 32-column loads in flight, one wait (the K2 softmax pattern)
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tm + la + ((col0 + c * 32) & 511), r[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_wait_ld(r[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc += __uint_as_float(r[c][0]) + __uint_as_float(r[c][31]);
      continue;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      if (ST) {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(acc + i);
        tmem_st32(tm + la + ((col0 + c * 32) & 511), r);
      } else {
        tmem_ld32(tm + la + ((col0 + c * 32) & 511), r);
        tmem_wait_ld(r);
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
      }
    }
    if (ST) tmem_wait_st();
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  if (acc == 12345.f) *sink = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

template <bool ST, bool BATCH = false>
void run(int warps, int iters) {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 4);
  tmem_kernel<ST, BATCH><<<148, warps * 32>>>(10, d, s);
  cudaDeviceSynchronize();
  tmem_kernel<ST, BATCH><<<148, warps * 32>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = double(warps) * 32 * 4 * 32 * 4 * iters;  // per CTA
  printf("%s%s warps=%2d: %.1f bytes/clk/SM  (%s)\n", ST ? "tcgen05.st" : "tcgen05.ld", BATCH ? " (4 in flight)" : "", warps,
         bytes / double(cyc), cudaGetErrorString(e));
  fflush(stdout);
}

int main() {
  for (int w : {4, 8, 16}) run<false>(w, 2000);
  for (int w : {4, 8, 16}) run<false, true>(w, 2000);
  for (int w : {4, 8, 16}) run<true>(w, 2000);
  return 0;
}
