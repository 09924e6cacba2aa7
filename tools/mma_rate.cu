// Microbenchmark: sustained tcgen05.mma (kind::f16, cta_group::1) throughput per shape, operands
// resident in shared memory (SS) or A in TMEM (TS).  One CTA per SM, one thread issuing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2605_28691_b200/csrc mma_rate.cu
#include <cstdio>
#include <cstdlib>

#include "../paper_2605_28691_b200/csrc/osp_common.cuh"

using namespace osp;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  // zero the operands
  for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
      constexpr uint32_t id = idesc_bf16(128, N, 0, 0);
      long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          if (TS)
            mma_ts(tm + 256, tm + kk * 8, sdesc_sw128(b + off, 16, 1024), id, 1);
          else
            mma_ss(tm + 256, sdesc_sw128(a + off, 16, 1024), sdesc_sw128(b + off, 16, 1024), id, 1);
        }
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
      long long t1 = clock64();
      if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tm, 512);
  }
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      fflush(stdout);                                                           \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <int N, bool TS>
void run(int iters) {
  unsigned long long* d = nullptr;
  printf("run N=%d TS=%d\n", N, int(TS));
  fflush(stdout);
  CK(cudaMalloc(&d, 8));
  auto k = rate_kernel<N, TS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024));
  k<<<148, 128, 131072 + 1024>>>(10, d);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 131072 + 1024>>>(iters, d);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double flops = 148.0 * iters * 8 * 2.0 * 128 * N * 16;
  const double per_mma = double(cyc) / (iters * 8.0);
  printf("%s M=128 N=%3d K=16: %7.1f TFLOP/s  %6.1f cycles/MMA (ideal %5.1f)  err=%s\n",
         TS ? "TS" : "SS", N, flops / ms / 1e9, per_mma, 128.0 * N / 256.0,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main(int argc, char** argv) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  printf("devices %d\n", n);
  fflush(stdout);
  const int iters = 4000;
  const int which = argc > 1 ? atoi(argv[1]) : -1;
  if (which < 0 || which == 0) run<64, false>(iters);
  if (which < 0 || which == 1) run<128, false>(iters);
  if (which < 0 || which == 2) run<256, false>(iters);
  if (which < 0 || which == 3) run<64, true>(iters);
  if (which < 0 || which == 4) run<128, true>(iters);
  if (which < 0 || which == 5) run<256, true>(iters);
  return 0;
}
