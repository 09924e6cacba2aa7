// Microbenchmark: fp32 reduction throughput into a hot (L2-resident) global region.
//   mode 0: red.global.add.v4.f32, each warp instruction covers 512 contiguous bytes
//   mode 1: cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 of 16 KB from smem
// 148 CTAs x 128 threads; every CTA adds `iters` times into its slice of a `region_mb` region.
#include <cstdio>
#include <cstdlib>

#include "../paper_2605_28691_b200/csrc/osp_common.cuh"

using namespace osp;

__global__ void __launch_bounds__(128, 1) red_kernel(float* dst, size_t region_floats, int iters, int mode) {
  extern __shared__ __align__(128) float stage[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) stage[i] = 1.0f;
  __syncthreads();
  fence_proxy_async_smem();
  const size_t chunk = 4096;  // floats per op group (16 KB)
  const size_t n_chunks = region_floats / chunk;
  for (int it = 0; it < iters; ++it) {
    const size_t c = (static_cast<size_t>(blockIdx.x) * 7 + it) % n_chunks;
    float* base = dst + c * chunk;
    if (mode == 0) {
      // 128 threads x 8 x v4 = 16 KB
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float* p = base + (j * 128 + threadIdx.x) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f),
                     "f"(1.f), "f"(1.f)
                     : "memory");
      }
    } else if (threadIdx.x == 0) {
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(base),
          "r"(smem_u32(stage)), "r"(16384)
          : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
  }
  if (mode == 1 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  for (int mb : {10, 64, 1024}) {
    const size_t n = static_cast<size_t>(mb) << 18;  // floats
    float* d;
    cudaMalloc(&d, n * 4);
    cudaMemset(d, 0, n * 4);
    for (int mode = 0; mode < 2; ++mode) {
      const int iters = 2000;
      red_kernel<<<148, 128, 16384>>>(d, n, 10, mode);
      cudaDeviceSynchronize();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      red_kernel<<<148, 128, 16384>>>(d, n, iters, mode);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = 148.0 * iters * 16384;
      printf("region %5d MB  %-28s %8.1f GB/s of fp32 adds  (%s)\n", mb,
             mode == 0 ? "red.global.add.v4.f32" : "cp.reduce.async.bulk add.f32", bytes / ms / 1e6,
             cudaGetErrorString(e));
      fflush(stdout);
    }
    cudaFree(d);
  }
  return 0;
}
