// Probe: do per-row (box {64,1}) and tile::gather4 TMA loads with 128B swizzle produce the same
// shared-memory image as one 128-row box?  (Decides whether K2/K3 can gather rows by TMA.)
// nvcc -gencode arch=compute_100a,code=sm_100a -o tma_gather_probe tools/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap m, const int* rows, uint8_t* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(16384) : "memory");
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(sm)), "l"(&m), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
    } else if (mode == 1) {
      for (int r = 0; r < 128; ++r)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sa(sm + r * 128)), "l"(&m), "r"(0), "r"(rows[r]), "r"(sa(&bar)) : "memory");
    } else {
      for (int r = 0; r < 128; r += 4)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(sa(sm + r * 128)), "l"(&m), "r"(0), "r"(rows[r]), "r"(rows[r + 1]), "r"(rows[r + 2]),
                       "r"(rows[r + 3]), "r"(sa(&bar)) : "memory");
    }
  }
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.b32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(sa(&bar)) : "memory");
  }
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 512, C = 64;
  uint16_t* h = (uint16_t*)malloc(R * C * 2);
  for (int i = 0; i < R * C; ++i) h[i] = (uint16_t)(i * 2654435761u >> 16);
  void* d;
  cudaMalloc(&d, R * C * 2);
  cudaMemcpy(d, h, R * C * 2, cudaMemcpyHostToDevice);
  int hr[128];
  for (int r = 0; r < 128; ++r) hr[r] = r;  // identity rows first: images must match mode 0
  int* dr;
  cudaMalloc(&dr, sizeof(hr));
  uint8_t* dout;
  cudaMalloc(&dout, 16384);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fn;
  uint8_t img[3][16384];
  for (int mode = 0; mode < 3; ++mode) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, mode == 0 ? 128u : (mode == 1 ? 1u : 1u)};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr) { printf("encode mode %d failed %d\n", mode, (int)cr); continue; }
    cudaMemcpy(dr, hr, sizeof(hr), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 17408);
    probe<<<1, 128, 17408>>>(m, dr, dout, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e) return 1;
    cudaMemcpy(img[mode], dout, 16384, cudaMemcpyDeviceToHost);
  }
  printf("per-row == tile: %s\n", memcmp(img[0], img[1], 16384) ? "NO" : "yes");
  printf("gather4 == tile: %s\n", memcmp(img[0], img[2], 16384) ? "NO" : "yes");
  // permuted rows with out-of-range entries (-> zero rows) vs a tile load of the permuted copy
  uint16_t* h2 = (uint16_t*)malloc(R * C * 2);
  memset(h2, 0, R * C * 2);
  for (int r = 0; r < 128; ++r) {
    hr[r] = (r % 13 == 5) ? R + 7 : (r * 37 + 11) % R;
    if (hr[r] < R) memcpy(h2 + r * C, h + hr[r] * C, C * 2);
  }
  void* d2;
  cudaMalloc(&d2, R * C * 2);
  cudaMemcpy(d2, h2, R * C * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, hr, sizeof(hr), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 3; mode += 2) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, mode == 0 ? 128u : 1u};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mode == 0 ? d2 : d, dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    probe<<<1, 128, 17408>>>(m, dr, dout, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("permuted mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(img[mode], dout, 16384, cudaMemcpyDeviceToHost);
  }
  printf("gather4 permuted+OOB == tile of permuted copy: %s\n", memcmp(img[0], img[2], 16384) ? "NO" : "yes");
  return 0;
}
