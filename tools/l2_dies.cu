// Does the B200 L2 keep one copy of a line for both dies, or does each die cache (and fetch from
// DRAM) its own?  Every participating CTA (one per SM) reads the same buffer once; ncu's
// dram__bytes_read then shows one or two copies.  Modes: all SMs, SMs [0,74), even SMs, SMs
// [74,148), and the ids of the SMs' %smid are printed for reference.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void __launch_bounds__(1024) rd(const uint4* buf, size_t n16, int mode, unsigned long long* sink) {
  const uint32_t s = smid();
  bool on = true;
  if (mode == 1) on = s < 74;
  if (mode == 2) on = (s & 1) == 0;
  if (mode == 3) on = s >= 74;
  if (!on) return;
  uint32_t acc = 0;
  for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
    uint4 v = __ldcg(buf + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const size_t bytes = 48ull << 20;
  uint4* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  // evict: touch a 256 MB buffer
  void* big;
  cudaMalloc(&big, 256ull << 20);
  cudaMemset(big, 0, 256ull << 20);
  cudaDeviceSynchronize();
  rd<<<148, 1024>>>(buf, bytes / 16, mode, sink);
  cudaDeviceSynchronize();
  printf("mode %d done (%s)\n", mode, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
