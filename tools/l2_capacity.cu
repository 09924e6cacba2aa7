// Effective L2 capacity: every SM reads a shared buffer of S MB once (launch 1), then again
// (launch 2); ncu with --cache-control none on launch 2 shows how much of it survived in L2.
// Mode 1: each SM reads only its 1/148 slice (no sharing between SMs).
#include <cstdio>
#include <cstdint>
#include <cstdlib>

__global__ void __launch_bounds__(1024) rd(const uint4* buf, size_t n16, int mode, unsigned* sink) {
  uint32_t acc = 0;
  size_t lo = 0, hi = n16;
  if (mode == 1) {
    lo = n16 * blockIdx.x / gridDim.x;
    hi = n16 * (blockIdx.x + 1) / gridDim.x;
  }
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    uint4 v = __ldcg(buf + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1u);
}

int main(int argc, char** argv) {
  const size_t mb = argc > 1 ? atoi(argv[1]) : 48;
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  const size_t bytes = mb << 20;
  uint4* buf;
  unsigned* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  void* big;
  cudaMalloc(&big, 512ull << 20);
  cudaMemset(big, 0, 512ull << 20);
  cudaDeviceSynchronize();
  rd<<<148, 1024>>>(buf, bytes / 16, mode, sink);
  rd<<<148, 1024>>>(buf, bytes / 16, mode, sink);
  cudaDeviceSynchronize();
  printf("S=%zu MB mode %d (%s)\n", mb, mode, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
