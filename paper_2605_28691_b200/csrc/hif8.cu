// HiF8 8-bit codec and per-tensor current-scaling quantizer on sm_100a.
//
// Replaces hif8.py encode_array / decode_array (hif8.py:171-193) and quantize_tensor's
// amax / scale (hif8.py:223-246).  The 256 values are ascending with code 127 = 0; encoding
// is nearest value, ties to the even code, saturating.  Every midpoint between adjacent values
// has <= 5 significant bits, so comparing x against midpoints is exact in fp32 and fp64 and
// reproduces the reference's |x - v| comparison.  float64 inputs are scaled and compared in
// fp64 (bit-exact with the reference); bf16 / fp32 inputs in fp32 (transport use).
#include <cuda_bf16.h>

#include "osp_common.cuh"
#include "osp_internal.h"

namespace osp {
namespace {

enum Dtype : int { kBf16 = 0, kF32 = 1, kF64 = 2 };

template <typename T>
__device__ __forceinline__ T load_as(const void* p, int64_t i, int dtype) {
  if (dtype == kBf16) return static_cast<T>(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
  if (dtype == kF32) return static_cast<T>(static_cast<const float*>(p)[i]);
  return static_cast<T>(static_cast<const double*>(p)[i]);
}

template <typename T>
__global__ void __launch_bounds__(256) hif8_encode_kernel(const void* __restrict__ x, int dtype, int64_t n,
                                                         const double* __restrict__ scale, int64_t group,
                                                         const double* __restrict__ table,
                                                         uint8_t* __restrict__ codes, int* nonfinite) {
  __shared__ T mids[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    mids[i] = i < 255 ? static_cast<T>((table[i] + table[i + 1]) * 0.5) : static_cast<T>(INFINITY);
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T s = scale ? static_cast<T>(scale[group > 0 ? i / group : 0]) : static_cast<T>(1);
    const T v = load_as<T>(x, i, dtype) * s;
    if (!isfinite(v)) {
      if (nonfinite) atomicOr(nonfinite, 1);
      codes[i] = 0;
      continue;
    }
    int c = 0;  // number of midpoints strictly below v
#pragma unroll
    for (int step = 128; step >= 1; step >>= 1)
      if (mids[c + step - 1] < v) c += step;
    if (c < 255 && mids[c] == v && (c & 1)) ++c;  // exact tie -> even code
    codes[i] = static_cast<uint8_t>(c);
  }
}

template <typename TOut>
__global__ void __launch_bounds__(256) hif8_decode_kernel(const uint8_t* __restrict__ codes, int64_t n,
                                                         const double* __restrict__ scale, int64_t group,
                                                         const double* __restrict__ table,
                                                         TOut* __restrict__ out) {
  __shared__ double vals[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) vals[i] = table[i];
  __syncthreads();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double s = scale ? scale[group > 0 ? i / group : 0] : 1.0;
    const double v = vals[codes[i]] / s;
    if constexpr (sizeof(TOut) == 2)
      out[i] = __float2bfloat16(static_cast<float>(v));
    else
      out[i] = static_cast<TOut>(v);
  }
}

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  // non-negative doubles order like their bit patterns; NaN (all ones exponent + mantissa)
  // sorts above +inf and therefore propagates, as np.max does.
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

__global__ void __launch_bounds__(256) absmax_kernel(const void* __restrict__ x, int dtype, int64_t n,
                                                     double* out) {
  double m = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double v = fabs(load_as<double>(x, i, dtype));
    m = (v > m || v != v) ? v : m;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_xor_sync(0xFFFFFFFFu, m, off);
    m = (o > m || o != o) ? o : m;
  }
  __shared__ double wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) b = (wm[w] > b || wm[w] != wm[w]) ? wm[w] : b;
    atomic_max_nonneg(out, b);
  }
}

__global__ void scale_kernel(const double* amax, int64_t count, double target, double eps, double* scale) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < count) scale[i] = target / (amax[i] + eps);
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

}  // namespace

int launch_hif8_encode(const void* x, int dtype, int64_t n, const double* scale, int64_t group,
                       const double* table, uint8_t* codes, int* nonfinite, cudaStream_t stream) {
  if (n == 0) return kOk;
  if (dtype == kF64)
    hif8_encode_kernel<double><<<grid_for(n), 256, 0, stream>>>(x, dtype, n, scale, group, table, codes, nonfinite);
  else if (dtype == kBf16 || dtype == kF32)
    hif8_encode_kernel<float><<<grid_for(n), 256, 0, stream>>>(x, dtype, n, scale, group, table, codes, nonfinite);
  else {
    set_error("hif8 encode supports bf16, fp32 and fp64 inputs");
    return kUnsupported;
  }
  return check_cuda(cudaGetLastError(), "hif8_encode launch");
}

int launch_hif8_decode(const uint8_t* codes, int64_t n, const double* scale, int64_t group,
                       const double* table, void* out, int dtype, cudaStream_t stream) {
  if (n == 0) return kOk;
  if (dtype == kF64)
    hif8_decode_kernel<double><<<grid_for(n), 256, 0, stream>>>(codes, n, scale, group, table,
                                                                 static_cast<double*>(out));
  else if (dtype == kF32)
    hif8_decode_kernel<float><<<grid_for(n), 256, 0, stream>>>(codes, n, scale, group, table,
                                                               static_cast<float*>(out));
  else if (dtype == kBf16)
    hif8_decode_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, stream>>>(codes, n, scale, group, table,
                                                                       static_cast<__nv_bfloat16*>(out));
  else {
    set_error("hif8 decode supports bf16, fp32 and fp64 outputs");
    return kUnsupported;
  }
  return check_cuda(cudaGetLastError(), "hif8_decode launch");
}

int launch_absmax(const void* x, int dtype, int64_t n, double* out, cudaStream_t stream) {
  int rc = check_cuda(cudaMemsetAsync(out, 0, sizeof(double), stream), "absmax memset");
  if (rc != kOk || n == 0) return rc;
  if (dtype < kBf16 || dtype > kF64) {
    set_error("absmax supports bf16, fp32 and fp64");
    return kUnsupported;
  }
  absmax_kernel<<<grid_for(n), 256, 0, stream>>>(x, dtype, n, out);
  return check_cuda(cudaGetLastError(), "absmax launch");
}

int launch_hif8_scale(const double* amax, int64_t count, double target, double eps, double* scale,
                      cudaStream_t stream) {
  scale_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, stream>>>(amax, count, target, eps, scale);
  return check_cuda(cudaGetLastError(), "hif8_scale launch");
}

}  // namespace osp
