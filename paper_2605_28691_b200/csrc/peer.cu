// K7: the SSP pattern switch as one pull over peer memory (NVLink / NVSwitch).
//
// The reference switch is pack -> all-to-all -> unpack (ssp.py:139-180): two local HBM passes
// around one collective.  Here every rank exposes its source rows in a CUDA-IPC buffer, and the
// destination rank gathers its rows straight out of its peers' HBM with one warp per row --
// no pack, no unpack, no staging buffer, no NCCL.  The row table composes the whole move
// (expand the compacted attention output -> pattern switch -> compact for the next
// attention), so the switch moves only real tokens and costs one read of each row over the
// fabric plus one local write.
//
// Ordering: a rank's source rows must be complete before any peer pulls them, and nobody may
// overwrite a source buffer a peer is still reading.  peer_barrier is one flag exchange: each
// rank publishes `epoch` into every peer's flag block (fence.sys + st.release.sys) and spins on
// its own block with ld.acquire.sys.  The host alternates two source slots, so the barrier in
// front of switch i+1 also proves every rank finished pulling switch i-1's slot.
#include "osp_common.cuh"
#include "osp_internal.h"
#include "osp_skiparse.h"

#include <cstring>

namespace osp {

constexpr int kMaxPeers = 64;

struct PeerPtrs {
  const uint8_t* p[kMaxPeers];
};

__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// flags.p[j] = rank j's flag block (uint32[n]); slot i of a block is written by rank i only.
// A rank that has not arrived after timeout_ns is reported through *status (1 + rank, first
// timeout wins) and the kernel returns: no __trap, so the context survives for a diagnosis.
__global__ void peer_barrier_kernel(const PeerPtrs flags, int rank, int n, uint32_t epoch,
                                    uint64_t timeout_ns, int* status) {
  const int t = threadIdx.x;
  if (t >= n) return;
  __threadfence_system();
  st_release_sys(reinterpret_cast<uint32_t*>(const_cast<uint8_t*>(flags.p[t])) + rank, epoch);
  const uint32_t* mine = reinterpret_cast<const uint32_t*>(flags.p[rank]) + t;
  const uint64_t t0 = global_ns();
  // epochs only grow; compare modulo 2^32
  while (static_cast<int32_t>(ld_acquire_sys(mine) - epoch) < 0) {
    if (global_ns() - t0 > timeout_ns) {  // rank t never arrived
      if (status) {
        atomicCAS_system(status, 0, 1 + t);
        __threadfence_system();
      }
      return;
    }
  }
}

// dst[i] = src rank (table[i] / stride), row (table[i] % stride); table[i] < 0 -> zero row.
template <typename V>
__global__ void __launch_bounds__(256) peer_gather_kernel(const PeerPtrs srcs, int n_src,
                                                          int64_t stride, const int64_t* __restrict__ table,
                                                          uint8_t* __restrict__ dst, int64_t n_rows,
                                                          int64_t row_vecs) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n_rows;
       row += nwarps) {
    const int64_t e = __ldg(table + row);
    V* out = reinterpret_cast<V*>(dst) + row * row_vecs;
    const int64_t j = e >= 0 ? e / stride : -1;
    if (j < 0 || j >= n_src) {
      V z;
      memset(&z, 0, sizeof(V));
      for (int64_t i = lane; i < row_vecs; i += 32) out[i] = z;
      continue;
    }
    // peer rows are read with plain loads (not .nc): they were written by another GPU
    const V* in = reinterpret_cast<const V*>(srcs.p[j]) + (e - j * stride) * row_vecs;
    int64_t i = lane;
    for (; i + 224 < row_vecs; i += 256) {  // 8 loads in flight per lane across the fabric
      V a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = in[i + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; ++u) out[i + 32 * u] = a[u];
    }
    for (; i < row_vecs; i += 32) out[i] = in[i];
  }
}

static int fill_ptrs(PeerPtrs& pp, const void* const* ptrs, int n) {
  if (n < 1 || n > kMaxPeers) {
    set_error("peer count must be in [1, " + std::to_string(kMaxPeers) + "]");
    return kValue;
  }
  std::memset(&pp, 0, sizeof(pp));
  for (int i = 0; i < n; ++i) pp.p[i] = static_cast<const uint8_t*>(ptrs[i]);
  return kOk;
}

template <typename V>
static void launch_gather_v(const PeerPtrs& pp, int n, int64_t stride, const int64_t* table, void* dst,
                            int64_t n_rows, int64_t row_bytes, cudaStream_t st) {
  int64_t blocks = (n_rows + 7) / 8;
  blocks = blocks < 148 * 16 ? blocks : 148 * 16;
  if (blocks < 1) blocks = 1;
  peer_gather_kernel<V><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      pp, n, stride, table, static_cast<uint8_t*>(dst), n_rows, row_bytes / static_cast<int64_t>(sizeof(V)));
}

}  // namespace osp

using namespace osp;

static cudaStream_t peer_stream(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

int osp_peer_alloc(int64_t bytes, void** ptr) {
  if (bytes <= 0 || ptr == nullptr) {
    set_error("peer buffer size must be positive");
    return kValue;
  }
  void* p = nullptr;
  int rc = check_cuda(cudaMalloc(&p, static_cast<size_t>(bytes)), "peer cudaMalloc");
  if (rc != kOk) return rc;
  rc = check_cuda(cudaMemset(p, 0, static_cast<size_t>(bytes)), "peer cudaMemset");
  if (rc != kOk) {
    cudaFree(p);
    return rc;
  }
  *ptr = p;
  return kOk;
}

int osp_peer_free(void* ptr) { return check_cuda(cudaFree(ptr), "peer cudaFree"); }

int osp_peer_export(void* ptr, uint8_t* handle64) {
  cudaIpcMemHandle_t h;
  int rc = check_cuda(cudaIpcGetMemHandle(&h, ptr), "cudaIpcGetMemHandle");
  if (rc != kOk) return rc;
  static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
  std::memcpy(handle64, &h, sizeof(h));
  return kOk;
}

int osp_peer_import(const uint8_t* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  return check_cuda(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess),
                    "cudaIpcOpenMemHandle");
}

int osp_peer_close(void* ptr) { return check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); }

int osp_peer_barrier(const void* const* flag_blocks, int rank, int n, uint32_t epoch,
                     int64_t timeout_ms, int* status, void* stream) {
  PeerPtrs pp;
  int rc = fill_ptrs(pp, flag_blocks, n);
  if (rc != kOk) return rc;
  if (rank < 0 || rank >= n) {
    set_error("rank out of range");
    return kValue;
  }
  const uint64_t timeout_ns =
      timeout_ms > 0 ? static_cast<uint64_t>(timeout_ms) * 1000000ull : 60ull * 1000000000ull;
  peer_barrier_kernel<<<1, 32 * ((n + 31) / 32), 0, peer_stream(stream)>>>(pp, rank, n, epoch,
                                                                          timeout_ns, status);
  return check_cuda(cudaGetLastError(), "peer_barrier launch");
}

int osp_peer_gather(const void* const* srcs, int n_src, int64_t stride_rows, const int64_t* table,
                    int64_t n_rows, void* dst, int64_t row_bytes, void* stream) {
  if (n_rows < 0 || row_bytes < 0 || stride_rows < 1) {
    set_error("negative sizes or non-positive stride");
    return kValue;
  }
  PeerPtrs pp;
  int rc = fill_ptrs(pp, srcs, n_src);
  if (rc != kOk) return rc;
  if (n_rows == 0 || row_bytes == 0) return kOk;
  uintptr_t al = reinterpret_cast<uintptr_t>(dst) | static_cast<uintptr_t>(row_bytes);
  for (int i = 0; i < n_src; ++i) al |= reinterpret_cast<uintptr_t>(srcs[i]);
  cudaStream_t st = peer_stream(stream);
  if ((al & 15) == 0) launch_gather_v<uint4>(pp, n_src, stride_rows, table, dst, n_rows, row_bytes, st);
  else if ((al & 7) == 0) launch_gather_v<uint2>(pp, n_src, stride_rows, table, dst, n_rows, row_bytes, st);
  else if ((al & 3) == 0) launch_gather_v<uint32_t>(pp, n_src, stride_rows, table, dst, n_rows, row_bytes, st);
  else if ((al & 1) == 0) launch_gather_v<uint16_t>(pp, n_src, stride_rows, table, dst, n_rows, row_bytes, st);
  else launch_gather_v<uint8_t>(pp, n_src, stride_rows, table, dst, n_rows, row_bytes, st);
  return check_cuda(cudaGetLastError(), "peer_gather launch");
}

}  // extern "C"
