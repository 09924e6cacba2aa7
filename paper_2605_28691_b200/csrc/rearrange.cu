// K1 Skiparse Rearrange, K4 SSP pack/unpack and K5 coordinate masks on sm_100a.
//
// Every map of the reference (skiparse.py:68-140 built by gridseq.py:198-229 and applied by
// IndexMap.apply gridseq.py:161-169; pad_tensor / strip_padding anyres.py:69-89; the SSP
// local steps ssp.py:166-178) permutes whole channel vectors between (batch, seq) addresses.
// Here each map is a closed-form function dst_row -> src_row (no index table in HBM), and
// one copy engine moves the channel vectors with 16-byte vector loads/stores, one warp per
// token row (thread per row for rows shorter than 32 vectors).  Pad slots (src = -1) are
// written as zeros, which fuses pad_tensor into the gather and strip_padding into the
// inverse gather.
#include "osp_common.cuh"
#include "osp_internal.h"

namespace osp {

enum MapKind : int {
  kIdentity = 0,
  kO2T = 1,
  kT2O = 2,
  kO2G = 3,
  kG2O = 4,
  kT2G = 5,
  kG2T = 6,
  kPad = 7,
  kStrip = 8,
  kSspPack = 10,
  kSspUnpack = 11,
  kTable = 12,
};



struct Tok {
  int64_t b, t, r, c;
};

// (row, pos) in the token-wise layout -> token.  row = (p*k+q)*B + b, pos = (t*H/k+hh)*W/k+ww.
__device__ __forceinline__ Tok tsa_token(int64_t row, int64_t pos, int64_t B, int64_t H, int64_t W,
                                         int64_t k) {
  const int64_t pq = row / B, b = row - pq * B;
  const int64_t p = pq / k, q = pq - p * k;
  const int64_t Hk = H / k, Wk = W / k;
  const int64_t ww = pos % Wk;
  const int64_t x = pos / Wk;
  const int64_t hh = x % Hk, t = x / Hk;
  return {b, t, hh * k + p, ww * k + q};
}
__device__ __forceinline__ void tsa_addr(const Tok& o, int64_t B, int64_t T, int64_t H, int64_t W,
                                         int64_t k, int64_t& row, int64_t& pos) {
  row = ((o.r % k) * k + (o.c % k)) * B + o.b;
  pos = (o.t * (H / k) + o.r / k) * (W / k) + o.c / k;
}
// (row, pos) in the group-wise layout -> token.  r = hg*k^2 + p1*k + p2, c = wg*k^2 + q1*k + q2,
// txh = t*H/k^2 + hg; row = (p1*k+q1)*B + b, pos = ((txh*k + p2)*W/k^2 + wg)*k + q2.
__device__ __forceinline__ Tok gsa_token(int64_t row, int64_t pos, int64_t B, int64_t H, int64_t W,
                                         int64_t k) {
  const int64_t k2 = k * k;
  const int64_t pq = row / B, b = row - pq * B;
  const int64_t p1 = pq / k, q1 = pq - p1 * k;
  const int64_t Wg = W / k2, Hg = H / k2;
  const int64_t q2 = pos % k;
  int64_t x = pos / k;
  const int64_t wg = x % Wg;
  x /= Wg;
  const int64_t p2 = x % k;
  const int64_t txh = x / k;
  const int64_t t = txh / Hg, hg = txh - t * Hg;
  return {b, t, hg * k2 + p1 * k + p2, wg * k2 + q1 * k + q2};
}
__device__ __forceinline__ void gsa_addr(const Tok& o, int64_t B, int64_t T, int64_t H, int64_t W,
                                         int64_t k, int64_t& row, int64_t& pos) {
  const int64_t k2 = k * k;
  const int64_t hg = o.r / k2, p1 = (o.r / k) % k, p2 = o.r % k;
  const int64_t wg = o.c / k2, q1 = (o.c / k) % k, q2 = o.c % k;
  const int64_t txh = o.t * (H / k2) + hg;
  row = (p1 * k + q1) * B + o.b;
  pos = ((txh * k + p2) * (W / k2) + wg) * k + q2;
}

__device__ __forceinline__ int64_t orig_src(const MapParams& p, const Tok& o) {
  if (o.r >= p.H0 || o.c >= p.W0) return -1;
  return o.b * (p.T * p.H0 * p.W0) + (o.t * p.H0 + o.r) * p.W0 + o.c;
}

__device__ __forceinline__ Tok orig_token(int64_t d, int64_t T, int64_t H, int64_t W) {
  const int64_t S = T * H * W;
  const int64_t b = d / S;
  int64_t s = d - b * S;
  const int64_t c = s % W;
  s /= W;
  return {b, s / H, s % H, c};
}

__device__ __forceinline__ int64_t map_src(const MapParams& p, int64_t d) {
  const int64_t L = p.T * p.H * p.W / (p.k * p.k);
  int64_t row, pos;
  switch (p.kind) {
    case kIdentity:
      return d;
    case kTable: {
      const int64_t s = __ldg(p.table + d);
      return (s >= 0 && s < p.n_in_rows) ? s : -1;
    }
    case kO2T: {
      Tok o = tsa_token(d / L, d % L, p.B, p.H, p.W, p.k);
      return orig_src(p, o);
    }
    case kO2G: {
      Tok o = gsa_token(d / L, d % L, p.B, p.H, p.W, p.k);
      return orig_src(p, o);
    }
    case kT2O: {
      Tok o = orig_token(d, p.T, p.H0, p.W0);
      tsa_addr(o, p.B, p.T, p.H, p.W, p.k, row, pos);
      return row * L + pos;
    }
    case kG2O: {
      Tok o = orig_token(d, p.T, p.H0, p.W0);
      gsa_addr(o, p.B, p.T, p.H, p.W, p.k, row, pos);
      return row * L + pos;
    }
    case kT2G: {
      Tok o = gsa_token(d / L, d % L, p.B, p.H, p.W, p.k);
      tsa_addr(o, p.B, p.T, p.H, p.W, p.k, row, pos);
      return row * L + pos;
    }
    case kG2T: {
      Tok o = tsa_token(d / L, d % L, p.B, p.H, p.W, p.k);
      gsa_addr(o, p.B, p.T, p.H, p.W, p.k, row, pos);
      return row * L + pos;
    }
    case kPad: {
      Tok o = orig_token(d, p.T, p.H, p.W);
      return orig_src(p, o);
    }
    case kStrip: {
      Tok o = orig_token(d, p.T, p.H0, p.W0);
      return o.b * (p.T * p.H * p.W) + (o.t * p.H + o.r) * p.W + o.c;
    }
    case kSspPack: {
      // Alg. 1 step 1 (ssp.py:156-166): orig_to_tsa on the reduced grid (T, H/k, W/k) with
      // batch G*b; the local shard is (G*b, L) in the current pattern layout.
      const int64_t Hr = p.H / p.k, Wr = p.W / p.k;
      const int64_t base = L / (p.k * p.k);
      Tok o = tsa_token(d / base, d % base, p.B, Hr, Wr, p.k);
      return o.b * L + (o.t * Hr + o.r) * Wr + o.c;
    }
    case kSspUnpack: {
      // Alg. 1 steps 3-4 (ssp.py:172-178) fused: z = recv.view(N,G,G,b,base).permute(0,2,1,3,4)
      // then tsa_to_orig on the reduced grid with batch G*b.
      const int64_t Hr = p.H / p.k, Wr = p.W / p.k;
      const int64_t base = L / (p.k * p.k);
      Tok o = orig_token(d, p.T, Hr, Wr);
      int64_t zrow, zpos;
      tsa_addr(o, p.B, p.T, Hr, Wr, p.k, zrow, zpos);
      const int64_t bb = zrow % p.bsub;
      int64_t x = zrow / p.bsub;
      const int64_t g1 = x % p.G;
      x /= p.G;
      const int64_t g2 = x % p.G;
      const int64_t n = x / p.G;
      const int64_t rrow = ((n * p.G + g1) * p.G + g2) * p.bsub + bb;
      return rrow * base + zpos;
    }
  }
  return -1;
}

template <typename V>
__global__ void __launch_bounds__(256) permute_rows_warp(const MapParams p, const uint8_t* __restrict__ src,
                                                         uint8_t* __restrict__ dst, int64_t n_rows,
                                                         int64_t row_vecs) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n_rows;
       row += nwarps) {
    const int64_t s = map_src(p, row);
    V* out = reinterpret_cast<V*>(dst) + row * row_vecs;
    if (s < 0) {
      V z;
      memset(&z, 0, sizeof(V));
      for (int64_t i = lane; i < row_vecs; i += 32) out[i] = z;
      continue;
    }
    const V* in = reinterpret_cast<const V*>(src) + s * row_vecs;
    int64_t i = lane;
    for (; i + 96 < row_vecs; i += 128) {
      V a0 = __ldg(in + i), a1 = __ldg(in + i + 32), a2 = __ldg(in + i + 64), a3 = __ldg(in + i + 96);
      out[i] = a0;
      out[i + 32] = a1;
      out[i + 64] = a2;
      out[i + 96] = a3;
    }
    for (; i < row_vecs; i += 32) out[i] = __ldg(in + i);
  }
}

template <typename V>
__global__ void __launch_bounds__(256) permute_rows_thread(const MapParams p, const uint8_t* __restrict__ src,
                                                           uint8_t* __restrict__ dst, int64_t n_rows,
                                                           int64_t row_vecs) {
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; row < n_rows;
       row += nthreads) {
    const int64_t s = map_src(p, row);
    V* out = reinterpret_cast<V*>(dst) + row * row_vecs;
    if (s < 0) {
      V z;
      memset(&z, 0, sizeof(V));
      for (int64_t i = 0; i < row_vecs; ++i) out[i] = z;
    } else {
      const V* in = reinterpret_cast<const V*>(src) + s * row_vecs;
      for (int64_t i = 0; i < row_vecs; ++i) out[i] = __ldg(in + i);
    }
  }
}

template <typename V>
int launch_permute_v(const MapParams& p, const void* src, void* dst, int64_t n_rows, int64_t row_bytes,
                     cudaStream_t stream) {
  const int64_t vecs = row_bytes / static_cast<int64_t>(sizeof(V));
  const int threads = 256;
  if (vecs >= 32) {
    int64_t blocks = (n_rows + 7) / 8;
    blocks = blocks < 148 * 32 ? blocks : 148 * 32;
    if (blocks < 1) blocks = 1;
    permute_rows_warp<V><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        p, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n_rows, vecs);
  } else {
    int64_t blocks = (n_rows + threads - 1) / threads;
    blocks = blocks < 148 * 32 ? blocks : 148 * 32;
    if (blocks < 1) blocks = 1;
    permute_rows_thread<V><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(
        p, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n_rows, vecs);
  }
  return check_cuda(cudaGetLastError(), "permute_rows launch");
}

int launch_permute(const MapParams& p, const void* src, void* dst, int64_t n_rows, int64_t row_bytes,
                   cudaStream_t stream) {
  if (n_rows == 0 || row_bytes == 0) return kOk;
  const uintptr_t al = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                       static_cast<uintptr_t>(row_bytes);
  if ((al & 15) == 0) return launch_permute_v<uint4>(p, src, dst, n_rows, row_bytes, stream);
  if ((al & 7) == 0) return launch_permute_v<uint2>(p, src, dst, n_rows, row_bytes, stream);
  if ((al & 3) == 0) return launch_permute_v<uint32_t>(p, src, dst, n_rows, row_bytes, stream);
  if ((al & 1) == 0) return launch_permute_v<uint16_t>(p, src, dst, n_rows, row_bytes, stream);
  return launch_permute_v<uint8_t>(p, src, dst, n_rows, row_bytes, stream);
}

// ------------------------------------------------------------------------- chunked table gather
// dst row r, channel chunk c  <-  src row index[r], chunk c, for layouts that store the channel
// chunks either inline (row stride = whole row, chunk stride = chunk width) or as separate
// contiguous blocks (row stride = chunk width, chunk stride = rows x chunk width).  This is the
// SSP switch's local step when the all-to-all runs per head chunk (overlapped with attention):
// the unpack (+ compaction) of all received chunks into one row-major activation, and the pack of
// a gradient into per-chunk send blocks.  index[r] < 0 (or >= n_in_rows) writes zeros.
template <typename V>
__global__ void __launch_bounds__(256) gather_chunks_warp(const int64_t* __restrict__ index,
                                                          const uint8_t* __restrict__ src,
                                                          uint8_t* __restrict__ dst, int64_t n_rows,
                                                          int64_t n_in_rows, int n_chunks, int64_t chunk_vecs,
                                                          int64_t src_rs, int64_t src_cs, int64_t dst_rs,
                                                          int64_t dst_cs) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; row < n_rows;
       row += nwarps) {
    int64_t s = __ldg(index + row);
    if (s >= n_in_rows) s = -1;
    for (int c = 0; c < n_chunks; ++c) {
      V* out = reinterpret_cast<V*>(dst + c * dst_cs + row * dst_rs);
      if (s < 0) {
        V z;
        memset(&z, 0, sizeof(V));
        for (int64_t i = lane; i < chunk_vecs; i += 32) out[i] = z;
        continue;
      }
      const V* in = reinterpret_cast<const V*>(src + c * src_cs + s * src_rs);
      int64_t i = lane;
      for (; i + 96 < chunk_vecs; i += 128) {
        V a0 = __ldg(in + i), a1 = __ldg(in + i + 32), a2 = __ldg(in + i + 64), a3 = __ldg(in + i + 96);
        out[i] = a0;
        out[i + 32] = a1;
        out[i + 64] = a2;
        out[i + 96] = a3;
      }
      for (; i < chunk_vecs; i += 32) out[i] = __ldg(in + i);
    }
  }
}

template <typename V>
static int launch_gather_chunks_v(const int64_t* index, const void* src, void* dst, int64_t n_rows,
                                  int64_t n_in_rows, int n_chunks, int64_t chunk_bytes, int64_t src_rs,
                                  int64_t src_cs, int64_t dst_rs, int64_t dst_cs, cudaStream_t stream) {
  int64_t blocks = (n_rows + 7) / 8;
  blocks = blocks < 148 * 32 ? blocks : 148 * 32;
  if (blocks < 1) blocks = 1;
  gather_chunks_warp<V><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      index, static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), n_rows, n_in_rows, n_chunks,
      chunk_bytes / static_cast<int64_t>(sizeof(V)), src_rs, src_cs, dst_rs, dst_cs);
  return check_cuda(cudaGetLastError(), "gather_chunks launch");
}

int launch_gather_chunks(const int64_t* index, const void* src, void* dst, int64_t n_rows, int64_t n_in_rows,
                         int n_chunks, int64_t chunk_bytes, int64_t src_rs, int64_t src_cs, int64_t dst_rs,
                         int64_t dst_cs, cudaStream_t stream) {
  if (n_rows == 0 || chunk_bytes == 0 || n_chunks == 0) return kOk;
  const uint64_t al = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                      static_cast<uint64_t>(chunk_bytes) | static_cast<uint64_t>(src_rs) |
                      static_cast<uint64_t>(src_cs) | static_cast<uint64_t>(dst_rs) | static_cast<uint64_t>(dst_cs);
  if ((al & 15) == 0)
    return launch_gather_chunks_v<uint4>(index, src, dst, n_rows, n_in_rows, n_chunks, chunk_bytes, src_rs,
                                         src_cs, dst_rs, dst_cs, stream);
  if ((al & 3) == 0)
    return launch_gather_chunks_v<uint32_t>(index, src, dst, n_rows, n_in_rows, n_chunks, chunk_bytes, src_rs,
                                            src_cs, dst_rs, dst_cs, stream);
  if ((al & 1) == 0)
    return launch_gather_chunks_v<uint16_t>(index, src, dst, n_rows, n_in_rows, n_chunks, chunk_bytes, src_rs,
                                            src_cs, dst_rs, dst_cs, stream);
  return launch_gather_chunks_v<uint8_t>(index, src, dst, n_rows, n_in_rows, n_chunks, chunk_bytes, src_rs,
                                         src_cs, dst_rs, dst_cs, stream);
}

// ------------------------------------------------------------------------- K5 masks
// bits[row][w] bit i <=> the source token of (row, 32*w+i) is real (r < H0 and c < W0).
// pattern: 0 original, 1 token-wise, 2 group-wise (anyres.py:92-96 with attention.py:121-125
// batch nesting (pattern id, batch item)).
__global__ void pattern_mask_bits_kernel(uint32_t* bits, int64_t n_rows, int64_t L, int64_t words,
                                         int pattern, int64_t B, int64_t T, int64_t H, int64_t W,
                                         int64_t k, int64_t H0, int64_t W0) {
  const int64_t total = n_rows * words;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / words, w = i - row * words;
    uint32_t m = 0;
    for (int j = 0; j < 32; ++j) {
      const int64_t pos = w * 32 + j;
      if (pos >= L) break;
      Tok o;
      if (pattern == 1) o = tsa_token(row, pos, B, H, W, k);
      else if (pattern == 2) o = gsa_token(row, pos, B, H, W, k);
      else o = orig_token(row * L + pos, T, H, W);
      if (o.r < H0 && o.c < W0) m |= 1u << j;
    }
    bits[i] = m;
  }
}

__global__ void bytes_to_bits_kernel(const uint8_t* valid, uint32_t* bits, int64_t n_rows, int64_t L,
                                     int64_t words) {
  const int64_t total = n_rows * words;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / words, w = i - row * words;
    uint32_t m = 0;
    for (int j = 0; j < 32; ++j) {
      const int64_t pos = w * 32 + j;
      if (pos >= L) break;
      if (valid[row * L + pos]) m |= 1u << j;
    }
    bits[i] = m;
  }
}

__global__ void bits_to_bytes_kernel(const uint32_t* bits, uint8_t* valid, int64_t n_rows, int64_t L,
                                     int64_t words) {
  const int64_t total = n_rows * L;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / L, pos = i - row * L;
    valid[i] = (bits[row * words + (pos >> 5)] >> (pos & 31)) & 1u;
  }
}

__global__ void invert_index_kernel(const int64_t* index, int64_t* inv, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = index[i];
    if (s >= 0 && s < n) inv[s] = i;
  }
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 64) b = 148 * 64;
  if (b < 1) b = 1;
  return static_cast<unsigned>(b);
}

int launch_pattern_mask_bits(uint32_t* bits, int64_t B, int64_t T, int64_t H, int64_t W, int64_t k,
                             int pattern, int64_t H0, int64_t W0, cudaStream_t stream) {
  const int64_t n_sub = pattern == 0 ? 1 : k * k;
  const int64_t L = T * H * W / n_sub;
  const int64_t words = (L + 31) / 32;
  const int64_t n_rows = n_sub * B;
  pattern_mask_bits_kernel<<<grid_for(n_rows * words, 256), 256, 0, stream>>>(
      bits, n_rows, L, words, pattern, B, T, H, W, k, H0, W0);
  return check_cuda(cudaGetLastError(), "pattern_mask_bits launch");
}

int launch_bytes_to_bits(const uint8_t* valid, uint32_t* bits, int64_t n_rows, int64_t L,
                         cudaStream_t stream) {
  const int64_t words = (L + 31) / 32;
  bytes_to_bits_kernel<<<grid_for(n_rows * words, 256), 256, 0, stream>>>(valid, bits, n_rows, L, words);
  return check_cuda(cudaGetLastError(), "bytes_to_bits launch");
}

int launch_bits_to_bytes(const uint32_t* bits, uint8_t* valid, int64_t n_rows, int64_t L,
                         cudaStream_t stream) {
  const int64_t words = (L + 31) / 32;
  bits_to_bytes_kernel<<<grid_for(n_rows * L, 256), 256, 0, stream>>>(bits, valid, n_rows, L, words);
  return check_cuda(cudaGetLastError(), "bits_to_bytes launch");
}

int launch_invert_index(const int64_t* index, int64_t* inv, int64_t n, cudaStream_t stream) {
  if (n == 0) return kOk;
  invert_index_kernel<<<grid_for(n, 256), 256, 0, stream>>>(index, inv, n);
  return check_cuda(cudaGetLastError(), "invert_index launch");
}

}  // namespace osp
