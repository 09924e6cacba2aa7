// extern "C" entry points of libosp_skiparse.so (declared in include/osp_skiparse.h):
// argument validation with the reference's error semantics, TMA descriptor encoding, and
// dispatch to the kernels.
#include <cstdio>
#include <string>

#include "../../include/osp_skiparse.h"
#include "osp_internal.h"

namespace osp {

int launch_permute(const MapParams& p, const void* src, void* dst, int64_t n_rows,
                   int64_t row_bytes, cudaStream_t stream);
int launch_pattern_mask_bits(uint32_t* bits, int64_t B, int64_t T, int64_t H, int64_t W,
                             int64_t k, int pattern, int64_t H0, int64_t W0, cudaStream_t stream);
int launch_bytes_to_bits(const uint8_t* valid, uint32_t* bits, int64_t n_rows, int64_t L,
                         cudaStream_t stream);
int launch_bits_to_bytes(const uint32_t* bits, uint8_t* valid, int64_t n_rows, int64_t L,
                         cudaStream_t stream);
int launch_invert_index(const int64_t* index, int64_t* inv, int64_t n, cudaStream_t stream);
int launch_gather_chunks(const int64_t* index, const void* src, void* dst, int64_t n_rows, int64_t n_in_rows,
                         int n_chunks, int64_t chunk_bytes, int64_t src_rs, int64_t src_cs, int64_t dst_rs,
                         int64_t dst_cs, cudaStream_t stream);
int launch_hif8_encode(const void* x, int dtype, int64_t n, const double* scale, int64_t group,
                       const double* table, uint8_t* codes, int* nonfinite, cudaStream_t stream);
int launch_hif8_decode(const uint8_t* codes, int64_t n, const double* scale, int64_t group,
                       const double* table, void* out, int dtype, cudaStream_t stream);
int launch_absmax(const void* x, int dtype, int64_t n, double* out, cudaStream_t stream);
int launch_hif8_scale(const double* amax, int64_t count, double target, double eps, double* scale,
                      cudaStream_t stream);

int debug_counters(unsigned long long* host, int n, int reset);
int debug_counters_bwd(unsigned long long* host, int n, int reset);

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return kOk;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return kCuda;
}

int set_smem_attr(const void* kernel, int bytes, std::atomic<uint64_t>& done, const char* what) {
  int dev = 0;
  int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != kOk) return rc;
  const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return kOk;
  rc = check_cuda(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
  if (rc != kOk) return rc;
  if (bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return kOk;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

int make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                      int64_t row_stride_elems, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return kCuda;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (row_stride_elems * 2) % 16 != 0) {
    set_error("attention operands need 16-byte aligned base pointers and row strides");
    return kValue;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(row_stride_elems * 2)};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled (2d) failed (%d) cols=%lld rows=%lld",
             static_cast<int>(r), static_cast<long long>(cols), static_cast<long long>(rows));
    set_error(buf);
    return kCuda;
  }
  return kOk;
}

int make_tmap_bf16_3d(CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                      int64_t n_seq, int64_t row_stride_elems, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
    return kCuda;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (row_stride_elems * 2) % 16 != 0) {
    set_error("attention operands need 16-byte aligned base pointers and row strides");
    return kValue;
  }
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(n_seq)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(row_stride_elems * 2),
                           static_cast<cuuint64_t>(rows * row_stride_elems * 2)};
  cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d) cols=%lld rows=%lld stride=%lld",
             static_cast<int>(r), static_cast<long long>(cols), static_cast<long long>(rows),
             static_cast<long long>(row_stride_elems));
    set_error(buf);
    return kCuda;
  }
  return kOk;
}

}  // namespace osp

using namespace osp;

static cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

static int grid_error(int64_t t, int64_t h, int64_t w, int64_t k) {
  if (t < 1 || h < 1 || w < 1 || k < 1) {
    set_error("grid extents and k must be positive integers");
    return kValue;
  }
  return kOk;
}

static int need_tsa(int64_t h, int64_t w, int64_t k) {
  if (h % k || w % k) {
    set_error("token-wise pattern needs h and w divisible by k=" + std::to_string(k) + ", got " +
              std::to_string(h) + "x" + std::to_string(w));
    return kPattern;
  }
  return kOk;
}

static int need_gsa(int64_t h, int64_t w, int64_t k) {
  if (h % (k * k) || w % (k * k)) {
    set_error("group-wise pattern needs h and w divisible by k^2=" + std::to_string(k * k) +
              ", got " + std::to_string(h) + "x" + std::to_string(w));
    return kPattern;
  }
  return kOk;
}

extern "C" {

const char* osp_last_error(void) { return g_err.c_str(); }

int osp_abi_version(void) { return OSP_ABI_VERSION; }

int osp_device_check(void) {
  int dev = 0;
  int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc != kOk) return rc;
  cudaDeviceProp prop;
  rc = check_cuda(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
  if (rc != kOk) return rc;
  if (prop.major != 10 || prop.minor != 0) {
    set_error("libosp_skiparse is built for sm_100a (B200); device is sm_" +
              std::to_string(prop.major) + std::to_string(prop.minor));
    return kUnsupported;
  }
  return kOk;
}

int osp_rearrange(const void* src, void* dst, int64_t elem_bytes, int64_t chan, int64_t batch,
                  int64_t t, int64_t h, int64_t w, int64_t k, int map_id, int64_t h_orig,
                  int64_t w_orig, void* stream) {
  int rc = grid_error(t, h, w, k);
  if (rc != kOk) return rc;
  if (elem_bytes < 1 || chan < 0 || batch < 1) {
    set_error("bad element size / chan / batch");
    return kValue;
  }
  if (h_orig <= 0) h_orig = h;
  if (w_orig <= 0) w_orig = w;
  if (h_orig > h || w_orig > w) {
    set_error("original extents exceed the padded grid");
    return kShape;
  }
  const bool padded = h_orig != h || w_orig != w;
  switch (map_id) {
    case OSP_MAP_O2T:
    case OSP_MAP_T2O:
      rc = need_tsa(h, w, k);
      break;
    case OSP_MAP_O2G:
    case OSP_MAP_G2O:
    case OSP_MAP_T2G:
    case OSP_MAP_G2T:
      rc = need_gsa(h, w, k);
      break;
    case OSP_MAP_IDENTITY:
    case OSP_MAP_PAD:
    case OSP_MAP_STRIP:
      break;
    default:
      set_error("unknown map id " + std::to_string(map_id));
      return kValue;
  }
  if (rc != kOk) return rc;
  if (padded && (map_id == OSP_MAP_T2G || map_id == OSP_MAP_G2T || map_id == OSP_MAP_IDENTITY)) {
    set_error("pattern-to-pattern maps run on the padded grid; pass h_orig=h, w_orig=w");
    return kValue;
  }
  MapParams p{};
  p.kind = map_id;
  p.B = batch;
  p.T = t;
  p.H = h;
  p.W = w;
  p.k = k;
  p.H0 = h_orig;
  p.W0 = w_orig;
  int64_t n_rows;
  const int64_t S = t * h * w, S0 = t * h_orig * w_orig;
  switch (map_id) {
    case OSP_MAP_T2O:
    case OSP_MAP_G2O:
    case OSP_MAP_STRIP:
      n_rows = batch * S0;
      break;
    default:
      n_rows = batch * S;
  }
  return launch_permute(p, src, dst, n_rows, elem_bytes * chan, as_stream(stream));
}

int osp_gather_rows(const void* src, void* dst, const int64_t* index, int64_t n_out_rows,
                    int64_t n_in_rows, int64_t row_bytes, void* stream) {
  if (n_out_rows < 0 || n_in_rows < 0 || row_bytes < 0) {
    set_error("negative sizes");
    return kValue;
  }
  MapParams p{};
  p.kind = 12;
  p.table = index;
  p.n_in_rows = n_in_rows;
  p.T = p.H = p.W = p.k = 1;
  return launch_permute(p, src, dst, n_out_rows, row_bytes, as_stream(stream));
}

int osp_gather_rows_chunked(const void* src, void* dst, const int64_t* index, int64_t n_out_rows,
                            int64_t n_in_rows, int64_t n_chunks, int64_t chunk_bytes,
                            int64_t src_row_stride, int64_t src_chunk_stride, int64_t dst_row_stride,
                            int64_t dst_chunk_stride, void* stream) {
  if (n_out_rows < 0 || n_in_rows < 0 || chunk_bytes < 0 || n_chunks < 0 || n_chunks > (1 << 20) ||
      src_row_stride < 0 || src_chunk_stride < 0 || dst_row_stride < 0 || dst_chunk_stride < 0) {
    set_error("negative sizes / strides");
    return kValue;
  }
  if (n_out_rows && !index) {
    set_error("missing index table");
    return kValue;
  }
  return launch_gather_chunks(index, src, dst, n_out_rows, n_in_rows, static_cast<int>(n_chunks), chunk_bytes,
                              src_row_stride, src_chunk_stride, dst_row_stride, dst_chunk_stride,
                              as_stream(stream));
}

int osp_invert_index(const int64_t* index, int64_t* inv, int64_t n, void* stream) {
  return launch_invert_index(index, inv, n, as_stream(stream));
}

int osp_pattern_mask_bits(uint32_t* bits, int64_t batch, int64_t t, int64_t h, int64_t w,
                          int64_t k, int pattern, int64_t h_orig, int64_t w_orig, void* stream) {
  int rc = grid_error(t, h, w, k);
  if (rc != kOk) return rc;
  if (pattern == OSP_PATTERN_TSA) rc = need_tsa(h, w, k);
  else if (pattern == OSP_PATTERN_GSA) rc = need_gsa(h, w, k);
  else if (pattern != OSP_PATTERN_ORIGINAL) {
    set_error("unknown pattern");
    return kValue;
  }
  if (rc != kOk) return rc;
  if (h_orig <= 0) h_orig = h;
  if (w_orig <= 0) w_orig = w;
  return launch_pattern_mask_bits(bits, batch, t, h, w, k, pattern, h_orig, w_orig, as_stream(stream));
}

int osp_mask_bytes_to_bits(const uint8_t* valid, uint32_t* bits, int64_t n_rows, int64_t len,
                           void* stream) {
  return launch_bytes_to_bits(valid, bits, n_rows, len, as_stream(stream));
}

int osp_mask_bits_to_bytes(const uint32_t* bits, uint8_t* valid, int64_t n_rows, int64_t len,
                           void* stream) {
  return launch_bits_to_bytes(bits, valid, n_rows, len, as_stream(stream));
}

static int attn_checks(int64_t n_seq, int64_t seq_len, int64_t heads, int64_t head_dim) {
  if (head_dim != 64 && head_dim != 128) {
    set_error("B200 attention kernels support head_dim 64 or 128, got " +
              std::to_string(head_dim));
    return kUnsupported;
  }
  if (n_seq < 1 || seq_len < 1 || heads < 1 || n_seq > 65535 || heads > 65535 ||
      seq_len > (int64_t(1) << 30)) {
    set_error("attention shape out of range");
    return kShape;
  }
  return kOk;
}

int osp_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n_seq,
                 int64_t seq_len, int64_t heads, int64_t head_dim, int64_t q_stride,
                 int64_t k_stride, int64_t v_stride, int64_t o_stride, const uint32_t* valid_bits,
                 const int32_t* seq_lens, int zero_invalid_queries, float scale, void* stream) {
  int rc = attn_checks(n_seq, seq_len, heads, head_dim);
  if (rc != kOk) return rc;
  if ((o_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(o) & 15)) {
    set_error("output needs 16-byte aligned base and row stride");
    return kValue;
  }
  AttnShape s{n_seq, seq_len, heads, head_dim, seq_lens};
  return launch_attn_fwd(q, k, v, o, lse, s, q_stride, k_stride, v_stride, o_stride, valid_bits,
                         zero_invalid_queries, scale, as_stream(stream));
}

size_t osp_attn_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t heads,
                                    int64_t head_dim) {
  AttnShape s{n_seq, seq_len, heads, head_dim};
  return attn_bwd_workspace_bytes(s);
}

int osp_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, void* dq, void* dk, void* dv, int64_t n_seq, int64_t seq_len,
                 int64_t heads, int64_t head_dim, int64_t q_stride, int64_t k_stride,
                 int64_t v_stride, int64_t o_stride, int64_t do_stride, int64_t dq_stride,
                 int64_t dk_stride, int64_t dv_stride, const uint32_t* valid_bits,
                 const int32_t* seq_lens, int zero_invalid_queries, float scale, void* workspace,
                 size_t workspace_bytes, void* stream) {
  int rc = attn_checks(n_seq, seq_len, heads, head_dim);
  if (rc != kOk) return rc;
  AttnShape s{n_seq, seq_len, heads, head_dim, seq_lens};
  if (workspace_bytes < attn_bwd_workspace_bytes(s)) {
    set_error("attention backward workspace too small");
    return kValue;
  }
  return launch_attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, s, q_stride, k_stride, v_stride,
                         o_stride, do_stride, dq_stride, dk_stride, dv_stride, valid_bits,
                         zero_invalid_queries, scale, workspace, workspace_bytes, as_stream(stream));
}

int osp_attn_fwd_gather(const void* q, const void* k, const void* v, void* o, float* lse,
                        int64_t n_rows, const int32_t* row_index, const int32_t* seq_lens,
                        int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                        int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                        float scale, void* stream) {
  int rc = attn_checks(n_seq, capacity, heads, head_dim);
  if (rc != kOk) return rc;
  if (!row_index || !seq_lens || n_rows <= 0 || capacity % 4) {
    set_error("gather attention needs row_index, seq_lens, n_rows > 0 and capacity % 4 == 0");
    return kValue;
  }
  if ((o_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(o) & 15)) {
    set_error("output needs 16-byte aligned base and row stride");
    return kValue;
  }
  AttnShape s{n_seq, capacity, heads, head_dim, seq_lens, row_index, n_rows};
  return launch_attn_fwd(q, k, v, o, lse, s, q_stride, k_stride, v_stride, o_stride, nullptr, 0,
                         scale, as_stream(stream));
}

int osp_attn_bwd_gather(const void* q, const void* k, const void* v, const void* o,
                        const void* dout, const float* lse, void* dq, void* dk, void* dv,
                        int64_t n_rows, const int32_t* row_index, const int32_t* seq_lens,
                        int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                        int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                        int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                        float scale, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = attn_checks(n_seq, capacity, heads, head_dim);
  if (rc != kOk) return rc;
  if (!row_index || !seq_lens || n_rows <= 0 || capacity % 4) {
    set_error("gather attention needs row_index, seq_lens, n_rows > 0 and capacity % 4 == 0");
    return kValue;
  }
  AttnShape s{n_seq, capacity, heads, head_dim, seq_lens, row_index, n_rows};
  if (workspace_bytes < attn_bwd_workspace_bytes(s)) {
    set_error("attention backward workspace too small");
    return kValue;
  }
  return launch_attn_bwd(q, k, v, o, dout, lse, dq, dk, dv, s, q_stride, k_stride, v_stride,
                         o_stride, do_stride, dq_stride, dk_stride, dv_stride, nullptr, 0, scale,
                         workspace, workspace_bytes, as_stream(stream));
}

static int scatter_checks(const int32_t* seq_lens, const int32_t* out_index, int64_t n_out_rows,
                          int64_t out_stride, const void* out) {
  if (!seq_lens || !out_index || n_out_rows <= 0 || n_out_rows >= (int64_t(1) << 31)) {
    set_error("scatter attention needs seq_lens, out_index and 0 < n_out_rows < 2^31");
    return kValue;
  }
  if ((out_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(out) & 15)) {
    set_error("output needs 16-byte aligned base and row stride");
    return kValue;
  }
  return kOk;
}

int osp_attn_fwd_scatter(const void* q, const void* k, const void* v, void* out, float* lse,
                         int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                         int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t out_stride,
                         const int32_t* seq_lens, const int32_t* out_index, int64_t n_out_rows,
                         const int32_t* zero_rows, int64_t n_zero_rows, float scale, void* stream) {
  int rc = attn_checks(n_seq, capacity, heads, head_dim);
  if (rc != kOk) return rc;
  if ((rc = scatter_checks(seq_lens, out_index, n_out_rows, out_stride, out)) != kOk) return rc;
  if (n_zero_rows < 0 || n_zero_rows > n_out_rows || (n_zero_rows && !zero_rows)) {
    set_error("zero_rows must list 0 <= n_zero_rows <= n_out_rows rows");
    return kValue;
  }
  AttnShape s{n_seq, capacity, heads, head_dim, seq_lens};
  s.out_index = out_index;
  s.zero_rows = zero_rows;
  s.n_zero = n_zero_rows;
  return launch_attn_fwd(q, k, v, out, lse, s, q_stride, k_stride, v_stride, out_stride, nullptr, 0,
                         scale, as_stream(stream));
}

size_t osp_attn_bwd_scatter_workspace_bytes(int64_t n_seq, int64_t capacity, int64_t heads,
                                            int64_t head_dim) {
  AttnShape s{n_seq, capacity, heads, head_dim};
  return attn_bwd_workspace_bytes(s) + static_cast<size_t>(n_seq * capacity * heads * head_dim * 2);
}

int osp_attn_bwd_scatter(const void* q, const void* k, const void* v, const void* out,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv,
                         int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                         int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t out_stride,
                         int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                         const int32_t* seq_lens, const int32_t* out_index, int64_t n_out_rows,
                         float scale, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = attn_checks(n_seq, capacity, heads, head_dim);
  if (rc != kOk) return rc;
  if ((rc = scatter_checks(seq_lens, out_index, n_out_rows, out_stride, out)) != kOk) return rc;
  if ((do_stride * 2) % 16 || (reinterpret_cast<uintptr_t>(dout) & 15)) {
    set_error("dout needs 16-byte aligned base and row stride");
    return kValue;
  }
  AttnShape s{n_seq, capacity, heads, head_dim, seq_lens};
  const size_t base = attn_bwd_workspace_bytes(s);
  if (workspace_bytes < osp_attn_bwd_scatter_workspace_bytes(n_seq, capacity, heads, head_dim)) {
    set_error("attention backward workspace too small (osp_attn_bwd_scatter_workspace_bytes)");
    return kValue;
  }
  s.out_index = out_index;
  s.do_image = static_cast<uint8_t*>(workspace) + base;
  return launch_attn_bwd(q, k, v, out, dout, lse, dq, dk, dv, s, q_stride, k_stride, v_stride,
                         out_stride, do_stride, dq_stride, dk_stride, dv_stride, nullptr, 0, scale,
                         workspace, workspace_bytes, as_stream(stream));
}

static int ssp_params(MapParams& p, int kind, int64_t group_size, int64_t local_batch, int64_t t,
                      int64_t h, int64_t w, int64_t k) {
  int rc = grid_error(t, h, w, k);
  if (rc != kOk) return rc;
  if (group_size < 1) {
    set_error("group size must be positive");
    return kValue;
  }
  const int64_t k2 = k * k;
  if (k2 % group_size) {  // ssp.py:147-148
    set_error("k^2=" + std::to_string(k2) + " not divisible by group size " +
              std::to_string(group_size));
    return kSharding;
  }
  const int64_t G = k2 / group_size;
  if (local_batch % G) {  // ssp.py:150-153
    set_error("local batch " + std::to_string(local_batch) + " not divisible by G=" +
              std::to_string(G));
    return kProtocol;
  }
  rc = need_gsa(h, w, k);
  if (rc != kOk) return rc;
  p = MapParams{};
  p.kind = kind;
  p.B = local_batch;
  p.T = t;
  p.H = h;
  p.W = w;
  p.k = k;
  p.H0 = h;
  p.W0 = w;
  p.G = G;
  p.bsub = local_batch / G;
  return kOk;
}

int osp_ssp_pack(const void* src, void* dst, int64_t elem_bytes, int64_t chan,
                 int64_t group_size, int64_t local_batch, int64_t t, int64_t h, int64_t w,
                 int64_t k, void* stream) {
  MapParams p;
  int rc = ssp_params(p, 10, group_size, local_batch, t, h, w, k);
  if (rc != kOk) return rc;
  const int64_t L = t * h * w / (k * k);
  return launch_permute(p, src, dst, local_batch * L, elem_bytes * chan, as_stream(stream));
}

int osp_ssp_unpack(const void* recv, void* dst, int64_t elem_bytes, int64_t chan,
                   int64_t group_size, int64_t local_batch, int64_t t, int64_t h, int64_t w,
                   int64_t k, void* stream) {
  MapParams p;
  int rc = ssp_params(p, 11, group_size, local_batch, t, h, w, k);
  if (rc != kOk) return rc;
  const int64_t L = t * h * w / (k * k);
  return launch_permute(p, recv, dst, local_batch * L, elem_bytes * chan, as_stream(stream));
}

int osp_absmax(const void* x, int dtype, int64_t n, double* amax, void* stream) {
  if (n < 0) {
    set_error("negative size");
    return kValue;
  }
  return launch_absmax(x, dtype, n, amax, as_stream(stream));
}

int osp_hif8_scale(const double* amax, int64_t count, double target, double eps, double* scale,
                   void* stream) {
  if (count < 1) {
    set_error("scale count must be positive");
    return kValue;
  }
  return launch_hif8_scale(amax, count, target, eps, scale, as_stream(stream));
}

int osp_hif8_encode(const void* x, int dtype, int64_t n, const double* scale,
                    int64_t scale_group, const double* table, uint8_t* codes, int* nonfinite_flag,
                    void* stream) {
  if (n < 0 || scale_group < 0 || !table) {
    set_error("hif8 encode: bad size / group / missing value table");
    return kValue;
  }
  return launch_hif8_encode(x, dtype, n, scale, scale_group, table, codes, nonfinite_flag,
                            as_stream(stream));
}

int osp_hif8_decode(const uint8_t* codes, int64_t n, const double* scale, int64_t scale_group,
                    const double* table, void* out, int dtype, void* stream) {
  if (n < 0 || scale_group < 0 || !table) {
    set_error("hif8 decode: bad size / group / missing value table");
    return kValue;
  }
  return launch_hif8_decode(codes, n, scale, scale_group, table, out, dtype, as_stream(stream));
}

int osp_qkv_project(const void* x, const void* w_t, void* out, int64_t rows, int64_t chan,
                    int64_t out_stride, int norm, const float* gamma_q, const float* gamma_k,
                    float eps, float* sumsq, const float* rope_table, int64_t t, int64_t h,
                    int64_t w, int64_t k, int pattern, int64_t batch, int64_t row_offset,
                    void* stream) {
  if (rows < 0 || chan <= 0 || !x || !w_t || !out) {
    set_error("qkv projection: bad sizes or null pointers");
    return kValue;
  }
  return launch_qkv_project(x, w_t, out, rows, chan, out_stride, norm, gamma_q, gamma_k, eps, sumsq,
                            rope_table, t, h, w, k, pattern, batch, row_offset, as_stream(stream));
}

int osp_qk_norm_rope_bwd(void* g, int64_t g_stride, const void* y, int64_t y_stride, int64_t rows,
                         int64_t chan, int norm, const float* gamma_q, const float* gamma_k, float eps,
                         const float* rope_table, int64_t t, int64_t h, int64_t w, int64_t k,
                         int pattern, int64_t batch, int64_t row_offset, void* stream) {
  if (rows < 0 || chan <= 0 || !g) {
    set_error("qk norm/rope backward: bad sizes or null pointers");
    return kValue;
  }
  return launch_qk_norm_rope_bwd(g, g_stride, y, y_stride, rows, chan, norm, gamma_q, gamma_k, eps,
                                 rope_table, t, h, w, k, pattern, batch, row_offset, as_stream(stream));
}

int osp_debug_counters_bwd(uint64_t* host_out, int n, int reset) {
  return debug_counters_bwd(reinterpret_cast<unsigned long long*>(host_out), n, reset);
}

int osp_debug_counters(uint64_t* host_out, int n, int reset) {
  return debug_counters(reinterpret_cast<unsigned long long*>(host_out), n, reset);
}

int osp_debug_mma(const void* a, const void* b, const void* v, float* s_out, float* o_out,
                  int64_t head_dim, void* stream) {
  return launch_debug_mma(a, b, v, s_out, o_out, static_cast<int>(head_dim), as_stream(stream));
}

}  // extern "C"
