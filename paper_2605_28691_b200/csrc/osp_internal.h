// Internal (non-ABI) declarations shared by the .cu translation units.
#pragma once

#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

namespace osp {

// Integer tuning / experiment switch from the environment (read by the callers into function-local
// statics, i.e. once per process); dflt when unset.
inline int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Thread-local error message backing osp_last_error().
void set_error(const std::string& msg);

// Status codes (mirror include/osp_skiparse.h).
enum Status : int {
  kOk = 0,
  kPattern = 1,
  kShape = 2,
  kCoordinate = 3,
  kSharding = 4,
  kCollective = 5,
  kProtocol = 6,
  kValue = 7,
  kUnsupported = 8,
  kCuda = 9,
};

int check_cuda(cudaError_t e, const char* what);

// Raise a kernel's dynamic shared-memory limit on the CURRENT device, once per (kernel, device).
// The attribute is per device context, so a process that drives several GPUs (the survey's
// single-process multi-device path) must set it on each; `done` is the call site's per-device
// bitmask (one bit per device ordinal < 64).  Concurrent first calls may both set the attribute,
// which is idempotent.
int set_smem_attr(const void* kernel, int bytes, std::atomic<uint64_t>& done, const char* what);

// Build a 3-D bf16 TMA descriptor over a (n_seq, rows, cols) row-strided matrix with a
// (64 x box_rows x 1) box and 128-byte swizzle.
int make_tmap_bf16_3d(CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                      int64_t n_seq, int64_t row_stride_elems, int box_rows);

// 2-D bf16 TMA descriptor over a (rows, cols) row-strided matrix with a (64 x box_rows) box and
// 128-byte swizzle (box_rows = 1 for tile::gather4 row gathers).
int make_tmap_bf16_2d(CUtensorMap* map, const void* base, int64_t cols, int64_t rows,
                      int64_t row_stride_elems, int box_rows);

// Closed-form row map of the rearrange engine (rearrange.cu).
struct MapParams {
  int kind;
  int64_t B;              // batch items (for SSP: local batch G*b)
  int64_t T, H, W, k;     // padded grid (for SSP: the global padded grid)
  int64_t H0, W0;         // original extents (== H, W when no padding)
  int64_t G, bsub;        // SSP: subsequences per rank, batch items per subsequence group
  const int64_t* table;   // kTable
  int64_t n_in_rows;      // kTable bound
};

struct AttnShape {
  int64_t n_seq, seq_len, heads, head_dim;  // seq_len = capacity (row stride of a sequence)
  const int32_t* seq_lens = nullptr;         // optional per-sequence valid lengths (<= seq_len)
  // gather mode: q/k/v/o/dO/dq/dk/dv are (n_rows, >= heads*head_dim) tensors in any token
  // layout; row j of sequence s is row row_index[s * seq_len + j] (-1 = none)
  const int32_t* row_index = nullptr;
  int64_t n_rows = 0;
  // scatter mode (operands contiguous, output through a row table): o row j of sequence s is row
  // out_index[s * seq_len + j] of an (n_out_rows, >= heads*head_dim) tensor (-1 = not stored),
  // zero_rows the rows of that tensor no sequence row lands on (zero-filled by the forward).  The
  // backward reads O and dO through the same table; its prologue writes the contiguous dO operand
  // image do_image (n_seq, seq_len, heads*head_dim) on the way.
  const int32_t* out_index = nullptr;
  const int32_t* zero_rows = nullptr;
  int64_t n_zero = 0;
  void* do_image = nullptr;
};

int launch_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                    const AttnShape& s, int64_t q_stride, int64_t k_stride, int64_t v_stride,
                    int64_t o_stride, const uint32_t* valid_bits, int zero_invalid_queries,
                    float scale, cudaStream_t stream);

int launch_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                    const float* lse, void* dq, void* dk, void* dv, const AttnShape& s,
                    int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                    int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                    const uint32_t* valid_bits, int zero_invalid_queries, float scale,
                    void* workspace, size_t workspace_bytes, cudaStream_t stream);
size_t attn_bwd_workspace_bytes(const AttnShape& s);

int launch_qkv_project(const void* x, const void* w_t, void* out, int64_t rows, int64_t chan,
                       int64_t out_stride, int norm, const float* gamma_q, const float* gamma_k,
                       float eps, float* sumsq, const float* rope_table, int64_t t, int64_t h,
                       int64_t w, int64_t k, int pattern, int64_t batch, int64_t row_offset,
                       cudaStream_t stream);
int launch_qk_norm_rope_bwd(void* g, int64_t g_stride, const void* y, int64_t y_stride, int64_t rows,
                            int64_t chan, int norm, const float* gamma_q, const float* gamma_k, float eps,
                            const float* rope_table, int64_t t, int64_t h, int64_t w, int64_t k, int pattern,
                            int64_t batch, int64_t row_offset, cudaStream_t stream);

int launch_debug_mma(const void* a, const void* b, const void* v, float* s_out, float* o_out,
                     int d, cudaStream_t stream);

}  // namespace osp
