/*
 * osp_skiparse.h -- C ABI of the B200-native Skiparse-2D Attention hot path.
 *
 * The reference (arxiv 2605.28691 "OSP-Next", package `osp`, pure Python/numpy) has no FFI;
 * its hot-path entry points are Python functions.  Each function below is the device-side
 * replacement of one of them and cites the reference interface it replaces
 * (path:line under /root/reference/pkg/src/osp/).  The Python shim
 * `paper_2605_28691_b200` binds these with ctypes and keeps the reference names and
 * signatures.
 *
 * Conventions
 *   - All pointers are device pointers; buffers are caller-owned; nothing is allocated.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy default) and
 *     never synchronises the host.
 *   - Tensors are dense (batch, seq, chan) row-major unless a row stride (in elements) is
 *     given.  Rearranges move whole channel vectors of `chan * elem_bytes` bytes and are
 *     dtype-agnostic (1/2/4/8-byte elements, bit-exact).
 *   - Return value: OSP_OK or an OSP_E_* code; osp_last_error() gives a thread-local message.
 *     Codes map 1:1 onto the reference's exception classes.
 *   - Re-entrant; the only global state is a once-per-kernel shared-memory attribute.
 */
#ifndef OSP_SKIPARSE_H_
#define OSP_SKIPARSE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSP_ABI_VERSION 2

enum osp_status {
  OSP_OK = 0,
  OSP_E_PATTERN = 1,     /* skiparse.PatternError   skiparse.py:33-34 */
  OSP_E_SHAPE = 2,       /* gridseq.ShapeError      gridseq.py:37 */
  OSP_E_COORDINATE = 3,  /* gridseq.CoordinateError gridseq.py:33 */
  OSP_E_SHARDING = 4,    /* ssp.ShardingError       ssp.py:33 */
  OSP_E_COLLECTIVE = 5,  /* ssp.CollectiveError     ssp.py:37 */
  OSP_E_PROTOCOL = 6,    /* ssp.ProtocolError       ssp.py:41 */
  OSP_E_VALUE = 7,       /* ValueError (bad argument) */
  OSP_E_UNSUPPORTED = 8, /* dtype / head_dim outside the B200 kernels' support */
  OSP_E_CUDA = 9         /* CUDA runtime / driver failure -> RuntimeError */
};

/* Map ids: the six maps of skiparse.py:68-140 plus pad / strip (anyres.py:69-89). */
enum osp_map_id {
  OSP_MAP_IDENTITY = 0, /* IndexMap.identity            gridseq.py:192-195 */
  OSP_MAP_O2T = 1,      /* orig_to_tsa                  skiparse.py:68-77  */
  OSP_MAP_T2O = 2,      /* tsa_to_orig                  skiparse.py:80-88  */
  OSP_MAP_O2G = 3,      /* orig_to_gsa                  skiparse.py:91-102 */
  OSP_MAP_G2O = 4,      /* gsa_to_orig                  skiparse.py:105-114 */
  OSP_MAP_T2G = 5,      /* tsa_to_gsa                   skiparse.py:117-128 */
  OSP_MAP_G2T = 6,      /* gsa_to_tsa                   skiparse.py:131-140 */
  OSP_MAP_PAD = 7,      /* pad_tensor (zero pad)        anyres.py:69-82    */
  OSP_MAP_STRIP = 8     /* strip_padding                anyres.py:85-89    */
};

enum osp_pattern { OSP_PATTERN_ORIGINAL = 0, OSP_PATTERN_TSA = 1, OSP_PATTERN_GSA = 2 };

const char* osp_last_error(void);
int osp_abi_version(void);
/* OSP_OK iff the current device is a Blackwell sm_100 part the kernels were built for. */
int osp_device_check(void);

/*
 * K1: Skiparse Rearrange.  Replaces IndexMap.apply (gridseq.py:161-169) of the maps built by
 * skiparse.py:68-140 (and pad_tensor / strip_padding, anyres.py:69-89).
 * (t, h, w, k) is the PADDED grid.  h_orig/w_orig (<= h/w; 0 = same as h/w) are the original
 * extents: O2T/O2G then read the UNPADDED original tensor and write zero pad slots (fused
 * pad_tensor), T2O/G2O write the UNPADDED original tensor (fused strip_padding).
 * T2G/G2T/IDENTITY require h_orig == h, w_orig == w.
 * Divisibility is checked exactly as skiparse.py:53-65 (OSP_E_PATTERN).
 */
int osp_rearrange(const void* src, void* dst, int64_t elem_bytes, int64_t chan, int64_t batch,
                  int64_t t, int64_t h, int64_t w, int64_t k, int map_id, int64_t h_orig,
                  int64_t w_orig, void* stream);

/* Table-driven gather for arbitrary IndexMaps (gridseq.py:161-169):
 * dst[i] = src[index[i]] over rows of row_bytes; index entries outside [0, n_in_rows) give
 * zero rows (the Python shim validates tables as gridseq.py:140-150 does). */
int osp_gather_rows(const void* src, void* dst, const int64_t* index, int64_t n_out_rows,
                    int64_t n_in_rows, int64_t row_bytes, void* stream);

/*
 * Table gather over channel-chunked layouts (bytes strides): for every output row r and chunk
 * c < n_chunks, chunk_bytes are copied from src + c*src_chunk_stride + index[r]*src_row_stride to
 * dst + c*dst_chunk_stride + r*dst_row_stride (index[r] < 0 or >= n_in_rows: zeros).  The SSP
 * switch's local step when its all-to-all runs per head chunk overlapped with attention
 * (ssp.py:166-178 unpack, composed with the block's compaction; and the pack of a gradient into
 * per-chunk send blocks); the channel-split identity (pkg/tests/test_ssp.py:167-178) makes the
 * chunked switch equal the whole one.
 */
int osp_gather_rows_chunked(const void* src, void* dst, const int64_t* index, int64_t n_out_rows,
                            int64_t n_in_rows, int64_t n_chunks, int64_t chunk_bytes,
                            int64_t src_row_stride, int64_t src_chunk_stride, int64_t dst_row_stride,
                            int64_t dst_chunk_stride, void* stream);
/* IndexMap.invert (gridseq.py:179-185): inv[index[i]] = i. */
int osp_invert_index(const int64_t* index, int64_t* inv, int64_t n, void* stream);

/*
 * K5: 1-D validity masks as bit words, bits[row * ceil(L/32) + pos/32] bit (pos%32).
 * osp_pattern_mask_bits: subsequence_mask (anyres.py:92-96) for `batch` items in the enlarged
 * batch order (pattern id, batch item) of attention.py:121-125; pattern ORIGINAL gives the
 * flat padded-grid mask (anyres.py:61-64) per batch item.  (t,h,w,k) padded, h_orig/w_orig
 * original extents.
 */
int osp_pattern_mask_bits(uint32_t* bits, int64_t batch, int64_t t, int64_t h, int64_t w,
                          int64_t k, int pattern, int64_t h_orig, int64_t w_orig, void* stream);
int osp_mask_bytes_to_bits(const uint8_t* valid, uint32_t* bits, int64_t n_rows, int64_t len,
                           void* stream);
int osp_mask_bits_to_bytes(const uint32_t* bits, uint8_t* valid, int64_t n_rows, int64_t len,
                           void* stream);

/*
 * K2: per-subsequence attention forward.  Replaces dense_attention (attention.py:47-67) as
 * called per subsequence by skiparse_attention (attention.py:126-130), extended to `heads`
 * heads of `head_dim` channels each (head_dim in {64, 128}; bf16 in/out, fp32 accumulate).
 *   q,k,v,o : (n_seq, seq_len, >= heads*head_dim) bf16 with row strides q_stride.. (elements)
 *   lse     : (n_seq, heads, seq_len) fp32 natural-log softmax normaliser; +inf for rows with
 *             no valid key or (zero_invalid_queries) an invalid query.
 *   valid_bits: NULL or (n_seq, ceil(seq_len/32)) key validity (attention.py:35-44 rules:
 *             masked keys weigh 0, an all-masked row outputs 0).
 *   seq_lens: NULL or (n_seq) int32 per-sequence lengths <= seq_len: sequence s uses only its
 *             first seq_lens[s] rows as queries and keys; its rows beyond get o = 0, lse = +inf.
 *             This runs subsequences with their padding compacted away.
 *   zero_invalid_queries: rows whose own bit is 0 output 0 (attention.py:127-130).
 *   scale   : softmax scale (reference: 1/sqrt(chan) with one head, attention.py:57).
 */
int osp_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int64_t n_seq,
                 int64_t seq_len, int64_t heads, int64_t head_dim, int64_t q_stride,
                 int64_t k_stride, int64_t v_stride, int64_t o_stride, const uint32_t* valid_bits,
                 const int32_t* seq_lens, int zero_invalid_queries, float scale, void* stream);

/*
 * K3: backward of osp_attn_fwd (no reference counterpart: attention.py has no backward).
 * Writes dq, dk, dv (bf16, own row strides; with seq_lens, rows beyond a sequence's length are
 * 0).  workspace >= osp_attn_bwd_workspace_bytes().
 */
size_t osp_attn_bwd_workspace_bytes(int64_t n_seq, int64_t seq_len, int64_t heads,
                                    int64_t head_dim);
int osp_attn_bwd(const void* q, const void* k, const void* v, const void* o, const void* dout,
                 const float* lse, void* dq, void* dk, void* dv, int64_t n_seq, int64_t seq_len,
                 int64_t heads, int64_t head_dim, int64_t q_stride, int64_t k_stride,
                 int64_t v_stride, int64_t o_stride, int64_t do_stride, int64_t dq_stride,
                 int64_t dk_stride, int64_t dv_stride, const uint32_t* valid_bits,
                 const int32_t* seq_lens, int zero_invalid_queries, float scale, void* workspace,
                 size_t workspace_bytes, void* stream);

/*
 * K2/K3 with the Skiparse Rearrange fused into the TMA prologue / epilogue (gather mode): q, k,
 * v, o, dout, dq, dk, dv are (n_rows, >= heads*head_dim) row-strided tensors in ANY token layout
 * (e.g. the original, unpadded latent); sequence s (a subsequence of a pattern) consists of rows
 * row_index[s*capacity + j], j < seq_lens[s] (entries beyond are -1).  Q/K/V/dO tiles are fetched
 * with tile::gather4 TMA loads and O, dK, dV, dQ rows are stored through the same table, so no
 * rearranged copy of the activations ever lands in HBM.  lse is (n_seq, heads, capacity) in
 * sequence order.  capacity % 4 == 0; the backward needs head_dim 128.
 */
int osp_attn_fwd_gather(const void* q, const void* k, const void* v, void* o, float* lse,
                        int64_t n_rows, const int32_t* row_index, const int32_t* seq_lens,
                        int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                        int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                        float scale, void* stream);
int osp_attn_bwd_gather(const void* q, const void* k, const void* v, const void* o,
                        const void* dout, const float* lse, void* dq, void* dk, void* dv,
                        int64_t n_rows, const int32_t* row_index, const int32_t* seq_lens,
                        int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                        int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t o_stride,
                        int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                        float scale, void* workspace, size_t workspace_bytes, void* stream);

/*
 * K2/K3 with the Skiparse Rearrange fused into the output side (scatter mode), the production
 * single-GPU block path.  q, k, v are contiguous per-sequence tiles as in osp_attn_fwd (each
 * operand tile is re-read by many CTAs, so the loads stay plain TMA tiles), but output row j of
 * sequence s is STORED to row out_index[s*capacity + j] of `out` (n_out_rows x >= heads*head_dim,
 * row stride out_stride; -1 = not stored): the attention epilogue itself performs the pattern
 * switch / padding expansion that follows attention (reference attention.py:131 and the block's
 * tsa_to_gsa / gsa_to_tsa, skiparse.py:117-140), so no permuted copy is written by a separate
 * pass.  zero_rows lists the n_zero_rows rows of `out` no sequence row lands on (pad tokens of
 * the destination layout); the forward zero-fills them.  lse is (n_seq, heads, capacity).
 * The backward reads O and dO through the same table: its Delta pre-pass (which reads both rows
 * anyway) gathers dO into a contiguous operand image inside the workspace
 * (>= osp_attn_bwd_scatter_workspace_bytes), and dq, dk, dv are written contiguously.
 * Replaces: attention.py:119-131 (gather -> dense_attention -> zero pads -> inverse gather).
 */
int osp_attn_fwd_scatter(const void* q, const void* k, const void* v, void* out, float* lse,
                         int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                         int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t out_stride,
                         const int32_t* seq_lens, const int32_t* out_index, int64_t n_out_rows,
                         const int32_t* zero_rows, int64_t n_zero_rows, float scale, void* stream);
size_t osp_attn_bwd_scatter_workspace_bytes(int64_t n_seq, int64_t capacity, int64_t heads,
                                            int64_t head_dim);
int osp_attn_bwd_scatter(const void* q, const void* k, const void* v, const void* out,
                         const void* dout, const float* lse, void* dq, void* dk, void* dv,
                         int64_t n_seq, int64_t capacity, int64_t heads, int64_t head_dim,
                         int64_t q_stride, int64_t k_stride, int64_t v_stride, int64_t out_stride,
                         int64_t do_stride, int64_t dq_stride, int64_t dk_stride, int64_t dv_stride,
                         const int32_t* seq_lens, const int32_t* out_index, int64_t n_out_rows,
                         float scale, void* workspace, size_t workspace_bytes, void* stream);

/*
 * K4: Sparse Sequence Parallel pattern switch, local steps of ssp_pattern_switch
 * (ssp.py:139-180; Alg. 1).  One rank's shard is (local_batch, L, chan) with
 * L = t*h*w/k^2, local_batch = G*b, G = k^2/group_size; (t,h,w,k) the padded global grid.
 *   osp_ssp_pack:   step 1 (ssp.py:166): orig_to_tsa on the reduced grid (t, h/k, w/k) with
 *                   batch G*b -> send buffer (k^2*G*b, L/k^2, chan) = group_size equal chunks.
 *   osp_ssp_unpack: steps 3+4 (ssp.py:172-178): view the received buffer as
 *                   (N, G, G, b, L/k^2, chan), swap axes 1 and 2, tsa_to_orig on the reduced
 *                   grid -> (G*b, L, chan) in the switched pattern layout.
 * Step 2 is one all-to-all of equal chunks (ssp.py:168), done by NCCL between the two.
 * Errors: OSP_E_SHARDING (k^2 % group_size), OSP_E_PROTOCOL (local_batch % G), as ssp.py:145-160.
 */
int osp_ssp_pack(const void* src, void* dst, int64_t elem_bytes, int64_t chan,
                 int64_t group_size, int64_t local_batch, int64_t t, int64_t h, int64_t w,
                 int64_t k, void* stream);
int osp_ssp_unpack(const void* recv, void* dst, int64_t elem_bytes, int64_t chan,
                   int64_t group_size, int64_t local_batch, int64_t t, int64_t h, int64_t w,
                   int64_t k, void* stream);

/*
 * HiF8 codec: replaces hif8.py encode_array / decode_array
 * (hif8.py:171-193) and the amax / scale of quantize_tensor (hif8.py:223-246).
 * dtype: 0 = bf16, 1 = fp32, 2 = fp64.  `table` = device pointer to the 256 ascending values
 * (code 127 = 0).  `scale` (device, nullable = 1.0): element i uses scale[i / scale_group]
 * (scale_group 0 = one scale).  encode stores code(x * scale) -- nearest value, ties to the
 * even code, saturating; fp64 inputs are scaled and compared in fp64 (bit-exact with the
 * reference), bf16/fp32 in fp32.  Non-finite inputs set *nonfinite_flag (device, nullable)
 * and encode as code 0 (the reference raises EncodeError, hif8.py:174-175).
 * decode stores table[code] / scale.  osp_absmax: *amax = max |x| (device, NaN propagates).
 * osp_hif8_scale: scale[i] = target / (amax[i] + eps).
 */
int osp_absmax(const void* x, int dtype, int64_t n, double* amax, void* stream);
int osp_hif8_scale(const double* amax, int64_t count, double target, double eps, double* scale,
                   void* stream);
int osp_hif8_encode(const void* x, int dtype, int64_t n, const double* scale,
                    int64_t scale_group, const double* table, uint8_t* codes, int* nonfinite_flag,
                    void* stream);
int osp_hif8_decode(const uint8_t* codes, int64_t n, const double* scale, int64_t scale_group,
                    const double* table, void* out, int dtype, void* stream);

/*
 * K6: QKV projection with the QK-RMSNorm + 3-D RoPE prologue; with
 * norm = 0 and rope_table = NULL it is the reference's fixed projection (attention.py:20-32).
 *   x     : (rows, chan) bf16, rows in the pattern layout `pattern` (0 original, 1 TSA, 2 GSA)
 *           of `batch` items on the padded grid (t, h, w, k)
 *   w_t   : (3*chan, chan) bf16 = [Wq | Wk | Wv]^T (K-major)
 *   out   : (rows, >= 3*chan) bf16 q | k | v, row stride out_stride (elements)
 *   norm  : 0 none; 1 RMSNorm over each 128-channel head of q and k; 2 RMSNorm of q and k over
 *           all chan channels (needs sumsq, (rows, 2) fp32 workspace); gamma_q / gamma_k (chan)
 *           fp32 or NULL (= 1)
 *   rope_table: NULL or (t + h + w, 32) float2 (cos, sin) per axis position and pair; head pairs
 *           (2i, 2i+1) split over (t, h, w) as 22 / 21 / 21 (Wan 3-D RoPE for head_dim 128)
 *   row_offset: pattern-layout row of x's first row (an SSP shard starts mid-layout)
 * head_dim is 128 (chan % 128 == 0).
 */
int osp_qkv_project(const void* x, const void* w_t, void* out, int64_t rows, int64_t chan,
                    int64_t out_stride, int norm, const float* gamma_q, const float* gamma_k,
                    float eps, float* sumsq, const float* rope_table, int64_t t, int64_t h,
                    int64_t w, int64_t k, int pattern, int64_t batch, int64_t row_offset,
                    void* stream);
/*
 * Backward of osp_qkv_project's q/k epilogue, IN PLACE on g (rows x >= 2*chan bf16, the gradient
 * of the normalised + rotated q | k): transpose of the RoPE rotation, then (norm 1 / 2) the
 * RMSNorm backward r*gamma*g - y*r^3*mean(gamma*g*y) per head / per row, y being the pre-norm
 * GEMM output (rows x >= 2*chan bf16; may be NULL with norm 0).  Same grid / pattern / row_offset
 * arguments as the forward.  No reference counterpart (SURVEY.md sec. 8f row 2 is beyond
 * attention.py:20-32).
 */
int osp_qk_norm_rope_bwd(void* g, int64_t g_stride, const void* y, int64_t y_stride, int64_t rows,
                         int64_t chan, int norm, const float* gamma_q, const float* gamma_k, float eps,
                         const float* rope_table, int64_t t, int64_t h, int64_t w, int64_t k,
                         int pattern, int64_t batch, int64_t row_offset, void* stream);

/*
 * K7: the SSP pattern switch as one pull over peer memory (replaces pack -> all_to_all -> unpack,
 * ssp.py:156-178, for the block's switches).
 *   osp_peer_alloc / osp_peer_free: a zeroed cudaMalloc buffer that can be exported over CUDA IPC.
 *   osp_peer_export: its 64-byte cudaIpcMemHandle; osp_peer_import opens a peer's handle
 *                    (lazy peer access), osp_peer_close releases it.
 *   osp_peer_barrier: flag_blocks = host array of n device pointers, rank j's uint32[n] flag
 *                    block; publishes `epoch` to slot `rank` of every block and waits until every
 *                    slot of this rank's block reached it (epochs increase by one per barrier).
 *                    timeout_ms > 0 bounds the wait: a rank that never arrives makes the kernel
 *                    write (1 + that rank) into *status (host-mapped pinned memory, first
 *                    timeout wins) and EXIT instead of trapping, so the context survives and the
 *                    host raises CollectiveError when it reads the word (status may be NULL:
 *                    then the kernel just exits).
 *   osp_peer_gather: dst[i] = row (table[i] % stride_rows) of srcs[table[i] / stride_rows]
 *                    (srcs = host array of n_src device pointers, local or peer-mapped);
 *                    table[i] < 0 gives a zero row.  table is a device int64 array of n_rows.
 */
int osp_peer_alloc(int64_t bytes, void** ptr);
int osp_peer_free(void* ptr);
int osp_peer_export(void* ptr, uint8_t* handle64);
int osp_peer_import(const uint8_t* handle64, void** ptr);
int osp_peer_close(void* ptr);
int osp_peer_barrier(const void* const* flag_blocks, int rank, int n, uint32_t epoch,
                     int64_t timeout_ms, int* status, void* stream);
int osp_peer_gather(const void* const* srcs, int n_src, int64_t stride_rows, const int64_t* table,
                    int64_t n_rows, void* dst, int64_t row_bytes, void* stream);

/* Profiling counters of instrumented builds (-DOSP_FWD_TIMING=1): copies n <= 64 uint64 into
 * host_out (zeros in normal builds) and optionally resets them.  Not part of the hot path. */
int osp_debug_counters(uint64_t* host_out, int n, int reset);
/* The same for the K3 backward's phase counters (OSP_BWD_TIMING=1 builds). */
int osp_debug_counters_bwd(uint64_t* host_out, int n, int reset);

/* Self-test of the tcgen05 instruction forms (S = A B^T, O = bf16(S) V for one 128-row tile). */
int osp_debug_mma(const void* a, const void* b, const void* v, float* s_out, float* o_out,
                  int64_t head_dim, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OSP_SKIPARSE_H_ */
