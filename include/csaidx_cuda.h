/*
 * csaidx_cuda.h — the C-ABI boundary of the B200 indexer (libcsaidx_cuda.so).
 *
 * Plain C: POD arguments, device or host pointers plus sizes, no C++ types,
 * no exceptions. Every entry point returns a status code; the C++ drop-in
 * layer (include/csaidx/ headers, libcsaidx.so) maps those codes 1:1 onto the
 * exception types the reference throws, and csaidx_cuda_last_error() returns
 * the (thread-local) message.
 *
 * The reference (proj/, CPU-only C++20) has no FFI of its own: its boundary
 * is the C++ API in proj/include/csaidx/. Each function below replaces one
 * step of that API's hot path; the comment on each cites the reference
 * interface it stands in for.
 *
 * Work is enqueued on the engine's stream (asynchronous) unless a function
 * says otherwise. Data-dependent failures (non-finite score, sentinel
 * contract) are latched in device flags and reported by
 * csaidx_engine_check(), which synchronizes.
 */
#ifndef CSAIDX_CUDA_H
#define CSAIDX_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; one per reference exception type (types.cpp, score.cpp,
 * topk.cpp, driver.cpp, memory_ledger.cpp). */
#define CSAIDX_OK 0
#define CSAIDX_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define CSAIDX_RUNTIME_ERROR 2    /* std::runtime_error    */
#define CSAIDX_OVERFLOW_ERROR 3   /* std::overflow_error   */
#define CSAIDX_LOGIC_ERROR 4      /* std::logic_error      */
#define CSAIDX_CUDA_ERROR 5       /* CUDA failure (mapped to runtime_error) */

/* Score kernel request, mirrors ScoreKernel (score.hpp:19-27). */
#define CSAIDX_KERNEL_AUTO 0   /* tcgen05 when the shape allows, else exact */
#define CSAIDX_KERNEL_EXACT 1  /* CUDA-core kernel in the reference op order */
#define CSAIDX_KERNEL_TENSOR 2 /* tcgen05 also for fp16_emulated: the reference's binary16 rounding points
                                  (score_scalar.cpp:29-32, half.cpp:84-91) applied to the MMA's dot
                                  products, so agreement is to binary16 rounding, not bit for bit */

/* AccumulationMode (score.hpp:11-17). */
#define CSAIDX_MODE_FP32 0
#define CSAIDX_MODE_FP16_EMULATED 1

/* ProblemDims (types.hpp:19-34). */
typedef struct csaidx_dims {
    int64_t batch;
    int64_t seq_len;
    int64_t key_blocks;
    int64_t heads;
    int64_t head_dim;
    int64_t ratio;
    int64_t top_k;
} csaidx_dims;

typedef struct csaidx_engine csaidx_engine;

const char* csaidx_cuda_last_error(void);
int csaidx_cuda_abi_version(void);
int csaidx_cuda_device_count(int* count);

/* Engine: device ordinal, stream, error flags, allocation accounting. */
int csaidx_engine_create(int device, csaidx_engine** out);
int csaidx_engine_destroy(csaidx_engine* e);
/* Enqueue on an external cudaStream_t (e.g. torch's current stream; NULL is
 * the legacy default stream). csaidx_engine_use_own_stream restores the
 * engine's private non-blocking stream (the default after create). */
int csaidx_engine_set_stream(csaidx_engine* e, void* stream);
int csaidx_engine_use_own_stream(csaidx_engine* e);
int csaidx_engine_get_stream(csaidx_engine* e, void** stream);
/* Lanes for overlapping host transfers and kernels: subsequent calls
 * enqueue on lane 0 (the main stream set above), 1 (copy-in), 2 (copy-out)
 * or 3 (a second compute stream). signal records event `slot` (0..191) on the current lane;
 * await makes the current lane wait for the slot's latest signal. */
int csaidx_engine_use_lane(csaidx_engine* e, int lane);
int csaidx_engine_signal(csaidx_engine* e, int slot);
int csaidx_engine_await(csaidx_engine* e, int slot);
/* Host-side wait for the slot's latest signal (e.g. before reusing a pinned
 * staging buffer whose copy was enqueued before the signal). */
int csaidx_engine_sync_slot(csaidx_engine* e, int slot);
/* A copy enqueued on an existing lane (1..3) without switching the current
 * lane, then (slot >= 0) the slot's event recorded after it on that lane.
 * For a second host thread feeding a lane while the calling thread drives
 * the engine (the host-rounding ring of csaidx_host_run_chunked_*); the two
 * threads must use disjoint slots. */
int csaidx_engine_copy_on_lane(csaidx_engine* e, int lane, int slot, void* dst, const void* src, size_t bytes);
/* The current lane waits (on the device) for all work enqueued so far on
 * `stream` (a cudaStream_t; NULL = the legacy default stream, which itself
 * orders after every blocking stream). The device-pointer driver entries
 * call it with NULL on entry, so operands produced on the default stream
 * need no host synchronisation before the call. */
int csaidx_engine_await_stream(csaidx_engine* e, void* stream);
/* Index sink: from now on every final output row written by
 * csaidx_cuda_select_final / csaidx_cuda_finalize for query position s of
 * batch b is also stored as int32 indices at dst[(b * seq_len + s) * k ..]
 * (a [batch, seq_len, k] buffer; a final launch whose batch count, k or
 * rows do not fit it fails with CSAIDX_INVALID_ARGUMENT). dst may be another GPU's memory mapped with
 * csaidx_cuda_ipc_open: then the final kernels of a query-sharded run write
 * their rows straight into the collecting rank over NVLink, fusing the
 * gather of the driver's result (reference run_chunked, driver.cpp:115-165,
 * assembles TopKResult rows; SURVEY §8e's gather) into the select.
 * NULL disables. */
int csaidx_engine_set_index_sink(csaidx_engine* e, int32_t* dst, int64_t batch, int64_t seq_len, int64_t k);
/* CUDA IPC of a device pointer for the index sink: a 64-byte handle of the
 * allocation that holds dev_ptr plus dev_ptr's offset inside it (caching
 * allocators hand out blocks inside larger allocations). open maps the
 * allocation in this process and returns the same byte; close takes the
 * pointer open returned and the same offset. */
int csaidx_cuda_ipc_handle(csaidx_engine* e, void* dev_ptr, void* handle, uint64_t* offset);
int csaidx_cuda_ipc_open(csaidx_engine* e, const void* handle, uint64_t offset, void** dev_ptr);
int csaidx_cuda_ipc_close(csaidx_engine* e, void* dev_ptr, uint64_t offset);
int csaidx_engine_num_sms(csaidx_engine* e, int* num_sms);
/* SM partition for running a select beside the score kernel: score launches
 * use at most score_sms CTAs (one per SM) and select launches run as
 * select_sms persistent CTAs of several rows each (one per SM). 0, 0 = the
 * whole GPU for every launch (the default). Results do not depend on it. */
int csaidx_engine_set_partition(csaidx_engine* e, int score_sms, int select_sms);
/* Synchronizes the stream, then reports (and clears) latched data errors. */
int csaidx_engine_check(csaidx_engine* e);
/* Synchronizes, then reports in *seen (and clears) whether a non-strict
 * csaidx_cuda_to_bf16 since the last call met a value bf16 cannot represent.
 * The host driver then re-runs on fp32 operands with the exact-order kernel,
 * so ScoreKernel::auto_detect gives the reference's scores on any fp32 input
 * (score.cpp:18-43 resolves auto to a kernel bit-identical to the scalar one). */
int csaidx_engine_take_inexact(csaidx_engine* e, int* seen);
/* Device bytes currently held / high-water through csaidx_cuda_alloc. */
int csaidx_engine_mem_stats(csaidx_engine* e, uint64_t* live, uint64_t* peak);
int csaidx_engine_reset_peak(csaidx_engine* e);

/* Kernel accounting: every launch is counted per class; with profiling on,
 * CUDA events on the launching stream bracket each launch and
 * csaidx_engine_kernel_stats resolves them into summed device milliseconds. */
#define CSAIDX_KIND_SCORE 0
#define CSAIDX_KIND_SELECT 1
#define CSAIDX_KIND_MERGE 2
#define CSAIDX_KIND_FINALIZE 3
#define CSAIDX_KIND_PREP 4
#define CSAIDX_KIND_ATTENTION 5
#define CSAIDX_NUM_KINDS 6
int csaidx_engine_set_profiling(csaidx_engine* e, int enabled);
int csaidx_engine_kernel_stats(csaidx_engine* e, int kind, int64_t* launches, double* total_ms);
int csaidx_engine_reset_stats(csaidx_engine* e);
/* Rows whose select took the exact global-memory fallback (the sampled
 * threshold mispredicted) since the last reset; synchronizes. */
int csaidx_engine_select_fallbacks(csaidx_engine* e, int64_t* rows, int reset);
/* Rows the select finished from a fused pre-filter candidate bitmap
 * (csaidx_cuda_select_from_candidates) since the last reset; synchronizes. */
int csaidx_engine_candidate_hits(csaidx_engine* e, int64_t* rows, int reset);
/* Profiling hook: when non-NULL, select launches of batch 0 write per-row
 * clock64 stamps [rows][8] = {start, threshold, filtered, sorted, n} into
 * this device buffer. */
int csaidx_engine_set_select_probe(csaidx_engine* e, long long* device_clocks);
/* Profiling hook: when non-NULL, tcgen05 score launches write per-CTA
 * clock64 wait counters [grid][8] = {MMA wait k_full, MMA wait acc_empty,
 * MMA wait q_full, MMA span, epilogue wait acc_full, epilogue span,
 * producer wait k_empty, producer wait q_empty} (grid = SM count). */
int csaidx_engine_set_score_probe(csaidx_engine* e, long long* device_counters);

/* Stream-ordered device memory from a cached pool. */
int csaidx_cuda_alloc(csaidx_engine* e, size_t bytes, void** ptr);
int csaidx_cuda_free(csaidx_engine* e, void* ptr);
int csaidx_cuda_copy(csaidx_engine* e, void* dst, const void* src, size_t bytes);
int csaidx_cuda_memset(csaidx_engine* e, void* dst, int value, size_t bytes);
/* Page-locked host staging memory (cudaHostAlloc) for asynchronous copies. */
int csaidx_cuda_host_alloc(csaidx_engine* e, size_t bytes, void** ptr);
int csaidx_cuda_host_free(csaidx_engine* e, void* ptr);
/* *pinned = 1 when ptr lies in page-locked host memory known to CUDA
 * (cudaHostAlloc / cudaHostRegister), else 0. */
int csaidx_cuda_host_is_pinned(const void* ptr, int* pinned);

/* fp32 -> bf16 (RNE) staging of q / kc (IndexerInputs::validated,
 * types.cpp:73-92: rejects non-finite; strict also rejects values that are
 * not bf16-representable, otherwise they are only noted for
 * csaidx_engine_take_inexact). src/dst are device pointers. */
int csaidx_cuda_to_bf16(csaidx_engine* e, const float* src, uint16_t* dst, int64_t n, int strict);

/* Operand element type of q / kc on device. */
#define CSAIDX_DTYPE_BF16 0 /* tcgen05 path (KERNEL_AUTO, fp32 mode, H_I=64, d_h=128) */
#define CSAIDX_DTYPE_F32 1  /* exact CUDA-core path only; bit-exact vs the CPU reference */

/* score_tile (score.hpp:61-64, score.cpp:54-101) on device operands:
 * out[b, i, j] for i < rows, j < cols, row stride ld (multiple of 4).
 * apply_mask folds mask_tile (causal.cpp:30-41) into the same pass and skips
 * key tiles that are causally dead for the whole query block. The tcgen05
 * kernel runs when kernel == AUTO, mode == FP32, dtype == BF16 and the shape
 * is the V4 indexer's; everything else runs the exact-order kernel. */
int csaidx_cuda_score(csaidx_engine* e, const void* q, const void* kc, int dtype, const float* w,
                      const csaidx_dims* dims, int64_t s0, int64_t rows, int64_t t0, int64_t cols,
                      int mode, int kernel, int apply_mask, float* out, int64_t ld);
/* Same tile over rank-local operands: q / w hold op_rows query rows per
 * batch ([B, op_rows, H_I, d_h] / [B, op_rows, H_I]) and query s0 + i lives
 * at operand row op_row0 + i. csaidx_cuda_score == op_rows = S,
 * op_row0 = s0. Lets a query-sharded rank keep only its own q / w rows. */
int csaidx_cuda_score_rows(csaidx_engine* e, const void* q, const void* kc, int dtype, const float* w,
                           const csaidx_dims* dims, int64_t s0, int64_t rows, int64_t t0, int64_t cols,
                           int mode, int kernel, int apply_mask, float* out, int64_t ld,
                           int64_t op_rows, int64_t op_row0);
/* csaidx_cuda_score_rows on the tcgen05 path that also writes, per row, the
 * maximum legal score of every 32-key group: gmax[(b * rows + i) * gmax_ld +
 * j / 32] (-inf when the group has no legal key; gmax_ld >= ceil(cols/32)).
 * A select given these maxima (csaidx_cuda_select_final's gmax) reads only
 * the groups that can hold a top-k score on long rows: two-level select. */
int csaidx_cuda_score_gmax(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                           const csaidx_dims* dims, int64_t s0, int64_t rows, int64_t t0, int64_t cols,
                           float* out, int64_t ld, int64_t op_rows, int64_t op_row0,
                           float* gmax, int64_t gmax_ld);
/* 1 when csaidx_cuda_score would take the tcgen05 path for these arguments. */
int csaidx_cuda_score_uses_tensor_cores(const csaidx_dims* dims, int dtype, int mode, int kernel);

/* build_mask_tile / apply_mask_tile (causal.cpp:43-79). */
int csaidx_cuda_bool_mask(csaidx_engine* e, uint8_t* keep, int64_t s0, int64_t t0, int64_t rows,
                          int64_t cols, int64_t ratio);
int csaidx_cuda_apply_bool_mask(csaidx_engine* e, float* scores, int64_t ld, const uint8_t* keep,
                                int64_t batch, int64_t rows, int64_t cols);

/* tile_topk (topk.hpp:71, topk.cpp:105-132): per (b, row) top-min(k, n)
 * under succ, n = legal columns (apply_mask) or cols; output rows of
 * width = min(k, cols) at stride cand_ld, indices offset by t0, padded with
 * (-inf, -1). Any k: takes up to csaidx_cuda_select_capacity() run in
 * shared memory (sampled threshold + bucket finish); larger takes run an
 * exact radix select + bitonic sort over global scratch owned by the engine
 * (the merge stages k > capacity rows in that scratch too). */
int csaidx_cuda_select(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows,
                       int64_t ld, int64_t cols, int64_t s0, int64_t t0, int64_t ratio,
                       int apply_mask, int64_t k, float* cand_val, int32_t* cand_idx,
                       int64_t cand_ld);
/* Sparse attention over the indexer's top-k (the CSA step
 * that consumes TopK(t), outside the reference's scope,
 * SPEC.md:8). For every (b, t) and head h:
 *   out[b,t,h,:dv] = sum_j softmax_j(sm_scale * q[b,t,h,:] . kv[b,i_j,:]) kv[b,i_j,:dv]
 *   lse[b,t,h]     = log sum_j exp(sm_scale * q[b,t,h,:] . kv[b,i_j,:])
 * over the entries i_j of indices[b,t,0:k] with 0 <= i_j < kv_len (others,
 * e.g. the -1 padding, are skipped; a row with none gets out = 0 and
 * lse = -inf). One shared latent KV head (MQA, the sparse-MLA layout):
 * q bf16 [B, S, heads, dqk], kv bf16 [B, kv_len, dqk], indices int32
 * [B, S, idx_ld], out bf16 [B, S, heads, dv] (rows of out_ld >= dv), lse
 * fp32 [B, S, heads] or NULL. Compiled shape: heads = a multiple of 128,
 * dqk = 576, dv = 512 (else CSAIDX_INVALID_ARGUMENT). tcgen05 kernel, one
 * work item per (query, group of 128 heads, half of dv). */
int csaidx_cuda_sparse_attention(csaidx_engine* e, const void* q_bf16, const void* kv_bf16,
                                 const int32_t* indices, int64_t batch, int64_t seq_len,
                                 int64_t kv_len, int64_t heads, int64_t dqk, int64_t dv, int64_t k,
                                 int64_t idx_ld, float sm_scale, void* out_bf16, int64_t out_ld,
                                 float* lse);
/* Largest take of the shared-memory select (4096). */
int csaidx_cuda_select_capacity(void);
/* 1 when the persistent multi-row select (csaidx_engine_set_partition) fits
 * shared memory for this k (k <= 1365 with 3 rows per CTA). */
int csaidx_cuda_select_overlap_capable(int64_t k);

/* Fused select pre-filter (an implementation of the same tile_topk
 * contract; results are identical to csaidx_cuda_select on every input):
 *   1. score_sampled scores every kt_stride-th 128-key tile of the masked
 *      tile into sample[b, i, 0..lds) (compacted columns, illegal = -inf);
 *   2. row_threshold turns each row's sample into a threshold tau[b*rows+i]
 *      chosen so that ~2k of the row's scores are expected to be >= tau
 *      (-inf when the legal row fits the candidate list outright);
 *   3. score_filtered is csaidx_cuda_score (apply_mask on) that also writes
 *      the candidate bitmap: bit (j % 32) of
 *      pass_bits[(b*rows + i) * bits_ld + j / 32] = (column j legal and
 *      score >= tau). Words of key tiles that are causally dead for the
 *      whole query block are left unwritten (no row reads them);
 *   4. select_from_candidates finishes each row from its flagged entries
 *      when min(k, n) <= flagged <= csaidx_cuda_candidate_capacity(k) (they
 *      then hold every score >= tau, hence the exact top) and streams the
 *      score row otherwise.
 * Tensor-core shape only (csaidx_cuda_score_uses_tensor_cores with BF16 /
 * FP32 / AUTO). bits_ld >= csaidx_cuda_candidate_words(cols). */
int csaidx_cuda_candidate_capacity(int64_t k);
int64_t csaidx_cuda_candidate_words(int64_t cols);
int csaidx_cuda_score_sampled(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                              const csaidx_dims* dims, int64_t s0, int64_t rows, int64_t t0, int64_t cols,
                              int kt_stride, float* sample, int64_t lds);
int csaidx_cuda_row_threshold(csaidx_engine* e, const float* sample, int64_t lds, int64_t batch, int64_t rows,
                              int64_t cols, int64_t s0, int64_t t0, int64_t ratio, int kt_stride, int64_t k,
                              float* tau);
int csaidx_cuda_score_filtered(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                               const csaidx_dims* dims, int64_t s0, int64_t rows, int64_t t0, int64_t cols,
                               float* out, int64_t ld, const float* tau, uint32_t* pass_bits, int64_t bits_ld);
int csaidx_cuda_select_from_candidates(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows,
                                       int64_t ld, int64_t cols, int64_t s0, int64_t t0, int64_t ratio, int64_t k,
                                       const uint32_t* pass_bits, int64_t bits_ld, float* out_val,
                                       int32_t* out_idx, int64_t out_ld);

/* tile_topk (topk.cpp:105-132) fused with the sentinel pass of
 * process_query_tile (driver.cpp:84-105), for query tiles whose single key
 * tile covers every key (t0 = 0, cols = T): with one tile the merge into the
 * all-sentinel TopKBuffer is a copy, so each row's exact top-min(k, n) goes
 * straight to out_idx/out_val[b, out_row0 + i, 0..k) (int64, fp32), sorted
 * under succ, the rest (-inf, -1). pass_bits: optional candidate bitmap of
 * csaidx_cuda_score_filtered (NULL = stream the scores); gmax: optional group
 * maxima of csaidx_cuda_score_gmax (NULL = one-level select). Replaces
 * select + finalize (two launches and the int32 run buffer round trip). */
int csaidx_cuda_select_final(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows,
                             int64_t ld, int64_t cols, int64_t s0, int64_t t0, int64_t ratio,
                             int64_t k, const uint32_t* pass_bits, int64_t bits_ld,
                             const float* gmax, int64_t gmax_ld,
                             int64_t* out_idx, float* out_val, int64_t out_rows, int64_t out_row0);

/* merge_topk / overwrite_topk (topk.hpp:73-82, topk.cpp:134-191) over nrows
 * running rows of k entries. check_overlap latches the reference's
 * overlapping-index error. */
int csaidx_cuda_merge(csaidx_engine* e, float* run_val, int32_t* run_idx, int64_t nrows, int64_t k,
                      const float* cand_val, const int32_t* cand_idx, int64_t cand_ld,
                      int64_t width, int overwrite, int check_overlap);

/* TopKBuffer initialisation (types.cpp:125-134): (-inf, -1). */
int csaidx_cuda_fill_sentinel(csaidx_engine* e, float* val, int32_t* idx, int64_t n);

/* Sentinel pass (driver.cpp:84-105) into int64/fp32 output rows
 * [b, out_row0 + i] of an [batch, out_rows, k] result. */
int csaidx_cuda_finalize(csaidx_engine* e, const float* run_val, const int32_t* run_idx,
                         int64_t batch, int64_t rows, int64_t s0, int64_t ratio, int64_t k,
                         int check_keff, int64_t* out_idx, float* out_val, int64_t out_rows,
                         int64_t out_row0);

/* One query chunk x one key tile of process_query_tile (driver.cpp:57-77):
 * masked score -> select -> merge (or copy when first_tile). score_buf must
 * hold batch*rows*ld floats, cand_* batch*rows*min(k, cols) entries. */
int csaidx_cuda_chunk_step(csaidx_engine* e, const void* q, const void* kc, int dtype,
                           const float* w, const csaidx_dims* dims, int64_t s0, int64_t rows,
                           int64_t t0, int64_t cols, int mode, int kernel, float* score_buf,
                           int64_t ld, float* cand_val, int32_t* cand_idx, float* run_val,
                           int32_t* run_idx, int first_tile, int overwrite);

/* Synthetic operand generator for large shapes (counter-based, same
 * distribution as synth.cpp:66-81, different stream). */
int csaidx_cuda_gen_normal_bf16(csaidx_engine* e, uint16_t* dst, int64_t n, double stddev,
                                uint64_t seed, uint64_t stream_id, int64_t offset);
int csaidx_cuda_gen_normal_f32(csaidx_engine* e, float* dst, int64_t n, double stddev,
                               uint64_t seed, uint64_t stream_id, int64_t offset);

/* ------------------------------------------------------------ multi-GPU
 * Transport of the query-sharded driver (csaidx_multi_*, csaidx_host.h): one
 * process per GPU; the driver broadcasts the keys, exchanges small host blobs
 * (the peer-sink IPC handle), synchronizes, and optionally gathers the int32
 * index rows. The reference parallelizes the same query-tile loop over host
 * threads (driver.cpp:131-161, DriverConfig::threads); its ranks are GPUs here.
 * All callbacks return CSAIDX_OK or an error code. */
typedef struct csaidx_collectives {
    void* ctx;
    int rank;
    int world;
    /* 1: bcast / gatherv take device pointers and are ordered on `stream`
     * (NCCL); 0: they take host pointers and complete before returning (the
     * driver stages device data through host memory around them). */
    int device_buffers;
    /* bytes at buf on rank `root` -> buf on every rank (in place) */
    int (*bcast)(void* ctx, void* buf, size_t bytes, int root, void* stream);
    /* every rank's `bytes` at in -> out[world * bytes] on every rank (host pointers) */
    int (*allgather_host)(void* ctx, const void* in, void* out, size_t bytes);
    /* returns on every rank once all ranks called it and the work queued on
     * `stream` (this rank's kernels, incl. their peer stores) has completed */
    int (*barrier)(void* ctx, void* stream);
    /* rank r's send_bytes at send -> root's recv + recv_off[r] (recv_bytes[r]
     * bytes; recv / recv_* only significant on root) */
    int (*gatherv)(void* ctx, const void* send, size_t send_bytes, void* recv, const size_t* recv_bytes,
                   const size_t* recv_off, int root, void* stream);
} csaidx_collectives;

/* NCCL transport (libnccl.so.2 resolved at run time with dlopen: the copy the
 * process already loaded, e.g. PyTorch's, or the system library). The
 * 128-byte unique id is created on one rank and handed to all others by the
 * caller (any out-of-band channel). ncclBroadcast / ncclAllGather /
 * ncclAllReduce / grouped ncclSend+ncclRecv on the caller's stream. */
int csaidx_nccl_unique_id(uint8_t id[128]);
int csaidx_nccl_collectives_create(int rank, int world, const uint8_t id[128], int device,
                                   csaidx_collectives** out);
int csaidx_nccl_collectives_destroy(csaidx_collectives* c);

/* int64 -> int32 index rows (indices < 2^31) and a row scatter: row r of
 * src (row_elems int32) -> dst + dst_row[r] * row_elems (dst_row on device). */
int csaidx_cuda_narrow_indices(csaidx_engine* e, const int64_t* src, int32_t* dst, int64_t n);
int csaidx_cuda_scatter_rows(csaidx_engine* e, const int32_t* src, int32_t* dst, const int64_t* dst_row,
                             int64_t nrows, int64_t row_elems);
/* Synchronizes the engine's current stream (no flag check). */
int csaidx_engine_sync(csaidx_engine* e);

#ifdef __cplusplus
}
#endif

#endif /* CSAIDX_CUDA_H */
