/*
 * csaidx_host.h — C entry points of libcsaidx.so, the drop-in C++ driver.
 *
 * The reference-facing call with HOST buffers (what a ctypes / cgo / JNI
 * binding of the reference's run_chunked / run_materialize / dispatch would
 * bind; proj/include/csaidx/driver.hpp:64-89), plus the device-resident
 * chunk scheduler used for multi-GPU sharding. Same status codes as
 * csaidx_cuda.h; csaidx_host_last_error() holds the exception message.
 */
#ifndef CSAIDX_HOST_H
#define CSAIDX_HOST_H

#include <stdint.h>

#include "csaidx_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Ablation (driver.hpp:11-20) */
#define CSAIDX_ABLATION_NONE 0
#define CSAIDX_ABLATION_A1_NO_MERGE 1
#define CSAIDX_ABLATION_A2_SKIP_NARROW 2

/* ScoreKernel (score.hpp:19-27) */
#define CSAIDX_SCORE_AUTO 0
#define CSAIDX_SCORE_SCALAR 1
#define CSAIDX_SCORE_AVX2 2

/* DriverConfig (driver.hpp:25-48) + gpu::Options. */
typedef struct csaidx_run_config {
    int64_t query_tile;            /* c_S */
    int64_t key_tile;              /* c_T */
    int mode;                      /* CSAIDX_MODE_* */
    int ablation;                  /* CSAIDX_ABLATION_* */
    int kernel;                    /* CSAIDX_SCORE_* */
    int causal_early_exit;
    int bool_mask_tile;
    int threads;
    uint64_t auto_threshold_bytes;
    int device;
    int strict_bf16;
    void* stream;                  /* cudaStream_t or NULL (engine stream) */
    int fp16_tensor_cores;         /* gpu::Options::fp16_tensor_cores */
} csaidx_run_config;

/* RunStats (driver.hpp:55-59) + the path taken and both peaks. */
typedef struct csaidx_run_stats {
    int64_t dispatch_count;
    int64_t tiles_skipped_masked;
    int64_t tiles_skipped_narrow;
    uint64_t ledger_peak_bytes;
    uint64_t device_peak_bytes;
    int path; /* 0 materialize, 1 chunked */
} csaidx_run_stats;

const char* csaidx_host_last_error(void);
void csaidx_host_default_config(csaidx_run_config* cfg);
/* The engine the driver uses for `device` (for profiling / memory stats). */
int csaidx_host_engine(int device, csaidx_engine** out);

/* run_chunked / run_materialize / dispatch on host fp32 buffers
 * q [B,S,H,D], kc [B,T,D], w [B,S,H]; results into host [B,S,k]. */
int csaidx_host_run_chunked(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                            const csaidx_run_config* cfg, int64_t* out_idx, float* out_val,
                            csaidx_run_stats* stats);
int csaidx_host_run_materialize(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                const csaidx_run_config* cfg, int64_t* out_idx, float* out_val,
                                csaidx_run_stats* stats);
int csaidx_host_dispatch(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                         const csaidx_run_config* cfg, int64_t* out_idx, float* out_val,
                         csaidx_run_stats* stats);

/* run_chunked on host buffers for a subset of query chunks (starts must be
 * multiples of the clamped c_S; NULL / 0 = all): only those q / w rows
 * cross PCIe; results packed into host [B, out_rows, k]. The per-rank entry
 * of a query-sharded multi-GPU run. */
int csaidx_host_run_chunked_rows(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                 const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                                 int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats);

/* Same with rank-local host operands: q / w hold only the listed chunks'
 * rows, stacked in list order like the outputs ([B, out_rows, H_I, d_h],
 * [B, out_rows, H_I]); kc is the full [B, T, d_h]. */
int csaidx_host_run_chunked_local(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                  const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                                  int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats);

/* Algorithm 2 over device-resident operands (dtype CSAIDX_DTYPE_*), for the
 * listed query chunks (NULL / 0 = all), outputs device [B, out_rows, k]. */
int csaidx_device_run_chunked(const void* q, const void* kc, int dtype, const float* w,
                              const csaidx_dims* dims, const csaidx_run_config* cfg,
                              const int64_t* chunk_starts, int64_t n_chunks, int64_t* out_idx,
                              float* out_val, int64_t out_rows, csaidx_run_stats* stats);

/* Same over rank-local operands: q / w hold only the listed chunks' rows,
 * stacked in list order like the outputs ([B, out_rows, H_I, d_h] and
 * [B, out_rows, H_I]); kc is the full [B, T, d_h]. A query-sharded rank's
 * HBM then scales with its share of S. */
int csaidx_device_run_chunked_local(const void* q, const void* kc, int dtype, const float* w,
                                    const csaidx_dims* dims, const csaidx_run_config* cfg,
                                    const int64_t* chunk_starts, int64_t n_chunks, int64_t* out_idx,
                                    float* out_val, int64_t out_rows, csaidx_run_stats* stats);

/* CSAT input dump (tensor_io.hpp:10-41, tensor_io.cpp:28-140). */
typedef struct csaidx_section_info {
    uint8_t tag;      /* 0 q, 1 kc, 2 w */
    uint8_t rank;
    uint32_t dims[4];
    uint64_t elems;
    uint64_t offset;  /* payload byte offset in the file */
} csaidx_section_info;
/* write_inputs_file: q / kc / w host fp32 arrays of `dims`. */
int csaidx_host_write_inputs_file(const char* path, const float* q, const float* kc, const float* w,
                                  const csaidx_dims* dims, uint64_t* bytes);
/* Header scan (read_sections' checks and error messages, without loading
 * payloads): up to max_sections infos, *n_sections = sections in the file. */
int csaidx_host_scan_sections(const char* path, csaidx_section_info* out, int max_sections, int* n_sections);
/* read_sections + shape check against dims into host fp32 arrays. */
int csaidx_host_read_inputs(const char* path, const csaidx_dims* dims, float* q, float* kc, float* w);
/* CSAT dump -> device buffers (gpu.hpp load_inputs_device): q / kc as dtype
 * (CSAIDX_DTYPE_BF16 rounds on device; strict rejects non-representable),
 * w fp32; only the listed query chunks' q / w rows (NULL / 0 = all), stacked
 * in list order ([B, out_rows, ...]), for the *_run_chunked_local entries. */
int csaidx_host_load_inputs_device(const char* path, const csaidx_dims* dims, int64_t query_tile,
                                   const int64_t* chunk_starts, int64_t n_chunks, int dtype, int strict,
                                   int device, void* q, void* kc, float* w);

/* Pure host arithmetic of the API (types.cpp / driver.cpp), no GPU needed. */
int csaidx_host_problem_dims(int64_t batch, int64_t seq_len, int64_t ratio, int64_t heads,
                             int64_t head_dim, int64_t top_k, csaidx_dims* out);
int csaidx_host_dispatch_count_model(const csaidx_dims* dims, int64_t query_tile, int64_t key_tile,
                                     int64_t* out);
int csaidx_host_chunked_peak_model_bytes(int64_t batch, int64_t query_tile, int64_t key_tile,
                                         int64_t top_k, int bool_mask_tile, uint64_t* out);
int csaidx_host_materialize_bytes(const csaidx_dims* dims, uint64_t* out);
int csaidx_host_choose_path(const csaidx_dims* dims, uint64_t threshold, int* path,
                            uint64_t* predicted);
int64_t csaidx_host_t_legal(int64_t t, int64_t ratio);
int64_t csaidx_host_k_eff(int64_t t, int64_t ratio, int64_t top_k);
/* The host rounding of the pipelined entry (csaidx_host_run_chunked*):
 * fp32 -> bf16, round to nearest even (bit-identical to the device's
 * csaidx_cuda_to_bf16 for finite inputs), on the host worker pool
 * (CSAIDX_HOST_THREADS). Flags: any non-finite entry / any entry that is not
 * bf16-representable (the checks of IndexerInputs::validated,
 * types.cpp:73-92, and of strict mode). */
int csaidx_host_round_bf16(const float* src, uint16_t* dst, uint64_t n, int* nonfinite, int* inexact);

/* Host <-> device bytes the calling thread's last host-buffer chunked call
 * moved (inputs in, index / value rows out) and how many of its query chunks
 * crossed PCIe as fp32 rather than host-rounded bf16. */
int csaidx_host_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes, int64_t* fp32_chunks, int64_t* chunks);

/* ------------------------------------------------------------ multi-GPU
 * The query-sharded driver (csaidx::gpu::MultiRank, include/csaidx/gpu.hpp):
 * one process per GPU over a csaidx_collectives transport (NCCL:
 * csaidx_nccl_collectives_create, or the caller's own). Replaces the
 * reference's threaded run_chunked (driver.cpp:115-165, DriverConfig::threads)
 * for ranks = GPUs. */
#define CSAIDX_GATHER_PEER 0       /* final kernels store rows into rank 0's buffer over a CUDA IPC mapping */
#define CSAIDX_GATHER_COLLECTIVE 1 /* rows gathered after the compute (transport gatherv) */

/* LPT plan: rank's ascending chunk starts (up to cap) and their count; loads
 * (optional, [world]) = per-rank causal pairs per batch. */
int csaidx_host_plan_shards(const csaidx_dims* dims, int64_t query_tile, int world, int rank, int64_t* starts,
                            int64_t cap, int64_t* n_chunks, uint64_t* loads);

typedef struct csaidx_multi csaidx_multi;
/* root_out: rank 0's device [B, S, k] int32 result (NULL elsewhere). Sets up
 * the plan and, for the peer gather, maps rank 0's buffer on every rank. */
int csaidx_multi_create(const csaidx_collectives* comm, const csaidx_dims* dims, const csaidx_run_config* cfg,
                        int gather_mode, int32_t* root_out, csaidx_multi** out);
/* This rank's chunk starts (valid until destroy) and rows per batch. */
int csaidx_multi_chunks(const csaidx_multi* m, const int64_t** starts, int64_t* n_chunks, int64_t* rows);
/* One step: q / w this rank's rows (chunks order, [B, rows, ...]); kc
 * [B, T, d_h] read on rank 0 and broadcast into kc elsewhere; local_idx /
 * local_val this rank's [B, rows, k] outputs, or both NULL (peer gather:
 * rank 0's int32 rows are then the only output). Returns when rank 0's
 * root_out holds every rank's rows. */
int csaidx_multi_run(csaidx_multi* m, const void* q, void* kc, int dtype, const float* w, int64_t* local_idx,
                     float* local_val, csaidx_run_stats* stats);
int csaidx_multi_destroy(csaidx_multi* m);

#ifdef __cplusplus
}
#endif

#endif /* CSAIDX_HOST_H */
