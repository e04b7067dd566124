// Kernel-side parameter blocks and launchers. Internal to libcsaidx_cuda;
// the public boundary is include/csaidx_cuda.h.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

// ------------------------------------------------------------------ score
constexpr int kScoreMaxPieces = 256;

struct ScoreTcParams {
    const float* w;     // [B, S, 64] fp32 mixing weights
    float* out;         // [B, rows, ld] fp32 scores
    int* nonfinite;     // set to 1 when an unmasked score is not finite
    int* sched;         // [2] work counter + exit counter (zero between launches)
    int64_t ld;
    int64_t seq_len, key_blocks, ratio;
    int64_t s0, rows, t0, cols;
    // Operand row layout: q / w hold op_rows query rows per batch and query
    // s lives at operand row s + op_shift (op_rows = seq_len, op_shift = 0
    // for the full [B, S, ...] tensors; rank-local stacks otherwise).
    int64_t op_rows, op_shift;
    int batch;
    int apply_mask;
    int fp16;  // AccumulationMode::fp16_emulated epilogue (binary16 rounding points)
    // Sample mode: tile kt of the launch covers physical key tile
    // kt * kt_stride; outputs use the compacted (virtual) column kt*128+lane.
    int kt_stride;
    // Fused candidate filter (optional): bit (j & 31) of
    // pass_bits[(b*rows + r) * bits_ld + j / 32] = (column j legal and its
    // score >= tau[b*rows + r]); one ballot + one word store per warp.
    // Words of causally dead key tiles are not written.
    const float* tau;
    uint32_t* pass_bits;
    int64_t bits_ld;
    // Optional group maxima (two-level select): gmax[(b*rows + r) * gmax_ld +
    // j / 32] = max of the legal scores of key columns [32 (j/32), +32) of
    // row r (-inf when none is legal).
    float* gmax;
    int64_t gmax_ld;
    // Optional profiling counters, [grid][8] clock64 cycles: MMA waits on
    // k_full / acc_empty / q_full, MMA span, epilogue (warp 4) wait on
    // acc_full, epilogue span, producer waits on k_empty / q_empty.
    long long* probe;
    // filled by the launcher: dense piece-major work list. Piece p (key tiles
    // [p*tpp, (p+1)*tpp)) is live for the query blocks qb >= nqb - count_p,
    // count_p = (piece_start[p+1] - piece_start[p]) / batch.
    int nqb, tpp, npieces, nitems;
    int piece_start[kScoreMaxPieces + 1];
};

struct ScoreExactParams {
    const void* q;            // [B, S, H, D], bf16 or fp32 (operand_f32)
    const void* kc;           // [B, T, D]
    const float* w;           // [B, S, H]
    float* out;               // [B, rows, ld]
    int* nonfinite;
    int64_t ld;
    int64_t seq_len, key_blocks, heads, head_dim, ratio;
    int64_t s0, rows, t0, cols;
    int64_t op_rows, op_shift;  // operand row layout (see ScoreTcParams)
    int batch;
    int apply_mask;
    int fp16;  // emulate binary16 rounding points (score_scalar.cpp:29-32)
    int operand_f32;  // 1: q/kc are fp32 (bit-exact vs the CPU reference on any input)
};

// ------------------------------------------------------------------ select
// Per (b, row): exact top-min(k, n) of the row's first n columns under the
// reference order (score desc, index asc), n = legal columns of that row
// (or all cols when apply_mask == 0). Output rows are `width` wide, sorted,
// padded with (-inf, -1).
struct SelectParams {
    const float* scores;  // [B, rows, ld]
    int64_t ld;
    int64_t rows, cols, s0, t0, ratio;
    int batch;
    int apply_mask;
    int k;
    int width;
    float* out_val;       // [B, rows, out_ld]
    int32_t* out_idx;
    int64_t out_ld;
    int* fallbacks;       // rows that took the exact global fallback (telemetry)
    long long* phase_clk; // optional [rows * 8] clock64 stamps per phase (profiling)
    // Optional candidate bitmap from the score epilogue (bit j of row r =
    // legal score j >= tau[r]): when the row's flagged count is within
    // [min(k, n), list capacity] the row is finished from the flagged
    // entries; otherwise it streams `scores` as usual.
    const uint32_t* pass_bits;  // [B, rows, bits_ld]
    int64_t bits_ld;
    int* cand_hits;       // rows finished from the bitmap (telemetry)
    // Optional fused sentinel pass (the finalize_kernel contract, for plans
    // whose one key tile covers every key): row r of batch b is written to
    // out_val / final_idx + (b * final_rows + final_row0 + r) * out_ld with
    // int64 indices; entries past min(k, n) are (-inf, -1).
    int64_t* final_idx;
    int64_t final_rows, final_row0;
    // Optional group maxima of the rows (ScoreTcParams::gmax): rows whose
    // legal length spans many more groups than k take the two-level path
    // (read the maxima, then only the groups that can hold a top-k score).
    const float* gmax;
    int64_t gmax_ld;
    // > 0: run as that many persistent CTAs, one per SM, each with several
    // row groups (to share the GPU with a concurrently running score kernel)
    int persistent_ctas;
    // Optional index sink (with final_idx): row r of batch b is also stored
    // as int32 indices at sink + (b * sink_seq + s0 + r) * out_ld — a [B, S, k]
    // buffer that may live in another GPU's memory (CUDA IPC peer mapping)
    int32_t* sink;
    int64_t sink_seq;
    int sink_only;  // final rows go to the sink only (final_idx / out_val unused)
    // Global scratch for takes above the shared-memory capacity (k > 4096):
    // per-row slots of select_large_scratch_bytes(); required then, else unused
    void* scratch;
    size_t scratch_bytes;
};

// Per-row candidate threshold from a strided sample of the row's scores
// (the sample pass of score_tc, kt_stride > 1): the sample's rank-r key with
// r chosen so ~2k entries of the whole row are expected to pass; -inf when
// the row's legal length fits the candidate list outright.
struct TauParams {
    const float* sample;  // [B, rows, lds] virtual columns (illegal = -inf)
    int64_t lds;
    int64_t rows, cols, s0, t0, ratio;
    int batch;
    int kt_stride;
    int k;
    int cand_cap;
    float* tau;           // [B * rows]
};

// ------------------------------------------------------------------ merge
// Per row: run := top-k(run U cand) (merge) or run := cand (overwrite, A1).
struct MergeParams {
    float* run_val;        // [nrows, k], sorted
    int32_t* run_idx;
    const float* cand_val; // [nrows, cand_ld], sorted, width valid
    const int32_t* cand_idx;
    int64_t cand_ld;
    int64_t nrows;
    int k;
    int width;
    int overwrite;
    int check_overlap;
    int* overlap_flag;
    // k above the shared-memory merge (4096): both rows are staged as
    // composites in global scratch, stage_rows rows of (k + width) at a time
    uint64_t* stage;
    int64_t stage_rows;
};

// ------------------------------------------------------------------ finalize
// Sentinel pass (driver.cpp:84-105): -inf -> index -1, trailing check,
// valid == k_eff check; widen to int64 into the output rows.
struct FinalizeParams {
    const float* run_val;   // [B, rows, k]
    const int32_t* run_idx;
    int64_t rows, s0, ratio;
    int batch;
    int k;
    int check_keff;
    int64_t* out_idx;       // [B, out_rows, k] at row offset out_row0
    float* out_val;
    int64_t out_rows, out_row0;
    int* trail_flag;        // sentinel entries do not trail
    int* keff_flag;         // valid != k_eff
    int32_t* sink;          // optional [B, sink_seq, k] int32 copy (SelectParams::sink)
    int64_t sink_seq;       // (out_idx / out_val null: the sink is the only output)
};

// ------------------------------------------------------------------ sparse attention (f4)
// out[b,t,h,:Dv] = softmax over the valid indices[b,t,:] of
// sm_scale * q[b,t,h,:] . kv[b,i,:], applied to kv[b,i,:Dv]; H = 128 g,
// Dqk = 576, Dv = 512 (one shared latent KV head). q is read through a TMA
// map built by the C-ABI entry, the gathered kv rows by cp.async.
struct SparseMlaParams {
    const __nv_bfloat16* q;  // [B, S, H, 576]
    const __nv_bfloat16* kv; // [B, kv_len, 576]
    const int32_t* indices;  // [B, S, idx_ld], -1 = padding
    int64_t idx_ld;
    __nv_bfloat16* out;      // [B, S, H, out_ld]
    int64_t out_ld;
    float* lse;              // optional [B, S, H]
    int64_t seq_len, kv_len;
    int batch;
    int k;
    int head_groups;         // H / 128
    float sm_scale;
};

// ------------------------------------------------------------------ prep
struct ConvertParams {
    const float* src;
    __nv_bfloat16* dst;
    int64_t n;
    int* inexact_flag;  // set when an element is not bf16-representable
    int* nonfinite_flag;
};

namespace csaidx_kern {

// Function attributes (cudaFuncSetAttribute) belong to a device context:
// launchers keep one "already set" flag per device.
constexpr int kMaxDevices = 64;
inline int attr_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 ? 0 : (d >= kMaxDevices ? kMaxDevices - 1 : d);
}


bool score_tc_supported(int64_t heads, int64_t head_dim);
size_t score_tc_smem_bytes();
int score_tc_q_box_rows();  // rows of the q TMA box (one query group x 64 heads)
cudaError_t launch_score_tc(const CUtensorMap& qmap, const CUtensorMap& kmap, ScoreTcParams p,
                            int num_sms, cudaStream_t stream);
cudaError_t launch_score_exact(const ScoreExactParams& p, cudaStream_t stream);

int select_max_take();
int select_cand_capacity(int k);  // candidate-list length the select kernel accepts for this k
bool select_fat_fits(int k);      // the persistent multi-row form fits shared memory for this k
cudaError_t launch_select(const SelectParams& p, cudaStream_t stream);
int sparse_mla_smem_bytes();
cudaError_t launch_sparse_mla(const CUtensorMap& qmap, const SparseMlaParams& p, cudaStream_t stream);
int sparse_mla_pair_smem_bytes();
// CTA-pair form (attn_pair_sm100.cu): same operator, Dqk split across a cluster of 2
cudaError_t launch_sparse_mla_pair(const CUtensorMap& qmap, const SparseMlaParams& p, cudaStream_t stream);
// Scratch the select needs for takes above select_max_take() (rows = B * rows).
size_t select_large_scratch_bytes(int k, int64_t cols, int64_t rows);
// Staging scratch the merge needs for k above select_max_take().
size_t merge_stage_bytes(int k, int width, int64_t nrows);
cudaError_t launch_tau(const TauParams& p, cudaStream_t stream);
cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream);
cudaError_t launch_finalize(const FinalizeParams& p, cudaStream_t stream);

cudaError_t launch_convert_bf16(const ConvertParams& p, cudaStream_t stream);
cudaError_t launch_fill_sentinel(float* val, int32_t* idx, int64_t n, cudaStream_t stream);
cudaError_t launch_bool_mask(uint8_t* keep, int64_t rows, int64_t cols, int64_t s0, int64_t t0,
                             int64_t ratio, cudaStream_t stream);
cudaError_t launch_apply_bool_mask(float* scores, int64_t ld, const uint8_t* keep, int64_t batch,
                                   int64_t rows, int64_t cols, cudaStream_t stream);
cudaError_t launch_narrow(const int64_t* src, int32_t* dst, int64_t n, cudaStream_t stream);
cudaError_t launch_scatter_rows(const int32_t* src, int32_t* dst, const int64_t* dst_row, int64_t nrows,
                                int64_t row_elems, cudaStream_t stream);
// Counter-based synthetic normal generator (splitmix64 hash of the element
// index + Box-Muller), rounded to bf16 or kept fp32.
cudaError_t launch_gen_normal_bf16(__nv_bfloat16* dst, int64_t n, double stddev, uint64_t seed,
                                   uint64_t stream_id, int64_t offset, cudaStream_t stream);
cudaError_t launch_gen_normal_f32(float* dst, int64_t n, double stddev, uint64_t seed,
                                  uint64_t stream_id, int64_t offset, cudaStream_t stream);

}  // namespace csaidx_kern
