/*
 * csaidx_oracle — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPU algorithm for the indexer step
 * (/root/reference/proj/src: synth.cpp, half.cpp, score_scalar.cpp,
 * causal.cpp, topk.cpp, driver.cpp, recall.cpp). It is the checker the GPU
 * path is compared against; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. The product path never calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 * (a) the known-answer vectors in the reference's own tests and (b) golden
 * fixtures produced by the reference itself (oracle/_ref, compiled from the
 * reference sources by oracle/Makefile; tests/golden/make_golden.py).
 */
#ifndef CSAIDX_ORACLE_H
#define CSAIDX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* synth.cpp:10-16 / 22-48 */
uint64_t orc_splitmix64(uint64_t* state);
typedef struct orc_xoshiro { uint64_t s[4]; } orc_xoshiro;
void orc_xoshiro_init(orc_xoshiro* g, uint64_t seed, uint64_t stream);
uint64_t orc_xoshiro_next(orc_xoshiro* g);
/* synth.cpp:50-64 */
void orc_fill_gaussian(float* out, int64_t n, double stddev, uint64_t seed, uint64_t stream);
/* synth.cpp:66-81 (q, kc ~ N(0, 1/d_h); w ~ N(0, 1/(d_h H_I))) */
void orc_generate_inputs(int64_t batch, int64_t seq_len, int64_t ratio, int64_t heads, int64_t head_dim,
                         uint64_t seed, float* q, float* kc, float* w);
/* bf16 round-to-nearest-even of an fp32 value (input staging rule). */
float orc_bf16_round(float x);
void orc_bf16_round_array(float* x, int64_t n);

/* half.cpp:21-91 */
uint16_t orc_float_to_half_bits(float x);
float orc_half_bits_to_float(uint16_t h);
float orc_half_round(float x);

/* causal.cpp:9-28 */
int64_t orc_t_legal(int64_t t, int64_t ratio);
int64_t orc_k_eff(int64_t t, int64_t ratio, int64_t top_k);

/* score_scalar.cpp:20-34 over one tile: out[b, i, j], fp16 = emulated mode. */
void orc_score_tile(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                    int64_t key_blocks, int64_t heads, int64_t head_dim, int64_t s0, int64_t t0, int64_t rows,
                    int64_t cols, int fp16, float* out);

/* topk.hpp:23-26 */
int orc_succ(float sa, int64_t ia, float sb, int64_t ib);

/* topk.cpp:193-206: top-min(k, legal) of row[0, legal) sorted under succ. */
int64_t orc_oracle_topk(const float* row, int64_t legal, int64_t k, float* out_v, int64_t* out_i);

/* driver.cpp:167-192 (results pre-filled with (-1, -inf) by the callee). */
void orc_run_materialize(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                         int64_t ratio, int64_t heads, int64_t head_dim, int64_t top_k, int fp16,
                         int64_t* out_idx, float* out_val);

/* driver.cpp:36-165 (serial schedule). ablation: 0 none, 1 a1_no_merge,
 * 2 a2_skip_narrow. stats3 = {dispatch_count, tiles_skipped_masked,
 * tiles_skipped_narrow}. Returns 0, or 4 (logic_error) when the sentinel
 * contract breaks. */
int orc_run_chunked(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                    int64_t ratio, int64_t heads, int64_t head_dim, int64_t top_k, int64_t query_tile,
                    int64_t key_tile, int fp16, int ablation, int causal_early_exit, int64_t* out_idx,
                    float* out_val, int64_t* stats3);

/* One full causal row (query t, batch b) with the reference op order, then
 * its top-(k+1) under succ: the sampled-row oracle for large shapes. q_row
 * is [heads, head_dim] of that query, w_row [heads], kc [key_blocks, d]. */
int64_t orc_row_topk(const float* q_row, const float* w_row, const float* kc, int64_t key_blocks,
                     int64_t heads, int64_t head_dim, int64_t legal, int64_t k, float* out_v,
                     int64_t* out_i);

/* Many full causal rows at once (the sampled-row oracle at scale): row r is
 * query q_rows[r] ([heads, head_dim]) with weights w_rows[r] ([heads])
 * against keys kc + kc_row0[r] * head_dim, over its first legal[r] keys;
 * scores land at out + offset[r] (offset[r] = sum of legal[<r]). Each score
 * follows score_scalar.cpp:20-34 exactly (score_span); the work is split in
 * 4096-key pieces over nthreads POSIX threads, so results do not depend on
 * the thread count. */
void orc_score_rows(const float* q_rows, const float* w_rows, const float* kc, const int64_t* kc_row0,
                    const int64_t* legal, int64_t nrows, int64_t heads, int64_t head_dim, int nthreads,
                    float* out);

/* recall.cpp:9-64 — returns rows evaluated; fills mean/min/pct_perfect. */
int64_t orc_recall(const int64_t* ref_idx, const int64_t* test_idx, int64_t nrows, int64_t top_k,
                   double* mean, double* min_r, double* pct_perfect, double* pct_below99);

#ifdef __cplusplus
}
#endif

#endif
