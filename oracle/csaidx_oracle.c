/*
 * csaidx_oracle.c — TEST INFRASTRUCTURE ONLY (see csaidx_oracle.h).
 *
 * CPU restatement of the reference indexer path, compiled with
 * -ffp-contract=off like the reference (CMakeLists.txt:12-15) so every fp32
 * operation rounds exactly where the reference's does. Each function cites
 * the reference lines it restates.
 */
#include "csaidx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORC_NEG_INF (-INFINITY)

/* ------------------------------------------------------------ synth.cpp */

/* synth.cpp:11-16 */
uint64_t orc_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* synth.cpp:22-28 */
void orc_xoshiro_init(orc_xoshiro* g, uint64_t seed, uint64_t stream) {
    uint64_t sm = seed + stream * 0x9E3779B97F4A7C15ULL;
    for (int i = 0; i < 4; ++i) g->s[i] = orc_splitmix64(&sm);
    if ((g->s[0] | g->s[1] | g->s[2] | g->s[3]) == 0) g->s[0] = 1;
}

/* synth.cpp:30-40 (xoshiro256++) */
uint64_t orc_xoshiro_next(orc_xoshiro* g) {
    uint64_t* s = g->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* synth.cpp:50-64: Box-Muller in double, u1 in (0, 1], u2 in [0, 1). */
void orc_fill_gaussian(float* out, int64_t n, double stddev, uint64_t seed, uint64_t stream) {
    orc_xoshiro g;
    orc_xoshiro_init(&g, seed, stream);
    const double two_pi = 2.0 * 3.14159265358979323846;
    int64_t i = 0;
    while (i < n) {
        const double u1 = (double)((orc_xoshiro_next(&g) >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(orc_xoshiro_next(&g) >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1));
        out[i++] = (float)(r * cos(two_pi * u2) * stddev);
        if (i < n) out[i++] = (float)(r * sin(two_pi * u2) * stddev);
    }
}

/* synth.cpp:66-81 with stream ids q=1, kc=2, w=3 (synth.hpp:29-31). */
void orc_generate_inputs(int64_t batch, int64_t seq_len, int64_t ratio, int64_t heads, int64_t head_dim,
                         uint64_t seed, float* q, float* kc, float* w) {
    const int64_t T = seq_len / ratio;
    const double unit = 1.0 / sqrt((double)head_dim);
    const double wscale = 1.0 / sqrt((double)head_dim * (double)heads);
    orc_fill_gaussian(q, batch * seq_len * heads * head_dim, unit, seed, 1);
    orc_fill_gaussian(kc, batch * T * head_dim, unit, seed, 2);
    orc_fill_gaussian(w, batch * seq_len * heads, wscale, seed, 3);
}

float orc_bf16_round(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return x; /* inf / nan unchanged */
    const uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

void orc_bf16_round_array(float* x, int64_t n) {
    for (int64_t i = 0; i < n; ++i) x[i] = orc_bf16_round(x[i]);
}

/* ------------------------------------------------------------ half.cpp */

static inline uint32_t rne_shift(uint32_t v, int shift) {
    const uint32_t bias = ((1u << (shift - 1)) - 1u) + ((v >> shift) & 1u);
    return (v + bias) >> shift;
}

/* half.cpp:21-55 */
uint16_t orc_float_to_half_bits(float x) {
    uint32_t bits;
    memcpy(&bits, &x, 4);
    const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
    const uint32_t a = bits & 0x7FFFFFFFu;
    if (a >= 0x7F800000u) return a > 0x7F800000u ? (uint16_t)(sign | 0x7E00u) : (uint16_t)(sign | 0x7C00u);
    const int exp32 = (int)(a >> 23) - 127;
    const int exp16 = exp32 + 15;
    const uint32_t mant = a & 0x7FFFFFu;
    if (exp16 >= 31) return (uint16_t)(sign | 0x7C00u);
    if (exp16 <= 0) {
        if (exp16 < -17 || (a >> 23) == 0) return sign;
        const int shift = -1 - exp32;
        if (shift >= 32) return sign;
        return (uint16_t)(sign | rne_shift(mant | 0x800000u, shift));
    }
    return (uint16_t)(sign | (((uint32_t)exp16 << 10) + rne_shift(mant, 13)));
}

/* half.cpp:57-82 */
float orc_half_bits_to_float(uint16_t h) {
    const uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu;
    uint32_t mant = h & 0x3FFu;
    uint32_t bits;
    if (e == 0) {
        if (mant == 0) {
            bits = sign;
        } else {
            int k = -1;
            do {
                mant <<= 1;
                ++k;
            } while ((mant & 0x400u) == 0);
            bits = sign | ((uint32_t)(127 - 15 - k) << 23) | ((mant & 0x3FFu) << 13);
        }
    } else if (e == 31) {
        bits = sign | 0x7F800000u | (mant << 13);
    } else {
        bits = sign | ((e - 15 + 127) << 23) | (mant << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* half.cpp:84-91: RNE to binary16, saturate at +/-65504. */
float orc_half_round(float x) {
    const uint16_t h = orc_float_to_half_bits(x);
    if ((h & 0x7FFFu) == 0x7C00u) return (h & 0x8000u) ? -65504.0f : 65504.0f;
    return orc_half_bits_to_float(h);
}

/* ------------------------------------------------------------ causal.cpp */

int64_t orc_t_legal(int64_t t, int64_t ratio) { return (t + 1) / ratio; }

int64_t orc_k_eff(int64_t t, int64_t ratio, int64_t top_k) {
    const int64_t l = orc_t_legal(t, ratio);
    return top_k < l ? top_k : l;
}

/* ------------------------------------------------------------ score */

/* score_scalar.cpp:20-34 for one query row against ncols consecutive key
 * rows. Keys are processed in panels of ORC_PANEL lanes (transposed once per
 * panel) so the compiler can vectorise ACROSS keys; every lane still runs the
 * reference's exact per-score sequence: ascending-d dot as mul then add,
 * x<0?0:x, ascending-h acc = acc + w*r (contraction is off for this TU). */
#define ORC_PANEL 16
typedef float orc_v8 __attribute__((vector_size(32)));
static void score_span(const float* qrow, const float* wrow, const float* krows, int64_t ncols, int64_t heads,
                       int64_t head_dim, int fp16, float* out) {
    float* kt = (float*)malloc((size_t)(head_dim * ORC_PANEL) * sizeof(float));
    for (int64_t j0 = 0; j0 < ncols; j0 += ORC_PANEL) {
        const int64_t nb = ncols - j0 < ORC_PANEL ? ncols - j0 : ORC_PANEL;
        for (int64_t d = 0; d < head_dim; ++d)
            for (int64_t jj = 0; jj < ORC_PANEL; ++jj)
                kt[d * ORC_PANEL + jj] = jj < nb ? krows[(j0 + jj) * head_dim + d] : 0.0f;
        float acc[ORC_PANEL];
        for (int jj = 0; jj < ORC_PANEL; ++jj) acc[jj] = 0.0f;
        for (int64_t h = 0; h < heads; ++h) {
            const float* qh = qrow + h * head_dim;
            /* 2 x 8 independent lanes; separate mul and add (no contraction). */
            orc_v8 d0 = {0, 0, 0, 0, 0, 0, 0, 0}, d1 = d0;
            for (int64_t d = 0; d < head_dim; ++d) {
                const float qv = qh[d];
                const orc_v8 qb = {qv, qv, qv, qv, qv, qv, qv, qv};
                orc_v8 k0, k1;
                memcpy(&k0, kt + d * ORC_PANEL, sizeof(k0));
                memcpy(&k1, kt + d * ORC_PANEL + 8, sizeof(k1));
                d0 = d0 + qb * k0;
                d1 = d1 + qb * k1;
            }
            float dot[ORC_PANEL];
            memcpy(dot, &d0, sizeof(d0));
            memcpy(dot + 8, &d1, sizeof(d1));
            const float wh = wrow[h];
            for (int jj = 0; jj < ORC_PANEL; ++jj) {
                float dv = dot[jj];
                if (fp16) dv = orc_half_round(dv);
                const float rect = (dv < 0.0f) ? 0.0f : dv;
                float a = acc[jj] + wh * rect;
                if (fp16) a = orc_half_round(a);
                acc[jj] = a;
            }
        }
        for (int64_t jj = 0; jj < nb; ++jj) out[j0 + jj] = acc[jj];
    }
    free(kt);
}

void orc_score_tile(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                    int64_t key_blocks, int64_t heads, int64_t head_dim, int64_t s0, int64_t t0, int64_t rows,
                    int64_t cols, int fp16, float* out) {
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t i = 0; i < rows; ++i) {
            const int64_t s = s0 + i;
            score_span(q + ((b * seq_len + s) * heads) * head_dim, w + (b * seq_len + s) * heads,
                       kc + (b * key_blocks + t0) * head_dim, cols, heads, head_dim, fp16,
                       out + (b * rows + i) * cols);
        }
    }
}

/* Threaded driver of score_span over independent rows (test infrastructure:
 * the reference scores one row per call; the per-score op order is the
 * same, so the split only changes which thread computes a score). */
#define ORC_PIECE 4096
typedef struct {
    const float *q, *w, *kc;
    const int64_t *kc_row0, *legal, *piece0, *offset;
    int64_t nrows, npieces, heads, head_dim;
    float* out;
    int64_t next;
    pthread_mutex_t mu;
} rows_job;

static void* rows_worker(void* arg) {
    rows_job* j = (rows_job*)arg;
    for (;;) {
        pthread_mutex_lock(&j->mu);
        const int64_t p = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (p >= j->npieces) break;
        int64_t r = 0; /* row owning piece p: piece0 is ascending */
        int64_t lo = 0, hi = j->nrows - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) / 2;
            if (j->piece0[mid] <= p) lo = mid; else hi = mid - 1;
        }
        r = lo;
        const int64_t c0 = (p - j->piece0[r]) * ORC_PIECE;
        const int64_t n = j->legal[r] - c0 < ORC_PIECE ? j->legal[r] - c0 : ORC_PIECE;
        score_span(j->q + r * j->heads * j->head_dim, j->w + r * j->heads,
                   j->kc + (j->kc_row0[r] + c0) * j->head_dim, n, j->heads, j->head_dim, 0,
                   j->out + j->offset[r] + c0);
    }
    return NULL;
}

void orc_score_rows(const float* q_rows, const float* w_rows, const float* kc, const int64_t* kc_row0,
                    const int64_t* legal, int64_t nrows, int64_t heads, int64_t head_dim, int nthreads,
                    float* out) {
    if (nrows <= 0) return;
    int64_t* piece0 = (int64_t*)malloc((size_t)nrows * sizeof(int64_t));
    int64_t* offset = (int64_t*)malloc((size_t)nrows * sizeof(int64_t));
    int64_t np = 0, off = 0;
    for (int64_t r = 0; r < nrows; ++r) {
        piece0[r] = np;
        offset[r] = off;
        np += (legal[r] + ORC_PIECE - 1) / ORC_PIECE;
        off += legal[r];
    }
    rows_job j = {q_rows, w_rows, kc, kc_row0, legal, piece0, offset, nrows, np, heads, head_dim, out, 0,
                  PTHREAD_MUTEX_INITIALIZER};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, rows_worker, &j);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(piece0);
    free(offset);
}

/* ------------------------------------------------------------ topk.cpp */

/* topk.hpp:23-26 */
int orc_succ(float sa, int64_t ia, float sb, int64_t ib) {
    if (sa != sb) return sa > sb;
    return ia < ib;
}

typedef struct {
    float s;
    int64_t i;
} entry_t;

static int cmp_succ(const void* a, const void* b) {
    const entry_t* x = (const entry_t*)a;
    const entry_t* y = (const entry_t*)b;
    if (orc_succ(x->s, x->i, y->s, y->i)) return -1;
    if (orc_succ(y->s, y->i, x->s, x->i)) return 1;
    return 0;
}

/* topk.cpp:193-206 */
int64_t orc_oracle_topk(const float* row, int64_t legal, int64_t k, float* out_v, int64_t* out_i) {
    if (legal <= 0) return 0;
    entry_t* all = (entry_t*)malloc((size_t)legal * sizeof(entry_t));
    for (int64_t j = 0; j < legal; ++j) {
        all[j].s = row[j];
        all[j].i = j;
    }
    qsort(all, (size_t)legal, sizeof(entry_t), cmp_succ);
    const int64_t take = k < legal ? k : legal;
    for (int64_t n = 0; n < take; ++n) {
        out_v[n] = all[n].s;
        out_i[n] = all[n].i;
    }
    free(all);
    return take;
}

/* driver.cpp:167-192 */
void orc_run_materialize(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                         int64_t ratio, int64_t heads, int64_t head_dim, int64_t top_k, int fp16,
                         int64_t* out_idx, float* out_val) {
    const int64_t T = seq_len / ratio;
    float* row = (float*)malloc((size_t)(T > 0 ? T : 1) * sizeof(float));
    for (int64_t n = 0; n < batch * seq_len * top_k; ++n) {
        out_idx[n] = -1;
        out_val[n] = ORC_NEG_INF;
    }
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t t = 0; t < seq_len; ++t) {
            const int64_t legal = orc_t_legal(t, ratio);
            const float* qrow = q + ((b * seq_len + t) * heads) * head_dim;
            const float* wrow = w + (b * seq_len + t) * heads;
            score_span(qrow, wrow, kc + b * T * head_dim, legal, heads, head_dim, fp16, row);
            orc_oracle_topk(row, legal, top_k, out_val + (b * seq_len + t) * top_k,
                            out_idx + (b * seq_len + t) * top_k);
        }
    }
    free(row);
}

/* merge_topk (topk.cpp:134-172): top-k of (run U tile) under succ, in
 * order. Both inputs sorted; a front-to-back merge yields the same list the
 * reference's in-place backward merge does. */
static void merge_row(float* bv, int64_t* bi, int64_t k, const entry_t* tile, int64_t tn, entry_t* scratch) {
    int64_t a = 0, c = 0;
    for (int64_t pos = 0; pos < k; ++pos) {
        const int take_tile = c < tn && (a >= k || orc_succ(tile[c].s, tile[c].i, bv[a], bi[a]));
        if (take_tile) {
            scratch[pos] = tile[c++];
        } else {
            scratch[pos].s = bv[a];
            scratch[pos].i = bi[a];
            ++a;
        }
    }
    for (int64_t pos = 0; pos < k; ++pos) {
        bv[pos] = scratch[pos].s;
        bi[pos] = scratch[pos].i;
    }
}

/* overwrite_topk (topk.cpp:174-191) */
static void overwrite_row(float* bv, int64_t* bi, int64_t k, const entry_t* tile, int64_t tn) {
    int64_t n = 0;
    for (int64_t e = 0; e < tn && n < k; ++e) {
        if (tile[e].s == ORC_NEG_INF) continue;
        bv[n] = tile[e].s;
        bi[n] = tile[e].i;
        ++n;
    }
    for (; n < k; ++n) {
        bv[n] = ORC_NEG_INF;
        bi[n] = -1;
    }
}

/* driver.cpp:36-106 (process_query_tile) + 115-165 (serial run_chunked) */
int orc_run_chunked(const float* q, const float* kc, const float* w, int64_t batch, int64_t seq_len,
                    int64_t ratio, int64_t heads, int64_t head_dim, int64_t top_k, int64_t query_tile,
                    int64_t key_tile, int fp16, int ablation, int causal_early_exit, int64_t* out_idx,
                    float* out_val, int64_t* stats3) {
    const int64_t T = seq_len / ratio;
    const int64_t cs = query_tile < seq_len ? query_tile : seq_len;
    const int64_t ct = key_tile < T ? key_tile : T;
    const int64_t k = top_k;
    int rc = 0;
    stats3[0] = stats3[1] = stats3[2] = 0;
    for (int64_t n = 0; n < batch * seq_len * k; ++n) {
        out_idx[n] = -1;
        out_val[n] = ORC_NEG_INF;
    }
    float* run_v = (float*)malloc((size_t)(batch * cs * k) * sizeof(float));
    int64_t* run_i = (int64_t*)malloc((size_t)(batch * cs * k) * sizeof(int64_t));
    float* tile = (float*)malloc((size_t)(batch * cs * ct) * sizeof(float));
    entry_t* ent = (entry_t*)malloc((size_t)(ct > k ? ct : k) * sizeof(entry_t));
    entry_t* scratch = (entry_t*)malloc((size_t)k * sizeof(entry_t));
    for (int64_t s0 = 0; s0 < seq_len && rc == 0; s0 += cs) {
        const int64_t rows = cs < seq_len - s0 ? cs : seq_len - s0;
        for (int64_t n = 0; n < batch * rows * k; ++n) {
            run_v[n] = ORC_NEG_INF;
            run_i[n] = -1;
        }
        for (int64_t t0 = 0; t0 < T; t0 += ct) {
            const int64_t cols = ct < T - t0 ? ct : T - t0;
            if (ablation == 2 && cols < k) {
                ++stats3[2];
                continue;
            }
            if (causal_early_exit && t0 >= orc_t_legal(s0 + rows - 1, ratio)) {
                stats3[1] += (T - t0 + ct - 1) / ct;
                break;
            }
            orc_score_tile(q, kc, w, batch, seq_len, T, heads, head_dim, s0, t0, rows, cols, fp16, tile);
            ++stats3[0];
            for (int64_t b = 0; b < batch; ++b) {
                for (int64_t i = 0; i < rows; ++i) {
                    const int64_t legal = orc_t_legal(s0 + i, ratio);
                    float* sc = tile + (b * rows + i) * cols;
                    for (int64_t j = 0; j < cols; ++j) {
                        if (t0 + j >= legal) sc[j] = ORC_NEG_INF; /* mask_tile */
                        ent[j].s = sc[j];
                        ent[j].i = t0 + j;
                    }
                    /* tile_topk: top-min(k, cols) under succ, descending */
                    qsort(ent, (size_t)cols, sizeof(entry_t), cmp_succ);
                    const int64_t width = k < cols ? k : cols;
                    float* bv = run_v + (b * rows + i) * k;
                    int64_t* bi = run_i + (b * rows + i) * k;
                    if (ablation == 1)
                        overwrite_row(bv, bi, k, ent, width);
                    else
                        merge_row(bv, bi, k, ent, width, scratch);
                }
            }
        }
        /* sentinel pass, driver.cpp:84-105 */
        for (int64_t b = 0; b < batch && rc == 0; ++b) {
            for (int64_t i = 0; i < rows; ++i) {
                float* bv = run_v + (b * rows + i) * k;
                int64_t* bi = run_i + (b * rows + i) * k;
                int64_t valid = 0;
                while (valid < k && bv[valid] != ORC_NEG_INF) ++valid;
                for (int64_t n = valid; n < k; ++n) {
                    if (bv[n] != ORC_NEG_INF) rc = 4;
                    bi[n] = -1;
                }
                if (ablation == 0 && valid != orc_k_eff(s0 + i, ratio, k)) rc = 4;
                memcpy(out_idx + (b * seq_len + s0 + i) * k, bi, (size_t)k * sizeof(int64_t));
                memcpy(out_val + (b * seq_len + s0 + i) * k, bv, (size_t)k * sizeof(float));
            }
        }
    }
    free(run_v);
    free(run_i);
    free(tile);
    free(ent);
    free(scratch);
    return rc;
}

int64_t orc_row_topk(const float* q_row, const float* w_row, const float* kc, int64_t key_blocks, int64_t heads,
                     int64_t head_dim, int64_t legal, int64_t k, float* out_v, int64_t* out_i) {
    if (legal > key_blocks) legal = key_blocks;
    if (legal <= 0) return 0;
    float* row = (float*)malloc((size_t)legal * sizeof(float));
    score_span(q_row, w_row, kc, legal, heads, head_dim, 0, row);
    const int64_t n = orc_oracle_topk(row, legal, k, out_v, out_i);
    free(row);
    return n;
}

/* ------------------------------------------------------------ recall.cpp */

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

static int64_t valid_count(const int64_t* row, int64_t k) {
    int64_t n = 0;
    while (n < k && row[n] != -1) ++n;
    return n;
}

/* recall.cpp:9-64 */
int64_t orc_recall(const int64_t* ref_idx, const int64_t* test_idx, int64_t nrows, int64_t top_k, double* mean,
                   double* min_r, double* pct_perfect, double* pct_below99) {
    int64_t* a = (int64_t*)malloc((size_t)top_k * sizeof(int64_t));
    int64_t* c = (int64_t*)malloc((size_t)top_k * sizeof(int64_t));
    double sum = 0.0, mn = 1.0;
    int64_t rows = 0, perfect = 0, below = 0;
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t nref = valid_count(ref_idx + r * top_k, top_k);
        if (nref == 0) continue;
        const int64_t ntest = valid_count(test_idx + r * top_k, top_k);
        memcpy(a, ref_idx + r * top_k, (size_t)nref * sizeof(int64_t));
        memcpy(c, test_idx + r * top_k, (size_t)ntest * sizeof(int64_t));
        qsort(a, (size_t)nref, sizeof(int64_t), cmp_i64);
        qsort(c, (size_t)ntest, sizeof(int64_t), cmp_i64);
        int64_t hits = 0, x = 0, y = 0;
        while (x < nref && y < ntest) {
            if (a[x] == c[y]) {
                ++hits;
                ++x;
                ++y;
            } else if (a[x] < c[y]) {
                ++x;
            } else {
                ++y;
            }
        }
        const double rr = (double)hits / (double)nref;
        sum += rr;
        if (rr < mn) mn = rr;
        if (rr == 1.0) ++perfect;
        if (rr < 0.99) ++below;
        ++rows;
    }
    free(a);
    free(c);
    *mean = rows ? sum / (double)rows : 1.0;
    *min_r = rows ? mn : 1.0;
    *pct_perfect = rows ? 100.0 * (double)perfect / (double)rows : 100.0;
    *pct_below99 = rows ? 100.0 * (double)below / (double)rows : 0.0;
    return rows;
}
