// Per-row exact top-k selection over one score tile (the GPU tile_topk,
// reference topk.cpp:105-132 + causal.cpp:30-41).
//
// One 256-thread CTA per (batch, query row), several rows per SM; n = the
// row's legal columns. Every entry is packed into a unique 64-bit composite
// (ord_key(score) << 32 | ~(col + 1)): ord_key is monotone in the float order
// with -0.0 folded onto +0.0, and the low word makes ties go to the smaller
// index, so descending composite order is exactly the reference's succ()
// order (topk.hpp:23-26).
//
// Fast path (one streaming pass over the row):
//   1. sample: evenly spaced 512-byte segments (~64 above the threshold), held in
//      registers; a value-linear histogram over the sample's range (plus a
//      refinement pass inside a coarse rank bin) picks a threshold expected
//      to keep ~2k entries of the row;
//   2. filter: the row is streamed once (4 x float4 per thread in flight);
//      survivors' columns are appended to a shared list with one warp scan
//      and one shared atomic per warp; their scores are then gathered back
//      (L2 hits) into 64-bit composites;
//   3. if the list holds between k and its capacity, the bucket finish
//      (descending scan, scatter of the buckets above rank k, rank inside
//      each small bucket) writes the top k sorted. Degenerate buckets (heavy
//      ties) take a shared-memory radix select + bitonic sort instead.
// When the sample mispredicts (fewer than k or more than capacity survivors)
// the row falls back to an exact MSB-first radix select over global memory
// with index-ordered tie collection. Rows with n <= capacity skip sampling.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// A CTA may host several row groups of kThreads threads (the persistent
// select_fat_kernel); every row-stage helper works on its group: gtid() is
// the thread's index in the group and csync() the group's own barrier.
__device__ __forceinline__ int gtid() { return static_cast<int>(threadIdx.x) & (kThreads - 1); }
__device__ __forceinline__ int gidx() { return static_cast<int>(threadIdx.x) / kThreads; }
__device__ __forceinline__ void csync() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + gidx()), "n"(kThreads) : "memory");
}
constexpr int kBins = 2048;
constexpr int kMaxRowGroups = 4;  // row groups per CTA (select_fat_kernel uses kFatGroups)
constexpr int kMaxTake = 4096;    // largest min(k, n) a row may select
constexpr int kMaxCand = 8192;    // largest shared candidate list
constexpr int kGatherPer = 16;     // survivors per thread the fused gather handles (4096)
// two-level select only pays when a row spans many more 32-key groups than
// k (it reads ~k groups instead of the whole row)
constexpr int kTwoLevelMinGroupsPerK = 2;
constexpr int kSampleSegs = 64;    // 512-byte segments: <= 8192 sampled keys per row
// Sample size: by default enough 128-key segments that the threshold sits
// near rank CSAIDX_SAMPLE_RANK of the sample (n / (2 target) keys per
// segment: 1/16 of the row at k = 512, 1/32 at k = 1024, 1/8 at k = 256);
// CSAIDX_SAMPLE_DIV > 0 fixes one segment per that many keys instead (round
// 1: 2048). Measured (profiles/r02_experiments.md): k = 256 rows 0.149 ->
// 0.071 ms (sampled-threshold misses 12 -> 0 per 2048 rows), C3 select -2-3%,
// C2 unchanged.
#ifndef CSAIDX_SAMPLE_DIV
#define CSAIDX_SAMPLE_DIV 0
#endif
#ifndef CSAIDX_SAMPLE_RANK
#define CSAIDX_SAMPLE_RANK 64        // (CSAIDX_SAMPLE_DIV == 0) expected sample rank of the threshold
#endif
#ifndef CSAIDX_TARGET_X4
#define CSAIDX_TARGET_X4 8           // expected survivors of the threshold = k * this / 4
#endif
#ifndef CSAIDX_TAU_BINS
#define CSAIDX_TAU_BINS 1024         // value-linear bins of the sampled threshold
#endif
constexpr int kTauBins = CSAIDX_TAU_BINS;

#ifndef CSAIDX_FIN_BINS
#define CSAIDX_FIN_BINS 1024
#endif
constexpr int kFinBins = CSAIDX_FIN_BINS;  // value-linear buckets of the bucket finish
// histogram region: the threshold's kBins bins, or the finish's start + cur
constexpr int kHistWords = 2 * kFinBins > kBins ? 2 * kFinBins : kBins;
constexpr int kMaxBucket = 128;  // largest bucket the finish ranks pairwise

struct Layout {
    int cand_cap;  // power of two, >= 2k
    int buf_cap;   // >= pow2(k) (radix path) and >= k + kMaxBucket (bucket finish)
};

__host__ __device__ inline int pow2_at_least(int x) {
#ifdef __CUDA_ARCH__
    return x <= 1 ? 1 : 1 << (32 - __clz(x - 1));  // one instruction instead of a loop per call
#else
    int p = 1;
    while (p < x) p <<= 1;
    return p;
#endif
}

__host__ __device__ inline Layout layout_for(int k) {
    Layout l;
    int c = pow2_at_least(3 * k);
    l.cand_cap = c < 2048 ? 2048 : (c > kMaxCand ? kMaxCand : c);
    l.buf_cap = pow2_at_least(k);
    if (l.buf_cap < k + kMaxBucket) l.buf_cap = k + kMaxBucket;
    return l;
}

__host__ __device__ inline size_t smem_bytes_for(int k) {
    const Layout l = layout_for(k);
    return static_cast<size_t>(l.cand_cap + l.buf_cap) * sizeof(uint64_t) + kHistWords * sizeof(uint32_t) +
           (4 * kWarps + 16) * sizeof(uint32_t);
}

__device__ __forceinline__ uint64_t composite(uint32_t key, int64_t col) {
    return (static_cast<uint64_t>(key) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(col + 1));
}

__device__ __forceinline__ int64_t composite_col(uint64_t c) {
    return static_cast<int64_t>(~static_cast<uint32_t>(c)) - 1;
}

// Descending bitonic sort of a[0, P), P a power of two, whole block.
__device__ void bitonic_sort_desc(uint64_t* a, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = gtid(); i < P / 2; i += kThreads) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint64_t x = a[lo], y = a[hi];
                if (desc ? (x < y) : (x > y)) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            csync();
        }
    }
}

// Descending bitonic sort of a[0, P) with P == E * kThreads: each thread
// holds E consecutive elements in registers; strides < E are in-register,
// strides < 32E go through warp shuffles, and only the strides that cross
// warps touch shared memory (6 barrier stages for P = 1024 instead of 55).
// Fully unrolled (size and stride are compile-time), so every per-stage
// predicate is one bit test of the thread index and each element costs a
// shuffle pair, one 64-bit compare and one select.
template <int E>
__device__ __forceinline__ void bitonic_sort_desc_regs(uint64_t* a) {
    constexpr int P = E * kThreads;
    const int t = gtid();
    uint64_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = a[t * E + e];
#pragma unroll
    for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride < E) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int pe = e ^ stride;
                    if (pe > e) {
                        const bool desc = ((t * E + e) & size) == 0;
                        const uint64_t lo = x[e], hi = x[pe];
                        const bool swap = desc ? (lo < hi) : (lo > hi);
                        x[e] = swap ? hi : lo;
                        x[pe] = swap ? lo : hi;
                    }
                }
            } else {
                // both bits come from the thread index: uniform over e
                const bool lower = (t & (stride / E)) == 0;
                const bool desc = (t & (size / E)) == 0 || size >= P;
                const bool keep_max = lower == desc;
                if (stride < 32 * E) {
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint64_t other = __shfl_xor_sync(0xffffffffu, x[e], stride / E);
                        x[e] = ((x[e] > other) == keep_max) ? x[e] : other;
                    }
                } else {
                    csync();
#pragma unroll
                    for (int e = 0; e < E; ++e) a[t * E + e] = x[e];
                    csync();
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const uint64_t other = a[(t * E + e) ^ stride];
                        x[e] = ((x[e] > other) == keep_max) ? x[e] : other;
                    }
                }
            }
        }
    }
    csync();
#pragma unroll
    for (int e = 0; e < E; ++e) a[t * E + e] = x[e];
    csync();
}

__device__ void sort_desc(uint64_t* a, int P) {
    switch (P / kThreads) {
        case 1: bitonic_sort_desc_regs<1>(a); break;
        case 2: bitonic_sort_desc_regs<2>(a); break;
        case 4: bitonic_sort_desc_regs<4>(a); break;
        case 8: bitonic_sort_desc_regs<8>(a); break;
        default: bitonic_sort_desc(a, P); break;  // P < blockDim or very large
    }
}

// Block-parallel search of the bin (counting from the top) holding the
// kk-th largest element: every thread sums a run of bins, a block scan
// locates the run, its owner walks it. out3 = {bin, count above, bin count}.
__device__ void find_bin(const uint32_t* hist, int nbins, uint32_t kk, uint32_t* out3, uint32_t* wsum) {
    const int lane = gtid() & 31, warp = gtid() >> 5;
    const int per = nbins >= kThreads ? nbins / kThreads : 1;
    const int hi = nbins - gtid() * per;  // thread 0 owns the highest bins
    uint32_t sum = 0;
    for (int b = hi - 1; b >= hi - per && b >= 0; --b) sum += hist[b];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    csync();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const uint32_t excl = before + incl - sum;
    if (sum > 0 && excl < kk && kk <= excl + sum) {
        uint32_t cum = excl;
        for (int b = hi - 1; b >= hi - per && b >= 0; --b) {
            const uint32_t c = hist[b];
            if (cum + c >= kk) {
                out3[0] = static_cast<uint32_t>(b);
                out3[1] = cum;
                out3[2] = c;
                break;
            }
            cum += c;
        }
    }
    csync();
}

// Exactly the kk largest of the unique 64-bit values a[0, n) (shared memory)
// into dst[0, kk), unordered. MSB-first radix select starting below the
// common prefix of the list's min and max (candidates are the top few percent
// of a row and share their leading bits); usually two 11-bit passes.
__device__ void smem_take_top(const uint64_t* a, int n, uint32_t kk, uint64_t* dst, uint32_t* hist, uint32_t* res,
                              uint32_t* wsum, uint32_t* counter) {
    // one min/max pair per row group (the persistent kernel's groups share
    // the CTA's static shared memory)
    __shared__ unsigned long long s_mm_all[kMaxRowGroups][2];
    unsigned long long* s_mm = s_mm_all[gidx()];
    const int lane = gtid() & 31;
    if (gtid() == 0) {
        s_mm[0] = ~0ull;
        s_mm[1] = 0ull;
        *counter = 0;
    }
    csync();
    unsigned long long mn = ~0ull, mx = 0ull;
    for (int i = gtid(); i < n; i += kThreads) {
        mn = min(mn, static_cast<unsigned long long>(a[i]));
        mx = max(mx, static_cast<unsigned long long>(a[i]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
        atomicMin(&s_mm[0], mn);
        atomicMax(&s_mm[1], mx);
    }
    csync();
    const uint64_t lo = s_mm[0], hi = s_mm[1];
    int pbits = lo == hi ? 64 : __clzll(static_cast<long long>(lo ^ hi));
    uint64_t prefix = pbits == 0 ? 0ull : (pbits == 64 ? lo : (lo >> (64 - pbits)));
    while (pbits < 64) {
        const int wbits = 64 - pbits < 11 ? 64 - pbits : 11;
        const int shift = 64 - pbits - wbits;
        for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
        csync();
        for (int i = gtid(); i < n; i += kThreads) {
            const uint64_t v = a[i];
            if (pbits == 0 || (v >> (64 - pbits)) == prefix)
                atomicAdd(&hist[static_cast<uint32_t>(v >> shift) & ((1u << wbits) - 1u)], 1u);
        }
        csync();
        find_bin(hist, 1 << wbits, kk, res, wsum);
        const uint32_t bin = res[0], above = res[1], cnt = res[2];
        csync();
        kk -= above;
        prefix = (pbits == 0 ? 0ull : (prefix << wbits)) | bin;
        pbits += wbits;
        if (cnt == kk) break;  // the whole bucket is in: exactly kk remain
    }
    // keep the values whose top pbits are >= prefix (exactly the requested count)
    const int nr = (n + 31) & ~31;
    for (int i = gtid(); i < nr; i += kThreads) {
        const uint64_t v = i < n ? a[i] : 0ull;
        const bool keep = i < n && (pbits >= 64 ? v >= prefix : (v >> (64 - pbits)) >= prefix);
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        uint32_t base = 0;
        if (lane == 0 && m != 0) base = atomicAdd(counter, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) dst[base + __popc(m & ((1u << lane) - 1u))] = v;
    }
    csync();
}

// Value-linear bucket of a composite between the list's min (lo) and max.
__device__ __forceinline__ int fin_bin(uint64_t c, float lo, float scale) {
    const float v = ord_key_to_float(static_cast<uint32_t>(c >> 32));
    return static_cast<int>(fminf(fmaxf((v - lo) * scale, 0.f), static_cast<float>(kFinBins - 1)));
}

// The top `take` of the unique composites a[0, n), sorted best first, into
// a[0, take): one histogram over kFinBins buckets linear in the score value
// (monotone, so bucket order is score order), a descending scan, a scatter
// of only the buckets that start above rank `take` into tmp[], and each
// scattered element's rank inside its bucket by pairwise comparison (buckets
// hold a few entries). Replaces a radix select + a k-wide bitonic sort.
// Returns false with a[] untouched when a needed bucket exceeds kMaxBucket
// or tmp[] (heavy ties, degenerate ranges); the caller then takes the radix
// path. start/cur: kFinBins words each; sc: 4 scratch words. With
// `prebuilt` the caller has already counted a[] into start[] over the bins
// (plo, pscale).
__device__ bool bucket_finish(uint64_t* a, int n, int take, uint64_t* tmp, int tmp_cap, uint32_t* start,
                              uint32_t* cur, uint32_t* wsum, uint32_t* sc, bool prebuilt, float plo, float pscale) {
    const int lane = gtid() & 31, warp = gtid() >> 5;
    if (gtid() == 0) {
        sc[0] = 0xffffffffu;  // min key
        sc[1] = 0u;           // max key
        sc[2] = 0u;           // overflow flag
        sc[3] = 0u;           // scattered extent
    }
    float lo = plo, scale = pscale;  // prebuilt: start[] already holds the histogram over (plo, pscale)
    if (!prebuilt) {
        for (int i = gtid(); i < kFinBins; i += kThreads) start[i] = 0;
        uint32_t kmin = 0xffffffffu, kmax = 0u;
        for (int i = gtid(); i < n; i += kThreads) {
            const uint32_t key = static_cast<uint32_t>(a[i] >> 32);
            kmin = min(kmin, key);
            kmax = max(kmax, key);
        }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        kmax = __reduce_max_sync(0xffffffffu, kmax);
        csync();
        if (lane == 0) {
            atomicMin(&sc[0], kmin);
            atomicMax(&sc[1], kmax);
        }
        csync();
        lo = ord_key_to_float(sc[0]);
        const float hi = ord_key_to_float(sc[1]);
        scale = static_cast<float>(kFinBins) / (hi - lo);
        if (!(hi > lo) || !isfinite(scale)) scale = 0.f;
        for (int i = gtid(); i < n; i += kThreads) atomicAdd(&start[fin_bin(a[i], lo, scale)], 1u);
    }
    csync();
    // descending exclusive scan: thread t owns bins [NB-4t-4, NB-4t), highest first
    constexpr int kPer = kFinBins / 256;
    static_assert(kFinBins % 256 == 0, "bins per thread");
    uint32_t c[kPer];
    uint32_t sum = 0;
    const int top = kFinBins - 1 - kPer * gtid();
    if (gtid() < 256) {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            c[u] = start[top - u];
            sum += c[u];
        }
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    csync();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (gtid() < 256) {
        uint32_t run = before + incl - sum;
        const uint32_t tk = static_cast<uint32_t>(take);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int b = top - u;
            start[b] = run;
            cur[b] = run;
            if (run < tk) {
                if (c[u] > static_cast<uint32_t>(kMaxBucket) || run + c[u] > static_cast<uint32_t>(tmp_cap)) sc[2] = 1u;
                if (run + c[u] >= tk) sc[3] = run + c[u];  // the bucket holding rank `take`
            }
            run += c[u];
        }
    }
    csync();
    if (sc[2] != 0u) return false;
    const uint32_t extent = sc[3];
    for (int i = gtid(); i < n; i += kThreads) {
        const uint64_t v = a[i];
        const int b = fin_bin(v, lo, scale);
        if (start[b] < static_cast<uint32_t>(take)) tmp[atomicAdd(&cur[b], 1u)] = v;
    }
    csync();
    for (uint32_t s = gtid(); s < extent; s += kThreads) {
        const uint64_t v = tmp[s];
        const int b = fin_bin(v, lo, scale);
        const uint32_t b0 = start[b], b1 = cur[b];
        uint32_t r = 0;
        for (uint32_t j = b0; j < b1; ++j) r += tmp[j] > v ? 1u : 0u;
        if (b0 + r < static_cast<uint32_t>(take)) a[b0 + r] = v;
    }
    csync();
    return true;
}

// ------------------------------------------------------------------ fallback
// Exact MSB-first radix select over global memory (any n, any ties): the
// selected composites (unsorted) land in buf[0, k).

__device__ __forceinline__ bool prefix_match(uint32_t key, uint32_t prefix, int pbits) {
    return pbits == 0 || (key >> (32 - pbits)) == prefix;
}

__device__ void histogram_pass(const float* row, int64_t n, uint32_t prefix, int pbits, int wbits, uint32_t* hist) {
    for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
    csync();
    const int shift = 32 - pbits - wbits;
    const uint32_t mask = (1u << wbits) - 1u;
    for (int64_t i = gtid(); i < n; i += kThreads) {
        const uint32_t key = ord_key(__ldg(row + i));
        if (prefix_match(key, prefix, pbits)) atomicAdd(&hist[(key >> shift) & mask], 1u);
    }
    csync();
}

// Ordered (index-ascending) block compaction: entries above the prefix go to
// above_dst, entries equal to it to eq_dst (first eq_limit in index order).
__device__ void collect_pass(const float* row, int64_t n, uint32_t prefix, int pbits, uint64_t* above_dst,
                             uint64_t* eq_dst, uint32_t eq_limit, uint32_t* wtot) {
    const int lane = gtid() & 31;
    const int warp = gtid() >> 5;
    uint32_t run_above = 0, run_eq = 0;
    int parity = 0;
    for (int64_t base = 0; base < n; base += kThreads) {
        const int64_t i = base + gtid();
        uint32_t key = 0;
        int cls = 0;
        if (i < n) {
            key = ord_key(__ldg(row + i));
            const uint32_t top = key >> (32 - pbits);
            cls = top > prefix ? 1 : (top == prefix ? 2 : 0);
        }
        const uint32_t ma = __ballot_sync(0xffffffffu, cls == 1);
        const uint32_t me = __ballot_sync(0xffffffffu, cls == 2);
        uint32_t* wt = wtot + parity * 2 * kWarps;
        if (lane == 0) {
            wt[warp] = __popc(ma);
            wt[kWarps + warp] = __popc(me);
        }
        csync();
        uint32_t off_a = 0, off_e = 0, tot_a = 0, tot_e = 0;
        for (int w = 0; w < kWarps; ++w) {
            if (w < warp) {
                off_a += wt[w];
                off_e += wt[kWarps + w];
            }
            tot_a += wt[w];
            tot_e += wt[kWarps + w];
        }
        const uint32_t lt = (1u << lane) - 1u;
        if (cls == 1) above_dst[run_above + off_a + __popc(ma & lt)] = composite(key, i);
        if (cls == 2) {
            const uint32_t pe = run_eq + off_e + __popc(me & lt);
            if (pe < eq_limit) eq_dst[pe] = composite(key, i);
        }
        run_above += tot_a;
        run_eq += tot_e;
        parity ^= 1;
    }
    csync();
}

__device__ void exact_global_select(const float* row, int64_t n, int k, uint64_t* buf, uint64_t* cand, int cand_cap,
                                    uint32_t* hist, uint32_t* wtot, uint32_t* res, uint32_t* wsum) {
    uint32_t prefix = 0;
    int pbits = 0;
    uint32_t kk = static_cast<uint32_t>(k);
    uint32_t bin_count = 0;
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
        const int wbits = pass == 2 ? 10 : 11;
        histogram_pass(row, n, prefix, pbits, wbits, hist);
        find_bin(hist, 1 << wbits, kk, res, wsum);
        kk -= res[1];
        bin_count = res[2];
        prefix = (pbits == 0 ? 0u : (prefix << wbits)) | res[0];
        pbits += wbits;
        csync();
        if (bin_count <= static_cast<uint32_t>(cand_cap)) break;
    }
    const uint32_t above = static_cast<uint32_t>(k) - kk;
    if (pbits == 32) {
        // a single key value: its first kk entries in index order
        collect_pass(row, n, prefix, pbits, buf, buf + above, kk, wtot);
    } else {
        collect_pass(row, n, prefix, pbits, buf, cand, static_cast<uint32_t>(cand_cap), wtot);
        const int P = pow2_at_least(static_cast<int>(bin_count));
        for (int i = static_cast<int>(bin_count) + gtid(); i < P; i += kThreads) cand[i] = 0;
        csync();
        sort_desc(cand, P);
        for (uint32_t i = gtid(); i < kk; i += kThreads) buf[above + i] = cand[i];
    }
    csync();
}

// ------------------------------------------------------------------ shared row stages

// Survivor columns idx_list[0, count) of `row` -> 64-bit composites in
// cand[0, count) (their scores were just streamed: L2 hits; each thread's
// loads are all in flight at once). When count fits the fused form the
// finish buckets over [lo_f, hi_f] (threshold, sample max) are counted into
// hist[0, kFinBins) on the way (prebuilt). count < 0: nothing to do.
__device__ void gather_candidates(const float* row, const uint32_t* idx_list, int count, uint64_t* cand,
                                  uint32_t* hist, float lo_f, uint32_t* max_slot, bool& prebuilt, float& pb_lo,
                                  float& pb_scale, bool build_hist = true) {
    if (build_hist && count >= 0 && count <= kGatherPer * kThreads) {
        // every survivor's score in registers first: the finish buckets span
        // [threshold, the survivors' true maximum] (the sample maximum would
        // leave the scores above it in one clamped top bucket, whose pairwise
        // ranking is quadratic and which can overflow into the slow path)
        uint32_t cc[kGatherPer];
        float vv[kGatherPer];
#pragma unroll
        for (int g = 0; g < kGatherPer; ++g) {
            const int i = gtid() + g * kThreads;
            cc[g] = i < count ? idx_list[i] : 0u;
        }
#pragma unroll
        for (int g = 0; g < kGatherPer; ++g)
            vv[g] = gtid() + g * kThreads < count ? __ldg(row + cc[g]) : -INFINITY;
        float vmax = -INFINITY;
#pragma unroll
        for (int g = 0; g < kGatherPer; ++g) vmax = fmaxf(vmax, vv[g]);
        const uint32_t kmax = __reduce_max_sync(0xffffffffu, vmax > -INFINITY ? ord_key(vmax) : 0u);
        if (gtid() == 0) *max_slot = 0u;
        csync();  // the list (it may alias hist) is consumed; max_slot reset
        for (int i = gtid(); i < kFinBins; i += kThreads) hist[i] = 0;
        if ((gtid() & 31) == 0) atomicMax(max_slot, kmax);
        csync();
        const float hi_f = ord_key_to_float(*max_slot);
        pb_lo = lo_f;
        pb_scale = static_cast<float>(kFinBins) / (hi_f - lo_f);
        if (!(hi_f > lo_f) || !isfinite(pb_scale)) pb_scale = 0.f;
#pragma unroll
        for (int g = 0; g < kGatherPer; ++g) {
            const int i = gtid() + g * kThreads;
            if (i < count) {
                const uint64_t c = composite(ord_key(vv[g]), cc[g]);
                cand[i] = c;
                atomicAdd(&hist[fin_bin(c, pb_lo, pb_scale)], 1u);
            }
        }
        prebuilt = true;
    } else if (count >= 0) {
        constexpr int G = 8;
        for (int base = gtid(); base < count; base += G * kThreads) {
            uint32_t cc[G];
            float vv[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int i = base + g * kThreads;
                cc[g] = i < count ? idx_list[i] : 0u;
            }
#pragma unroll
            for (int g = 0; g < G; ++g) vv[g] = base + g * kThreads < count ? __ldg(row + cc[g]) : 0.f;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int i = base + g * kThreads;
                if (i < count) cand[i] = composite(ord_key(vv[g]), cc[g]);
            }
        }
    }
    csync();
}

// The sorted top `take` of a row. count >= 0: from the unique candidates
// cand[0, count) (bucket finish, or for heavy ties a shared-memory radix
// select + register bitonic sort); count < 0 (the threshold mispredicted):
// exact radix select over the row in global memory. Returns the array that
// holds the result (cand or buf).
__device__ const uint64_t* finish_row(const float* row, int64_t n, int take, int count, const Layout& L,
                                      uint64_t* cand, uint64_t* buf, uint32_t* hist, uint32_t* wtot,
                                      uint32_t* wsum, uint32_t* res, uint32_t* counter, bool prebuilt, float pb_lo,
                                      float pb_scale, int* fallbacks) {
    if (count >= 0) {
        if (bucket_finish(cand, count, take, buf, L.buf_cap, hist, hist + kFinBins, wsum, res, prebuilt, pb_lo,
                          pb_scale))
            return cand;
        if (count > take) {
            smem_take_top(cand, count, static_cast<uint32_t>(take), buf, hist, res, wsum, counter);
        } else {
            for (int i = gtid(); i < count; i += kThreads) buf[i] = cand[i];
        }
    } else {
        if (gtid() == 0 && fallbacks != nullptr) atomicAdd(fallbacks, 1);
        exact_global_select(row, n, take, buf, cand, L.cand_cap, hist, wtot, res, wsum);
    }
    const int P = pow2_at_least(take);
    for (int i = take + gtid(); i < P; i += kThreads) buf[i] = 0;
    csync();
    sort_desc(buf, P);
    return buf;
}

// Output row: the first `take` entries of result (best first), the rest
// (-inf, -1); int32 candidate rows, or with final_idx the int64 output rows
// of the fused sentinel pass (finalize_kernel semantics).
__device__ void write_row(const SelectParams& p, int b, int64_t row_id, int take, const uint64_t* result) {
    const bool final_out = p.final_idx != nullptr || p.sink_only;
    const int64_t orow = final_out ? static_cast<int64_t>(b) * p.final_rows + p.final_row0 + row_id
                                   : static_cast<int64_t>(b) * p.rows + row_id;
    const float neg_inf = -__int_as_float(0x7f800000);
    if (final_out) {
        // sink_only: the int32 sink row is the only output (a query-sharded
        // rank whose rows are collected in rank 0's buffer)
        float* ov = p.sink_only ? nullptr : p.out_val + orow * p.out_ld;
        int64_t* oi = p.sink_only ? nullptr : p.final_idx + orow * p.out_ld;
        int32_t* si = p.sink != nullptr ? p.sink + (static_cast<int64_t>(b) * p.sink_seq + p.s0 + row_id) * p.out_ld
                                        : nullptr;
        for (int e = gtid(); e < p.width; e += kThreads) {
            int64_t idx = -1;
            float v = neg_inf;
            if (e < take) {
                const uint64_t c = result[e];
                v = ord_key_to_float(static_cast<uint32_t>(c >> 32));
                idx = v == neg_inf ? -1 : composite_col(c) + p.t0;
            }
            if (ov != nullptr) ov[e] = v;
            if (oi != nullptr) oi[e] = idx;
            if (si != nullptr) si[e] = static_cast<int32_t>(idx);  // peer store when the sink is remote
        }
        if (si != nullptr) __threadfence_system();  // the peer stores are performed before the kernel retires
        return;
    }
    float* ov = p.out_val + orow * p.out_ld;
    int32_t* oi = p.out_idx + orow * p.out_ld;
    for (int e = gtid(); e < p.width; e += kThreads) {
        if (e < take) {
            const uint64_t c = result[e];
            ov[e] = ord_key_to_float(static_cast<uint32_t>(c >> 32));
            oi[e] = static_cast<int32_t>(composite_col(c) + p.t0);
        } else {
            ov[e] = neg_inf;
            oi[e] = -1;
        }
    }
}

// Sampled threshold of a long row (n > cand_cap): evenly spaced 512-byte
// segments (one float4 per lane, <= 8192 values; about 64 sampled scores lie
// above the threshold) held in registers, value-linear histograms over the
// sample's range (plus one refinement pass inside a coarse rank bin) -> a
// threshold expected to keep ~2k of the row's entries. Uses hist (kTauBins
// words), res, wsum, counter.
__device__ __forceinline__ float sample_threshold(const float* row, int64_t n, int k, const Layout& L, uint32_t* hist,
                                               uint32_t* res, uint32_t* wsum, uint32_t* counter) {
    const int lane = gtid() & 31;
    // sample evenly spaced 512-byte segments (one float4 per lane,
    //    ~1/16 of the row, <= 8192 values), held in registers; each
    //    warp issues all of its loads before consuming them
    // 32-bit arithmetic: a row's legal length is < 2^31 (n <= T)
    const int n32 = static_cast<int>(n);
    // ~2k survivors: a comfortable margin over k (misses -> the slow
    // exact fallback) while the shared list stays at <= 4k entries
    const int want = (k * CSAIDX_TARGET_X4) / 4;
    const int target = (want < (L.cand_cap * 3) / 4) ? want : (L.cand_cap * 3) / 4;
#if CSAIDX_SAMPLE_DIV > 0
    int nseg = static_cast<int>(n / CSAIDX_SAMPLE_DIV);
#else
    // sample size for a rank of ~CSAIDX_SAMPLE_RANK inside the sample,
    // whatever k: segments of 128 keys, ns / n = rank / target
    int nseg = static_cast<int>((static_cast<int64_t>(n32) * CSAIDX_SAMPLE_RANK) / (128 * static_cast<int64_t>(target)));
#endif
    if (nseg > kSampleSegs) nseg = kSampleSegs;
    if (nseg < 1) nseg = 1;
    const int64_t seg_stride = (n32 / nseg) & ~3;
    constexpr int kSegsPerWarp = kSampleSegs / kWarps;  // 8
    const int w = gtid() >> 5;
    float4 sv[kSegsPerWarp];
#pragma unroll
    for (int u = 0; u < kSegsPerWarp; ++u) {
        const int sg = w + u * kWarps;
        sv[u] = sg < nseg ? __ldg(reinterpret_cast<const float4*>(row + sg * seg_stride) + lane)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int u = 0; u < kSegsPerWarp; ++u) {
        if (w + u * kWarps < nseg) {
            const uint32_t k0 = ord_key(sv[u].x), k1 = ord_key(sv[u].y);
            const uint32_t k2 = ord_key(sv[u].z), k3 = ord_key(sv[u].w);
            kmin = min(kmin, min(min(k0, k1), min(k2, k3)));
            kmax = max(kmax, max(max(k0, k1), max(k2, k3)));
        }
    }
    if (gtid() == 0) {
        *counter = 0;
        res[0] = res[1] = res[2] = 0u;  // find_bin leaves them when the rank is out of range
        res[6] = 0xffffffffu;
        res[7] = 0u;
    }
    for (int i = gtid(); i < kTauBins; i += kThreads) hist[i] = 0;
    csync();
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) {
        atomicMin(&res[6], kmin);
        atomicMax(&res[7], kmax);
    }
    csync();
    const int ns = 128 * nseg;
    int r = (target * ns) / n32;  // <= 6144 * 8192: no overflow
    if (r < 1) r = 1;
    // The sample's rank-r value by value-linear histograms over
    // [sample min, sample max]: one pass, plus a refinement pass
    // inside the rank-r bin when that bin is coarse (outliers,
    // heavy tails). tau = the lower edge of the final bin.
    const float smin = ord_key_to_float(res[6]), smax = ord_key_to_float(res[7]);
    float lo = smin, hi = smax;
    uint32_t rr = static_cast<uint32_t>(r);
    float tau_f = smin;
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        float scale = static_cast<float>(kTauBins) / (hi - lo);
        if (!(hi > lo) || !isfinite(scale)) break;  // degenerate: keep tau = lo
        if (pass > 0) {
            for (int i = gtid(); i < kTauBins; i += kThreads) hist[i] = 0;
            if (gtid() == 0) res[0] = res[1] = res[2] = 0u;
            csync();
        }
#pragma unroll
        for (int u = 0; u < kSegsPerWarp; ++u) {
            if (w + u * kWarps < nseg) {
                const float vs[4] = {sv[u].x, sv[u].y, sv[u].z, sv[u].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float v = vs[c];
                    if (v >= lo && v <= hi)
                        atomicAdd(&hist[static_cast<int>(fminf((v - lo) * scale, static_cast<float>(kTauBins - 1)))],
                                  1u);
                }
            }
        }
        csync();
        find_bin(hist, kTauBins, rr, res, wsum);
        const uint32_t bin = res[0], above = res[1], cnt = res[2];
        csync();
        const float width = (hi - lo) / static_cast<float>(kTauBins);
        const float blo = lo + static_cast<float>(bin) * width;
        tau_f = blo > lo ? blo : lo;
        if (cnt * 8u <= rr || cnt <= 4u) break;  // fine enough
        rr -= above;
        hi = fminf(hi, blo + width);
        lo = tau_f;
    }
    // scores are compared as floats: ord_key is monotone and folds
    // -0.0 onto +0.0 exactly like the float order
    if (tau_f == 0.f) tau_f = 0.f;  // -0.0 -> +0.0

    return tau_f;
}

// One streaming pass over a long row keeping the entries >= tau_f: survivor
// columns listed in the buf + hist region (warp scan + one shared atomic per
// warp), then gathered back (L2 hits) into the composites cand[0, count) with
// the finish histogram prebuilt. Returns count (-1: the threshold kept fewer
// than k or more than the list holds -> exact fallback).
template <int kUnroll>
__device__ __forceinline__ int stream_collect(const float* row, int64_t n, int k, float tau_f, const Layout& L,
                                              uint64_t* cand, uint64_t* buf, uint32_t* hist, uint32_t* res,
                                              uint32_t* counter, bool& prebuilt, float& pb_lo, float& pb_scale) {
    const int lane = gtid() & 31;
    const uint32_t tau = ord_key(tau_f);
    if (gtid() == 0) *counter = 0;
    csync();
    int count = -1;
    // survivors are recorded as column indices only (the composites
    // are gathered after the pass); the list aliases buf + hist
    uint32_t* idx_list = reinterpret_cast<uint32_t*>(buf);

    // 2. stream the row once; keep entries >= tau
    const float4* row4 = reinterpret_cast<const float4*>(row);
    const int64_t n4 = n >> 2;
    const int64_t step = kUnroll * static_cast<int64_t>(kThreads);
    const int64_t n4r = (n4 + step - 1) / step * step;
    const uint32_t cap = static_cast<uint32_t>(
        min(L.cand_cap, 2 * L.buf_cap + kHistWords));  // idx list capacity
    for (int64_t it = gtid(); it < n4r; it += step) {
        float4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int64_t i4 = it + u * kThreads;
            v[u] = i4 < n4 ? __ldg(row4 + i4) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
        // one bit per entry: 4 * kUnroll bits (64-bit mask above 8 float4)
        using Mask = typename std::conditional<(kUnroll > 8), unsigned long long, uint32_t>::type;
        Mask m = 0;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            m |= static_cast<Mask>(v[u].x >= tau_f ? 1u : 0u) << (4 * u + 0);
            m |= static_cast<Mask>(v[u].y >= tau_f ? 1u : 0u) << (4 * u + 1);
            m |= static_cast<Mask>(v[u].z >= tau_f ? 1u : 0u) << (4 * u + 2);
            m |= static_cast<Mask>(v[u].w >= tau_f ? 1u : 0u) << (4 * u + 3);
        }
        if (!__any_sync(0xffffffffu, m != 0)) continue;
        const uint32_t c = kUnroll > 8 ? __popcll(m) : __popc(static_cast<uint32_t>(m));
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t base = 0;
        if (lane == 31) base = atomicAdd(counter, incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint32_t pos = base + incl - c;
        // Survivors are ~6% of entries: walk only the set bits (the
        // warp iterates max-popc times, usually 2-4) and record the
        // column only: the divergent body stays a handful of
        // instructions.
        while (m != 0) {
            const int bit = kUnroll > 8 ? __ffsll(static_cast<long long>(m)) - 1
                                        : __ffs(static_cast<int>(m)) - 1;
            m &= m - 1;
            if (pos < cap)
                idx_list[pos] = static_cast<uint32_t>(4 * (it + (bit >> 2) * kThreads) + (bit & 3));
            ++pos;
        }
    }
    if (gtid() < 32) {  // the < 4 entries past the last float4
        const int64_t i = 4 * n4 + lane;
        const bool inb = i < n;
        const uint32_t key = inb ? ord_key(__ldg(row + i)) : 0u;
        const bool pass = inb && key >= tau;
        const uint32_t mm = __ballot_sync(0xffffffffu, pass);
        if (mm != 0) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(counter, __popc(mm));
            base = __shfl_sync(0xffffffffu, base, 0);
            const uint32_t pos = base + __popc(mm & ((1u << lane) - 1u));
            if (pass && pos < cap) idx_list[pos] = static_cast<uint32_t>(i);
        }
    }
    csync();
    const uint32_t total = *counter;
    count = (total >= static_cast<uint32_t>(k) && total <= cap) ? static_cast<int>(total) : -1;
    gather_candidates(row, idx_list, count, cand, hist, tau_f, res + 5, prebuilt, pb_lo, pb_scale);
    return count;
}

// ------------------------------------------------------------------ kernel


// One row (b, row_id) on one row group, with that group's shared memory.
template <int kUnroll>
__device__ __forceinline__ void select_row(const SelectParams& p, int b, int64_t row_id, uint8_t* smem_raw) {
    const int k = p.k;
    const Layout L = layout_for(k);
    uint64_t* cand = reinterpret_cast<uint64_t*>(smem_raw);  // [cand_cap]
    uint64_t* buf = cand + L.cand_cap;                       // [buf_cap]
    uint32_t* hist = reinterpret_cast<uint32_t*>(buf + L.buf_cap);
    uint32_t* wtot = hist + kHistWords;                           // [2][2*kWarps]
    uint32_t* wsum = wtot + 4 * kWarps;                      // [kWarps] (find_bin)
    uint32_t* res = wsum + kWarps;                           // [8]
    uint32_t* counter = res + 4;

    int64_t n = p.cols;
    if (p.apply_mask) {
        n = (p.s0 + row_id + 1) / p.ratio - p.t0;
        n = n < 0 ? 0 : (n > p.cols ? p.cols : n);
    }
    const float* row = p.scores + (static_cast<int64_t>(b) * p.rows + row_id) * p.ld;
    const int take = static_cast<int>(n < k ? n : k);
    const int lane = gtid() & 31;

    const uint64_t* result = buf;  // sorted selection, best first (buf or cand)
    long long* clk = p.phase_clk != nullptr && gtid() == 0 && b == 0 ? p.phase_clk + row_id * 8 : nullptr;
    if (clk) clk[0] = clock64();
    if (take > 0) {
        int count = -1;  // candidates in cand[], or -1 -> fallback
        int pre = -1;    // candidates flagged by the score epilogue, if usable
        bool prebuilt = false;  // finish histogram built by the gather
        float pb_lo = 0.f, pb_scale = 0.f;
        if (p.pass_bits != nullptr) {
            // The bitmap flags every legal score >= the row's tau; when the
            // flagged count lies in [take, cand_cap] the flagged entries
            // contain the exact top-take and fit the list.
            const uint32_t* bits = p.pass_bits + (static_cast<int64_t>(b) * p.rows + row_id) * p.bits_ld;
            const int nw = static_cast<int>((n + 31) >> 5);
            if (gtid() == 0) *counter = 0;
            csync();
            uint32_t loc = 0;
            for (int i = gtid(); i < nw; i += kThreads) loc += __popc(__ldg(bits + i));
            loc = __reduce_add_sync(0xffffffffu, loc);
            if (lane == 0 && loc != 0) atomicAdd(counter, loc);
            csync();
            const uint32_t tot = *counter;
            csync();
            if (tot >= static_cast<uint32_t>(take) && tot <= static_cast<uint32_t>(L.cand_cap)) {
                if (gtid() == 0) *counter = 0;
                csync();
                for (int i = gtid(); i < nw; i += kThreads) {
                    uint32_t m = __ldg(bits + i);
                    if (m == 0) continue;
                    uint32_t pos = atomicAdd(counter, static_cast<uint32_t>(__popc(m)));
                    while (m != 0) {
                        const int j = i * 32 + __ffs(m) - 1;
                        m &= m - 1;
                        cand[pos++] = composite(ord_key(__ldg(row + j)), j);
                    }
                }
                pre = static_cast<int>(tot);
                if (gtid() == 0 && p.cand_hits != nullptr) atomicAdd(p.cand_hits, 1);
                csync();
            }
        }
        bool have = false;  // candidates ready in cand[0, count)
        if (pre >= 0) {
            count = pre;
            have = true;
        } else if (n <= L.cand_cap) {
            for (int64_t i = gtid(); i < n; i += kThreads) cand[i] = composite(ord_key(__ldg(row + i)), i);
            count = static_cast<int>(n);
            csync();
            have = true;
        }
        const int ngroups = static_cast<int>((n + 31) >> 5);
        if (!have && p.gmax != nullptr && ngroups >= kTwoLevelMinGroupsPerK * k && ngroups <= 2 * L.cand_cap) {
            // Two-level select: with g_k the k-th largest 32-key group
            // maximum, at least k scores are >= g_k and every score >= g_k
            // lies in a group whose maximum is >= g_k. So only those groups
            // (about k of them) are read, and their entries >= g_k (about
            // 1.1-1.3 k) are the candidates. A threshold that admits fewer
            // than `take` or more than the list holds falls through to the
            // sampled path below (exact either way).
            const float* gmr = p.gmax + (static_cast<int64_t>(b) * p.rows + row_id) * p.gmax_ld;
            float* gsm = reinterpret_cast<float*>(cand);  // the row's group maxima
            if (gtid() == 0) {
                *counter = 0;
                res[0] = res[1] = res[2] = 0u;
                res[6] = 0xffffffffu;
                res[7] = 0u;
            }
            for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
            uint32_t kmin = 0xffffffffu, kmax = 0u;
            for (int g = gtid(); g < ngroups; g += kThreads) {
                const float v = __ldg(gmr + g);
                gsm[g] = v;
                const uint32_t key = ord_key(v);
                kmin = min(kmin, key);
                kmax = max(kmax, key);
            }
            kmin = __reduce_min_sync(0xffffffffu, kmin);
            kmax = __reduce_max_sync(0xffffffffu, kmax);
            csync();
            if (lane == 0) {
                atomicMin(&res[6], kmin);
                atomicMax(&res[7], kmax);
            }
            csync();
            const float gmin = ord_key_to_float(res[6]), gmaxv = ord_key_to_float(res[7]);
            float lo = gmin, hi = gmaxv, tau_g = gmin;
            uint32_t rr = static_cast<uint32_t>(take);
#pragma unroll 1
            for (int pass = 0; pass < 2; ++pass) {
                const float scale = static_cast<float>(kBins) / (hi - lo);
                if (!(hi > lo) || !isfinite(scale)) break;
                if (pass > 0) {
                    for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
                    if (gtid() == 0) res[0] = res[1] = res[2] = 0u;
                    csync();
                }
                for (int g = gtid(); g < ngroups; g += kThreads) {
                    const float v = gsm[g];
                    if (v >= lo && v <= hi)
                        atomicAdd(&hist[static_cast<int>(fminf((v - lo) * scale, static_cast<float>(kBins - 1)))], 1u);
                }
                csync();
                find_bin(hist, kBins, rr, res, wsum);
                const uint32_t bin = res[0], above = res[1], cnt = res[2];
                csync();
                const float width = (hi - lo) / static_cast<float>(kBins);
                const float blo = lo + static_cast<float>(bin) * width;
                tau_g = blo > lo ? blo : lo;
                if (cnt * 8u <= rr || cnt <= 4u) break;
                rr -= above;
                hi = fminf(hi, blo + width);
                lo = tau_g;
            }
            if (tau_g == 0.f) tau_g = 0.f;  // -0.0 -> +0.0
            // groups that can hold a score >= tau_g, listed in buf
            uint32_t* glist = reinterpret_cast<uint32_t*>(buf);
            const uint32_t gcap = static_cast<uint32_t>(2 * L.buf_cap);
            for (int g0 = 0; g0 < ngroups; g0 += kThreads) {
                const int g = g0 + gtid();
                const bool keep = g < ngroups && gsm[g] >= tau_g;
                const uint32_t m = __ballot_sync(0xffffffffu, keep);
                uint32_t base = 0;
                if (lane == 0 && m != 0) base = atomicAdd(counter, __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
                if (keep && pos < gcap) glist[pos] = static_cast<uint32_t>(g);
            }
            csync();
            const uint32_t ng = *counter;
            csync();
            if (ng <= gcap) {
                // one group (128 B, 8 x float4) per thread in flight; the
                // survivors' columns go to the list in the histogram region
                if (gtid() == 0) *counter = 0;
                csync();
                uint32_t* idx2 = hist;
                const uint32_t cap2 = static_cast<uint32_t>(kHistWords);
                for (uint32_t t = gtid(); t < ng; t += kThreads) {
                    const uint32_t g = glist[t];
                    const float4* src = reinterpret_cast<const float4*>(row + static_cast<int64_t>(g) * 32);
                    const int64_t lim = n - static_cast<int64_t>(g) * 32;  // valid columns in the group
                    // a partial last group loads only the float4s holding legal
                    // columns (the rest may lie past the row's allocation)
                    float4 v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = 4 * u < lim ? __ldg(src + u) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                    uint32_t m = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        m |= (v[u].x >= tau_g && 4 * u + 0 < lim ? 1u : 0u) << (4 * u + 0);
                        m |= (v[u].y >= tau_g && 4 * u + 1 < lim ? 1u : 0u) << (4 * u + 1);
                        m |= (v[u].z >= tau_g && 4 * u + 2 < lim ? 1u : 0u) << (4 * u + 2);
                        m |= (v[u].w >= tau_g && 4 * u + 3 < lim ? 1u : 0u) << (4 * u + 3);
                    }
                    if (m != 0) {
                        uint32_t pos = atomicAdd(counter, static_cast<uint32_t>(__popc(m)));
                        while (m != 0) {
                            const int bit = __ffs(m) - 1;
                            m &= m - 1;
                            if (pos < cap2) idx2[pos] = g * 32 + static_cast<uint32_t>(bit);
                            ++pos;
                        }
                    }
                }
                csync();
                const uint32_t total = *counter;
                csync();
                if (total >= static_cast<uint32_t>(take) && total <= cap2) {
                    count = static_cast<int>(total);
                    gather_candidates(row, idx2, count, cand, hist, tau_g, res + 5, prebuilt, pb_lo, pb_scale);
                    have = true;
                    if (gtid() == 0 && p.cand_hits != nullptr) atomicAdd(p.cand_hits, 1);
                }
            }
        }
        if (!have) {
            const float tau_f = sample_threshold(row, n, k, L, hist, res, wsum, counter);
            count = stream_collect<kUnroll>(row, n, k, tau_f, L, cand, buf, hist, res, counter, prebuilt, pb_lo,
                                            pb_scale);
        }

        if (clk) clk[2] = clock64();
        if (clk) {
            clk[6] = count;
            clk[7] = clock64();
        }
        result = finish_row(row, n, take, count, L, cand, buf, hist, wtot, wsum, res, counter, prebuilt, pb_lo,
                            pb_scale, p.fallbacks);
    }

    if (clk) {
        clk[3] = clock64();
        clk[4] = n;
    }
    write_row(p, b, row_id, take, result);
}

template <int kUnroll, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks) select_kernel(const SelectParams p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    select_row<kUnroll>(p, static_cast<int>(blockIdx.y), blockIdx.x, smem_raw);
}

// Persistent form for running beside the score kernel on a few SMs: one
// fat CTA per SM holding kFatGroups independent row groups (each its own
// shared memory slice and barrier) that walk the rows with a grid stride.
constexpr int kFatGroups = 3;
static_assert(kFatGroups <= kMaxRowGroups, "per-group static shared slots");

__global__ void __launch_bounds__(kThreads * kFatGroups, 1) select_fat_kernel(const SelectParams p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* mine = smem_raw + static_cast<size_t>(gidx()) * smem_bytes_for(p.k);
    const int64_t nrows = p.rows * p.batch;
    for (int64_t rr = static_cast<int64_t>(blockIdx.x) * kFatGroups + gidx(); rr < nrows;
         rr += static_cast<int64_t>(gridDim.x) * kFatGroups) {
        const int b = static_cast<int>(rr / p.rows);
        select_row<8>(p, b, rr - static_cast<int64_t>(b) * p.rows, mine);
        csync();  // the group's shared memory is reused by its next row
    }
}

// ------------------------------------------------------------------ tau
constexpr int kTauMaxSamples = 8192;

__global__ void __launch_bounds__(kThreads) tau_kernel(const TauParams p) {
    __shared__ uint32_t s_keys[kTauMaxSamples];
    __shared__ uint32_t hist[kBins];
    __shared__ uint32_t wsum[kWarps];
    __shared__ uint32_t res[8];
    const int64_t row_id = blockIdx.x;
    const int b = blockIdx.y;
    const int lane = gtid() & 31;
    int64_t n = (p.s0 + row_id + 1) / p.ratio - p.t0;
    n = n < 0 ? 0 : (n > p.cols ? p.cols : n);
    float* out = p.tau + static_cast<int64_t>(b) * p.rows + row_id;
    const float neg_inf = -__int_as_float(0x7f800000);
    if (n <= p.cand_cap) {  // the whole legal row fits the candidate list
        if (gtid() == 0) *out = neg_inf;
        return;
    }
    const int64_t vt = ((n + 127) / 128 + p.kt_stride - 1) / p.kt_stride;
    int64_t nv = vt * 128;
    if (nv > p.lds) nv = p.lds;
    const float* srow = p.sample + (static_cast<int64_t>(b) * p.rows + row_id) * p.lds;
    if (gtid() == 0) {
        res[4] = 0;
        res[6] = 0xffffffffu;
        res[7] = 0u;
    }
    for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
    csync();
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    const int64_t nvr = (nv + 31) & ~int64_t{31};
    for (int64_t i = gtid(); i < nvr; i += kThreads) {
        const float v = i < nv ? __ldg(srow + i) : neg_inf;
        const bool keep = v != neg_inf;  // legal sampled entries (scores are finite)
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        uint32_t base = 0;
        if (lane == 0 && m != 0) base = atomicAdd(&res[4], __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
            const uint32_t key = ord_key(v);
            if (pos < static_cast<uint32_t>(kTauMaxSamples)) s_keys[pos] = key;
            kmin = min(kmin, key);
            kmax = max(kmax, key);
        }
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (lane == 0) {
        atomicMin(&res[6], kmin);
        atomicMax(&res[7], kmax);
    }
    csync();
    const int ns = static_cast<int>(min(res[4], static_cast<uint32_t>(kTauMaxSamples)));
    const int target = (2 * p.k < (p.cand_cap * 3) / 4) ? 2 * p.k : (p.cand_cap * 3) / 4;
    int r = static_cast<int>((static_cast<int64_t>(target) * ns) / n);
    if (r < 1) r = 1;
    if (ns == 0 || r > ns) {  // sample too thin to cut: keep everything (the select falls back)
        if (gtid() == 0) *out = neg_inf;
        return;
    }
    const uint32_t lo = res[6], hi_k = res[7];
    uint32_t prefix = 0;
    int pbits = lo == hi_k ? 32 : __clz(lo ^ hi_k);
    if (pbits > 0) prefix = pbits == 32 ? lo : (lo >> (32 - pbits));
    uint32_t rr = static_cast<uint32_t>(r);
#pragma unroll 1
    for (int pass = 0; pass < 2 && pbits < 32; ++pass) {
        const int wbits = 32 - pbits < 11 ? 32 - pbits : 11;
        const int shift = 32 - pbits - wbits;
        if (pass > 0) {
            for (int i = gtid(); i < kBins; i += kThreads) hist[i] = 0;
            csync();
        }
        for (int i = gtid(); i < ns; i += kThreads) {
            const uint32_t v = s_keys[i];
            if (pbits == 0 || (v >> (32 - pbits)) == prefix) atomicAdd(&hist[(v >> shift) & ((1u << wbits) - 1u)], 1u);
        }
        csync();
        find_bin(hist, 1 << wbits, rr, res, wsum);
        rr -= res[1];
        prefix = (pbits == 0 ? 0u : (prefix << wbits)) | res[0];
        pbits += wbits;
        csync();
    }
    if (gtid() == 0) *out = ord_key_to_float(pbits >= 32 ? prefix : (prefix << (32 - pbits)));
}

// ------------------------------------------------------------------ large take
// take = min(k, n) above the shared-memory select's capacity (k > 4096: the
// reference's tile_topk / oracle_topk accept any k, topk.cpp:105-132,
// 193-206). One CTA per row over global scratch: the exact MSB-first radix
// select (histogram passes over the row, index-ordered collection of the tied
// bin) picks the top take into the row's slot, a bitonic sort over the slot
// orders them under succ, and write_row emits the row. Exact for any n, k.
constexpr int kLargeCand = 8192;                          // tied-bin collection capacity
constexpr size_t kLargeScratchBudget = size_t{256} << 20;  // bytes of slots per launch slab

__host__ __device__ inline int64_t large_slot_elems(int k, int64_t cols) {
    const int64_t take = k < cols ? k : cols;
    int64_t p = 1;
    while (p < take) p <<= 1;
    return p + kLargeCand;
}

__global__ void __launch_bounds__(kThreads) select_large_kernel(const SelectParams p, int64_t fr0, int64_t slot_elems) {
    __shared__ uint32_t hist[kBins];
    __shared__ uint32_t wtot[4 * kWarps], wsum[kWarps], res[8];
    const int64_t fr = fr0 + blockIdx.x;
    const int b = static_cast<int>(fr / p.rows);
    const int64_t row_id = fr - static_cast<int64_t>(b) * p.rows;
    int64_t n = p.cols;
    if (p.apply_mask) {
        n = (p.s0 + row_id + 1) / p.ratio - p.t0;
        n = n < 0 ? 0 : (n > p.cols ? p.cols : n);
    }
    const int take = static_cast<int>(n < p.k ? n : p.k);
    const float* row = p.scores + (static_cast<int64_t>(b) * p.rows + row_id) * p.ld;
    uint64_t* buf = static_cast<uint64_t*>(p.scratch) + static_cast<int64_t>(blockIdx.x) * slot_elems;
    uint64_t* cand = buf + (slot_elems - kLargeCand);
    if (take > 0) {
        if (take == n) {
            for (int64_t i = gtid(); i < n; i += kThreads) buf[i] = composite(ord_key(__ldg(row + i)), i);
        } else {
            exact_global_select(row, n, take, buf, cand, kLargeCand, hist, wtot, res, wsum);
        }
        const int P = pow2_at_least(take);
        for (int i = take + gtid(); i < P; i += kThreads) buf[i] = 0;
        csync();
        sort_desc(buf, P);
    }
    write_row(p, b, row_id, take, buf);
}

}  // namespace

namespace csaidx_kern {

int select_max_take() { return kMaxTake; }

int select_cand_capacity(int k) { return layout_for(k).cand_cap; }

cudaError_t launch_tau(const TauParams& p, cudaStream_t stream) {
    if (p.rows <= 0 || p.batch <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(p.rows), static_cast<unsigned>(p.batch));
    tau_kernel<<<grid, kThreads, 0, stream>>>(p);
    return cudaGetLastError();
}

namespace {
template <int U, int MB>
cudaError_t launch_select_variant(const SelectParams& p, cudaStream_t stream) {
    static bool attr_set[kMaxDevices] = {};
    const int attr_set_dev = attr_device();
    if (!attr_set[attr_set_dev]) {
        cudaError_t e = cudaFuncSetAttribute(select_kernel<U, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem_bytes_for(kMaxTake)));
        if (e != cudaSuccess) return e;
        attr_set[attr_set_dev] = true;
    }
    const dim3 grid(static_cast<unsigned>(p.rows), static_cast<unsigned>(p.batch));
    select_kernel<U, MB><<<grid, kThreads, smem_bytes_for(p.k), stream>>>(p);
    return cudaGetLastError();
}

int select_variant() {
    static int v = [] {
        const char* s = getenv("CSAIDX_SELECT_VARIANT");  // A/B knob (dev): 0 = by k, 1 = 4 x float4 / 4 CTAs, 2 = 8 x float4 / 4 CTAs, 3 = 8 x float4 / 3 CTAs
        return s != nullptr ? atoi(s) : 0;
    }();
    return v;
}
}  // namespace

// 227 KiB of opt-in shared memory per block, less 1 KiB for static shared
// variables of the row stages
constexpr size_t kFatSmemMax = 226 * 1024;
bool select_fat_fits(int k) { return kFatGroups * smem_bytes_for(k) <= kFatSmemMax; }

size_t select_large_scratch_bytes(int k, int64_t cols, int64_t rows) {
    const size_t slot = static_cast<size_t>(large_slot_elems(k, cols)) * sizeof(uint64_t);
    int64_t R = static_cast<int64_t>(kLargeScratchBudget / slot);
    if (R < 1) R = 1;
    if (R > rows) R = rows;
    return static_cast<size_t>(R) * slot;
}

cudaError_t launch_select(const SelectParams& p, cudaStream_t stream) {
    if (p.rows <= 0 || p.batch <= 0) return cudaSuccess;
    if (p.k > kMaxTake || p.width > kMaxTake) {
        // large take: one CTA per row over global slots, in slabs of rows
        const int64_t total = p.rows * p.batch;
        const int64_t slot = large_slot_elems(p.k, p.cols);
        if (p.scratch == nullptr || p.scratch_bytes < select_large_scratch_bytes(p.k, p.cols, total))
            return cudaErrorInvalidValue;
        const int64_t R = static_cast<int64_t>(p.scratch_bytes / (static_cast<size_t>(slot) * sizeof(uint64_t)));
        for (int64_t fr0 = 0; fr0 < total; fr0 += R) {
            const int64_t nr = total - fr0 < R ? total - fr0 : R;
            select_large_kernel<<<static_cast<unsigned>(nr), kThreads, 0, stream>>>(p, fr0, slot);
        }
        return cudaGetLastError();
    }
    if (p.persistent_ctas > 0 && p.phase_clk == nullptr && select_fat_fits(p.k)) {
        static bool fat_attr[kMaxDevices] = {};
        const int fat_attr_dev = attr_device();
        if (!fat_attr[fat_attr_dev]) {
            cudaError_t e = cudaFuncSetAttribute(select_fat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kFatSmemMax));
            if (e != cudaSuccess) return e;
            fat_attr[fat_attr_dev] = true;
        }
        select_fat_kernel<<<p.persistent_ctas, kThreads * kFatGroups, kFatGroups * smem_bytes_for(p.k), stream>>>(p);
        return cudaGetLastError();
    }
    // 8 float4 in flight per thread, 3 CTAs per SM (measured faster than
    // 4 x float4 at 4 CTAs per SM: scripts/probe_select.py)
    // 8 float4 in flight per thread at 3 CTAs per SM measured faster than
    // 4 x float4 at 4 CTAs per SM (scripts/time_select.py). Also measured
    // slower and dropped: building the composites inside the filter loop
    // (re-reading the score from L1) instead of the L2 gather, and a
    // persistent warp-specialised form streaming rows through a TMA
    // bulk-copy ring (2 CTAs/SM; 3.7 vs 5.3 TB/s on long rows).
    if (select_variant() == 1) return launch_select_variant<4, 4>(p, stream);
    if (select_variant() == 3) return launch_select_variant<8, 3>(p, stream);
    // k <= 512 (<= 29 KB of shared memory per row): a 4th CTA per SM at 64
    // registers pays off (0.080 vs 0.087 ms on 2048 rows of 32K at k = 512);
    // at k = 1024 the register-starved stream loses (0.109 vs 0.102 ms)
    if (p.k <= 512 || select_variant() == 2) return launch_select_variant<8, 4>(p, stream);
    // 16 float4 (256 B) per thread per iteration at 3 CTAs per SM (80
    // registers, no spills): 2-3% faster than 8 (0.101 vs 0.104 ms at
    // n = 32K, 0.407 vs 0.418 ms at n = 256K; variant 3 = the 8-float4 form)
    return launch_select_variant<16, 3>(p, stream);
}

}  // namespace csaidx_kern
