// Per-row exact top-k selection over one score tile (the GPU tile_topk,
// reference topk.cpp:105-132 + causal.cpp:30-41).
//
// One CTA per (batch, query row). Scores are mapped to an orderable 32-bit
// key (ord_key: monotone, -0.0 == +0.0) and the k-th largest key is located
// by MSB-first radix refinement (11/11/10-bit digits, shared-memory
// histograms) over the row in HBM/L2. Once the threshold digit's bucket is
// small enough it is collected into shared memory; everything strictly above
// the bucket is collected directly. An ordered (index-ascending) block
// compaction makes ties on the exact threshold resolve to the smallest
// indices, so the selected set is exactly the reference's under succ()
// (score desc, then index asc; topk.hpp:23-26). The survivors are bitonic
// sorted on a 64-bit composite key (ord_key << 32 | ~(index + 1)), which is
// the same total order, and written as (value, index) rows of `width`,
// padded with the (-inf, -1) sentinel.
//
// Algorithmic traffic: 4 B per legal score per pass; the common case is one
// histogram pass plus one collection pass.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 2048;
constexpr int kMaxTake = 4096;  // largest min(k, n) one row may select
constexpr int kCandCap = 4096;  // threshold-bucket entries kept on chip
constexpr size_t kSmemBytes =
    kBins * sizeof(uint32_t) + (kMaxTake + kCandCap) * sizeof(uint64_t) + 2 * 2 * kWarps * sizeof(uint32_t) + 64;

__device__ __forceinline__ uint64_t composite(uint32_t key, int64_t col) {
    return (static_cast<uint64_t>(key) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(col + 1));
}

__device__ __forceinline__ int64_t composite_col(uint64_t c) {
    return static_cast<int64_t>(~static_cast<uint32_t>(c)) - 1;
}

__device__ __forceinline__ int pow2_ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Descending bitonic sort of a[0, P), P a power of two, whole block.
__device__ void bitonic_sort_desc(uint64_t* a, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool desc = (lo & size) == 0;
                const uint64_t x = a[lo], y = a[hi];
                if (desc ? (x < y) : (x > y)) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
            __syncthreads();
        }
    }
}

struct RowView {
    const float* row;
    int64_t n;
};

__device__ __forceinline__ bool prefix_match(uint32_t key, uint32_t prefix, int pbits) {
    return pbits == 0 || (key >> (32 - pbits)) == prefix;
}

// Histogram of the next `wbits` bits below a `pbits`-bit prefix.
__device__ void histogram_pass(const RowView& r, uint32_t prefix, int pbits, int wbits, uint32_t* hist) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int shift = 32 - pbits - wbits;
    const uint32_t mask = (1u << wbits) - 1u;
    const int64_t n4 = r.n >> 2;
    const float4* row4 = reinterpret_cast<const float4*>(r.row);
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 v = __ldg(row4 + i);
        const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t key = ord_key(e[u]);
            if (prefix_match(key, prefix, pbits)) atomicAdd(&hist[(key >> shift) & mask], 1u);
        }
    }
    for (int64_t i = (n4 << 2) + threadIdx.x; i < r.n; i += blockDim.x) {
        const uint32_t key = ord_key(__ldg(r.row + i));
        if (prefix_match(key, prefix, pbits)) atomicAdd(&hist[(key >> shift) & mask], 1u);
    }
    __syncthreads();
}

// Finds the bin (scanning from the top) that holds the kk-th largest key.
// Returns bin, count strictly above it, and the bin's own count.
__device__ void find_bin(const uint32_t* hist, int nbins, uint32_t kk, uint32_t* out3) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int per = nbins / 32;
        // lane 0 owns the highest bins
        const int hi = nbins - lane * per;  // exclusive upper bound
        uint32_t sum = 0;
        for (int b = hi - 1; b >= hi - per; --b) sum += hist[b];
        // exclusive scan over lanes (lane 0 first)
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - sum;
        const bool mine = excl < kk && kk <= incl;
        if (mine) {
            uint32_t cum = excl;
            for (int b = hi - 1; b >= hi - per; --b) {
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
    }
    __syncthreads();
}

// Ordered block compaction over the row: entries with top-pbits(key) above
// `prefix` go to above_dst (all of them), entries equal to it go to eq_dst
// (only the first eq_limit in index order).
__device__ void collect_pass(const RowView& r, uint32_t prefix, int pbits, uint64_t* above_dst,
                             uint64_t* eq_dst, uint32_t eq_limit, uint32_t* wtot /*[2][2*kWarps]*/) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t run_above = 0, run_eq = 0;
    int parity = 0;
    for (int64_t base = 0; base < r.n; base += 4 * static_cast<int64_t>(blockDim.x)) {
        const int64_t i0 = base + 4 * static_cast<int64_t>(threadIdx.x);
        uint32_t keys[4];
        int cls[4];
        uint32_t na = 0, ne = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u;
            cls[u] = 0;
            keys[u] = 0;
            if (i < r.n) {
                const uint32_t key = ord_key(__ldg(r.row + i));
                keys[u] = key;
                const uint32_t top = pbits == 0 ? 0u : (key >> (32 - pbits));
                if (pbits != 0 && top > prefix) {
                    cls[u] = 1;
                    ++na;
                } else if (pbits == 0 || top == prefix) {
                    cls[u] = 2;
                    ++ne;
                }
            }
        }
        // warp inclusive scan of the packed (above | eq << 16) counts
        uint32_t packed = na | (ne << 16);
        uint32_t incl = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        uint32_t* wt = wtot + parity * 2 * kWarps;
        if (lane == 31) {
            wt[warp] = incl & 0xffffu;
            wt[kWarps + warp] = incl >> 16;
        }
        __syncthreads();
        uint32_t woff_a = 0, woff_e = 0, tot_a = 0, tot_e = 0;
        for (int w = 0; w < kWarps; ++w) {
            const uint32_t a = wt[w], e = wt[kWarps + w];
            if (w < warp) {
                woff_a += a;
                woff_e += e;
            }
            tot_a += a;
            tot_e += e;
        }
        uint32_t pa = run_above + woff_a + ((incl - packed) & 0xffffu);
        uint32_t pe = run_eq + woff_e + ((incl - packed) >> 16);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (cls[u] == 1) {
                above_dst[pa++] = composite(keys[u], i0 + u);
            } else if (cls[u] == 2) {
                if (pe < eq_limit) eq_dst[pe] = composite(keys[u], i0 + u);
                ++pe;
            }
        }
        run_above += tot_a;
        run_eq += tot_e;
        parity ^= 1;  // next iteration writes the other wtot half; one barrier suffices
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) select_kernel(const SelectParams p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint64_t* buf = reinterpret_cast<uint64_t*>(smem_raw);     // [kMaxTake]
    uint64_t* cand = buf + kMaxTake;                            // [kCandCap]
    uint32_t* hist = reinterpret_cast<uint32_t*>(cand + kCandCap);
    uint32_t* wtot = hist + kBins;                              // [2][2*kWarps]
    uint32_t* res = wtot + 4 * kWarps;                          // [3] find_bin result

    const int64_t row = blockIdx.x;
    const int b = blockIdx.y;
    int64_t n = p.cols;
    if (p.apply_mask) {
        n = (p.s0 + row + 1) / p.ratio - p.t0;
        n = n < 0 ? 0 : (n > p.cols ? p.cols : n);
    }
    RowView r{p.scores + (static_cast<int64_t>(b) * p.rows + row) * p.ld, n};
    const int take = static_cast<int>(n < p.k ? n : p.k);

    if (take > 0) {
        if (n <= p.k) {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) buf[i] = composite(ord_key(__ldg(r.row + i)), i);
        } else {
            uint32_t prefix = 0;
            int pbits = 0;
            uint32_t kk = static_cast<uint32_t>(p.k);
            uint32_t bin_count = 0;
            const int widths[3] = {11, 11, 10};
            for (int pass = 0; pass < 3; ++pass) {
                const int wbits = widths[pass];
                histogram_pass(r, prefix, pbits, wbits, hist);
                find_bin(hist, 1 << wbits, kk, res);
                const uint32_t bin = res[0];
                kk -= res[1];
                bin_count = res[2];
                prefix = (pbits == 0 ? 0u : (prefix << wbits)) | bin;
                pbits += wbits;
                __syncthreads();  // everyone has read res before it is reused
                if (bin_count <= static_cast<uint32_t>(kCandCap)) break;
            }
            const uint32_t above = static_cast<uint32_t>(p.k) - kk;
            if (pbits == 32) {
                // The threshold bucket is a single key: keep its first kk
                // entries in index order (ties to the smaller index).
                collect_pass(r, prefix, pbits, buf, buf + above, kk, wtot);
            } else {
                collect_pass(r, prefix, pbits, buf, cand, static_cast<uint32_t>(kCandCap), wtot);
                const int P = pow2_ceil(static_cast<int>(bin_count));
                for (int i = static_cast<int>(bin_count) + threadIdx.x; i < P; i += blockDim.x) cand[i] = 0;
                __syncthreads();
                bitonic_sort_desc(cand, P);
                for (uint32_t i = threadIdx.x; i < kk; i += blockDim.x) buf[above + i] = cand[i];
            }
        }
        __syncthreads();
        const int P = pow2_ceil(take);
        for (int i = take + threadIdx.x; i < P; i += blockDim.x) buf[i] = 0;
        __syncthreads();
        bitonic_sort_desc(buf, P);
    }

    float* ov = p.out_val + (static_cast<int64_t>(b) * p.rows + row) * p.out_ld;
    int32_t* oi = p.out_idx + (static_cast<int64_t>(b) * p.rows + row) * p.out_ld;
    const float neg_inf = -__int_as_float(0x7f800000);
    for (int e = threadIdx.x; e < p.width; e += blockDim.x) {
        if (e < take) {
            const uint64_t c = buf[e];
            ov[e] = ord_key_to_float(static_cast<uint32_t>(c >> 32));
            oi[e] = static_cast<int32_t>(composite_col(c) + p.t0);
        } else {
            ov[e] = neg_inf;
            oi[e] = -1;
        }
    }
}

}  // namespace

namespace csaidx_kern {

int select_max_take() { return kMaxTake; }

cudaError_t launch_select(const SelectParams& p, cudaStream_t stream) {
    if (p.rows <= 0 || p.batch <= 0) return cudaSuccess;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const dim3 grid(static_cast<unsigned>(p.rows), static_cast<unsigned>(p.batch));
    select_kernel<<<grid, kThreads, kSmemBytes, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
