// Per-row exact top-k selection over one score tile (the GPU tile_topk,
// reference topk.cpp:105-132 + causal.cpp:30-41).
//
// One CTA per (batch, query row); n = the row's legal columns. Every entry is
// packed into a unique 64-bit composite (ord_key(score) << 32 | ~(col + 1)):
// ord_key is monotone in the float order with -0.0 folded onto +0.0, and the
// low word makes ties go to the smaller index, so descending composite order
// is exactly the reference's succ() order (topk.hpp:23-26).
//
// Fast path (one streaming pass over HBM/L2):
//   1. sample: every stride-th 32-byte sector of the row (1/16 of the row or
//      less) goes to shared memory; a shared-memory radix select finds the
//      sample key whose rank predicts ~2k survivors in the whole row;
//   2. filter: the row is streamed once (2 x float4 per thread in flight);
//      entries at or above that key are appended to a shared candidate list
//      with warp-aggregated atomics;
//   3. if the list holds between k and its capacity, the exact k-th largest
//      composite is found by shared-memory radix select (unique keys, so no
//      tie bookkeeping), the k survivors are bitonic-sorted and written.
// If the sample mispredicts (fewer than k or more than capacity survivors)
// the row falls back to an exact MSB-first radix select over global memory
// with index-ordered tie collection. Rows with n <= capacity skip sampling.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 2048;
constexpr int kMaxTake = 4096;    // largest min(k, n) a row may select
constexpr int kCandCap = 8192;    // shared candidate list (u64)
constexpr int kSampleSectors = 1024;
constexpr size_t kSmemBytes = kCandCap * sizeof(uint64_t) + kMaxTake * sizeof(uint64_t) + kBins * sizeof(uint32_t) +
                              4 * kWarps * sizeof(uint32_t) + 64;

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

// Finds the bin (scanning from the top) holding the kk-th largest element.
// out3 = {bin, count strictly above it, the bin's own count}.
__device__ void find_bin(const uint32_t* hist, int nbins, uint32_t kk, uint32_t* out3) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int per = nbins / 32;
        const int hi = nbins - lane * per;  // lane 0 owns the highest bins
        uint32_t sum = 0;
        for (int b = hi - 1; b >= hi - per; --b) sum += hist[b];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const uint32_t excl = incl - sum;
        if (excl < kk && kk <= incl) {
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

// kk-th largest of the unique 64-bit values a[0, n) in shared memory: returns
// (prefix, pbits) such that exactly kk values have their top pbits >= prefix.
__device__ void smem_radix_u64(const uint64_t* a, int n, uint32_t kk, uint32_t* hist, uint32_t* res,
                               uint64_t& prefix_out, int& pbits_out) {
    uint64_t prefix = 0;
    int pbits = 0;
    const int widths[6] = {11, 11, 10, 11, 11, 10};
#pragma unroll
    for (int pass = 0; pass < 6; ++pass) {
        const int wbits = widths[pass];
        const int shift = 64 - pbits - wbits;
        for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t v = a[i];
            if (pbits == 0 || (v >> (64 - pbits)) == prefix)
                atomicAdd(&hist[static_cast<uint32_t>(v >> shift) & ((1u << wbits) - 1u)], 1u);
        }
        __syncthreads();
        find_bin(hist, 1 << wbits, kk, res);
        const uint32_t bin = res[0], above = res[1], cnt = res[2];
        __syncthreads();
        kk -= above;
        prefix = (pbits == 0 ? 0ull : (prefix << wbits)) | bin;
        pbits += wbits;
        if (cnt == kk) break;  // the whole bucket is in; exactly kk remain
    }
    prefix_out = prefix;
    pbits_out = pbits;
}

__device__ __forceinline__ bool top_ge(uint64_t v, uint64_t prefix, int pbits) {
    return pbits >= 64 ? v >= prefix : (v >> (64 - pbits)) >= prefix;
}

// kk-th largest of the u32 sample s[0, n) (shared memory).
__device__ uint32_t smem_kth_u32(const uint32_t* s, int n, uint32_t kk, uint32_t* hist, uint32_t* res) {
    uint32_t prefix = 0;
    int pbits = 0;
    const int widths[3] = {11, 11, 10};
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
        const int wbits = widths[pass];
        const int shift = 32 - pbits - wbits;
        for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t v = s[i];
            if (pbits == 0 || (v >> (32 - pbits)) == prefix) atomicAdd(&hist[(v >> shift) & ((1u << wbits) - 1u)], 1u);
        }
        __syncthreads();
        find_bin(hist, 1 << wbits, kk, res);
        const uint32_t bin = res[0], above = res[1];
        __syncthreads();
        kk -= above;
        prefix = (pbits == 0 ? 0u : (prefix << wbits)) | bin;
        pbits += wbits;
    }
    return prefix;  // full 32-bit key of the kk-th largest sample
}

// ------------------------------------------------------------------ fallback
// Exact MSB-first radix select over global memory (any n, any ties): the
// selected composites (unsorted) land in buf[0, k).

__device__ __forceinline__ bool prefix_match(uint32_t key, uint32_t prefix, int pbits) {
    return pbits == 0 || (key >> (32 - pbits)) == prefix;
}

__device__ void histogram_pass(const float* row, int64_t n, uint32_t prefix, int pbits, int wbits, uint32_t* hist) {
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const int shift = 32 - pbits - wbits;
    const uint32_t mask = (1u << wbits) - 1u;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t key = ord_key(__ldg(row + i));
        if (prefix_match(key, prefix, pbits)) atomicAdd(&hist[(key >> shift) & mask], 1u);
    }
    __syncthreads();
}

// Ordered (index-ascending) block compaction: entries above the prefix go to
// above_dst, entries equal to it to eq_dst (first eq_limit in index order).
__device__ void collect_pass(const float* row, int64_t n, uint32_t prefix, int pbits, uint64_t* above_dst,
                             uint64_t* eq_dst, uint32_t eq_limit, uint32_t* wtot) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t run_above = 0, run_eq = 0;
    int parity = 0;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
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
        __syncthreads();
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
    __syncthreads();
}

__device__ void exact_global_select(const float* row, int64_t n, int k, uint64_t* buf, uint64_t* cand,
                                    uint32_t* hist, uint32_t* wtot, uint32_t* res) {
    uint32_t prefix = 0;
    int pbits = 0;
    uint32_t kk = static_cast<uint32_t>(k);
    uint32_t bin_count = 0;
    const int widths[3] = {11, 11, 10};
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
        const int wbits = widths[pass];
        histogram_pass(row, n, prefix, pbits, wbits, hist);
        find_bin(hist, 1 << wbits, kk, res);
        kk -= res[1];
        bin_count = res[2];
        prefix = (pbits == 0 ? 0u : (prefix << wbits)) | res[0];
        pbits += wbits;
        __syncthreads();
        if (bin_count <= static_cast<uint32_t>(kCandCap)) break;
    }
    const uint32_t above = static_cast<uint32_t>(k) - kk;
    if (pbits == 32) {
        // a single key value: its first kk entries in index order
        collect_pass(row, n, prefix, pbits, buf, buf + above, kk, wtot);
    } else {
        collect_pass(row, n, prefix, pbits, buf, cand, static_cast<uint32_t>(kCandCap), wtot);
        const int P = pow2_ceil(static_cast<int>(bin_count));
        for (int i = static_cast<int>(bin_count) + threadIdx.x; i < P; i += blockDim.x) cand[i] = 0;
        __syncthreads();
        bitonic_sort_desc(cand, P);
        for (uint32_t i = threadIdx.x; i < kk; i += blockDim.x) buf[above + i] = cand[i];
    }
    __syncthreads();
}

// ------------------------------------------------------------------ kernel

__global__ void __launch_bounds__(kThreads, 2) select_kernel(const SelectParams p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint64_t* cand = reinterpret_cast<uint64_t*>(smem_raw);  // [kCandCap]
    uint64_t* buf = cand + kCandCap;                         // [kMaxTake]
    uint32_t* hist = reinterpret_cast<uint32_t*>(buf + kMaxTake);
    uint32_t* wtot = hist + kBins;                           // [2][2*kWarps]
    uint32_t* res = wtot + 4 * kWarps;                       // find_bin result (3) + counter
    uint32_t* counter = res + 4;
    uint32_t* sample = reinterpret_cast<uint32_t*>(cand);    // aliases cand during sampling

    const int64_t row_id = blockIdx.x;
    const int b = blockIdx.y;
    int64_t n = p.cols;
    if (p.apply_mask) {
        n = (p.s0 + row_id + 1) / p.ratio - p.t0;
        n = n < 0 ? 0 : (n > p.cols ? p.cols : n);
    }
    const float* row = p.scores + (static_cast<int64_t>(b) * p.rows + row_id) * p.ld;
    const int k = p.k;
    const int take = static_cast<int>(n < k ? n : k);
    const int lane = threadIdx.x & 31;

    if (take > 0) {
        int count = -1;  // candidates in cand[], or -1 -> fallback
        if (n <= kCandCap) {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cand[i] = composite(ord_key(__ldg(row + i)), i);
            count = static_cast<int>(n);
            __syncthreads();
        } else {
            // 1. sample every stride-th 32-byte sector
            const int64_t sectors = n >> 3;
            int64_t stride = (sectors + kSampleSectors - 1) / kSampleSectors;
            if (stride < 16) stride = 16;
            const int nss = static_cast<int>((sectors + stride - 1) / stride);
            const float4* row4 = reinterpret_cast<const float4*>(row);
            for (int s = threadIdx.x; s < nss; s += blockDim.x) {
                const int64_t sec = static_cast<int64_t>(s) * stride;
                const float4 a = __ldg(row4 + 2 * sec), c = __ldg(row4 + 2 * sec + 1);
                uint32_t* dst = sample + 8 * s;
                dst[0] = ord_key(a.x); dst[1] = ord_key(a.y); dst[2] = ord_key(a.z); dst[3] = ord_key(a.w);
                dst[4] = ord_key(c.x); dst[5] = ord_key(c.y); dst[6] = ord_key(c.z); dst[7] = ord_key(c.w);
            }
            if (threadIdx.x == 0) *counter = 0;
            __syncthreads();
            const int ns = 8 * nss;
            const int target = (2 * k < (kCandCap * 3) / 4) ? 2 * k : (kCandCap * 3) / 4;
            int r = static_cast<int>((static_cast<int64_t>(target) * ns) / n);
            if (r < 1) r = 1;
            if (r > ns) r = ns;
            const uint32_t tau = smem_kth_u32(sample, ns, static_cast<uint32_t>(r), hist, res);
            // 2. stream the row once; keep entries with key >= tau. The test
            //    is a plain float compare (ord_key is monotone and maps -0.0
            //    onto +0.0, like the float order); survivors (~2k of n) are
            //    appended with one warp scan + one shared atomic per warp.
            const float tau_f = ord_key_to_float(tau);
            const int64_t n4 = n >> 2;
            constexpr int kUnroll = 4;
            const int64_t step = kUnroll * static_cast<int64_t>(blockDim.x);
            const int64_t n4r = (n4 + step - 1) / step * step;
            for (int64_t it = threadIdx.x; it < n4r; it += step) {
                float4 v[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int64_t i4 = it + u * blockDim.x;
                    v[u] = i4 < n4 ? __ldg(row4 + i4) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                }
                uint32_t m = 0;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    m |= (v[u].x >= tau_f ? 1u : 0u) << (4 * u + 0);
                    m |= (v[u].y >= tau_f ? 1u : 0u) << (4 * u + 1);
                    m |= (v[u].z >= tau_f ? 1u : 0u) << (4 * u + 2);
                    m |= (v[u].w >= tau_f ? 1u : 0u) << (4 * u + 3);
                }
                if (!__any_sync(0xffffffffu, m != 0)) continue;
                const uint32_t c = __popc(m);
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
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        if (m & (1u << (4 * u + x))) {
                            if (pos < static_cast<uint32_t>(kCandCap))
                                cand[pos] = composite(ord_key(e[x]), 4 * (it + u * blockDim.x) + x);
                            ++pos;
                        }
                    }
                }
            }
            if (threadIdx.x < 32) {  // the < 4 entries past the last float4
                const int64_t i = 4 * n4 + lane;
                const bool inb = i < n;
                const uint32_t key = inb ? ord_key(__ldg(row + i)) : 0u;
                const bool pass = inb && key >= tau;
                const uint32_t m = __ballot_sync(0xffffffffu, pass);
                if (m != 0) {
                    uint32_t base = 0;
                    if (lane == 0) base = atomicAdd(counter, __popc(m));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
                    if (pass && pos < static_cast<uint32_t>(kCandCap)) cand[pos] = composite(key, i);
                }
            }
            __syncthreads();
            const uint32_t total = *counter;
            count = (total >= static_cast<uint32_t>(k) && total <= static_cast<uint32_t>(kCandCap))
                        ? static_cast<int>(total)
                        : -1;
            __syncthreads();
        }

        if (count >= 0) {
            // 3. exact k-th largest composite among the candidates
            if (count > take) {
                uint64_t prefix;
                int pbits;
                smem_radix_u64(cand, count, static_cast<uint32_t>(take), hist, res, prefix, pbits);
                if (threadIdx.x == 0) *counter = 0;
                __syncthreads();
                for (int i = threadIdx.x; i < count; i += blockDim.x) {
                    const uint64_t v = cand[i];
                    if (top_ge(v, prefix, pbits)) buf[atomicAdd(counter, 1u)] = v;
                }
            } else {
                for (int i = threadIdx.x; i < count; i += blockDim.x) buf[i] = cand[i];
            }
            __syncthreads();
        } else {
            exact_global_select(row, n, take, buf, cand, hist, wtot, res);
        }
        const int P = pow2_ceil(take);
        for (int i = take + threadIdx.x; i < P; i += blockDim.x) buf[i] = 0;
        __syncthreads();
        bitonic_sort_desc(buf, P);
    }

    float* ov = p.out_val + (static_cast<int64_t>(b) * p.rows + row_id) * p.out_ld;
    int32_t* oi = p.out_idx + (static_cast<int64_t>(b) * p.rows + row_id) * p.out_ld;
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
