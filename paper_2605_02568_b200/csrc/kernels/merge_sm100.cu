// Partition-merge and sentinel pass (reference topk.cpp:134-191 and
// driver.cpp:84-105).
//
// merge_kernel: one CTA per query row. The running row (k entries, sorted
// under succ) and the candidate row (width entries, sorted) are packed to the
// 64-bit composite key (ord_key(score) << 32 | ~(index + 1)); the candidate
// row is laid down reversed behind the running row, which makes one bitonic
// sequence, and a single bitonic merge network (log2(2P) stages) sorts it.
// The first k entries are the top-k of the union, ordered. The "+1" in the
// composite makes the (-inf, -1) sentinel outrank a masked (-inf, j)
// placeholder exactly as succ() does (test_topk.cpp:48).
//
// finalize_kernel: one warp per row; turns -inf entries into (-inf, -1),
// checks sentinels trail and that exactly k_eff entries are real, and widens
// indices to int64 into the caller's output rows.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kMergeThreads = 256;
constexpr int kMaxK = 4096;

__device__ __forceinline__ uint64_t pack(float v, int32_t idx) {
    return (static_cast<uint64_t>(ord_key(v)) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(idx + 1));
}

__device__ __forceinline__ void unpack(uint64_t c, float& v, int32_t& idx) {
    v = ord_key_to_float(static_cast<uint32_t>(c >> 32));
    idx = static_cast<int32_t>(~static_cast<uint32_t>(c)) - 1;
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(const MergeParams p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint64_t* a = reinterpret_cast<uint64_t*>(smem_raw);
    const int64_t row = blockIdx.x;
    float* rv = p.run_val + row * p.k;
    int32_t* ri = p.run_idx + row * p.k;
    const float* cv = p.cand_val + row * p.cand_ld;
    const int32_t* ci = p.cand_idx + row * p.cand_ld;
    const float neg_inf = -__int_as_float(0x7f800000);

    if (p.overwrite) {
        // A1 ablation: the row becomes the tile row; placeholders -> sentinels.
        for (int e = threadIdx.x; e < p.k; e += blockDim.x) {
            if (e < p.width && cv[e] != neg_inf) {
                rv[e] = cv[e];
                ri[e] = ci[e];
            } else {
                rv[e] = neg_inf;
                ri[e] = -1;
            }
        }
        return;
    }

    if (p.check_overlap) {
        for (int e = threadIdx.x; e < p.width; e += blockDim.x) {
            const int32_t idx = ci[e];
            if (idx < 0) continue;
            for (int f = 0; f < p.k; ++f) {
                if (ri[f] == idx) {
                    atomicOr(p.overlap_flag, 1);
                    break;
                }
            }
        }
    }

    int P = 1;
    while (P < p.k) P <<= 1;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        a[i] = i < p.k ? pack(rv[i], ri[i]) : 0ull;
        a[2 * P - 1 - i] = i < p.width ? pack(cv[i], ci[i]) : 0ull;
    }
    __syncthreads();
    for (int stride = P; stride > 0; stride >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
            const int lo = 2 * i - (i & (stride - 1));
            const int hi = lo + stride;
            const uint64_t x = a[lo], y = a[hi];
            if (x < y) {
                a[lo] = y;
                a[hi] = x;
            }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < p.k; e += blockDim.x) {
        float v;
        int32_t idx;
        unpack(a[e], v, idx);
        rv[e] = v;
        ri[e] = idx;
    }
}

__global__ void finalize_kernel(const FinalizeParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nrows = static_cast<int64_t>(p.batch) * p.rows;
    if (gw >= nrows) return;
    const int b = static_cast<int>(gw / p.rows);
    const int64_t i = gw % p.rows;
    const float* rv = p.run_val + gw * p.k;
    const int32_t* ri = p.run_idx + gw * p.k;
    const float neg_inf = -__int_as_float(0x7f800000);
    int64_t* oi = p.out_idx + (static_cast<int64_t>(b) * p.out_rows + p.out_row0 + i) * p.k;
    float* ov = p.out_val + (static_cast<int64_t>(b) * p.out_rows + p.out_row0 + i) * p.k;
    int first_inf = p.k;
    int real = 0;
    for (int e = lane; e < p.k; e += 32) {
        const float v = rv[e];
        const bool inf = (v == neg_inf);
        if (inf && e < first_inf) first_inf = e;
        real += inf ? 0 : 1;
        ov[e] = v;
        oi[e] = inf ? -1 : static_cast<int64_t>(ri[e]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        first_inf = min(first_inf, __shfl_xor_sync(0xffffffffu, first_inf, o));
        real += __shfl_xor_sync(0xffffffffu, real, o);
    }
    if (lane == 0) {
        if (real != first_inf) atomicOr(p.trail_flag, 1);
        if (p.check_keff) {
            const int64_t legal = (p.s0 + i + 1) / p.ratio;
            const int64_t want = legal < p.k ? legal : p.k;
            if (first_inf != want) atomicOr(p.keff_flag, 1);
        }
    }
}

}  // namespace

namespace csaidx_kern {

cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream) {
    if (p.nrows <= 0) return cudaSuccess;
    if (p.k > kMaxK) return cudaErrorInvalidValue;
    int P = 1;
    while (P < p.k) P <<= 1;
    const size_t smem = 2 * static_cast<size_t>(P) * sizeof(uint64_t);
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(2 * kMaxK * sizeof(uint64_t)));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    merge_kernel<<<static_cast<unsigned>(p.nrows), kMergeThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeParams& p, cudaStream_t stream) {
    const int64_t nrows = static_cast<int64_t>(p.batch) * p.rows;
    if (nrows <= 0) return cudaSuccess;
    const int threads = 256;
    const int64_t blocks = (nrows * 32 + threads - 1) / threads;
    finalize_kernel<<<static_cast<unsigned>(blocks), threads, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
