// Partition-merge and sentinel pass (reference topk.cpp:134-191 and
// driver.cpp:84-105).
//
// merge_kernel: one CTA per query row. The running row (k entries, sorted
// under succ) and the candidate row (width entries, sorted) are packed to the
// 64-bit composite key (ord_key(score) << 32 | ~(index + 1)) and merged by a
// merge path: each thread binary-searches the split of its k/256 outputs and
// merges them sequentially (O(k) work, two barriers, instead of a bitonic
// network's log2(2k) stages). The first k entries are the top-k of the
// union, ordered. The "+1" in the
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
    const int64_t row = blockIdx.x;
    uint64_t* a = p.stage != nullptr ? p.stage + row * (static_cast<int64_t>(p.k) + p.width)
                                     : reinterpret_cast<uint64_t*>(smem_raw);
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

    // Merge path: both lists (sorted best first) are staged as composites;
    // thread t produces outputs [t*E, (t+1)*E) of the merged order after
    // locating its start by a binary search over the split (co-rank), then
    // merges E entries sequentially. Ties (identical sentinel composites)
    // go to the running row first; either way the output bytes are the same.
    const int nr = p.k, nc = p.width;
    uint64_t* run = a;
    uint64_t* cand = a + nr;
    if ((nr & 3) == 0 && (nc & 3) == 0 && (p.cand_ld & 3) == 0) {  // 16-byte loads, 4 entries each
        for (int i = 4 * threadIdx.x; i < nr + nc; i += 4 * blockDim.x) {
            const bool r = i < nr;
            const float4 v = *reinterpret_cast<const float4*>(r ? rv + i : cv + (i - nr));
            const int4 x = *reinterpret_cast<const int4*>(r ? ri + i : ci + (i - nr));
            a[i] = pack(v.x, x.x);
            a[i + 1] = pack(v.y, x.y);
            a[i + 2] = pack(v.z, x.z);
            a[i + 3] = pack(v.w, x.w);
        }
    } else {
        for (int i = threadIdx.x; i < nr; i += blockDim.x) run[i] = pack(rv[i], ri[i]);
        for (int i = threadIdx.x; i < nc; i += blockDim.x) cand[i] = pack(cv[i], ci[i]);
    }
    __syncthreads();
    // (rv / ri were consumed into shared memory above: outputs go straight
    // to global)
    const int E = (nr + kMergeThreads - 1) / kMergeThreads;
    const int d0 = threadIdx.x * E;
    if (d0 < nr) {
        int lo = d0 - nc > 0 ? d0 - nc : 0, hi = d0 < nr ? d0 : nr;
        int i = lo;
        while (lo <= hi) {
            i = (lo + hi) >> 1;
            const int j = d0 - i;
            if (i > 0 && j < nc && run[i - 1] < cand[j]) {
                hi = i - 1;
            } else if (j > 0 && i < nr && cand[j - 1] <= run[i]) {
                lo = i + 1;
            } else {
                break;
            }
        }
        int j = d0 - i;
#pragma unroll 1
        for (int e = 0; e < E && d0 + e < nr; ++e) {
            const bool take_run = j >= nc || (i < nr && run[i] >= cand[j]);
            float v;
            int32_t idx;
            unpack(take_run ? run[i++] : cand[j++], v, idx);
            rv[d0 + e] = v;
            ri[d0 + e] = idx;
        }
    }
}

// One CTA per row; 4 entries per thread per step (16 B loads, 2 x 16 B
// int64 stores) when k is a multiple of 4.
__global__ void __launch_bounds__(256) finalize_kernel(const FinalizeParams p) {
    __shared__ int s_first, s_real;
    const int64_t row = blockIdx.x;
    const int b = static_cast<int>(row / p.rows);
    const int64_t i = row % p.rows;
    const float* rv = p.run_val + row * p.k;
    const int32_t* ri = p.run_idx + row * p.k;
    const float neg_inf = -__int_as_float(0x7f800000);
    const bool outs = p.out_idx != nullptr;  // else the sink is the only output
    int64_t* oi = outs ? p.out_idx + (static_cast<int64_t>(b) * p.out_rows + p.out_row0 + i) * p.k : nullptr;
    float* ov = outs ? p.out_val + (static_cast<int64_t>(b) * p.out_rows + p.out_row0 + i) * p.k : nullptr;
    int32_t* si = p.sink != nullptr ? p.sink + (static_cast<int64_t>(b) * p.sink_seq + p.s0 + i) * p.k : nullptr;
    if (threadIdx.x == 0) {
        s_first = p.k;
        s_real = 0;
    }
    __syncthreads();
    int first_inf = p.k;
    int real = 0;
    if ((p.k & 3) == 0) {
        for (int e = 4 * threadIdx.x; e < p.k; e += 4 * blockDim.x) {
            const float4 v = *reinterpret_cast<const float4*>(rv + e);
            const int4 x = *reinterpret_cast<const int4*>(ri + e);
            const float vv[4] = {v.x, v.y, v.z, v.w};
            const int xx[4] = {x.x, x.y, x.z, x.w};
            long long o[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool inf = vv[u] == neg_inf;
                if (inf && e + u < first_inf) first_inf = e + u;
                real += inf ? 0 : 1;
                o[u] = inf ? -1ll : static_cast<long long>(xx[u]);
            }
            if (outs) {
                *reinterpret_cast<float4*>(ov + e) = v;
                *reinterpret_cast<longlong2*>(oi + e) = make_longlong2(o[0], o[1]);
                *reinterpret_cast<longlong2*>(oi + e + 2) = make_longlong2(o[2], o[3]);
            }
            if (si != nullptr)
                *reinterpret_cast<int4*>(si + e) = make_int4(static_cast<int>(o[0]), static_cast<int>(o[1]),
                                                             static_cast<int>(o[2]), static_cast<int>(o[3]));
        }
    } else {
        for (int e = threadIdx.x; e < p.k; e += blockDim.x) {
            const float v = rv[e];
            const bool inf = v == neg_inf;
            if (inf && e < first_inf) first_inf = e;
            real += inf ? 0 : 1;
            if (outs) {
                ov[e] = v;
                oi[e] = inf ? -1 : static_cast<int64_t>(ri[e]);
            }
            if (si != nullptr) si[e] = inf ? -1 : ri[e];
        }
    }
    if (si != nullptr) __threadfence_system();  // peer stores performed before the kernel retires
    if (first_inf < p.k) atomicMin(&s_first, first_inf);
    if (real != 0) atomicAdd(&s_real, real);
    __syncthreads();
    if (threadIdx.x == 0) {
        const int first = s_first;
        if (s_real != first) atomicOr(p.trail_flag, 1);
        if (p.check_keff) {
            const int64_t legal = (p.s0 + i + 1) / p.ratio;
            const int64_t want = legal < p.k ? legal : p.k;
            if (first != want) atomicOr(p.keff_flag, 1);
        }
    }
}

}  // namespace

namespace csaidx_kern {

constexpr size_t kStageBudget = size_t{256} << 20;  // bytes of global staging per launch slab

size_t merge_stage_bytes(int k, int width, int64_t nrows) {
    const size_t row = (static_cast<size_t>(k) + static_cast<size_t>(width)) * sizeof(uint64_t);
    int64_t R = static_cast<int64_t>(kStageBudget / row);
    if (R < 1) R = 1;
    if (R > nrows) R = nrows;
    return static_cast<size_t>(R) * row;
}

cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream) {
    if (p.nrows <= 0) return cudaSuccess;
    if (p.k > kMaxK && !p.overwrite) {
        // global staging, in slabs of stage_rows rows
        if (p.stage == nullptr || p.stage_rows < 1) return cudaErrorInvalidValue;
        for (int64_t r0 = 0; r0 < p.nrows; r0 += p.stage_rows) {
            MergeParams q = p;
            q.nrows = p.nrows - r0 < p.stage_rows ? p.nrows - r0 : p.stage_rows;
            q.run_val = p.run_val + r0 * p.k;
            q.run_idx = p.run_idx + r0 * p.k;
            q.cand_val = p.cand_val + r0 * p.cand_ld;
            q.cand_idx = p.cand_idx + r0 * p.cand_ld;
            merge_kernel<<<static_cast<unsigned>(q.nrows), kMergeThreads, 0, stream>>>(q);
        }
        return cudaGetLastError();
    }
    MergeParams q = p;
    q.stage = nullptr;
    if (p.overwrite) {  // A1: a row copy, no staging
        merge_kernel<<<static_cast<unsigned>(p.nrows), kMergeThreads, 0, stream>>>(q);
        return cudaGetLastError();
    }
    const size_t smem = (static_cast<size_t>(p.k) + static_cast<size_t>(p.width)) * sizeof(uint64_t);
    static bool attr_set[kMaxDevices] = {};
    const int attr_set_dev = attr_device();
    if (!attr_set[attr_set_dev]) {
        cudaError_t e = cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(2 * kMaxK * sizeof(uint64_t)));
        if (e != cudaSuccess) return e;
        attr_set[attr_set_dev] = true;
    }
    merge_kernel<<<static_cast<unsigned>(p.nrows), kMergeThreads, smem, stream>>>(q);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeParams& p, cudaStream_t stream) {
    const int64_t nrows = static_cast<int64_t>(p.batch) * p.rows;
    if (nrows <= 0) return cudaSuccess;
    finalize_kernel<<<static_cast<unsigned>(nrows), 256, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
