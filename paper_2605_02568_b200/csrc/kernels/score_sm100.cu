// Indexer score kernels for sm_100a.
//
//   scores[b, i, j] = sum_h w[b, s0+i, h] * relu(q[b, s0+i, h, :] . kc[b, t0+j, :])
//
// Reference semantics: score.hpp:51-64, score_scalar.cpp:20-34 (op order),
// causal.cpp:30-41 (mask). Two kernels:
//
//  * score_tc_kernel — the production path for the V4 indexer shape
//    (H_I = 64, d_h = 128). A warp-specialised tcgen05 GEMM with keys as M
//    (128 TMEM lanes) and (query x head) as N (4 queries x 64 heads = 256
//    columns). q and kc tiles are staged by TMA with 128-byte swizzle; the
//    fp32 accumulator lives in TMEM (2 x 256 columns, double buffered); the
//    epilogue warps read one key row per thread with tcgen05.ld and fold
//    ReLU, the w-weighted head reduction and the causal mask before the only
//    store, so the [B,S,H_I,T] per-head intermediate never exists.
//
//  * score_exact_kernel — any shape, CUDA cores, the reference's fp32 op
//    order exactly (ascending-d dot as mul-then-add, ReLU as x<0?0:x,
//    ascending-h acc = acc + w*r, optional binary16 rounding points). Given
//    bf16-representable inputs it is bit-identical to the CPU reference.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kHeads = 64;
constexpr int kDim = 128;
constexpr int kBlockKeys = 128;                 // UMMA M (TMEM lanes)
constexpr int kQPerGroup = 4;                   // queries per UMMA N
constexpr int kUmmaN = kQPerGroup * kHeads;     // 256
constexpr int kGroups = 2;                      // query groups per work item
constexpr int kQPerItem = kQPerGroup * kGroups; // 8
constexpr int kStages = 2;
constexpr int kKTilesPerPiece = 32;             // 4096 keys per work item
constexpr int kKSteps = kDim / 16;              // UMMA_K = 16 for bf16

constexpr uint32_t kHalfRowBytes = 128;                          // 64 bf16
constexpr uint32_t kQHalfBytes = kUmmaN * kHalfRowBytes;         // 32 KiB
constexpr uint32_t kQGroupBytes = 2 * kQHalfBytes;               // 64 KiB
constexpr uint32_t kKHalfBytes = kBlockKeys * kHalfRowBytes;     // 16 KiB
constexpr uint32_t kKStageBytes = 2 * kKHalfBytes;               // 32 KiB
constexpr uint32_t kQBytes = kGroups * kQGroupBytes;             // 128 KiB
constexpr uint32_t kSmemData = kQBytes + kStages * kKStageBytes; // 192 KiB
constexpr uint32_t kSmemBytes = kSmemData + 256 + 1024;          // + barriers + align slack

constexpr int kNumThreads = 384;  // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdesc = idesc_bf16_f32(kBlockKeys, kUmmaN);

struct Item {
    int b, r0, nrows, kt_begin, kt_end;
};

__device__ __forceinline__ int64_t t_legal_dev(int64_t t, int64_t ratio) { return (t + 1) / ratio; }

// Work item enumeration shared by every role. Items run heaviest-first: query
// blocks from the end of the chunk (longest causal prefix) downwards, each
// split into pieces of kKTilesPerPiece key tiles.
__device__ __forceinline__ bool decode_item(const ScoreTcParams& p, int idx, Item& it) {
    const int piece = idx % p.npieces;
    const int rest = idx / p.npieces;
    const int b = rest % p.batch;
    const int qb = p.nqb - 1 - rest / p.batch;
    it.b = b;
    it.r0 = qb * kQPerItem;
    it.nrows = min(kQPerItem, static_cast<int>(p.rows) - it.r0);
    int64_t kend = p.cols;
    if (p.apply_mask) {
        const int64_t s_last = p.s0 + it.r0 + it.nrows - 1;
        kend = t_legal_dev(s_last, p.ratio) - p.t0;
        kend = kend < 0 ? 0 : (kend > p.cols ? p.cols : kend);
    }
    const int ntiles = static_cast<int>((kend + kBlockKeys - 1) / kBlockKeys);
    it.kt_begin = piece * kKTilesPerPiece;
    it.kt_end = min(it.kt_begin + kKTilesPerPiece, ntiles);
    return it.kt_begin < it.kt_end;
}

__global__ void __launch_bounds__(kNumThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap qmap,
                    const __grid_constant__ CUtensorMap kmap, const ScoreTcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* q_smem = smem;
    uint8_t* k_smem = smem + kQBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemData);
    uint64_t* k_full = bars + 0;
    uint64_t* k_empty = bars + 2;
    uint64_t* q_full = bars + 4;
    uint64_t* q_empty = bars + 5;
    uint64_t* acc_full = bars + 6;
    uint64_t* acc_empty = bars + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

    const int warp = threadIdx.x / 32;

    if (warp == 0 && elect_one()) {
        tma_prefetch(&qmap);
        tma_prefetch(&kmap);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int a = 0; a < 2; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], kEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            const uint64_t keep = policy_evict_last();  // keys are re-read by every query block
            uint32_t kiter = 0, qiter = 0;
            for (int idx = blockIdx.x; idx < p.nitems; idx += gridDim.x) {
                Item it;
                if (!decode_item(p, idx, it)) continue;
                mbar_wait(q_empty, (qiter & 1) ^ 1);
                mbar_expect_tx(q_full, kQBytes);
                const int32_t qrow =
                    static_cast<int32_t>((static_cast<int64_t>(it.b) * p.seq_len + p.s0 + it.r0) * kHeads);
                for (int g = 0; g < kGroups; ++g) {
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_2d(q_smem + g * kQGroupBytes + hf * kQHalfBytes, &qmap, q_full,
                                    hf * 64, qrow + g * kUmmaN);
                    }
                }
                ++qiter;
                const int64_t krow0 = static_cast<int64_t>(it.b) * p.key_blocks + p.t0;
                for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                    const uint32_t s = kiter % kStages;
                    mbar_wait(&k_empty[s], ((kiter / kStages) & 1) ^ 1);
                    mbar_expect_tx(&k_full[s], kKStageBytes);
                    const int32_t krow = static_cast<int32_t>(krow0 + kt * kBlockKeys);
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_2d_hint(k_smem + s * kKStageBytes + hf * kKHalfBytes, &kmap,
                                         &k_full[s], hf * 64, krow, keep);
                    }
                    ++kiter;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (elect_one()) {
            uint32_t kiter = 0, qiter = 0, aiter = 0;
            const uint32_t q_base = smem_u32(q_smem);
            const uint32_t k_base = smem_u32(k_smem);
            for (int idx = blockIdx.x; idx < p.nitems; idx += gridDim.x) {
                Item it;
                if (!decode_item(p, idx, it)) continue;
                mbar_wait(q_full, qiter & 1);
                ++qiter;
                tc_fence_after();
                for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                    const uint32_t s = kiter % kStages;
                    mbar_wait(&k_full[s], (kiter / kStages) & 1);
                    tc_fence_after();
                    for (int g = 0; g < kGroups; ++g) {
                        const uint32_t a = aiter & 1;
                        mbar_wait(&acc_empty[a], ((aiter >> 1) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t d_tmem = tmem_base + a * kUmmaN;
#pragma unroll
                        for (int kk = 0; kk < kKSteps; ++kk) {
                            const uint32_t koff = (kk >> 2) * kKHalfBytes + (kk & 3) * 32;
                            const uint32_t qoff = g * kQGroupBytes + (kk >> 2) * kQHalfBytes + (kk & 3) * 32;
                            umma_bf16(d_tmem, sw128_kmajor_desc(k_base + s * kKStageBytes + koff),
                                      sw128_kmajor_desc(q_base + qoff), kIdesc, kk > 0 ? 1u : 0u);
                        }
                        umma_commit(&acc_full[a]);
                        ++aiter;
                    }
                    umma_commit(&k_empty[s]);
                    ++kiter;
                }
                umma_commit(q_empty);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue
        const int quarter = warp & 3;           // TMEM lane quarter this warp may touch
        const int qpair = (warp - 4) >> 2;      // which two queries of the group
        const uint32_t lane = lane_id();
        const uint32_t row_taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t aiter = 0;
        const float neg_inf = -__int_as_float(0x7f800000);
        for (int idx = blockIdx.x; idx < p.nitems; idx += gridDim.x) {
            Item it;
            if (!decode_item(p, idx, it)) continue;
            for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                const int64_t j = static_cast<int64_t>(kt) * kBlockKeys + quarter * 32 + lane;
                for (int g = 0; g < kGroups; ++g) {
                    const uint32_t a = aiter & 1;
                    mbar_wait(&acc_full[a], (aiter >> 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int qq = 0; qq < 2; ++qq) {
                        const int qi = g * kQPerGroup + qpair * 2 + qq;   // query within item
                        if (qi >= it.nrows) continue;                      // warp-uniform
                        const int64_t r = it.r0 + qi;
                        const int64_t s = p.s0 + r;
                        const float* wrow = p.w + (static_cast<int64_t>(it.b) * p.seq_len + s) * kHeads;
                        const uint32_t col = a * kUmmaN + (qpair * 2 + qq) * kHeads;
                        float acc = 0.0f;
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            float v[32];
                            tmem_ld32(row_taddr + col + half * 32, v);
                            tmem_ld_wait();
                            const float4* w4 = reinterpret_cast<const float4*>(wrow + half * 32);
#pragma unroll
                            for (int h4 = 0; h4 < 8; ++h4) {
                                const float4 wv = __ldg(w4 + h4);
                                acc = fmaf(wv.x, fmaxf(v[4 * h4 + 0], 0.0f), acc);
                                acc = fmaf(wv.y, fmaxf(v[4 * h4 + 1], 0.0f), acc);
                                acc = fmaf(wv.z, fmaxf(v[4 * h4 + 2], 0.0f), acc);
                                acc = fmaf(wv.w, fmaxf(v[4 * h4 + 3], 0.0f), acc);
                            }
                        }
                        if (j < p.cols) {
                            float outv = acc;
                            const bool legal = !p.apply_mask || (p.t0 + j) < t_legal_dev(s, p.ratio);
                            if (!legal) {
                                outv = neg_inf;
                            } else if (!isfinite(acc)) {
                                atomicOr(p.nonfinite, 1);
                            }
                            p.out[(static_cast<int64_t>(it.b) * p.rows + r) * p.ld + j] = outv;
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&acc_empty[a]);
                    ++aiter;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
    }
}

// Binary16 rounding with saturation, matching half.cpp:84-91 (RNE, overflow
// saturates to +/-65504 instead of producing infinity).
__device__ __forceinline__ float half_round_sat(float x) {
    const __half h = __float2half_rn(x);
    const float r = __half2float(h);
    if (isinf(r)) return r > 0.0f ? 65504.0f : -65504.0f;
    return r;
}

__device__ __forceinline__ float ld_operand(const void* base, int64_t i, bool f32) {
    return f32 ? static_cast<const float*>(base)[i]
               : __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
}

__device__ __forceinline__ void score_exact_one(const ScoreExactParams& p, int b, int64_t i, int64_t j) {
    const int64_t s = p.s0 + i;
    const int64_t t = p.t0 + j;
    const float neg_inf = -__int_as_float(0x7f800000);
    float* dst = p.out + (static_cast<int64_t>(b) * p.rows + i) * p.ld + j;
    if (p.apply_mask && t >= t_legal_dev(s, p.ratio)) {
        *dst = neg_inf;
        return;
    }
    const bool f32 = p.operand_f32 != 0;
    const int64_t qbase = ((static_cast<int64_t>(b) * p.seq_len + s) * p.heads) * p.head_dim;
    const int64_t kbase = (static_cast<int64_t>(b) * p.key_blocks + t) * p.head_dim;
    const float* wrow = p.w + (static_cast<int64_t>(b) * p.seq_len + s) * p.heads;
    float acc = 0.0f;
    for (int64_t h = 0; h < p.heads; ++h) {
        float dot = 0.0f;
        for (int64_t d = 0; d < p.head_dim; ++d) {
            dot = __fadd_rn(dot, __fmul_rn(ld_operand(p.q, qbase + h * p.head_dim + d, f32),
                                           ld_operand(p.kc, kbase + d, f32)));
        }
        if (p.fp16) dot = half_round_sat(dot);
        const float rect = (dot < 0.0f) ? 0.0f : dot;
        acc = __fadd_rn(acc, __fmul_rn(wrow[h], rect));
        if (p.fp16) acc = half_round_sat(acc);
    }
    if (!p.fp16 && !isfinite(acc)) atomicOr(p.nonfinite, 1);
    *dst = acc;
}

__global__ void score_exact_kernel(const ScoreExactParams p) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int b = blockIdx.z;
    if (j >= p.cols) return;
    for (int64_t i = blockIdx.y; i < p.rows; i += gridDim.y) {
        score_exact_one(p, b, i, j);
    }
}

}  // namespace

namespace csaidx_kern {

bool score_tc_supported(int64_t heads, int64_t head_dim) {
    return heads == kHeads && head_dim == kDim;
}

size_t score_tc_smem_bytes() { return kSmemBytes; }

cudaError_t launch_score_tc(const CUtensorMap& qmap, const CUtensorMap& kmap, ScoreTcParams p,
                            int num_sms, cudaStream_t stream) {
    p.nqb = static_cast<int>((p.rows + kQPerItem - 1) / kQPerItem);
    const int64_t max_tiles = (p.cols + kBlockKeys - 1) / kBlockKeys;
    p.npieces = static_cast<int>((max_tiles + kKTilesPerPiece - 1) / kKTilesPerPiece);
    if (p.npieces < 1) p.npieces = 1;
    p.nitems = p.nqb * p.batch * p.npieces;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(score_tc_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int grid = p.nitems < num_sms ? p.nitems : num_sms;
    if (grid <= 0) return cudaSuccess;
    score_tc_kernel<<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    return cudaGetLastError();
}

cudaError_t launch_score_exact(const ScoreExactParams& p, cudaStream_t stream) {
    if (p.rows <= 0 || p.cols <= 0) return cudaSuccess;
    const dim3 block(128);
    const dim3 grid(static_cast<unsigned>((p.cols + 127) / 128),
                    static_cast<unsigned>(p.rows < 65535 ? p.rows : 65535),
                    static_cast<unsigned>(p.batch));
    score_exact_kernel<<<grid, block, 0, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
