// Indexer score kernels for sm_100a.
//
//   scores[b, i, j] = sum_h w[b, s0+i, h] * relu(q[b, s0+i, h, :] . kc[b, t0+j, :])
//
// Reference semantics: score.hpp:51-64, score_scalar.cpp:20-34 (op order),
// causal.cpp:30-41 (mask). Two kernels:
//
//  * score_tc_kernel — the production path for the V4 indexer shape
//    (H_I = 64, d_h = 128). A warp-specialised, persistent tcgen05 GEMM with
//    keys as M (128 TMEM lanes) and (query x head) as N (2 queries x 64 heads
//    = 128 columns; CSAIDX_QGROUP=4 builds the 256-column form). q and kc
//    tiles are staged by TMA with 128-byte swizzle, w rows by a bulk copy;
//    the fp32 accumulators live in TMEM (4 x 128 columns); each is drained
//    by the 4 epilogue warps owning its query pair, which reduce both
//    queries together (the epilogue is latency bound, so the pair's
//    independent chains are what buys throughput); the epilogue warps read one key row per
//    thread with tcgen05.ld and fold ReLU, the w-weighted head reduction and
//    the causal mask before the only store, so the [B,S,H_I,T] per-head
//    intermediate never exists. Work items (8 queries x <= tpp key tiles)
//    form a dense piece-major list (causally dead tiles are never listed)
//    handed out by an atomic counter, so every SM stays busy to the end.
//
//  * score_exact_kernel — any shape, CUDA cores, the reference's fp32 op
//    order exactly (ascending-d dot as mul-then-add, ReLU as x<0?0:x,
//    ascending-h acc = acc + w*r, optional binary16 rounding points). Given
//    the same operands it is bit-identical to the CPU reference.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kHeads = 64;
constexpr int kDim = 128;
constexpr int kBlockKeys = 128;                 // UMMA M (TMEM lanes)
#ifndef CSAIDX_QGROUP
#define CSAIDX_QGROUP 2
#endif
#ifndef CSAIDX_EPI_REGS
#define CSAIDX_EPI_REGS 1  // next TMEM slice pair prefetched (needs the 576-thread register budget)
#endif
constexpr int kQPerGroup = CSAIDX_QGROUP;       // queries per UMMA N (4: N = 256, 2: N = 128)
constexpr int kUmmaN = kQPerGroup * kHeads;
constexpr int kQPerItem = 8;
constexpr int kGroups = kQPerItem / kQPerGroup; // query groups per work item
constexpr int kAcc = 512 / kUmmaN;              // TMEM accumulator buffers (512 columns)
static_assert(kQPerGroup == 4 || kQPerGroup == 2, "query group of 4 or 2");
constexpr int kStages = 2;
constexpr int kMinTilesPerPiece = 32;           // >= 4096 keys per work item
constexpr int kKSteps = kDim / 16;              // UMMA_K = 16 for bf16
constexpr int kItemSlots = 4;

constexpr uint32_t kHalfRowBytes = 128;                          // 64 bf16
constexpr uint32_t kQHalfBytes = kUmmaN * kHalfRowBytes;         // 32 / 16 KiB
constexpr uint32_t kQGroupBytes = 2 * kQHalfBytes;               // 64 / 32 KiB
constexpr uint32_t kKHalfBytes = kBlockKeys * kHalfRowBytes;     // 16 KiB
constexpr uint32_t kKStageBytes = 2 * kKHalfBytes;               // 32 KiB
constexpr uint32_t kQBytes = kGroups * kQGroupBytes;             // 128 KiB
constexpr uint32_t kWRowBytes = kHeads * 4;                      // 256 B per query
constexpr uint32_t kWBufBytes = kQPerItem * kWRowBytes;          // 2 KiB
constexpr uint32_t kWOffset = kQBytes + kStages * kKStageBytes;  // 192 KiB
constexpr int kWBufs = 3;                                        // see the producer's reuse proof
constexpr uint32_t kBarOffset = kWOffset + kWBufs * kWBufBytes;  // + 6 KiB
constexpr uint32_t kSmemBytes = kBarOffset + 512 + 1024;         // barriers, items, align slack

// Warp roles: 0 = scheduler + TMA producer, 1 = TMEM owner + MMA issuer,
// 2..17 = epilogue. Two control warps (not four) leave 576 threads, so the
// epilogue gets 112 registers (65536 / 576): room to keep the next TMEM
// slice pair in flight. TMEM lane access goes by warp % 4, so any 4
// consecutive epilogue warps cover the 4 lane quarters.
constexpr int kFirstEpiWarp = 2;
constexpr int kNumThreads = 576;
constexpr int kEpiWarps = 16;     // 4 per TMEM lane quarter, 2 queries of the item each
// Epilogue warps draining each accumulator: every warp (groups of 4) or the
// 4 warps, one per lane quarter, that own the group (groups of 2).
constexpr int kAccDrainers = kQPerGroup == 4 ? kEpiWarps : 4;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdesc = idesc_bf16_f32(kBlockKeys, kUmmaN);

struct Item {
    int b, r0, nrows, kt_begin, kt_end;  // kt_begin < 0: no more work
};

__device__ __forceinline__ int64_t t_legal_dev(int64_t t, int64_t ratio) { return (t + 1) / ratio; }

// Dense piece-major decode: idx -> (piece p, batch b, query block qb).
__device__ __forceinline__ void decode_item(const ScoreTcParams& p, int idx, Item& it) {
    int lo = 0, hi = p.npieces;  // largest piece with piece_start <= idx
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (p.piece_start[mid] <= idx) lo = mid; else hi = mid;
    }
    const int local = idx - p.piece_start[lo];
    it.b = local % p.batch;
    const int qb = p.nqb - 1 - local / p.batch;
    it.r0 = qb * kQPerItem;
    it.nrows = min(kQPerItem, static_cast<int>(p.rows) - it.r0);
    int64_t kend = p.cols;
    if (p.apply_mask) {
        kend = t_legal_dev(p.s0 + it.r0 + it.nrows - 1, p.ratio) - p.t0;
        kend = kend < 0 ? 0 : (kend > p.cols ? p.cols : kend);
    }
    const int ntiles_phys = static_cast<int>((kend + kBlockKeys - 1) / kBlockKeys);
    const int ntiles = (ntiles_phys + p.kt_stride - 1) / p.kt_stride;  // virtual tiles
    it.kt_begin = lo * p.tpp;
    it.kt_end = min(it.kt_begin + p.tpp, ntiles);
}

// Epilogue math for one query of one accumulator: 64 head partials of one
// key row -> sum_h w_h * relu(x_h): ReLU on the ALU pipe (FMNMX), products
// as packed FFMA2 on the FMA pipe into four independent chains.
//
// The epilogue paces the MMA: with the head math removed the kernel runs
// ~21% faster at C3 (energy/pacing probe, profiles/r01_ncu_history.md).
// Measured alternatives that shift ReLU onto the FMA pipe — 2 relu(x) =
// x + |x| as an FADD, or folded into a second FFMA2 with the |x| operand
// modifier — were equal (16 heads) or slower (16/32 heads as |x|-FFMA2):
// FFMA2 does not double the FMA pipe's rate, so the ALU pipe taking every
// ReLU is the balanced split.
//
// The 64 columns are read from TMEM in 8-column slices so the epilogue fits
// the 112 registers a 576-thread CTA allows; chain assignment and order do
// not depend on the slicing. ncu: the epilogue's top stall is the short
// scoreboard (w from shared memory / TMEM loads), then issue contention; it
// is latency bound, hence the paired form below.
// One query's 64 head partials in eight 8-column TMEM slices (the load of
// slice s+1 in flight while slice s is reduced), two packed FFMA2 chains.
// head_reduce_tmem2 below computes exactly this per query (same chains,
// same order), so a score never depends on whether its query was reduced
// alone or paired — the results stay tiling invariant bit for bit.
__device__ __forceinline__ void relu_fma8x(const float (&v)[8], const float* __restrict__ w8, float2& a0,
                                           float2& a1);

__device__ __forceinline__ float head_reduce_tmem(uint32_t taddr, const float* __restrict__ wq) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    float va[8], vb[8];
    tmem_ld8(taddr, va);
    tmem_ld_wait();
#pragma unroll
    for (int s = 0; s < 8; s += 2) {
        tmem_ld8(taddr + (s + 1) * 8, vb);
        relu_fma8x(va, wq + s * 8, a0, a1);
        tmem_ld_wait();
        if (s + 2 < 8) tmem_ld8(taddr + (s + 2) * 8, va);
        relu_fma8x(vb, wq + (s + 1) * 8, a0, a1);
        if (s + 2 < 8) tmem_ld_wait();
    }
    return (a0.x + a0.y) + (a1.x + a1.y);
}

// Two queries of the same accumulator (query groups of 2) reduced together:
// both 8-column slices are loaded before one wait, and the two independent
// chains interleave, halving the waits per pair and doubling the epilogue's
// instruction-level parallelism (it is latency bound: ~35% of issue slots).
__device__ __forceinline__ void relu_fma8x(const float (&v)[8], const float* __restrict__ w8, float2& a0,
                                           float2& a1) {
    const float4 wl = *reinterpret_cast<const float4*>(w8);
    const float4 wh = *reinterpret_cast<const float4*>(w8 + 4);
    a0 = __ffma2_rn(make_float2(fmaxf(v[0], 0.f), fmaxf(v[1], 0.f)), make_float2(wl.x, wl.y), a0);
    a1 = __ffma2_rn(make_float2(fmaxf(v[2], 0.f), fmaxf(v[3], 0.f)), make_float2(wl.z, wl.w), a1);
    a0 = __ffma2_rn(make_float2(fmaxf(v[4], 0.f), fmaxf(v[5], 0.f)), make_float2(wh.x, wh.y), a0);
    a1 = __ffma2_rn(make_float2(fmaxf(v[6], 0.f), fmaxf(v[7], 0.f)), make_float2(wh.z, wh.w), a1);
}

__device__ __forceinline__ float2 head_reduce_tmem2(uint32_t taddr0, uint32_t taddr1, const float* __restrict__ w0,
                                                    const float* __restrict__ w1) {
    float2 a0 = make_float2(0.f, 0.f), a1 = a0, b0 = a0, b1 = a0;
#if CSAIDX_EPI_REGS
    // the next slice pair's loads are in flight while the current pair is
    // reduced
    float va[8], vb[8], vc[8], vd[8];
    tmem_ld8(taddr0, va);
    tmem_ld8(taddr1, vb);
    tmem_ld_wait();
#pragma unroll
    for (int s = 0; s < 8; s += 2) {
        tmem_ld8(taddr0 + (s + 1) * 8, vc);
        tmem_ld8(taddr1 + (s + 1) * 8, vd);
        relu_fma8x(va, w0 + s * 8, a0, a1);
        relu_fma8x(vb, w1 + s * 8, b0, b1);
        tmem_ld_wait();
        if (s + 2 < 8) {
            tmem_ld8(taddr0 + (s + 2) * 8, va);
            tmem_ld8(taddr1 + (s + 2) * 8, vb);
        }
        relu_fma8x(vc, w0 + (s + 1) * 8, a0, a1);
        relu_fma8x(vd, w1 + (s + 1) * 8, b0, b1);
        if (s + 2 < 8) tmem_ld_wait();
    }
#else
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        float va[8], vb[8];
        tmem_ld8(taddr0 + s * 8, va);
        tmem_ld8(taddr1 + s * 8, vb);
        tmem_ld_wait();
        relu_fma8x(va, w0 + s * 8, a0, a1);
        relu_fma8x(vb, w1 + s * 8, b0, b1);
    }
#endif
    return make_float2((a0.x + a0.y) + (a1.x + a1.y), (b0.x + b0.y) + (b1.x + b1.y));
}

// fp16_emulated on the tensor cores (AccumulationMode::fp16_emulated,
// score_scalar.cpp:29-32 / half.cpp:84-91): each head's dot product (the
// MMA's fp32 value) is rounded to binary16 with saturation, ReLU'd as
// x < 0 ? 0 : x, and acc = half(acc + w * r) is accumulated in ascending h
// with the multiply and the add rounded separately — the reference's
// rounding points; only the dot product's own summation order differs from
// the scalar kernel (the MMA's), so results agree to binary16 rounding, not
// bit for bit (score_exact_kernel stays the bit-exact path). Both queries of
// an accumulator pair run in one packed chain: cvt.rn.satfinite.f16x2 +
// FMUL2 / FADD2.
__device__ __forceinline__ float2 half2_round_sat(float a, float b) {
    uint32_t h;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));  // b -> upper, a -> lower
    const __half2 v = *reinterpret_cast<const __half2*>(&h);
    return make_float2(__low2float(v), __high2float(v));
}

__device__ __forceinline__ float2 head_reduce_fp16_2(uint32_t taddr0, uint32_t taddr1, const float* __restrict__ w0,
                                                     const float* __restrict__ w1) {
    float2 acc = make_float2(0.f, 0.f);
    float va[8], vb[8], vc[8], vd[8];
    tmem_ld8(taddr0, va);
    tmem_ld8(taddr1, vb);
    tmem_ld_wait();
#pragma unroll
    for (int s = 0; s < 8; s += 2) {
        tmem_ld8(taddr0 + (s + 1) * 8, vc);
        tmem_ld8(taddr1 + (s + 1) * 8, vd);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float2 d = half2_round_sat(va[c], vb[c]);
            const float2 r = make_float2(d.x < 0.f ? 0.f : d.x, d.y < 0.f ? 0.f : d.y);
            acc = __fadd2_rn(acc, __fmul2_rn(make_float2(w0[s * 8 + c], w1[s * 8 + c]), r));
            acc = half2_round_sat(acc.x, acc.y);
        }
        tmem_ld_wait();
        if (s + 2 < 8) {
            tmem_ld8(taddr0 + (s + 2) * 8, va);
            tmem_ld8(taddr1 + (s + 2) * 8, vb);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float2 d = half2_round_sat(vc[c], vd[c]);
            const float2 r = make_float2(d.x < 0.f ? 0.f : d.x, d.y < 0.f ? 0.f : d.y);
            acc = __fadd2_rn(acc, __fmul2_rn(make_float2(w0[(s + 1) * 8 + c], w1[(s + 1) * 8 + c]), r));
            acc = half2_round_sat(acc.x, acc.y);
        }
        if (s + 2 < 8) tmem_ld_wait();
    }
    return acc;
}

// Instances: kMode 0 = plain masked score tile (production), 1 = strided
// key-tile sample (kt_stride > 1), 2 = plain + candidate bitmap against tau
// (the fused select pre-filter, CSAIDX_SELECT_PREFILTER=1), 3 = plain +
// per-32-key group maxima (two-level select for long rows), 4 = plain with
// the fp16_emulated epilogue (head_reduce_fp16_2); kProbe adds the
// per-role wait-cycle counters (dev). The production instance carries none
// of the optional code.
template <int kMode, bool kProbe>
__global__ void __launch_bounds__(kNumThreads, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap qmap,
                    const __grid_constant__ CUtensorMap kmap, const __grid_constant__ ScoreTcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // Align by offsetting the shared array itself (keeps the shared address
    // space visible to the compiler, so w reads are LDS, not generic loads).
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* q_smem = smem;
    uint8_t* k_smem = smem + kQBytes;
    float* w_smem = reinterpret_cast<float*>(smem + kWOffset);  // [kWBufs][8][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
    uint64_t* k_full = bars;                          // [kStages]
    uint64_t* k_empty = k_full + kStages;             // [kStages]
    uint64_t* q_full = k_empty + kStages;             // [kGroups] one per query-group buffer
    uint64_t* q_empty = q_full + kGroups;             // [kGroups]
    uint64_t* acc_full = q_empty + kGroups;           // [kAcc]
    uint64_t* acc_empty = acc_full + kAcc;            // [kAcc]
    uint64_t* item_full = acc_empty + kAcc;           // [kItemSlots]
    uint64_t* item_empty = item_full + kItemSlots;    // [kItemSlots]
    uint64_t* w_full = item_empty + kItemSlots;       // [kWBufs]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_full + kWBufs);
    Item* items = reinterpret_cast<Item*>(w_full + kWBufs + 2);  // [kItemSlots]

    const int warp = threadIdx.x / 32;
    constexpr bool kFilter = kMode == 2;
    constexpr bool kGmax = kMode == 3;
    constexpr bool kFp16 = kMode == 4;
    long long* const probe = kProbe ? p.probe : nullptr;  // per-CTA wait-cycle counters (profiling)
    const int64_t kts = kMode == 1 ? p.kt_stride : 1;  // key-tile stride (sample mode)

    if (warp == 0 && elect_one()) {
        tma_prefetch(&qmap);
        tma_prefetch(&kmap);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int g = 0; g < kGroups; ++g) {
            mbar_init(&q_full[g], 1);
            mbar_init(&q_empty[g], 1);
        }
        for (int a = 0; a < kAcc; ++a) {
            mbar_init(&acc_full[a], 1);
            mbar_init(&acc_empty[a], kAccDrainers);
        }
        for (int s = 0; s < kItemSlots; ++s) {
            mbar_init(&item_full[s], 1);
            mbar_init(&item_empty[s], 1 + kEpiWarps);  // MMA thread + epilogue warps
        }
        for (int wb = 0; wb < kWBufs; ++wb) mbar_init(&w_full[wb], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ scheduler + TMA producer
        if (elect_one()) {
            const uint64_t keep = policy_evict_last();  // keys are re-read by every query block
            uint32_t kiter = 0, qiter = 0;
            long long pw_k = 0, pw_q = 0;
            for (uint32_t it_iter = 0;; ++it_iter) {
                const uint32_t slot = it_iter % kItemSlots;
                mbar_wait(&item_empty[slot], ((it_iter / kItemSlots) & 1) ^ 1);
                const int idx = atomicAdd(p.sched, 1);
                Item it;
                if (idx >= p.nitems) {
                    it.kt_begin = -1;
                    items[slot] = it;
                    mbar_arrive(&item_full[slot]);
                    if (probe) {
                        probe[blockIdx.x * 8 + 6] = pw_k;
                        probe[blockIdx.x * 8 + 7] = pw_q;
                    }
                    break;
                }
                decode_item(p, idx, it);
                items[slot] = it;
                mbar_arrive(&item_full[slot]);

                // Query groups refill independently: group g of item i is
                // reloaded as soon as item i-1's last group-g MMA retires,
                // overlapping the other group's MMAs; group 1 is issued after
                // the item's first key tile so that tile is never delayed.
                const int64_t qrow64 = static_cast<int64_t>(it.b) * p.op_rows + p.s0 + p.op_shift + it.r0;
                const int32_t qrow = static_cast<int32_t>(qrow64 * kHeads);
                const uint32_t qpar = (qiter & 1) ^ 1;
                auto load_group = [&](int g) {
                    const long long c0 = probe ? clock64() : 0;
                    mbar_wait(&q_empty[g], qpar);
                    if (probe) pw_q += clock64() - c0;
                    mbar_expect_tx(&q_full[g], kQGroupBytes);
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_2d(q_smem + g * kQGroupBytes + hf * kQHalfBytes, &qmap, &q_full[g], hf * 64,
                                    qrow + g * kUmmaN);
                    }
                };
                load_group(0);
                // q_empty[0] of item i-1 retires after item i-1's first group-1
                // MMA, which waited for the epilogue to release item i-2's last
                // accumulator: so with 3 w buffers, buffer (i % 3) is free.
                const uint32_t wb = qiter % kWBufs;
                mbar_expect_tx(&w_full[wb], it.nrows * kWRowBytes);
                bulk_copy_g2s(w_smem + wb * (kQPerItem * kHeads), p.w + qrow64 * kHeads, it.nrows * kWRowBytes,
                              &w_full[wb]);
                const int64_t krow0 = static_cast<int64_t>(it.b) * p.key_blocks + p.t0;
                for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                    const uint32_t s = kiter % kStages;
                    const long long c0 = probe ? clock64() : 0;
                    mbar_wait(&k_empty[s], ((kiter / kStages) & 1) ^ 1);
                    if (probe) pw_k += clock64() - c0;
                    mbar_expect_tx(&k_full[s], kKStageBytes);
                    const int32_t krow = static_cast<int32_t>(krow0 + static_cast<int64_t>(kt) * kts * kBlockKeys);
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_2d_hint(k_smem + s * kKStageBytes + hf * kKHalfBytes, &kmap, &k_full[s], hf * 64,
                                         krow, keep);
                    }
                    ++kiter;
                    if (kt == it.kt_begin)
                        for (int g = 1; g < kGroups; ++g) load_group(g);
                }
                ++qiter;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (elect_one()) {
            uint32_t kiter = 0, qiter = 0, aiter = 0;
            long long mw_k = 0, mw_acc = 0, mw_q = 0;
            const long long m_start = probe ? clock64() : 0;
            const uint32_t q_base = smem_u32(q_smem);
            const uint32_t k_base = smem_u32(k_smem);
            for (uint32_t it_iter = 0;; ++it_iter) {
                const uint32_t slot = it_iter % kItemSlots;
                mbar_wait(&item_full[slot], (it_iter / kItemSlots) & 1);
                const Item it = items[slot];
                mbar_arrive(&item_empty[slot]);
                if (it.kt_begin < 0) {
                    if (probe) {
                        probe[blockIdx.x * 8 + 0] = mw_k;
                        probe[blockIdx.x * 8 + 1] = mw_acc;
                        probe[blockIdx.x * 8 + 2] = mw_q;
                        probe[blockIdx.x * 8 + 3] = clock64() - m_start;
                    }
                    break;
                }
                const uint32_t qpar = qiter & 1;
                ++qiter;
                for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                    const uint32_t s = kiter % kStages;
                    long long c0 = probe ? clock64() : 0;
                    mbar_wait(&k_full[s], (kiter / kStages) & 1);
                    if (probe) mw_k += clock64() - c0;
                    tc_fence_after();
                    for (int g = 0; g < kGroups; ++g) {
                        if (kt == it.kt_begin) {
                            if (probe) c0 = clock64();
                            mbar_wait(&q_full[g], qpar);
                            if (probe) mw_q += clock64() - c0;
                            tc_fence_after();
                        }
                        const uint32_t a = aiter % kAcc;
                        if (probe) c0 = clock64();
                        mbar_wait(&acc_empty[a], ((aiter / kAcc) & 1) ^ 1);
                        if (probe) mw_acc += clock64() - c0;
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
                        if (kt == it.kt_end - 1) umma_commit(&q_empty[g]);  // group g of this item retired
                        ++aiter;
                    }
                    umma_commit(&k_empty[s]);
                    ++kiter;
                }
            }
        }
    } else if (warp >= kFirstEpiWarp) {
        // ------------------------------------------------ epilogue
        // 16 warps: warp w reads TMEM lanes 32*(w % 4).. (its key quarter)
        // and owns slot qsel = (w - 2) / 4: query qsel of every 4-query group
        // (QG = 4) or the query pair of group qsel (QG = 2).
        const int quarter = warp & 3;
        const int qsel = (warp - kFirstEpiWarp) >> 2;
        const uint32_t lane = lane_id();
        const uint32_t quarter_taddr = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
        // The warp's two queries of every item: query qsel of each 4-query
        // group (groups of 4), or both queries of group qsel (groups of 2).
        int wq[2];
        for (int u = 0; u < 2; ++u) wq[u] = kQPerGroup == 4 ? u * kQPerGroup + qsel : qsel * kQPerGroup + u;
        uint32_t aiter = 0, qiter = 0;
        long long ew_acc = 0;
        const long long e_start = probe ? clock64() : 0;
        const float neg_inf = -__int_as_float(0x7f800000);
        for (uint32_t it_iter = 0;; ++it_iter) {
            const uint32_t slot = it_iter % kItemSlots;
            mbar_wait(&item_full[slot], (it_iter / kItemSlots) & 1);
            const Item it = items[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&item_empty[slot]);
            if (it.kt_begin < 0) {
                if (probe && warp == kFirstEpiWarp && lane == 0) {
                    probe[blockIdx.x * 8 + 4] = ew_acc;
                    probe[blockIdx.x * 8 + 5] = clock64() - e_start;
                }
                break;
            }
            const uint32_t wb = qiter % kWBufs;
            const float* w_item = w_smem + wb * (kQPerItem * kHeads);
            // Per-item constants of this warp's 2 queries: output row and the
            // causal limit (first illegal column, t0-relative).
            float* orow[2];
            int lim[2];
            float tq[2];  // candidate thresholds (filter mode)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int qi = wq[u];
                const int64_t r = it.r0 + qi;
                const int64_t grow = static_cast<int64_t>(it.b) * p.rows + r;
                orow[u] = p.out + grow * p.ld;
                int64_t l = p.cols;
                if (p.apply_mask) {
                    l = t_legal_dev(p.s0 + r, p.ratio) - p.t0;
                    l = l < 0 ? 0 : (l > p.cols ? p.cols : l);
                }
                lim[u] = static_cast<int>(l);
                tq[u] = (kFilter && qi < it.nrows) ? p.tau[grow] : 0.f;
            }
            mbar_wait(&w_full[wb], (qiter / kWBufs) & 1);
            ++qiter;
            const int cols = static_cast<int>(p.cols);
            const int out_cols = kts == 1 ? cols : static_cast<int>(p.ld);
            for (int kt = it.kt_begin; kt < it.kt_end; ++kt) {
                const int jo = kt * kBlockKeys + quarter * 32 + static_cast<int>(lane);  // output column
                const int j = jo + kt * (kts - 1) * kBlockKeys;                            // key column
                // groups of 4: one accumulator per query (both buffers per key
                // tile); groups of 2: the warp's group's buffer holds both
                constexpr int kUnits = kQPerGroup == 4 ? 2 : 1;
                constexpr int kPerUnit = 2 / kUnits;
#pragma unroll
                for (int un = 0; un < kUnits; ++un) {
                    const uint32_t a = kQPerGroup == 4 ? aiter % kAcc : static_cast<uint32_t>(qsel);
                    const uint32_t par = kQPerGroup == 4 ? (aiter / kAcc) & 1 : aiter & 1;
                    const long long c0 = probe ? clock64() : 0;
                    mbar_wait(&acc_full[a], par);
                    if (probe) ew_acc += clock64() - c0;
                    tc_fence_after();
                    // Drain the accumulator into registers, release it to the MMA
                    // warp, then do the stores (and mode epilogues) off its
                    // critical path.
                    float accv[kPerUnit];
                    if (kFp16) {  // the unit's queries in one packed chain (a missing second one repeats the first)
                        const int q0 = wq[un * kPerUnit];
                        const int q1 = (kPerUnit == 2 && wq[un * kPerUnit + kPerUnit - 1] < it.nrows)
                                           ? wq[un * kPerUnit + kPerUnit - 1]
                                           : q0;
                        const float2 pr = head_reduce_fp16_2(
                            quarter_taddr + a * kUmmaN + (q0 % kQPerGroup) * kHeads,
                            quarter_taddr + a * kUmmaN + (q1 % kQPerGroup) * kHeads, w_item + q0 * kHeads,
                            w_item + q1 * kHeads);
                        accv[0] = pr.x;
                        accv[kPerUnit - 1] = pr.y;
                    } else if (kPerUnit == 2 && wq[1] < it.nrows) {  // both queries of the accumulator at once
                        const uint32_t col = a * kUmmaN;
                        const float2 pr = head_reduce_tmem2(quarter_taddr + col, quarter_taddr + col + kHeads,
                                                            w_item + wq[0] * kHeads, w_item + wq[1] * kHeads);
                        accv[0] = pr.x;
                        accv[kPerUnit - 1] = pr.y;
                    } else {
#pragma unroll
                        for (int pu = 0; pu < kPerUnit; ++pu) {
                            const int qi = wq[un * kPerUnit + pu];
                            accv[pu] = qi < it.nrows  // warp-uniform
                                           ? head_reduce_tmem(quarter_taddr + a * kUmmaN + (qi % kQPerGroup) * kHeads,
                                                              w_item + qi * kHeads)
                                           : 0.f;
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&acc_empty[a]);
#pragma unroll
                    for (int pu = 0; pu < kPerUnit; ++pu) {
                        const int u = un * kPerUnit + pu;
                        const int qi = wq[u];
                        if (qi < it.nrows) {  // warp-uniform
                            const float acc = accv[pu];
                            const bool legal = j < lim[u];
                            if (jo < out_cols) {
                                if (!kFp16 && legal && !isfinite(acc)) atomicOr(p.nonfinite, 1);
                                orow[u][jo] = legal ? acc : neg_inf;
                            }
                            if (kGmax) {
                                // max over the warp's 32 key columns: one float redux.sync
                                // (sm_100a)
                                float gm;
                                asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;"
                                             : "=f"(gm)
                                             : "f"((legal && jo < out_cols) ? acc : neg_inf));
                                if (lane == 0 && jo < out_cols) {
                                    const int64_t grow = static_cast<int64_t>(it.b) * p.rows + it.r0 + qi;
                                    p.gmax[grow * p.gmax_ld + (jo >> 5)] = gm;
                                }
                            }
                            if (kFilter) {
                                // fused select pre-filter: one candidate word per
                                // warp (32 consecutive key columns)
                                const uint32_t m = __ballot_sync(0xffffffffu, legal && acc >= tq[u]);
                                if (lane == 0) {
                                    const int64_t grow = static_cast<int64_t>(it.b) * p.rows + it.r0 + qi;
                                    p.pass_bits[grow * p.bits_ld + (jo >> 5)] = m;
                                }
                            }
                        }
                    }
                    ++aiter;
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem_base);
    }
    if (threadIdx.x == 0) {
        // The last CTA out re-arms the work counter for the next launch.
        __threadfence();
        if (atomicAdd(p.sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            p.sched[0] = 0;
            p.sched[1] = 0;
            __threadfence();
        }
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
    // Causally illegal entries are scored too: the reference checks the
    // whole tile for non-finite fp32 scores before mask_tile
    // (score.cpp:90-97, then causal.cpp:30-41), so an overflow at a future
    // position raises runtime_error here as well.
    const bool masked = p.apply_mask && t >= t_legal_dev(s, p.ratio);
    const bool f32 = p.operand_f32 != 0;
    const int64_t orow = static_cast<int64_t>(b) * p.op_rows + s + p.op_shift;
    const int64_t qbase = (orow * p.heads) * p.head_dim;
    const int64_t kbase = (static_cast<int64_t>(b) * p.key_blocks + t) * p.head_dim;
    const float* wrow = p.w + orow * p.heads;
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
    *dst = masked ? neg_inf : acc;
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

int score_tc_q_box_rows() { return kUmmaN; }

cudaError_t launch_score_tc(const CUtensorMap& qmap, const CUtensorMap& kmap, ScoreTcParams p,
                            int num_sms, cudaStream_t stream) {
    // Dense piece-major work list: piece pc covers key tiles [pc*tpp,
    // (pc+1)*tpp); the query blocks for which it is causally live form a
    // suffix qb >= nqb - count[pc] because the live extent grows with qb.
    p.nqb = static_cast<int>((p.rows + kQPerItem - 1) / kQPerItem);
    if (p.kt_stride < 1) p.kt_stride = 1;
    const int64_t stride = p.kt_stride;
    const int64_t max_tiles = ((p.cols + kBlockKeys - 1) / kBlockKeys + stride - 1) / stride;  // virtual
    int64_t tpp = kMinTilesPerPiece;
    while ((max_tiles + tpp - 1) / tpp > kScoreMaxPieces) tpp *= 2;
    p.tpp = static_cast<int>(tpp);
    p.npieces = static_cast<int>((max_tiles + tpp - 1) / tpp);
    std::vector<int> live(static_cast<size_t>(p.npieces) + 1, 0);  // live[n] = #qb with exactly n pieces
    for (int qb = 0; qb < p.nqb; ++qb) {
        const int64_t r0 = static_cast<int64_t>(qb) * kQPerItem;
        const int64_t nrows = (p.rows - r0) < kQPerItem ? (p.rows - r0) : kQPerItem;
        int64_t kend = p.cols;
        if (p.apply_mask) {
            kend = (p.s0 + r0 + nrows) / p.ratio - p.t0;
            kend = kend < 0 ? 0 : (kend > p.cols ? p.cols : kend);
        }
        const int64_t ntiles = ((kend + kBlockKeys - 1) / kBlockKeys + stride - 1) / stride;
        ++live[static_cast<size_t>((ntiles + tpp - 1) / tpp)];
    }
    int above = 0;  // #qb with more than pc pieces, built from the top
    std::vector<int> count(static_cast<size_t>(p.npieces), 0);
    for (int pc = p.npieces - 1; pc >= 0; --pc) {
        above += live[static_cast<size_t>(pc) + 1];
        count[static_cast<size_t>(pc)] = above;
    }
    p.piece_start[0] = 0;
    for (int pc = 0; pc < p.npieces; ++pc) p.piece_start[pc + 1] = p.piece_start[pc] + count[pc] * p.batch;
    p.nitems = p.piece_start[p.npieces];
    if (p.nitems <= 0) return cudaSuccess;
    static bool attr_set[kMaxDevices] = {};
    const int attr_set_dev = attr_device();
    if (!attr_set[attr_set_dev]) {
        for (auto* fn : {score_tc_kernel<0, false>, score_tc_kernel<0, true>, score_tc_kernel<1, false>,
                         score_tc_kernel<2, false>, score_tc_kernel<3, false>, score_tc_kernel<4, false>}) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(kSmemBytes));
            if (e != cudaSuccess) return e;
        }
        attr_set[attr_set_dev] = true;
    }
    const int grid = p.nitems < num_sms ? p.nitems : num_sms;
    if (p.fp16)
        score_tc_kernel<4, false><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    else if (p.tau != nullptr)
        score_tc_kernel<2, false><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    else if (p.gmax != nullptr)
        score_tc_kernel<3, false><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    else if (p.kt_stride > 1)
        score_tc_kernel<1, false><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    else if (p.probe != nullptr)
        score_tc_kernel<0, true><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
    else
        score_tc_kernel<0, false><<<grid, kNumThreads, kSmemBytes, stream>>>(qmap, kmap, p);
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
