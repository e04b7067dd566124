// Sparse attention over the indexer's top-k, CTA-pair form (same operator
// and contract as sparse_mla_kernel in attn_sm100.cu; see there for the
// definition and the reference anchors).
//
// Why a pair: an M = 128 tcgen05.mma costs >= ~46 cycles for any N < 128
// (profiles/r02_mma_floor.md), so the single-CTA kernel is bound by its 36
// QK instructions per 32-key block, and both CTAs of a query (one per half
// of Dv) computed all of S. Here the two CTAs of a cluster split the
// contraction instead: CTA r computes the partial scores over Dqk dims
// [288 r, 288 r + 288) (18 MMAs per block), the pair swaps partials through
// distributed shared memory (st.async with mbarrier completion), and both
// form S = S_0 + S_1 (one fp32 add, commutative, so both CTAs hold the same
// bits and make the same softmax decisions). Each CTA then accumulates its
// half of Dv as before.
//  * Each CTA gathers only the 5 SW128 panels (320 dims) it reads: CTA 0
//    dims 0..319 (QK 0..287, V 0..255), CTA 1 dims 256..575 (QK 288..575,
//    V 256..511) — V is local panels 0..3 in both. 20 KiB per 32-key stage.
//  * Q's 288 dims live in TMEM (144 columns): every QK MMA is A-from-TMEM.
//    TMEM: Q 0..143 (of 192) + O 192..447 + S/P 448..511.
//  * The exchange per block and softmax warp: 32 heads x 32 fp32 = 4 KiB
//    each way, chunk-major so both the st.async writes and the shared loads
//    are conflict free; slot reuse is acknowledged by a remote arrive.
// Warp roles as in attn_sm100.cu: 0-3 softmax + epilogue, 4-7 KV
// producers, 8 TMEM owner + MMA issuer, 9-12 Q stagers.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kH = 128;
constexpr int kDqk = 576;
constexpr int kDvHalf = 256;
constexpr int kDqkHalf = 288;              // contraction dims per CTA
constexpr int kQkSteps = kDqkHalf / 16;    // 18 MMAs per block per CTA
constexpr int kCtaPanels = 5;              // SW128 panels gathered per CTA
constexpr int kBlk = 32;
constexpr int kStages = 6;
constexpr int kKvPanelBytes = kBlk * 128;                   // 4 KiB
constexpr int kKvStageBytes = kCtaPanels * kKvPanelBytes;   // 20 KiB
constexpr int kMaxK = 4096;
constexpr int kIdxOffset = kStages * kKvStageBytes;
constexpr int kXchgSlotBytes = kH * kBlk * 4;               // 16 KiB
constexpr int kXchgOffset = kIdxOffset + kMaxK * 4;
constexpr int kRedOffset = kXchgOffset + 2 * kXchgSlotBytes;  // row maxima [2][2][128] + row sums [2][128]
constexpr int kBarOffset = kRedOffset + 3072;
constexpr int kSmemBytes = kBarOffset + 1024 + 1024;
constexpr int kSmWarps = 8;                // softmax warps: 2 per TMEM lane quarter, 16 keys of a block each
constexpr int kCols = kBlk / 2;
constexpr int kThreads = 544;              // 8 softmax + 4 KV producer + 1 MMA + 4 Q-staging warps
constexpr int kProducers = 128;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColQ = 0, kColO = 192;
// three S/P slots: the softmax sends block j+1's partial before it works on
// block j, so S(j+1) must exist while P(j) is pending and S(j+2) is computed
constexpr int kSSlots = 3;
__device__ __forceinline__ uint32_t s_col(uint32_t g) {
    const uint32_t i = g % kSSlots;
    return i == 0 ? 448u : (i == 1 ? 480u : 144u);  // 144..175 lie past Q's 144 columns
}
constexpr float kRescaleLog2 = 8.0f;
#ifndef CSAIDX_ATTN_PROBE
#define CSAIDX_ATTN_PROBE 0  // (dev) clock64 stamps of CTA 0's softmax warp 0 and MMA issuer per block
#endif
#if CSAIDX_ATTN_PROBE
constexpr int kProbeBlocks = 2048;
__device__ long long g_attn_probe[kProbeBlocks * 8];
#define PROBE(slot) \
    if (blockIdx.x == 0 && g < kProbeBlocks) g_attn_probe[g * 8 + (slot)] = clock64();
#else
#define PROBE(slot)
#endif
#ifndef CSAIDX_PAIR_DBG
#define CSAIDX_PAIR_DBG 0  // (dev timing only) 1: no exchange at all, 2: send but never wait for the peer
#endif

__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// 2^y on the FMA pipe for half of each block's exponentials (as attn_sm100.cu)
__device__ __forceinline__ float2 exp2_poly2(float2 y) {
    const float2 magic = make_float2(12582912.f, 12582912.f);
    y.x = fmaxf(y.x, -127.f);
    y.y = fmaxf(y.y, -127.f);
    const float2 t = __fadd2_rn(y, magic);
    const float2 f = __fadd2_rn(y, __fadd2_rn(magic, make_float2(-t.x, -t.y)));
    float2 p = __ffma2_rn(make_float2(0.009591416f, 0.009591416f), f, make_float2(0.05587532f, 0.05587532f));
    p = __ffma2_rn(p, f, make_float2(0.24023689f, 0.24023689f));
    p = __ffma2_rn(p, f, make_float2(0.69312757f, 0.69312757f));
    p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;
    return d;
}

// ---- cluster helpers
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the peer CTA's shared::cluster address of a local shared::cta address
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(peer));
    return r;
}
__device__ __forceinline__ void remote_arrive(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t cluster_addr, float a, float b, float c, float d,
                                            uint32_t cluster_bar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            cluster_addr),
        "f"(a), "f"(b), "f"(c), "f"(d), "r"(cluster_bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

constexpr uint32_t kIdescQK = idesc_bf16_f32(kH, kBlk);
constexpr uint32_t kIdescPV = idesc_bf16_f32(kH, kDvHalf) | (1u << 16);  // B MN-major

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    sparse_mla_pair_kernel(const __grid_constant__ SparseMlaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // the same offset in both CTAs (the dynamic window starts at the same
    // address), so mapa of a local address names the peer's twin
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* kv_smem = smem;
    int32_t* idx_s = reinterpret_cast<int32_t*>(smem + kIdxOffset);
    uint8_t* xchg = smem + kXchgOffset;  // [2 slots][8 chunks][128 heads] x 16 B, written by the peer
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
    uint64_t* kv_full = bars;                    // [kStages]
    uint64_t* kv_empty = kv_full + kStages;      // [kStages]
    uint64_t* s_full = kv_empty + kStages;       // [kSSlots]
    uint64_t* p_full = s_full + kSSlots;         // [kSSlots]
    uint64_t* q_tmem = p_full + kSSlots;         // [1]
    uint64_t* q_free = q_tmem + 1;               // [1]
    uint64_t* o_free = q_free + 1;               // [1]
    uint64_t* vw_free = o_free + 1;              // [kStages]
    uint64_t* x_full = vw_free + kStages;        // [2][kSmWarps] the peer's partial landed (tx bytes)
    uint64_t* x_free = x_full + 2 * kSmWarps;    // [2][kSmWarps] the peer has read my partial
    uint32_t* valid_w = reinterpret_cast<uint32_t*>(x_free + 2 * kSmWarps);  // [kStages]
    float* mx_s = reinterpret_cast<float*>(smem + kRedOffset);  // [2 blocks][2 halves][128 heads]
    float* l_s = mx_s + 4 * kH;                                  // [2 halves][128 heads]
    uint32_t* tmem_slot = valid_w + kStages;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const uint32_t peer = rank ^ 1u;
    const int nb = (p.k + kBlk - 1) / kBlk;
    const int G = p.head_groups;
    const int64_t nitems = p.seq_len * p.batch * G;  // (b, query, head group); the pair splits Dqk / Dv
    const int64_t cid = cluster_id_x(), ncl = nclusters_x();

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], kProducers + 1);
            mbar_init(&kv_empty[s], 1);
            mbar_init(&vw_free[s], kSmWarps);
        }
        for (int s = 0; s < kSSlots; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], kSmWarps);
        }
        mbar_init(q_tmem, 4);
        mbar_init(q_free, 1);
        mbar_init(o_free, kSmWarps);
        for (int i = 0; i < 2 * kSmWarps; ++i) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_free[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 12) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote traffic
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    auto decode = [&](int64_t item, int& b, int64_t& tq, int64_t& hrow) {
        const int64_t qi = item / G;
        b = static_cast<int>(qi / p.seq_len);
        tq = qi - static_cast<int64_t>(b) * p.seq_len;
        hrow = item * kH;  // ((b * S + tq) * G + hg) * 128
    };

    if (warp >= 8 && warp < 12) {
        // ---------------------------------------------------------- KV producers
        const int pt = threadIdx.x - 256;
        constexpr int kPieces = (kBlk * kCtaPanels * 8) / kProducers;  // 10
        static_assert(kProducers == 4 * kBlk, "4 producer threads per gathered row");
        const int r = pt >> 2;
        uint32_t soff[kPieces];
#pragma unroll
        for (int u = 0; u < kPieces; ++u) {
            const int cc = (pt & 3) + 4 * u;
            soff[u] = (cc >> 3) * kKvPanelBytes + r * 128 + (((cc & 7) ^ (r & 7)) << 4);
        }
        uint32_t g = 0;
        for (int64_t item = cid; item < nitems; item += ncl) {
            int b;
            int64_t tq, hrow;
            decode(item, b, tq, hrow);
            const int32_t* idx_row = p.indices + (static_cast<int64_t>(b) * p.seq_len + tq) * p.idx_ld;
            asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
            for (int i = pt; i < nb * kBlk; i += kProducers) {
                const int32_t idx = i < p.k ? __ldg(idx_row + i) : -1;
                idx_s[i] = (idx >= 0 && idx < p.kv_len) ? idx : -1;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
            // this CTA's panels start at dim 256 * rank
            const char* kv_b = reinterpret_cast<const char*>(p.kv) + static_cast<int64_t>(b) * p.kv_len * (kDqk * 2) +
                               rank * 512 + (pt & 3) * 16;
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % kStages;
                const int32_t myidx = idx_s[j * kBlk + r];
                const char* src = kv_b + static_cast<int64_t>(myidx >= 0 ? myidx : 0) * (kDqk * 2);
                uint32_t vmask = 0;
                if (warp == 8) vmask = __ballot_sync(0xffffffffu, idx_s[j * kBlk + lane] >= 0);
                mbar_wait(&kv_empty[s], ((g / kStages) & 1) ^ 1);
                asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
                if (pt == 0) {
                    mbar_wait(&vw_free[s], ((g / kStages) & 1) ^ 1);
                    valid_w[s] = vmask;
                    mbar_arrive(&kv_full[s]);
                }
                const uint32_t st = smem_u32(kv_smem + s * kKvStageBytes);
#pragma unroll
                for (int u = 0; u < kPieces; ++u)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + soff[u]), "l"(src + 64 * u)
                                 : "memory");
                asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&kv_full[s]))
                             : "memory");
            }
        }
    } else if (warp >= 13) {
        // ---------------------------------------------------------- Q stagers
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        uint32_t it = 0;
        for (int64_t item = cid; item < nitems; item += ncl, ++it) {
            int b;
            int64_t tq, hrow;
            decode(item, b, tq, hrow);
            // this CTA's 288 dims of the head row
            const uint4* qsrc = reinterpret_cast<const uint4*>(p.q + (hrow + row) * kDqk + rank * kDqkHalf);
#pragma unroll
            for (int c = 0; c < kDqkHalf * 2; c += 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(qsrc) + c));
            if (it > 0) {
                mbar_wait(q_free, (it - 1) & 1);
                tc_fence_after();
            }
#pragma unroll 1
            for (int c0 = 0; c0 < 128; c0 += 64) {  // columns 0..127 (dims 0..255 of the half)
                uint32_t w[64];
                uint4* w4 = reinterpret_cast<uint4*>(w);
#pragma unroll
                for (int v = 0; v < 16; ++v) w4[v] = __ldg(qsrc + c0 / 4 + v);
                tmem_st16(lane_base + kColQ + c0, *reinterpret_cast<uint32_t(*)[16]>(w));
                tmem_st16(lane_base + kColQ + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(w + 16));
                tmem_st16(lane_base + kColQ + c0 + 32, *reinterpret_cast<uint32_t(*)[16]>(w + 32));
                tmem_st16(lane_base + kColQ + c0 + 48, *reinterpret_cast<uint32_t(*)[16]>(w + 48));
            }
            {  // columns 128..143 (dims 256..287 of the half)
                uint32_t w[16];
                uint4* w4 = reinterpret_cast<uint4*>(w);
#pragma unroll
                for (int v = 0; v < 4; ++v) w4[v] = __ldg(qsrc + 32 + v);
                tmem_st16(lane_base + kColQ + 128, w);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(q_tmem);
        }
    } else if (warp == 12) {
        // ---------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t kv_base = smem_u32(kv_smem);
            // K step kk of this CTA = global step 18 rank + kk: local panel
            // (global >> 2) - 4 rank, 32-byte step (global & 3) inside it
            uint32_t boff[kQkSteps];
#pragma unroll
            for (int kk = 0; kk < kQkSteps; ++kk) {
                const int gk = kQkSteps * static_cast<int>(rank) + kk;
                boff[kk] = ((gk >> 2) - 4 * static_cast<int>(rank)) * kKvPanelBytes + (gk & 3) * 32;
            }
            uint32_t g = 0, it = 0;
            for (int64_t item = cid; item < nitems; item += ncl, ++it) {
                mbar_wait(q_tmem, it & 1);
                tc_fence_after();
                auto issue_pv = [&](int j, uint32_t gj) {
                    const int s = gj % kStages;
                    if (j == 0 && it > 0) mbar_wait(o_free, (it - 1) & 1);
                    mbar_wait(&p_full[gj % kSSlots], (gj / kSSlots) & 1);
                    {
                        const uint32_t g = gj;
                        PROBE(5)
                    }
                    tc_fence_after();
                    const uint32_t vb = kv_base + s * kKvStageBytes;  // V = local panels 0..3
#pragma unroll
                    for (int kk = 0; kk < kBlk / 16; ++kk)
                        umma_bf16_ts(tmem + kColO, tmem + s_col(gj) + kk * 16,
                                     sw128_mnmajor_desc(vb + kk * 2048, kKvPanelBytes, 1024), kIdescPV,
                                     (j > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&kv_empty[s]);
                };
                auto issue_qk = [&](int j, uint32_t gj) {
                    const int s = gj % kStages;
                    mbar_wait(&kv_full[s], (gj / kStages) & 1);
                    {
                        const uint32_t g = gj;
                        PROBE(4)
                    }
                    fence_proxy_async();
                    tc_fence_after();
                    const uint32_t st = kv_base + s * kKvStageBytes;
                    const uint32_t d = tmem + s_col(gj);
#pragma unroll
                    for (int kk = 0; kk < kQkSteps; ++kk)
                        umma_bf16_ts(d, tmem + kColQ + kk * 8, sw128_kmajor_desc(st + boff[kk]), kIdescQK,
                                     kk > 0 ? 1u : 0u);
                    umma_commit(&s_full[gj % kSSlots]);
                    if (j == nb - 1) umma_commit(q_free);
                };
                // QK two blocks ahead of PV: the softmax of block j starts by
                // sending S(j+1), and QK(j+2) (the slot of P(j-1), whose PV
                // was issued one iteration earlier) runs while it waits for P(j)
                issue_qk(0, g);
                if (nb > 1) issue_qk(1, g + 1);
                for (int j = 0; j < nb; ++j) {
                    if (j + 2 < nb) issue_qk(j + 2, g + j + 2);
                    issue_pv(j, g + j);
                }
                g += nb;
            }
        }
    } else {
        // ---------------------------------------------------------- softmax + epilogue
        // warp = (half of the block's keys hf, TMEM lane quarter): the pair of
        // warps of a quarter share the row max through shared memory each
        // block and the row sum at the end
        const int quarter = warp & 3, hf = warp >> 2;
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float scale_log2 = p.sm_scale * 1.4426950408889634f;
        const float ninf = -INFINITY;
        auto pair_sync = [&] {  // the two warps of this quarter
            tc_fence_before();
            asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");
            tc_fence_after();
        };
        // exchange: my 16 columns of the partial go to the peer's slot,
        // chunk-major [chunk][head] x 16 B (conflict free both ways)
        const uint32_t x_local = smem_u32(xchg);
        const uint32_t x_peer = peer_addr(x_local, peer);
        const uint32_t xf_peer0 = peer_addr(smem_u32(&x_full[warp]), peer);
        const uint32_t xf_peer1 = peer_addr(smem_u32(&x_full[kSmWarps + warp]), peer);
        const uint32_t xr_peer0 = peer_addr(smem_u32(&x_free[warp]), peer);
        const uint32_t xr_peer1 = peer_addr(smem_u32(&x_free[kSmWarps + warp]), peer);
        const uint32_t xoff = ((4 * hf) * kH + row) * 16;  // first chunk of this warp's columns
        // own partial of block gs: read it, st.async it to the peer (after the
        // peer released the slot), post the receive of the peer's partial
        auto send = [&](uint32_t gs, float (&y)[kCols]) {
            const int sl = static_cast<int>(gs & 1);
            mbar_wait(&s_full[gs % kSSlots], (gs / kSSlots) & 1);
            tc_fence_after();
            tmem_ld16(lane_base + s_col(gs) + hf * kCols, y);
            if (lane == 0) mbar_expect_tx(&x_full[sl * kSmWarps + warp], 32 * kCols * 4);
            tmem_ld_wait();
            if (CSAIDX_PAIR_DBG == 1) return;
            if (CSAIDX_PAIR_DBG == 0) mbar_wait_cluster(&x_free[sl * kSmWarps + warp], ((gs >> 1) & 1) ^ 1);
#pragma unroll
            for (int q = 0; q < kCols / 4; ++q)
                st_async_v4(x_peer + sl * kXchgSlotBytes + xoff + q * kH * 16, y[4 * q], y[4 * q + 1], y[4 * q + 2],
                            y[4 * q + 3], sl ? xf_peer1 : xf_peer0);
        };
        uint32_t g = 0;
        for (int64_t item = cid; item < nitems; item += ncl) {
            int b;
            int64_t tq, hrow;
            decode(item, b, tq, hrow);
            float m = ninf, l = 0.f;  // l: this warp's keys only (same m in both warps)
            float nxt[kCols];
            send(g, nxt);
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % kStages;
                const int sl = static_cast<int>(g & 1);
                float x[kCols];
                if (warp == 0 && lane == 0) { PROBE(0) }
#pragma unroll
                for (int c = 0; c < kCols; ++c) x[c] = nxt[c];
                if (j + 1 < nb) send(g + 1, nxt);  // overlaps the exchange with this block's softmax
                if (warp == 0 && lane == 0) { PROBE(1) }
                mbar_wait(&kv_full[s], (g / kStages) & 1);  // completed: orders the valid word
                uint32_t vm = 0;
                if (lane == 0) {
                    vm = valid_w[s];
                    mbar_arrive(&vw_free[s]);
                }
                vm = (__shfl_sync(0xffffffffu, vm, 0) >> (kCols * hf)) & 0xffffu;
                // the peer's partial -> S = S_0 + S_1 (same bits in both CTAs)
                if (CSAIDX_PAIR_DBG == 0) mbar_wait_cluster(&x_full[sl * kSmWarps + warp], (g >> 1) & 1);
                if (warp == 0 && lane == 0) { PROBE(2) }
#pragma unroll
                for (int q = 0; q < kCols / 4 && CSAIDX_PAIR_DBG != 1; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(xchg + sl * kXchgSlotBytes + xoff + q * kH * 16);
                    x[4 * q] += v.x;
                    x[4 * q + 1] += v.y;
                    x[4 * q + 2] += v.z;
                    x[4 * q + 3] += v.w;
                }
                __syncwarp();
                if (lane == 0 && CSAIDX_PAIR_DBG == 0) remote_arrive(sl ? xr_peer1 : xr_peer0);  // the peer may refill my slot
                if (vm != 0xffffu) {
#pragma unroll
                    for (int c = 0; c < kCols; ++c) x[c] = ((vm >> c) & 1u) ? x[c] : ninf;
                }
                const float mh = max3f(max3f(max3f(x[0], x[1], x[2]), max3f(x[3], x[4], x[5]), max3f(x[6], x[7], x[8])),
                                       max3f(max3f(x[9], x[10], x[11]), max3f(x[12], x[13], x[14]), x[15]), ninf);
                mx_s[(sl * 2 + hf) * kH + row] = mh;
                pair_sync();
                const float mx = fmaxf(mh, mx_s[(sl * 2 + (hf ^ 1)) * kH + row]) * scale_log2;
                float alpha = 1.f;
                bool rescale = false;
                if (mx > m) {
                    if (m == ninf) {
                        m = mx;
                    } else if (mx > m + kRescaleLog2) {
                        alpha = ex2(m - mx);
                        l *= alpha;
                        m = mx;
                        rescale = true;
                    }
                }
                if (__any_sync(0xffffffffu, rescale)) {
                    // PV of block g-1 landed (exact parity wait: attn_sm100.cu);
                    // each warp of the quarter rescales its half of O's columns
                    mbar_wait(&kv_empty[(g - 1) % kStages], ((g - 1) / kStages) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = hf * (kDvHalf / 2); c0 < (hf + 1) * (kDvHalf / 2); c0 += 32) {
                        float o[32];
                        tmem_ld32(lane_base + kColO + c0, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] *= alpha;
                        tmem_st32(lane_base + kColO + c0, o);
                    }
                    tmem_st_wait();
                }
                uint32_t pk[kCols / 2];
                if (m != ninf) {
                    const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
                    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                    for (int c = 0; c < kCols; c += 2) {
                        const float2 a = __ffma2_rn(make_float2(x[c], x[c + 1]), sc2, nm2);
                        float2 pr;
                        if (c < kCols / 2) {
                            pr.x = ex2(a.x);
                            pr.y = ex2(a.y);
                        } else {
                            pr = exp2_poly2(a);
                        }
                        acc = __fadd2_rn(acc, pr);
                        const __nv_bfloat162 h2 = __floats2bfloat162_rn(pr.x, pr.y);
                        pk[c / 2] = *reinterpret_cast<const uint32_t*>(&h2);
                    }
                    l += acc.x + acc.y;
                } else {
#pragma unroll
                    for (int c = 0; c < kCols / 2; ++c) pk[c] = 0u;
                }
                // P of these 16 keys over the first 8 of the warp's own S columns
                tmem_st8(lane_base + s_col(g) + hf * kCols, pk);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[g % kSSlots]);
                if (warp == 0 && lane == 0) { PROBE(3) }
            }
            // the row sum over both warps' keys (same order in both: l_0 + l_1)
            l_s[hf * kH + row] = l;
            mbar_wait(&kv_empty[(g - 1) % kStages], ((g - 1) / kStages) & 1);  // the item's last PV landed
            pair_sync();
            const float lt = l_s[row] + l_s[kH + row];
            const float inv_l = lt > 0.f ? 1.f / lt : 0.f;
            __nv_bfloat16* orow = p.out + (hrow + row) * p.out_ld + rank * kDvHalf;
#pragma unroll 1
            for (int c0 = hf * (kDvHalf / 2); c0 < (hf + 1) * (kDvHalf / 2); c0 += 32) {
                float o[32];
                tmem_ld32(lane_base + kColO + c0, o);
                tmem_ld_wait();
                uint4 pk[4];
                uint32_t* pw = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    const __nv_bfloat162 h2 = __floats2bfloat162_rn(o[c] * inv_l, o[c + 1] * inv_l);
                    pw[c / 2] = *reinterpret_cast<const uint32_t*>(&h2);
                }
                uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
                for (int v = 0; v < 4; ++v) dst[v] = pk[v];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(o_free);
            if (rank == 0 && hf == 0 && p.lse != nullptr)
                p.lse[hrow + row] = lt > 0.f ? (m + __log2f(lt)) * 0.6931471805599453f : ninf;
            // l_s is rewritten only after the next item's blocks, which pass pair_sync
        }
    }

    tc_fence_before();
    cluster_sync_all();  // no remote arrive / st.async may target an exited CTA
    if (warp == 12) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

}  // namespace

#if CSAIDX_ATTN_PROBE
extern "C" int csaidx_dev_attn_probe(long long* out, int n) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, g_attn_probe, sizeof(long long) * n));
}
#endif

namespace csaidx_kern {

int sparse_mla_pair_smem_bytes() { return kSmemBytes; }

cudaError_t launch_sparse_mla_pair(const SparseMlaParams& p, cudaStream_t stream) {
    if (p.seq_len <= 0 || p.batch <= 0) return cudaSuccess;
    static bool attr_set[kMaxDevices] = {};
    const int dev = attr_device();
    if (!attr_set[dev]) {
        cudaError_t e =
            cudaFuncSetAttribute(sparse_mla_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    // persistent: one CTA pair per two SMs walks the (b, query, head group) items
    int sms = 0, cur = 0;
    cudaGetDevice(&cur);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur);
    const int64_t items = p.seq_len * p.batch * p.head_groups;
    const int64_t pairs = items < sms / 2 ? items : sms / 2;
    sparse_mla_pair_kernel<<<static_cast<unsigned>(2 * pairs), kThreads, kSmemBytes, stream>>>(p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
