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
//    V 256..511) — V is local panels 0..3 in both. 20 KiB per 32-key stage,
//    7 stages; indices read from global memory one block ahead.
//  * Q's 288 dims live in TMEM (144 columns; every QK MMA is A-from-TMEM),
//    brought in per item as 5 panels through a 2-slot TMA ring and
//    tcgen05.cp (in issue order with the MMAs). TMEM: Q 0..143, a third
//    S/P slot 144..175, O 192..447, S/P 448..511.
//  * Two softmax teams of 4 warps take alternate blocks (three S slots: QK
//    runs two blocks ahead of PV); the running max passes between teams
//    through shared memory, each team keeps its own row sum.
//  * The exchange per block and softmax warp: 32 heads x 32 fp32 = 4 KiB
//    each way, chunk-major so both the st.async writes and the shared loads
//    are conflict free; slot reuse is acknowledged by a remote arrive.
//  * The MMA issuer polls: QK and PV each in order, whichever has its inputs.
// Measured (profiles/r02_attention.md): correct, but no faster than the
// single-CTA kernel (0.42 vs 0.40-0.43 of the sustained peak at k = 1024):
// the per-block chain of a team (S -> exchange ~0.8-1K cycles -> max /
// exponentials -> P, ~3.1K cycles) over two teams sets a ~1.6K-cycle block
// period, above the ~1.1K of MMA work. Opt-in: CSAIDX_ATTN_PAIR=1.
// Warps: 0-7 softmax (team = warp / 4, TMEM quarter = warp % 4), 8-11 KV
// producers, 12 TMEM owner + MMA issuer, 13-16 epilogue (O / l -> bf16 rows
// of the previous item), 17 Q TMA.
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
constexpr int kStages = 7;
constexpr int kKvPanelBytes = kBlk * 128;                   // 4 KiB
constexpr int kKvStageBytes = kCtaPanels * kKvPanelBytes;   // 20 KiB
constexpr int kQPanelBytes = 128 * 128;                     // 128 heads x 64 dims
constexpr int kQSlots = 2;                                  // Q panels in flight (TMA -> tcgen05.cp ring)
constexpr int kKvOffset = kQSlots * kQPanelBytes;
constexpr int kXchgSlotBytes = kH * kBlk * 4;               // 16 KiB
constexpr int kXchgOffset = kKvOffset + kStages * kKvStageBytes;
constexpr int kRedOffset = kXchgOffset + 2 * kXchgSlotBytes;  // row maxima [2][2][128] + row sums [2][128]
constexpr int kBarOffset = kRedOffset + 3072;
constexpr int kSmemBytes = kBarOffset + 1024 + 1024;
constexpr int kSmWarps = 8;                // softmax warps: two teams of 4 (one per TMEM lane quarter), alternating blocks
constexpr int kThreads = 576;              // 8 softmax + 4 KV producer + 1 MMA + 4 epilogue + 1 Q-TMA warps
constexpr int kProducers = 128;
constexpr int kWarpMma = 12, kWarpEpi = 13, kWarpQ = 17;  // epilogue warps 13..16 cover TMEM lane quarters 1, 2, 3, 0
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
__device__ long long g_attn_probe[kProbeBlocks * 16];
#define PROBE(slot) \
    if (blockIdx.x == 0 && g < kProbeBlocks) g_attn_probe[g * 16 + (slot)] = clock64();
#else
#define PROBE(slot)
#endif
#ifndef CSAIDX_PAIR_L1PF
#define CSAIDX_PAIR_L1PF 0  // (measured slower) L1 prefetch of a block's rows before its stage frees (cp.async.ca then hits L1)
#endif
#ifndef CSAIDX_PAIR_POLL_NS
#define CSAIDX_PAIR_POLL_NS 64  // MMA issuer back-off when nothing is ready
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
    sparse_mla_pair_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ SparseMlaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // the same offset in both CTAs (the dynamic window starts at the same
    // address), so mapa of a local address names the peer's twin
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* q_smem = smem;  // ring of Q panels (TMA), copied into TMEM by tcgen05.cp
    uint8_t* kv_smem = smem + kKvOffset;
    uint8_t* xchg = smem + kXchgOffset;  // [2 slots][8 chunks][128 heads] x 16 B, written by the peer
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
    uint64_t* kv_full = bars;                    // [kStages]
    uint64_t* kv_empty = kv_full + kStages;      // [kStages]
    uint64_t* s_full = kv_empty + kStages;       // [kSSlots]
    uint64_t* p_full = s_full + kSSlots;         // [kSSlots]
    uint64_t* q_sfull = p_full + kSSlots;        // [kQSlots] a Q panel landed in shared memory (TMA)
    uint64_t* q_sfree = q_sfull + kQSlots;       // [kQSlots] its copy into TMEM completed (slot reusable)
    uint64_t* o_free = q_sfree + kQSlots;        // [1]
    uint64_t* vw_free = o_free + 1;              // [kStages]
    uint64_t* x_full = vw_free + kStages;        // [2][kSmWarps] the peer's partial landed (tx bytes)
    uint64_t* x_free = x_full + 2 * kSmWarps;    // [2][kSmWarps] the peer has read my partial
    uint32_t* valid_w = reinterpret_cast<uint32_t*>(x_free + 2 * kSmWarps);  // [kStages]
    float* m_s = reinterpret_cast<float*>(smem + kRedOffset);  // [team][128 heads] running max after its last block
    float* ml_s = m_s + 2 * kH;                                 // [team][2][128 heads] (m, l) at the item's end
    uint64_t* m_ready = reinterpret_cast<uint64_t*>(smem + kBarOffset + 768);  // [team][quarter] m_s published
    uint64_t* ml_ready = m_ready + kSmWarps;  // [quarter] both teams' (m, l) of an item written
    uint32_t* tmem_slot = valid_w + kStages;
    static_assert((3 * kStages + 2 * kSSlots + 2 * kQSlots + 1 + 4 * kSmWarps) * 8 + (kStages + 1) * 4 <= 768,
                  "barrier block overlaps m_ready");

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
            mbar_init(&vw_free[s], 4);
        }
        for (int s = 0; s < kSSlots; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 4);
        }
        for (int i = 0; i < kQSlots; ++i) {
            mbar_init(&q_sfull[i], 1);
            mbar_init(&q_sfree[i], 1);
        }
        mbar_init(o_free, 128);  // every lane of the 4 epilogue warps
        for (int i = 0; i < 2 * kSmWarps; ++i) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_free[i], 1);
        }
        // arrivals per lane (each lane's own shared-memory write, then its
        // arrive): the hand-offs stay ordered lane by lane
        // (m_ready: one arrive per warp after __syncwarp; per-lane arrivals
        // measured wrong results here, not understood — kept out)
        for (int i = 0; i < kSmWarps; ++i) mbar_init(&m_ready[i], 1);
        for (int i = 0; i < 4; ++i) mbar_init(&ml_ready[i], 64);  // both teams' warps of the quarter
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kWarpMma) tmem_alloc<kTmemCols>(tmem_slot);
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

    if (warp >= 8 && warp < kWarpMma) {
        // ---------------------------------------------------------- KV producers
        const int pt = threadIdx.x - 256;  // 0..127: four threads per gathered row
        constexpr int kPieces = (kBlk * kCtaPanels * 8) / kProducers;  // 10 pieces of 16 B
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
            auto load_idx = [&](int i) {  // -1: padding, past k or out of range
                const int32_t idx = i < p.k ? __ldg(idx_row + i) : -1;
                return (idx >= 0 && idx < p.kv_len) ? idx : -1;
            };
            // this CTA's panels start at dim 256 * rank
            const char* kv_b = reinterpret_cast<const char*>(p.kv) + static_cast<int64_t>(b) * p.kv_len * (kDqk * 2) +
                               rank * 512 + (pt & 3) * 16;
            int32_t nidx = load_idx(r), nval = warp == 8 ? load_idx(lane) : 0;  // block 0's, then one ahead
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % kStages;
                const int32_t myidx = nidx;
                const uint32_t vmask = warp == 8 ? __ballot_sync(0xffffffffu, nval >= 0) : 0u;
                if (j + 1 < nb) {
                    nidx = load_idx((j + 1) * kBlk + r);
                    if (warp == 8) nval = load_idx((j + 1) * kBlk + lane);
                }
                const char* src = kv_b + static_cast<int64_t>(myidx >= 0 ? myidx : 0) * (kDqk * 2);
#if CSAIDX_PAIR_L1PF
                {
                    // pull this block's rows toward the SM while the stage is
                    // still in use: the copies below then hit L1 instead of
                    // paying the L2 latency after the stage frees up
                    const char* line = src - (pt & 3) * 16;  // the row's 640 bytes: 5 lines of 128 B
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(line + (pt & 3) * 128));
                    if ((pt & 3) == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(line + 512));
                }
#endif
                mbar_wait(&kv_empty[s], ((g / kStages) & 1) ^ 1);
                if (pt == 0) { PROBE(6) }
                asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
                if (pt == 0) {
                    mbar_wait(&vw_free[s], ((g / kStages) & 1) ^ 1);
                    valid_w[s] = vmask;
                    mbar_arrive(&kv_full[s]);
                }
                const uint32_t st = smem_u32(kv_smem + s * kKvStageBytes);
#pragma unroll
                for (int u = 0; u < kPieces; ++u)
#if CSAIDX_PAIR_L1PF
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(st + soff[u]), "l"(src + 64 * u)
                                 : "memory");
#else
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(st + soff[u]), "l"(src + 64 * u)
                                 : "memory");
#endif
                asm volatile("cp.async.commit_group;" ::: "memory");
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&kv_full[s]))
                             : "memory");
                if (pt == 0) { PROBE(7) }
            }
        }
    } else if (warp == kWarpQ) {
        // ---------------------------------------------------------- Q panels by TMA
        // panel P = it * 5 + pn (64 of this CTA's 288 dims of the item's 128
        // head rows; the last one half used) into slot P % kQSlots once the
        // panel kQSlots back has been copied into TMEM
        if (lane == 0) {
            uint32_t P = 0;
            for (int64_t item = cid; item < nitems; item += ncl) {
                int b;
                int64_t tq, hrow;
                decode(item, b, tq, hrow);
                for (int pn = 0; pn < kCtaPanels; ++pn, ++P) {
                    const int sl = P % kQSlots;
                    mbar_wait(&q_sfree[sl], ((P / kQSlots) & 1) ^ 1);
                    mbar_expect_tx(&q_sfull[sl], kQPanelBytes);
                    tma_load_2d(q_smem + sl * kQPanelBytes, &qmap, &q_sfull[sl],
                                static_cast<int32_t>(rank * kDqkHalf + pn * 64), static_cast<int32_t>(hrow));
                }
            }
        }
    } else if (warp >= kWarpEpi) {
        // ---------------------------------------------------------- Q stagers + epilogue
        // Stage item it's Q once item it-1's S MMAs retired, then write item
        // it-1's output (O / l from TMEM) while the softmax teams already
        // work on item it; the next item's first PV waits for o_free.
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float ninf = -INFINITY;
        auto epilogue = [&](uint32_t ie, int64_t hrow_e) {
            mbar_wait(&ml_ready[quarter], ie & 1);  // both teams' (m, l) of item ie
            const float m0 = ml_s[row], l0 = ml_s[kH + row], m1 = ml_s[2 * kH + row], l1 = ml_s[3 * kH + row];
            const float M = fmaxf(m0, m1);
            const float L = (l0 > 0.f ? l0 * ex2(m0 - M) : 0.f) + (l1 > 0.f ? l1 * ex2(m1 - M) : 0.f);
            const float inv_l = L > 0.f ? 1.f / L : 0.f;
            const uint32_t gl = (ie + 1) * static_cast<uint32_t>(nb) - 1;  // the item's last block
            mbar_wait(&kv_empty[gl % kStages], (gl / kStages) & 1);       // its PV landed (exact: next phase needs o_free)
            tc_fence_after();
            __nv_bfloat16* orow = p.out + (hrow_e + row) * p.out_ld + rank * kDvHalf;
#pragma unroll 1
            for (int c0 = 0; c0 < kDvHalf; c0 += 32) {
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
            mbar_arrive(o_free);
            if (rank == 0 && p.lse != nullptr)
                p.lse[hrow_e + row] = L > 0.f ? (M + __log2f(L)) * 0.6931471805599453f : ninf;
        };
        uint32_t it = 0;
        int64_t prev_hrow = 0;
        for (int64_t item = cid; item < nitems; item += ncl, ++it) {
            int b;
            int64_t tq, hrow;
            decode(item, b, tq, hrow);
            if (it > 0) epilogue(it - 1, prev_hrow);
            prev_hrow = hrow;
        }
        if (it > 0) epilogue(it - 1, prev_hrow);
    } else if (warp == kWarpMma) {
        // ---------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t kv_base = smem_u32(kv_smem);
            // K step kk of this CTA = global step 18 rank + kk: local panel
            // (global >> 2) - 4 rank, 32-byte step (global & 3) inside it
            auto boff = [&](int kk) {
                const int gk = kQkSteps * static_cast<int>(rank) + kk;
                return static_cast<uint32_t>(((gk >> 2) - 4 * static_cast<int>(rank)) * kKvPanelBytes + (gk & 3) * 32);
            };
            // One global block sequence over this cluster's items (block G =
            // item G / nb, key block G % nb): QK runs two blocks ahead of PV
            // across item boundaries too, so the next item's first scores are
            // computed while the current item's last softmax blocks finish.
            const uint32_t my_items = cid < nitems ? static_cast<uint32_t>((nitems - 1 - cid) / ncl + 1) : 0u;
            const uint32_t total = my_items * static_cast<uint32_t>(nb);
            auto issue_pv = [&](uint32_t gj) {
                const uint32_t it = gj / nb;
                const int j = static_cast<int>(gj - it * nb);
                const int s = gj % kStages;
                if (j == 0 && it > 0) mbar_wait(o_free, (it - 1) & 1);  // the last epilogue has read O
                mbar_wait(&p_full[gj % kSSlots], (gj / kSSlots) & 1);
                {
                    const uint32_t g = gj;
                    PROBE(5)
                }
                tc_fence_after();
                const uint32_t vb = kv_base + s * kKvStageBytes;  // V = local panels 0..3
#pragma unroll
                for (int kk = 0; kk < kBlk / 16; ++kk)
                    umma_bf16_ts(tmem + kColO, tmem + s_col(gj) + kk * 8,
                                 sw128_mnmajor_desc(vb + kk * 2048, kKvPanelBytes, 1024), kIdescPV,
                                 (j > 0 || kk > 0) ? 1u : 0u);
                umma_commit(&kv_empty[s]);
            };
            auto issue_qk = [&](uint32_t gj) {
                const uint32_t it = gj / nb;
                const int j = static_cast<int>(gj - it * nb);
                const int s = gj % kStages;
                (void)j;
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
                    umma_bf16_ts(d, tmem + kColQ + kk * 8, sw128_kmajor_desc(st + boff(kk)), kIdescQK,
                                 kk > 0 ? 1u : 0u);
                umma_commit(&s_full[gj % kSSlots]);
            };
            // Polling issue: QK(nq) and PV(np) each in order, QK at most two
            // blocks ahead of PV (QK(G) reuses the S slot of P(G-3)), and
            // whichever has its inputs goes first, so a late gather does not
            // hold back a ready PV and a slow softmax does not hold back the
            // next scores.
            auto ready = [&](uint64_t* bar, uint32_t parity) {
                uint32_t ok;
                asm volatile(
                    "{\n\t.reg .pred P;\n\t"
                    "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, P;\n\t}"
                    : "=r"(ok)
                    : "r"(smem_u32(bar)), "r"(parity)
                    : "memory");
                return ok != 0;
            };
            // Q panel P: shared memory -> TMEM columns 8 * (4 pn + t), one
            // 128 x 256-bit copy per K step, in issue order with the MMAs (so
            // after the previous item's QK, which read the old Q)
            const uint32_t qb = smem_u32(q_smem);
            auto issue_qcopy = [&](uint32_t P) {
                const int sl = P % kQSlots;
                const int pn = static_cast<int>(P % kCtaPanels);
                mbar_wait(&q_sfull[sl], (P / kQSlots) & 1);
                tc_fence_after();
                const int steps = pn < 4 ? 4 : kQkSteps - 16;
                for (int t = 0; t < steps; ++t)
                    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + kColQ + (4 * pn + t) * 8),
                                 "l"(sw128_kmajor_desc(qb + sl * kQPanelBytes + t * 32))
                                 : "memory");
                umma_commit(&q_sfree[sl]);
            };
            const uint32_t total_q = my_items * kCtaPanels;
            uint32_t nc = 0;  // Q panels copied
            auto qk_ready = [&](uint32_t gj) {
                const uint32_t it = gj / nb;
                if (gj == it * nb && nc < (it + 1) * kCtaPanels) return false;  // the item's Q not all in TMEM yet
                return ready(&kv_full[gj % kStages], (gj / kStages) & 1);
            };
            auto pv_ready = [&](uint32_t gj) {
                const uint32_t it = gj / nb;
                if (gj == it * nb && it > 0 && !ready(o_free, (it - 1) & 1)) return false;
                return ready(&p_full[gj % kSSlots], (gj / kSSlots) & 1);
            };
            uint32_t nq = 0, np = 0;
            while (np < total) {
                bool did = false;
                // the next item's Q panels once every QK of the current item is issued
                if (nc < total_q && nq >= (nc / kCtaPanels) * nb &&
                    ready(&q_sfull[nc % kQSlots], (nc / kQSlots) & 1)) {
                    issue_qcopy(nc);
                    ++nc;
                    did = true;
                }
                if (nq < total && nq <= np + 2 && qk_ready(nq)) {
                    issue_qk(nq);
                    ++nq;
                    did = true;
                }
                if (np < nq && pv_ready(np)) {
                    issue_pv(np);
                    ++np;
                    did = true;
                }
                if (!did) __nanosleep(CSAIDX_PAIR_POLL_NS);  // leave the issue slots to the softmax warps
            }
        }
    } else {
        // ---------------------------------------------------------- softmax + epilogue
        // Two teams of four warps (one per TMEM lane quarter) take alternate
        // blocks of an item (team = j & 1), so two blocks' latency chains
        // (S load, exchange with the peer, max, exponentials, P store) run at
        // once. The running max passes from team to team through shared
        // memory (m_ready); each team keeps its own row sum relative to the
        // max it last used, and the two sums are combined at the item's end.
        const int quarter = warp & 3, team = warp >> 2;
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float scale_log2 = p.sm_scale * 1.4426950408889634f;
        const float ninf = -INFINITY;
        const int cnt0 = (nb + 1) / 2, cnt1 = nb / 2;  // blocks per item of team 0 / team 1
        const int mycnt = team ? cnt1 : cnt0;
        // exchange slot = team; chunk-major [chunk][head] x 16 B
        const uint32_t x_peer = peer_addr(smem_u32(xchg), peer) + team * kXchgSlotBytes;
        const uint8_t* x_mine = xchg + team * kXchgSlotBytes;
        const int xb = team * 4 + quarter;  // this warp's x_full / x_free
        const uint32_t xf_peer = peer_addr(smem_u32(&x_full[xb]), peer);
        const uint32_t xr_peer = peer_addr(smem_u32(&x_free[xb]), peer);
        uint32_t g = 0, it = 0;
        for (int64_t item = cid; item < nitems; item += ncl, ++it) {
            int b;
            int64_t tq, hrow;
            decode(item, b, tq, hrow);
            float m = ninf, l = 0.f;  // this team's max in use and its row sum relative to it
            for (int j = team; j < nb; j += 2) {
                const uint32_t gb = g + j;  // global block
                const uint32_t n = it * mycnt + (j >> 1);  // this team's block count: barrier phases
                const int s = gb % kStages;
                float x[kBlk];
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(0) }
                mbar_wait(&s_full[gb % kSSlots], (gb / kSSlots) & 1);
                tc_fence_after();
                tmem_ld32(lane_base + s_col(gb), x);
                if (lane == 0) mbar_expect_tx(&x_full[xb], 32 * kBlk * 4);
                tmem_ld_wait();
                if (CSAIDX_PAIR_DBG == 0) mbar_wait_cluster(&x_free[xb], (n & 1) ^ 1);
#pragma unroll
                for (int q = 0; q < kBlk / 4; ++q)
                    st_async_v4(x_peer + (q * kH + row) * 16, x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3],
                                xf_peer);
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(1) }
                mbar_wait(&kv_full[s], (gb / kStages) & 1);  // completed: orders the valid word
                uint32_t vm = 0;
                if (lane == 0) {
                    vm = valid_w[s];
                    mbar_arrive(&vw_free[s]);
                }
                vm = __shfl_sync(0xffffffffu, vm, 0);
                // the peer's partial -> S = S_0 + S_1 (same bits in both CTAs)
                if (CSAIDX_PAIR_DBG == 0) mbar_wait_cluster(&x_full[xb], n & 1);
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(2) }
#pragma unroll
                for (int q = 0; q < kBlk / 4; ++q) {
                    const float4 v = *reinterpret_cast<const float4*>(x_mine + (q * kH + row) * 16);
                    x[4 * q] += v.x;
                    x[4 * q + 1] += v.y;
                    x[4 * q + 2] += v.z;
                    x[4 * q + 3] += v.w;
                }
                __syncwarp();
                if (lane == 0 && CSAIDX_PAIR_DBG == 0) remote_arrive(xr_peer);  // the peer may refill my slot
                if (vm != 0xffffffffu) {
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) x[c] = ((vm >> c) & 1u) ? x[c] : ninf;
                }
                float t3[11];
#pragma unroll
                for (int c = 0; c < 10; ++c) t3[c] = max3f(x[3 * c], x[3 * c + 1], x[3 * c + 2]);
                t3[10] = fmaxf(x[30], x[31]);
                const float mx = max3f(max3f(max3f(t3[0], t3[1], t3[2]), max3f(t3[3], t3[4], t3[5]),
                                             max3f(t3[6], t3[7], t3[8])),
                                       t3[9], t3[10]) * scale_log2;
                // The max in use after block j-1 (the other team's) and the lazy
                // rule: move it only when this block exceeds it by 2^8. From
                // the third block on the max rarely moves, so the exponentials
                // are computed with the value this team last saw and checked
                // against the other team's published one afterwards (the rare
                // lanes that differ recompute), keeping the hand-off out of
                // the chain.
                const int ot = team ^ 1;
                auto wait_other = [&]() {
                    const uint32_t on = it * (ot ? cnt1 : cnt0) + ((j - 1) >> 1);
                    mbar_wait(&m_ready[ot * 4 + quarter], on & 1);
                    return m_s[ot * kH + row];
                };
                float mprev = j == 1 ? wait_other() : (j == 0 ? ninf : m);
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(8) }
                float mnew, alpha;
                bool rescale;
                auto decide = [&]() {
                    mnew = mprev;
                    rescale = false;
                    alpha = 1.f;
                    if (mx > mprev) {
                        if (mprev == ninf) {
                            mnew = mx;
                        } else if (mx > mprev + kRescaleLog2) {
                            alpha = ex2(mprev - mx);
                            mnew = mx;
                            rescale = true;
                        }
                    }
                };
                uint32_t pk[kBlk / 2];
                float psum = 0.f;
                auto exps = [&]() {  // P = 2^(s * scale_log2 - mnew) packed to bf16 pairs, and its sum
                    if (mnew != ninf) {
                        const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-mnew, -mnew);
                        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                        for (int c = 0; c < kBlk; c += 2) {
                            const float2 a = __ffma2_rn(make_float2(x[c], x[c + 1]), sc2, nm2);
                            float2 pr;
                            if (c < kBlk / 2) {
                                pr.x = ex2(a.x);
                                pr.y = ex2(a.y);
                            } else {
                                pr = exp2_poly2(a);
                            }
                            acc = __fadd2_rn(acc, pr);
                            const __nv_bfloat162 h2 = __floats2bfloat162_rn(pr.x, pr.y);
                            pk[c / 2] = *reinterpret_cast<const uint32_t*>(&h2);
                        }
                        psum = acc.x + acc.y;
                    } else {
#pragma unroll
                        for (int c = 0; c < kBlk / 2; ++c) pk[c] = 0u;
                        psum = 0.f;
                    }
                };
                decide();
                exps();
                if (j >= 2) {
                    const float mtrue = wait_other();
                    if (mtrue != mprev) {  // the other team moved the max at block j-1
                        mprev = mtrue;
                        decide();
                        exps();
                    }
                }
                m_s[team * kH + row] = mnew;  // the other team's next block reads it
                __syncwarp();
                if (lane == 0) mbar_arrive(&m_ready[team * 4 + quarter]);
                if (mnew != m) {  // this team's sum follows the max in use
                    if (m != ninf) l *= ex2(m - mnew);
                    m = mnew;
                }
                l += psum;
                if (__any_sync(0xffffffffu, rescale)) {
                    // PV of block gb-1 landed (exact parity wait: attn_sm100.cu)
                    mbar_wait(&kv_empty[(gb - 1) % kStages], ((gb - 1) / kStages) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = 0; c0 < kDvHalf; c0 += 32) {
                        float o[32];
                        tmem_ld32(lane_base + kColO + c0, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) o[c] *= alpha;
                        tmem_st32(lane_base + kColO + c0, o);
                    }
                    tmem_st_wait();
                }
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(9) }
                tmem_st16(lane_base + s_col(gb), pk);  // P over the S columns just read
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[gb % kSSlots]);
                if ((warp & 3) == 0 && lane == 0) { const uint32_t g = gb; PROBE(3) }
            }
            g += nb;
            // (m, l) of this team -> the stagers' epilogue, once the previous
            // item's epilogue has read ml_s (o_free; with nb >= 4 the blocks
            // above already waited for it through PV(0), with fewer blocks
            // this keeps ml_s and ml_ready one item deep)
            if (it > 0) mbar_wait(o_free, (it - 1) & 1);
            ml_s[(team * 2 + 0) * kH + row] = m;
            ml_s[(team * 2 + 1) * kH + row] = l;
            mbar_arrive(&ml_ready[quarter]);
        }
    }

    tc_fence_before();
    cluster_sync_all();  // no remote arrive / st.async may target an exited CTA
    if (warp == kWarpMma) {
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

cudaError_t launch_sparse_mla_pair(const CUtensorMap& qmap, const SparseMlaParams& p, cudaStream_t stream) {
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
    sparse_mla_pair_kernel<<<static_cast<unsigned>(2 * pairs), kThreads, kSmemBytes, stream>>>(qmap, p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
