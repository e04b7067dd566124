// Sparse attention over the indexer's top-k (the CSA step
// after the indexer: "a sparse attention kernel reads only
// TopK(t) ... for each query"; PAPER.md:360-375 composes the chunked indexer
// with TileLang's sparse MLA kernel). The reference stops at the index list
// (SPEC.md:8 puts the attention step out of its scope), so the operator here
// follows the sparse-MLA definition that kernel family implements:
//
//   out[b,t,h,:] = sum_j softmax_j(sm_scale * q[b,t,h,:] . kv[b,i_j,:]) * kv[b,i_j,:Dv]
//   lse[b,t,h]   = log sum_j exp(sm_scale * q[b,t,h,:] . kv[b,i_j,:])
//
// over the valid entries i_j of indices[b,t,:] (0 <= i_j < T; -1 = padding),
// with one shared latent KV head (MQA): kv rows of Dqk = 576 (the first
// Dv = 512 are also the values), H = 128 g query heads, bf16 in / fp32
// accumulate / bf16 out.
//
// B200 design (work item = (query, group of 128 heads, half of Dv); one
// persistent CTA per SM, shared memory and TMEM both full):
//  * heads are the UMMA M dimension (128 TMEM lanes), so every softmax
//    statistic of a head lives in one thread;
//  * S = Q K^T per block of 32 keys (M = 128, N = 32, K = 576). Q's first 384
//    dims are the TMEM A operand (tcgen05.mma ... [a_tmem], 192 columns of
//    packed bf16 pairs), the last 192 stay in shared memory (3 SW128 panels,
//    TMA). An M = 128 MMA costs >= ~46 cycles for any N < 128 (measured,
//    profiles/r02_mma_floor.md), so the 36 QK instructions per block bound
//    the kernel; wider blocks (N = 48 / 64) lost because shared memory then
//    holds fewer gather stages (profiles/r02_attention.md);
//  * the selected KV rows are gathered 32 per block by 128 producer threads
//    with cp.async (16-byte pieces written straight into the SW128 K-major
//    layout; completion tracked by the stage's mbarrier), 4 stages deep
//    (TMA tile::gather4 — 4 rows x 128 B per instruction — is bound by the
//    TMA unit's instruction rate);
//  * the softmax warps read S (tcgen05.ld), keep the running max / sum in
//    registers (exp2 domain, lazy rescale: O is only rescaled when the max
//    grows by more than 2^8), and write P as packed bf16 over the S columns
//    they just read (tcgen05.st) — P is the A operand of O += P V (A from
//    TMEM, M = 128, N = 256, K = 32), whose B operand is the same gathered KV
//    tile read MN-major (no transpose copy);
//  * O [128 x 256] fp32 stays in TMEM for the whole item; the two items of a
//    (query, head group) each own half of Dv and both compute S (65% of the
//    issued MMA work is useful at Dqk = 576, Dv = 512).
//    TMEM: Q 192 + O 256 + S/P 2 x 32 = 512 columns.
// Persistent: one CTA per SM walks the items round-robin and
// every barrier phase runs on across items, so the next item's Q staging,
// gathers and first S MMAs overlap the current item's last softmax blocks and
// epilogue (a CTA per item spent ~15K cycles per item in prologue / epilogue).
// Warp roles: 0-3 softmax + epilogue (TMEM lane quarters), 4-7 KV producers
// (cp.async gather), 8 TMEM owner + MMA issuer, 9-12 Q stagers (Q head into
// TMEM, Q tail by TMA, once the previous item's S MMAs are done).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "sm100_ptx.cuh"

using namespace csaidx_dev;

namespace {

constexpr int kH = 128;                    // query heads = UMMA M
constexpr int kDqk = 576;
constexpr int kDvHalf = 256;               // Dv columns per CTA = UMMA N of PV
constexpr int kPanels = kDqk / 64;         // 9 SW128 panels of 64 bf16
constexpr int kQTmemSteps = 24;            // K steps of 16 whose Q slice is in TMEM (dims 0..383)
constexpr int kQSmemPanels = kPanels - kQTmemSteps / 4;  // 3 panels in shared memory (dims 384..575)
constexpr int kBlk = 32;                   // keys per block = UMMA N of QK, K of PV
constexpr int kStages = 4;
constexpr int kQPanelBytes = kH * 128;                 // 16 KiB
constexpr int kQBytes = kQSmemPanels * kQPanelBytes;   // 48 KiB
constexpr int kKvPanelBytes = kBlk * 128;              // 4 KiB
constexpr int kKvStageBytes = kPanels * kKvPanelBytes; // 36 KiB
constexpr int kKvOffset = kQBytes;
constexpr int kMaxK = 4096;                            // indices staged in shared memory
constexpr int kIdxOffset = kKvOffset + kStages * kKvStageBytes;
constexpr int kBarOffset = kIdxOffset + kMaxK * 4;
constexpr int kMlOffset = kBarOffset + 256;             // (m, l) per head row at an item's end
constexpr int kSmemBytes = kMlOffset + 2 * kH * 4 + 1024;  // + align slack
constexpr int kThreads = 416;              // 4 softmax + 4 KV producer + 1 MMA + 4 Q-staging warps
constexpr int kProducers = 128;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColQ = 0, kColO = 192, kColS = 448;  // S (and P over it): 2 x 32 columns
constexpr float kRescaleLog2 = 8.0f;       // lazy rescale threshold (factor 256)

// D[tmem] (+)= A[tmem] * B[smem desc] (A = P, packed bf16 pairs per column).
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

// 2^y for a pair on the FMA / ALU pipes (y <= ~8 here): round-to-nearest
// split y = n + f (f in [-1/2, 1/2]) by the 1.5 * 2^23 trick, a quartic for
// 2^f (max relative error 5.3e-6: far below P's bf16 rounding, and l = sum p
// stays within the lse tolerance; a cubic's 1.7e-4 did not), 2^n added
// to the exponent field. Half of each block's exponentials take this path so
// the MUFU pipe is not the softmax's bound (the FA4 split).
__device__ __forceinline__ float2 exp2_poly2(float2 y) {
    const float2 magic = make_float2(12582912.f, 12582912.f);
    y.x = fmaxf(y.x, -127.f);
    y.y = fmaxf(y.y, -127.f);
    const float2 t = __fadd2_rn(y, magic);
    const float2 f = __fadd2_rn(y, __fadd2_rn(magic, make_float2(-t.x, -t.y)));  // y - (t - magic)
    float2 p = __ffma2_rn(make_float2(0.009591416f, 0.009591416f), f, make_float2(0.05587532f, 0.05587532f));
    p = __ffma2_rn(p, f, make_float2(0.24023689f, 0.24023689f));
    p = __ffma2_rn(p, f, make_float2(0.69312757f, 0.69312757f));
    p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
    return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                       __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// MN-major SW128 descriptor (B of O += P V): the gathered tile read with Dv
// as N: 64-element rows of 128 B, 8-row (key) atoms of 1 KiB (SBO), the
// next 64 Dv columns one panel further (LBO).
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;
    return d;
}

constexpr uint32_t kIdescQK = idesc_bf16_f32(kH, kBlk);
constexpr uint32_t kIdescPV = idesc_bf16_f32(kH, kDvHalf) | (1u << 16);  // B MN-major

__global__ void __launch_bounds__(kThreads, 1)
    sparse_mla_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ SparseMlaParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* q_smem = smem;
    uint8_t* kv_smem = smem + kKvOffset;
    int32_t* idx_s = reinterpret_cast<int32_t*>(smem + kIdxOffset);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOffset);
    uint64_t* q_full = bars;                    // [1] Q tail in shared memory (TMA), per item
    uint64_t* kv_full = q_full + 1;             // [kStages]
    uint64_t* kv_empty = kv_full + kStages;     // [kStages] committed after the block's PV
    uint64_t* s_full = kv_empty + kStages;      // [2]
    uint64_t* p_full = s_full + 2;              // [2]
    uint64_t* q_tmem = p_full + 2;              // [1] Q head staged into TMEM, per item
    uint64_t* q_free = q_tmem + 1;              // [1] every S MMA of the item done (Q reusable)
    uint64_t* o_free = q_free + 1;              // [1] the epilogue has read O
    uint64_t* vw_free = o_free + 1;             // [kStages] the softmax warps have read the valid word
    uint64_t* ml_ready = vw_free + kStages;     // [1] the softmax warps' (m, l) of an item written
    uint32_t* valid_w = reinterpret_cast<uint32_t*>(ml_ready + 1);  // [kStages]
    float* ml_s = reinterpret_cast<float*>(smem + kMlOffset);          // [m | l][128 heads]
    uint32_t* tmem_slot = valid_w + kStages;

    const int warp = threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    const int nb = (p.k + kBlk - 1) / kBlk;  // blocks per item
    const int G = p.head_groups;  // groups of 128 query heads
    const int64_t nitems = 2 * p.seq_len * p.batch * G;  // (b, query, head group, half of Dv)

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], kProducers + 1);  // one cp.async arrive per producer thread + the valid word
            mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&p_full[s], 4);  // one arrive per softmax warp
        }
        mbar_init(q_tmem, 4);    // one arrive per Q-staging warp
        mbar_init(q_free, 1);
        mbar_init(o_free, 256);  // every lane of the softmax and Q-staging warps (each writes half of O's columns)
        mbar_init(ml_ready, 128);
        for (int s = 0; s < kStages; ++s) mbar_init(&vw_free[s], 4);
        fence_barrier_init();
    }
    if (warp == 8) tmem_alloc<kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    // Items are handed out round-robin: item = blockIdx.x + i * gridDim.x,
    // (b, query, head group, half) = decoded below. Every role walks the same
    // sequence; barrier phases run on across items (block counter g = i * nb
    // + j). hrow = the item's first head row in the [B * S * H] q / out rows.
    auto decode = [&](int64_t item, int& b, int64_t& tq, int& half, int64_t& hrow) {
        half = static_cast<int>(item & 1);
        const int64_t qg = item >> 1;
        const int64_t qi = qg / G;
        b = static_cast<int>(qi / p.seq_len);
        tq = qi - static_cast<int64_t>(b) * p.seq_len;
        hrow = qg * kH;  // ((b * S + tq) * G + hg) * 128
    };

    if (warp >= 4 && warp < 8) {
        // ---------------------------------------------------------- KV producers
        const int pt = threadIdx.x - 128;  // 0..127
        // thread pt copies row r = pt / 4 of every block, 16-byte pieces
        // cc = pt % 4 + 4u (u < 18): one 64-bit row address per block, the
        // pieces at immediate offsets; smem offsets are the same every block
        constexpr int kPieces = (kBlk * kPanels * 8) / kProducers;  // 18
        static_assert(kProducers == 4 * kBlk, "4 producer threads per gathered row");
        const int r = pt >> 2;
        uint32_t soff[kPieces];
#pragma unroll
        for (int u = 0; u < kPieces; ++u) {
            const int cc = (pt & 3) + 4 * u;
            soff[u] = (cc >> 3) * kKvPanelBytes + r * 128 + (((cc & 7) ^ (r & 7)) << 4);
        }
        uint32_t g = 0, it = 0;
        for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
            int b, half;
            int64_t tq, hrow;
            decode(item, b, tq, half, hrow);
            // the item's k indices -> shared memory (row of the gather; -1 for
            // padding); idx_s is reused once the softmax has read every valid word
            const int32_t* idx_row = p.indices + (static_cast<int64_t>(b) * p.seq_len + tq) * p.idx_ld;
            asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");  // previous item's reads of idx_s done
            for (int i = pt; i < nb * kBlk; i += kProducers) {
                const int32_t idx = i < p.k ? __ldg(idx_row + i) : -1;
                idx_s[i] = (idx >= 0 && idx < p.kv_len) ? idx : -1;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory");
            const char* kv_b = reinterpret_cast<const char*>(p.kv) + static_cast<int64_t>(b) * p.kv_len * (kDqk * 2) +
                               (pt & 3) * 16;
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % kStages;
                const int32_t myidx = idx_s[j * kBlk + r];
                const char* src = kv_b + static_cast<int64_t>(myidx >= 0 ? myidx : 0) * (kDqk * 2);  // padding: row 0
                uint32_t vmask = 0;
                if (warp == 4) vmask = __ballot_sync(0xffffffffu, idx_s[j * kBlk + lane] >= 0);
                mbar_wait(&kv_empty[s], ((g / kStages) & 1) ^ 1);
                // this thread's copies into the stage for block g - 4 have landed
                // (the MMA consumed them, so this never waits); the group wait
                // makes that ordering visible to tools that track cp.async
                // (racecheck does not model the mbarrier completion)
                asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
                if (pt == 0) {
                    // the valid word of block g - 4 has been read (a thread-to-thread
                    // barrier, so the reuse is ordered without going through the
                    // tensor core's commits; it has always completed by now)
                    mbar_wait(&vw_free[s], ((g / kStages) & 1) ^ 1);
                    valid_w[s] = vmask;
                    mbar_arrive(&kv_full[s]);  // release: the softmax reads the word after kv_full
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
    } else if (warp >= 9) {
        // ---------------------------------------------------------- Q stagers
        // warps 9..12 cover TMEM lane quarters 1,2,3,0; thread = head
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float ninf = -INFINITY;
        // O columns 128..255 of item ie (the softmax warps write 0..127)
        auto epilogue_half = [&](uint32_t ie, int64_t hrow_e, int half_e) {
            mbar_wait(ml_ready, ie & 1);
            const float l = ml_s[kH + row];
            const float inv_l = l > 0.f ? 1.f / l : 0.f;
            const uint32_t gl = (ie + 1) * static_cast<uint32_t>(nb) - 1;  // the item's last block
            mbar_wait(&kv_empty[gl % kStages], (gl / kStages) & 1);       // its PV landed (next phase needs o_free)
            tc_fence_after();
            __nv_bfloat16* orow = p.out + (hrow_e + row) * p.out_ld + half_e * kDvHalf;
#pragma unroll 1
            for (int c0 = kDvHalf / 2; c0 < kDvHalf; c0 += 32) {
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
            (void)ninf;
        };
        int64_t prev_hrow = 0;
        int prev_half = 0;
        uint32_t it = 0;
        for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
            int b, half;
            int64_t tq, hrow;
            decode(item, b, tq, half, hrow);
            const int64_t qrow = hrow;
            const uint4* qsrc = reinterpret_cast<const uint4*>(p.q + (qrow + row) * kDqk);
            // warm L2 with this head's row while the previous item still owns Q
#pragma unroll
            for (int c = 0; c < kDqk * 2; c += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(qsrc) + c));
            if (it > 0) {
                mbar_wait(q_free, (it - 1) & 1);  // every S MMA of the previous item has completed
                tc_fence_after();
            }
            if (warp == 9 && lane == 0) {  // Q tail (dims 384..575) by TMA
                mbar_expect_tx(q_full, kQBytes);
                for (int pn = 0; pn < kQSmemPanels; ++pn)
                    tma_load_2d(q_smem + pn * kQPanelBytes, &qmap, q_full, (kQTmemSteps / 4 + pn) * 64,
                                static_cast<int32_t>(qrow));
            }
            // Q head (dims 0..383) -> TMEM lane `row`, columns 0..191 (bf16 pairs)
#pragma unroll 1
            for (int c0 = 0; c0 < kQTmemSteps * 8; c0 += 64) {
                uint32_t w[64];
                uint4* w4 = reinterpret_cast<uint4*>(w);
#pragma unroll
                for (int v = 0; v < 16; ++v) w4[v] = __ldg(qsrc + c0 / 4 + v);
                tmem_st16(lane_base + kColQ + c0, *reinterpret_cast<uint32_t(*)[16]>(w));
                tmem_st16(lane_base + kColQ + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(w + 16));
                tmem_st16(lane_base + kColQ + c0 + 32, *reinterpret_cast<uint32_t(*)[16]>(w + 32));
                tmem_st16(lane_base + kColQ + c0 + 48, *reinterpret_cast<uint32_t(*)[16]>(w + 48));
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(q_tmem);
            if (it > 0) epilogue_half(it - 1, prev_hrow, prev_half);
            prev_hrow = hrow;
            prev_half = half;
        }
        if (it > 0) epilogue_half(it - 1, prev_hrow, prev_half);
    } else if (warp == 8) {
        // ---------------------------------------------------------- MMA issuer
        if (elect_one()) {
            const uint32_t q_base = smem_u32(q_smem);
            const uint32_t kv_base = smem_u32(kv_smem);
            uint32_t g = 0, it = 0;
            for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
                const int half = static_cast<int>(item & 1);
                mbar_wait(q_full, it & 1);
                mbar_wait(q_tmem, it & 1);
                tc_fence_after();
                auto issue_pv = [&](int j, uint32_t gj) {
                    const int s = gj % kStages;
                    if (j == 0 && it > 0) mbar_wait(o_free, (it - 1) & 1);  // the last epilogue has read O
                    mbar_wait(&p_full[gj & 1], (gj >> 1) & 1);
                    tc_fence_after();
                    const uint32_t vb = kv_base + s * kKvStageBytes + (half * 4) * kKvPanelBytes;
#pragma unroll
                    for (int kk = 0; kk < kBlk / 16; ++kk)  // 16 keys per K step: 8 columns of P, 2 KiB of rows
                        umma_bf16_ts(tmem + kColO, tmem + kColS + (gj & 1) * kBlk + kk * 8,
                                     sw128_mnmajor_desc(vb + kk * 2048, kKvPanelBytes, 1024), kIdescPV,
                                     (j > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&kv_empty[s]);  // stage free and O holds PV of block j
                };
                for (int j = 0; j < nb; ++j) {
                    const uint32_t gj = g + j;
                    const int s = gj % kStages;
                    mbar_wait(&kv_full[s], (gj / kStages) & 1);
                    fence_proxy_async();  // cp.async (generic proxy) writes -> the tensor core's reads
                    tc_fence_after();
                    const uint32_t st = kv_base + s * kKvStageBytes;
                    const uint32_t d = tmem + kColS + (gj & 1) * kBlk;
#pragma unroll
                    for (int kk = 0; kk < kQTmemSteps; ++kk)  // Q head from TMEM: 8 columns per 16 dims
                        umma_bf16_ts(d, tmem + kColQ + kk * 8,
                                     sw128_kmajor_desc(st + (kk >> 2) * kKvPanelBytes + (kk & 3) * 32), kIdescQK,
                                     kk > 0 ? 1u : 0u);
#pragma unroll
                    for (int kk = kQTmemSteps; kk < kDqk / 16; ++kk) {  // Q tail from shared memory
                        const uint32_t qa = q_base + ((kk - kQTmemSteps) >> 2) * kQPanelBytes + (kk & 3) * 32;
                        const uint32_t kb = st + (kk >> 2) * kKvPanelBytes + (kk & 3) * 32;
                        umma_bf16(d, sw128_kmajor_desc(qa), sw128_kmajor_desc(kb), kIdescQK, 1u);
                    }
                    umma_commit(&s_full[gj & 1]);
                    if (j == nb - 1) umma_commit(q_free);  // Q (TMEM head, smem tail) reusable
                    if (j > 0) issue_pv(j - 1, gj - 1);
                }
                issue_pv(nb - 1, g + nb - 1);
                g += nb;
            }
        }
    } else {
        // ---------------------------------------------------------- softmax + epilogue
        const int row = warp * 32 + lane;  // head
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        const float scale_log2 = p.sm_scale * 1.4426950408889634f;
        const float ninf = -INFINITY;
        uint32_t g = 0, it = 0;
        for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
            int b, half;
            int64_t tq, hrow;
            decode(item, b, tq, half, hrow);
            float m = ninf, l = 0.f;
            for (int j = 0; j < nb; ++j, ++g) {
                const int s = g % kStages;
                mbar_wait(&s_full[g & 1], (g >> 1) & 1);
                mbar_wait(&kv_full[s], (g / kStages) & 1);  // completed: orders the valid word
                tc_fence_after();
                float x[kBlk];
                tmem_ld32(lane_base + kColS + (g & 1) * kBlk, x);
                // lane 0 reads the valid word and releases it (its own arrive orders
                // its own read), the warp gets it by shuffle
                uint32_t vm = 0;
                if (lane == 0) {
                    vm = valid_w[s];
                    mbar_arrive(&vw_free[s]);
                }
                vm = __shfl_sync(0xffffffffu, vm, 0);
                tmem_ld_wait();
                if (vm != 0xffffffffu) {  // block-uniform: padding / out-of-range keys -> -inf
#pragma unroll
                    for (int c = 0; c < kBlk; ++c) x[c] = ((vm >> c) & 1u) ? x[c] : ninf;
                }
                // raw block max (3-input FMNMX tree), then the exp2 domain
                float t3[11];
#pragma unroll
                for (int c = 0; c < 10; ++c) t3[c] = max3f(x[3 * c], x[3 * c + 1], x[3 * c + 2]);
                t3[10] = fmaxf(x[30], x[31]);
                const float mx = max3f(max3f(max3f(t3[0], t3[1], t3[2]), max3f(t3[3], t3[4], t3[5]),
                                             max3f(t3[6], t3[7], t3[8])),
                                       t3[9], t3[10]) * scale_log2;
                float alpha = 1.f;
                bool rescale = false;
                if (mx > m) {
                    if (m == ninf) {
                        m = mx;  // O is unwritten (j == 0) or all zero: nothing to rescale
                    } else if (mx > m + kRescaleLog2) {
                        alpha = ex2(m - mx);
                        l *= alpha;
                        m = mx;
                        rescale = true;
                    }
                }
                if (__any_sync(0xffffffffu, rescale)) {
                    // PV of block j-1 has landed in O. Its commit is kv_empty of
                    // that block's stage; the barrier's previous phase (PV of
                    // block g-5) completed before block g-1 was loaded and its
                    // next one (PV of block g+3) needs this warp's P of block
                    // g+3, so a parity wait here is exact even though this warp
                    // skips the blocks without a rescale. (tcgen05.commit
                    // completions are not ordered across barriers: a single
                    // o_done barrier waited only on rescaling blocks returned
                    // early and corrupted O.)
                    mbar_wait(&kv_empty[(g - 1) % kStages], ((g - 1) / kStages) & 1);
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
                // p = 2^(s * scale_log2 - m): one FFMA2 per pair for the argument,
                // MUFU.EX2 for the first half of the block, the FMA-pipe quartic for
                // the second; pairwise sums; packed to bf16 pairs for the PV MMA
                uint32_t pk[kBlk / 2];
                float sum = 0.f;
                if (m != ninf) {
                    const float2 sc2 = make_float2(scale_log2, scale_log2), nm2 = make_float2(-m, -m);
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
                    sum = acc.x + acc.y;
                } else {
#pragma unroll
                    for (int c = 0; c < kBlk / 2; ++c) pk[c] = 0u;
                }
                l += sum;
                tmem_st16(lane_base + kColS + (g & 1) * kBlk, pk);  // P over the S columns just read
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&p_full[g & 1]);
            }
            // epilogue: O / l -> bf16 rows of this head (columns 0..127 here,
            // 128..255 by the Q-staging warps, which read (m, l) from ml_s once
            // the previous item's epilogue has released it), lse (half 0)
            if (it > 0) mbar_wait(o_free, (it - 1) & 1);
            ml_s[row] = m;
            ml_s[kH + row] = l;
            mbar_arrive(ml_ready);
            mbar_wait(&kv_empty[(g - 1) % kStages], ((g - 1) / kStages) & 1);  // the item's last PV landed
            tc_fence_after();
            const float inv_l = l > 0.f ? 1.f / l : 0.f;
            __nv_bfloat16* orow =
                p.out + (hrow + row) * p.out_ld + half * kDvHalf;
#pragma unroll 1
            for (int c0 = 0; c0 < kDvHalf / 2; c0 += 32) {
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
            mbar_arrive(o_free);  // (with the Q-staging warps' arrivals) the next item's first PV may overwrite O
            if (half == 0 && p.lse != nullptr)
                p.lse[hrow + row] =
                    l > 0.f ? (m + __log2f(l)) * 0.6931471805599453f : ninf;
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 8) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

}  // namespace

namespace csaidx_kern {

int sparse_mla_smem_bytes() { return kSmemBytes; }

cudaError_t launch_sparse_mla(const CUtensorMap& qmap, const SparseMlaParams& p,
                              cudaStream_t stream) {
    if (p.seq_len <= 0 || p.batch <= 0) return cudaSuccess;
    static bool attr_set[kMaxDevices] = {};
    const int dev = attr_device();
    if (!attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(sparse_mla_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    // persistent: one CTA per SM walks the (b, query, half) items round-robin
    int sms = 0, cur = 0;
    cudaGetDevice(&cur);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur);
    const int64_t items = 2 * p.seq_len * p.batch;
    const unsigned grid = static_cast<unsigned>(items < sms ? items : sms);
    sparse_mla_kernel<<<grid, kThreads, kSmemBytes, stream>>>(qmap, p);
    return cudaGetLastError();
}

}  // namespace csaidx_kern
