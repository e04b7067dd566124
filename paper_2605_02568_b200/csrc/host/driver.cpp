// Host chunk scheduler (Algorithm 2) over the C-ABI. Reference semantics:
// driver.cpp:29-211. Each (s0, t0) host tile becomes one masked score launch
// plus one select (+ merge) launch on device; the running top-k rows live in
// HBM for the whole query chunk; the sentinel pass and the k_eff contract are
// checked on device. Ledger charges mirror the reference's labels, byte
// counts and scopes, so RunStats and ledger peaks are directly comparable.
#include "csaidx/driver.hpp"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <thread>

#include "csaidx/causal.hpp"
#include "device.hpp"
#include "host_convert.hpp"

namespace csaidx {

namespace detail {

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Clamped {
    int64_t cs, ct;
};

Clamped clamp(const ProblemDims& dims, const TileConfig& tile) {
    tile.validate();
    return {std::min(tile.query_tile, dims.seq_len), std::min(tile.key_tile, dims.key_blocks)};
}

}  // namespace

int64_t physical_key_tile(const ProblemDims& dims, const DriverConfig& config, const ChunkPlan& plan) {
    // Under production semantics the final rows are the top-k_eff of every
    // legal entry under one total order however the key range is split (the
    // reference's chunked == materialize contract, test_driver.cpp), so the
    // device widens the key tile up to the score-buffer budget: one score
    // launch and one select per chunk instead of a select + merge per
    // requested tile. Ablations and the boolean-mask tile keep the requested
    // tiles (their results or charges depend on them).
    const int64_t T = dims.key_blocks;
    if (plan.ct >= T || config.ablation != Ablation::none || config.bool_mask_tile) return plan.ct;
    const uint64_t per_tile = static_cast<uint64_t>(dims.batch * plan.cs * ((plan.ct + 3) / 4 * 4)) * sizeof(float);
    const int64_t tiles = ceil_div(T, plan.ct);
    const int64_t f = std::min<int64_t>(tiles, std::max<int64_t>(1, static_cast<int64_t>(key_tile_budget() / per_tile)));
    return f >= tiles ? T : plan.ct * f;
}

ChunkPlan plan_chunks(const ProblemDims& dims, const TileConfig& tile, const std::vector<int64_t>* starts) {
    const Clamped c = clamp(dims, tile);
    ChunkPlan plan;
    plan.cs = c.cs;
    plan.ct = c.ct;
    if (starts == nullptr) {
        for (int64_t s0 = 0; s0 < dims.seq_len; s0 += c.cs) plan.starts.push_back(s0);
    } else {
        for (int64_t s0 : *starts) {
            if (s0 < 0 || s0 >= dims.seq_len || s0 % c.cs != 0)
                throw std::invalid_argument("chunk start must be a multiple of the query tile inside the sequence");
            plan.starts.push_back(s0);
        }
    }
    int64_t row = 0;
    for (int64_t s0 : plan.starts) {
        plan.out_row0.push_back(row);
        row += std::min(c.cs, dims.seq_len - s0);
    }
    plan.order.resize(plan.starts.size());
    for (size_t i = 0; i < plan.order.size(); ++i) plan.order[i] = i;
    std::stable_sort(plan.order.begin(), plan.order.end(),
                     [&](size_t a, size_t b) { return plan.starts[a] > plan.starts[b]; });
    return plan;
}

void run_plan(csaidx_engine* e, const DeviceOps& ops, const ProblemDims& dims, const DriverConfig& config,
              const ChunkPlan& plan, int64_t* out_idx, float* out_val, int64_t out_rows, MemoryLedger& ledger,
              RunStats& stats, const ChunkHooks& hooks) {
    const int64_t B = dims.batch, k = dims.top_k, T = dims.key_blocks;
    const int kcode = kernel_code(config.kernel, config.mode);
    const int mcode = mode_code(config.mode);
    const csaidx_dims cd = to_c(dims);
    const int64_t ct = physical_key_tile(dims, config, plan);
    const int64_t ld = (ct + 3) / 4 * 4;
    const int64_t width_max = std::min(k, ct);

    // Device working set, sized once for the largest tile and reused.
    DeviceBuffer scores(e, static_cast<size_t>(B * plan.cs * ld) * sizeof(float));
    DeviceBuffer cand_v(e, static_cast<size_t>(B * plan.cs * width_max) * 4);
    DeviceBuffer cand_i(e, static_cast<size_t>(B * plan.cs * width_max) * 4);
    DeviceBuffer run_v(e, static_cast<size_t>(B * plan.cs * k) * 4);
    DeviceBuffer run_i(e, static_cast<size_t>(B * plan.cs * k) * 4);
    DeviceBuffer keep;
    if (config.bool_mask_tile) keep = DeviceBuffer(e, static_cast<size_t>(plan.cs * ct));

    // Fused select pre-filter (csaidx_cuda.h): tensor-core tiles whose longest
    // legal row exceeds the candidate list. Same results as the plain select;
    // device scratch only (the reference has no such buffers to charge).
    const int cap = csaidx_cuda_candidate_capacity(k);
    const bool prefilter = prefilter_enabled() && !config.bool_mask_tile && cap > 0 && ops.op_rows == 0 &&
                           csaidx_cuda_score_uses_tensor_cores(&cd, ops.dtype, mcode, kcode) != 0;
    const int64_t tiles_max = ceil_div(ct, 128);
    // per tile: stride = ceil(tiles / kPrefilterSampleTiles) -> at most
    // min(tiles, kPrefilterSampleTiles) sampled tiles
    const int64_t lds = std::min<int64_t>(tiles_max, kPrefilterSampleTiles) * 128;
    const int64_t bits_ld = csaidx_cuda_candidate_words(ct);
    DeviceBuffer pf_bits, pf_tau, pf_sample;
    if (prefilter) {
        pf_bits = DeviceBuffer(e, static_cast<size_t>(B * plan.cs * bits_ld) * sizeof(uint32_t));
        pf_tau = DeviceBuffer(e, static_cast<size_t>(B * plan.cs) * sizeof(float));
        pf_sample = DeviceBuffer(e, static_cast<size_t>(B * plan.cs * lds) * sizeof(float));
    }

    // Select beside score: with one key tile per query chunk (c_T >= T) on
    // the tensor-core path, chunk o's select runs on a few SMs (persistent,
    // several rows per CTA) on a second compute lane while chunk o+1's score
    // runs on the rest; the score tiles are double buffered. Results are
    // identical (the same kernels per row); only the SM assignment changes.
    // select_overlap_sms() < 0: no partition — both kernels take whole SMs
    // as they free up, the select lane first (stream priority), so each
    // kernel's tail is filled by the other's start.
    const int overlap_sms = select_overlap_sms();
    const bool overlap = ct >= T && !prefilter && !config.bool_mask_tile && plan.order.size() >= 2 &&
                         csaidx_cuda_score_uses_tensor_cores(&cd, ops.dtype, mcode, kcode) != 0 &&
                         (overlap_sms < 0 || (overlap_sms > 0 && csaidx_cuda_select_overlap_capable(k) != 0));
    // Two-level select (csaidx_cuda_score_gmax): when rows can span >= 4k
    // 32-key groups the score epilogue also writes each group's maximum, and
    // the select reads only the ~k groups that can hold a top-k score
    // (opt-in, CSAIDX_TWO_LEVEL=1: measured slower overall at C4).
    const bool two_level = ct >= T && !prefilter && !config.bool_mask_tile && two_level_enabled() &&
                           csaidx_cuda_score_uses_tensor_cores(&cd, ops.dtype, mcode, kcode) != 0 &&
                           ceil_div(ct, 32) >= 4 * k;
    const int64_t gmax_ld = ceil_div(ct, 32);
    DeviceBuffer gmax_buf[2];  // double buffered like the score tiles when the select runs beside the score
    if (two_level)
        for (int i = 0; i < (overlap ? 2 : 1); ++i)
            gmax_buf[i] = DeviceBuffer(e, static_cast<size_t>(B * plan.cs * gmax_ld) * sizeof(float));
    DeviceBuffer scores2;
    struct PartitionGuard {
        csaidx_engine* e = nullptr;
        ~PartitionGuard() {
            if (e != nullptr) csaidx_engine_set_partition(e, 0, 0);
        }
    } partition;
    if (overlap) {
        scores2 = DeviceBuffer(e, static_cast<size_t>(B * plan.cs * ld) * sizeof(float));
        if (overlap_sms > 0) {
            int nsm = 0;
            check(csaidx_engine_num_sms(e, &nsm));
            const int x = std::min(overlap_sms, nsm / 3);
            check(csaidx_engine_set_partition(e, nsm - x, x));
            partition.e = e;
        }
    }
    constexpr int kScoreDone = 64, kSelectDone = 96, kSideLane = 3;

    for (size_t o = 0; o < plan.order.size(); ++o) {
        const size_t c = plan.order[o];
        float* const sbuf = overlap && (o & 1) ? scores2.as<float>() : scores.as<float>();
        float* const gbuf = two_level ? gmax_buf[overlap ? (o & 1) : 0].as<float>() : nullptr;
        // (overlap) the buffer was last read by chunk o-2's select
        if (overlap && o >= 2) check(csaidx_engine_await(e, kSelectDone + static_cast<int>((o - 2) % 32)));
        const int64_t s0 = plan.starts[c];
        const int64_t rows = std::min(plan.cs, dims.seq_len - s0);
        const int64_t op_rows = ops.op_rows > 0 ? ops.op_rows : dims.seq_len;
        const int64_t op_row0 = ops.op_rows > 0 ? plan.out_row0[c] : s0;
        if (hooks.before) hooks.before(o);
        LedgerCharge buffer_charge(ledger, "topk_buffer", run_buffer_bytes(B, rows, k));
        // One key tile covering all T keys: its select is a copy into the
        // all-sentinel buffer followed by the sentinel pass, so it writes the
        // output rows directly (csaidx_cuda_select_final) and the buffer is
        // only initialised if the tile ends up skipped.
        const bool one_tile = ct >= T;
        bool finalized = false;
        if (!one_tile) check(csaidx_cuda_fill_sentinel(e, run_v.as<float>(), run_i.as<int32_t>(), B * rows * k));
        bool first = true;
        for (int64_t t0 = 0; t0 < T; t0 += ct) {
            // The requested (logical) key tiles inside this physical one, with
            // the reference's per-tile decisions and ledger charges in its
            // order (driver.cpp:44-69); `end` closes the dispatched ones.
            int64_t end = t0;
            bool exited = false;
            for (int64_t l0 = t0; l0 < std::min(T, t0 + ct); l0 += plan.ct) {
                const int64_t lcols = std::min(plan.ct, T - l0);
                if (config.ablation == Ablation::a2_skip_narrow && lcols < k) {
                    ++stats.tiles_skipped_narrow;
                    continue;
                }
                if (config.causal_early_exit && tile_fully_masked(s0, rows, l0, dims.ratio)) {
                    stats.tiles_skipped_masked += ceil_div(T - l0, plan.ct);
                    exited = true;
                    break;
                }
                LedgerCharge tile_charge(ledger, "score_tile", chunk_tile_bytes(B, rows, lcols));
                if (config.bool_mask_tile) {
                    LedgerCharge mask_charge(ledger, "mask_tile", static_cast<uint64_t>(rows) * static_cast<uint64_t>(lcols));
                }
                LedgerCharge scratch_charge(ledger, "tile_topk_scratch", tile_scratch_bytes(B, rows, lcols, k));
                ++stats.dispatch_count;
                end = l0 + lcols;
            }
            if (end == t0) {
                if (exited) break;
                continue;
            }
            const int64_t cols = end - t0;
            const int64_t legal_max = std::min(cols, (s0 + rows) / dims.ratio - t0);
            const bool filtered = prefilter && legal_max > cap;
            if (filtered) {
                const int64_t ntiles = ceil_div(cols, 128);
                const int stride = static_cast<int>(std::max<int64_t>(1, ceil_div(ntiles, kPrefilterSampleTiles)));
                check(csaidx_cuda_score_sampled(e, ops.q, ops.kc, ops.w, &cd, s0, rows, t0, cols, stride,
                                                pf_sample.as<float>(), lds));
                check(csaidx_cuda_row_threshold(e, pf_sample.as<float>(), lds, B, rows, cols, s0, t0, dims.ratio,
                                                stride, k, pf_tau.as<float>()));
                check(csaidx_cuda_score_filtered(e, ops.q, ops.kc, ops.w, &cd, s0, rows, t0, cols, sbuf,
                                                 ld, pf_tau.as<float>(), pf_bits.as<uint32_t>(), bits_ld));
            } else if (config.bool_mask_tile) {
                check(csaidx_cuda_score_rows(e, ops.q, ops.kc, ops.dtype, ops.w, &cd, s0, rows, t0, cols, mcode, kcode,
                                             0, sbuf, ld, op_rows, op_row0));
                check(csaidx_cuda_bool_mask(e, keep.as<uint8_t>(), s0, t0, rows, cols, dims.ratio));
                check(csaidx_cuda_apply_bool_mask(e, sbuf, ld, keep.as<uint8_t>(), B, rows, cols));
            } else if (two_level) {
                check(csaidx_cuda_score_gmax(e, ops.q, ops.kc, ops.w, &cd, s0, rows, t0, cols, sbuf, ld, op_rows, op_row0,
                                             gbuf, gmax_ld));
            } else {
                check(csaidx_cuda_score_rows(e, ops.q, ops.kc, ops.dtype, ops.w, &cd, s0, rows, t0, cols, mcode, kcode,
                                             1, sbuf, ld, op_rows, op_row0));
            }
            const int64_t width = std::min(k, cols);
            const bool overwrite = config.ablation == Ablation::a1_no_merge;
            auto select = [&](float* v, int32_t* i, int64_t out_ld) {
                if (filtered)
                    check(csaidx_cuda_select_from_candidates(e, sbuf, B, rows, ld, cols, s0, t0,
                                                             dims.ratio, k, pf_bits.as<uint32_t>(), bits_ld, v, i,
                                                             out_ld));
                else
                    check(csaidx_cuda_select(e, sbuf, B, rows, ld, cols, s0, t0, dims.ratio, 1, k, v, i,
                                             out_ld));
            };
            if (one_tile) {
                if (overlap) {  // select on the side lane once this chunk's score is done
                    check(csaidx_engine_signal(e, kScoreDone + static_cast<int>(o % 32)));
                    check(csaidx_engine_use_lane(e, kSideLane));
                    check(csaidx_engine_await(e, kScoreDone + static_cast<int>(o % 32)));
                }
                check(csaidx_cuda_select_final(e, sbuf, B, rows, ld, cols, s0, t0, dims.ratio, k,
                                               filtered ? pf_bits.as<uint32_t>() : nullptr, bits_ld,
                                               gbuf, two_level ? gmax_ld : 0,
                                               out_idx, out_val, out_rows, plan.out_row0[c]));
                if (overlap) check(csaidx_engine_signal(e, kSelectDone + static_cast<int>(o % 32)));
                finalized = true;
            } else if (first && width == k) {
                // merge into all-sentinel rows (or A1 overwrite) == copy
                select(run_v.as<float>(), run_i.as<int32_t>(), k);
            } else {
                select(cand_v.as<float>(), cand_i.as<int32_t>(), width);
                check(csaidx_cuda_merge(e, run_v.as<float>(), run_i.as<int32_t>(), B * rows, k, cand_v.as<float>(),
                                        cand_i.as<int32_t>(), width, width, overwrite ? 1 : 0, 0));
            }
            first = false;
            if (exited) break;
        }
        if (!finalized) {
            if (one_tile) check(csaidx_cuda_fill_sentinel(e, run_v.as<float>(), run_i.as<int32_t>(), B * rows * k));
            check(csaidx_cuda_finalize(e, run_v.as<float>(), run_i.as<int32_t>(), B, rows, s0, dims.ratio, k,
                                       config.ablation == Ablation::none ? 1 : 0, out_idx, out_val, out_rows,
                                       plan.out_row0[c]));
        }
        // (overlap) still on the side lane when this chunk's select was
        // enqueued there: hooks.after signals from it and returns to lane 0
        if (hooks.after)
            hooks.after(o);
        else
            check(csaidx_engine_use_lane(e, 0));
    }
    check(csaidx_engine_check(e));
}

void run_materialize_device(csaidx_engine* e, const DeviceOps& ops, const ProblemDims& dims, int mode, int kernel,
                            int64_t* out_idx, float* out_val, MemoryLedger& ledger) {
    const int64_t B = dims.batch, S = dims.seq_len, T = dims.key_blocks, k = dims.top_k;
    LedgerCharge charge(ledger, "score_tile", chunk_tile_bytes(B, S, T));
    const int64_t ld = (T + 3) / 4 * 4;
    const csaidx_dims cd = to_c(dims);
    DeviceBuffer scores(e, static_cast<size_t>(B * S * ld) * sizeof(float));
    // The whole [B, S, T] matrix as one masked tile, same kernel as chunked.
    check(csaidx_cuda_score(e, ops.q, ops.kc, ops.dtype, ops.w, &cd, 0, S, 0, T, mode, kernel, 1, scores.as<float>(),
                            ld));
    const int64_t width = std::min(k, T);
    DeviceBuffer run_v(e, static_cast<size_t>(B * S * k) * 4), run_i(e, static_cast<size_t>(B * S * k) * 4);
    check(csaidx_cuda_fill_sentinel(e, run_v.as<float>(), run_i.as<int32_t>(), B * S * k));
    // oracle_topk per row == top-min(k, legal) sorted under succ; rows are
    // written at stride k so the tail beyond `width` keeps its sentinels.
    check(csaidx_cuda_select(e, scores.as<float>(), B, S, ld, T, 0, 0, dims.ratio, 1, k, run_v.as<float>(),
                             run_i.as<int32_t>(), k));
    (void)width;
    check(csaidx_cuda_finalize(e, run_v.as<float>(), run_i.as<int32_t>(), B, S, 0, dims.ratio, k, 1, out_idx, out_val,
                               S, 0));
    check(csaidx_engine_check(e));
}

namespace {

void check_extents(const ProblemDims& dims, size_t nq, size_t nk, size_t nw) {
    validate_dims(dims);
    if (static_cast<int64_t>(nq) != dims.q_elems() || static_cast<int64_t>(nk) != dims.kc_elems() ||
        static_cast<int64_t>(nw) != dims.w_elems())
        throw std::invalid_argument("IndexerInputs: extent mismatch with ProblemDims");
}

void download_result(csaidx_engine* e, const DeviceBuffer& idx, const DeviceBuffer& val, TopKResult& out) {
    idx.download(out.indices.data(), out.indices.size() * sizeof(int64_t));
    val.download(out.values.data(), out.values.size() * sizeof(float));
    check(csaidx_engine_check(e));
}

}  // namespace

namespace {

// Pinned bf16 staging slabs of the host-rounding pipeline, kept across calls
// (pinning hundreds of MiB per call would cost more than the transfer).
// One set per calling thread (see engine()).
struct PinnedSlabs {
    std::vector<void*> ptr;
    size_t bytes = 0;
    uint16_t* get(csaidx_engine* e, int i, int count, size_t need) {
        if (need > bytes || static_cast<int>(ptr.size()) < count) {
            release(e);
            ptr.assign(static_cast<size_t>(count), nullptr);
            bytes = need;
            try {
                for (auto& p : ptr) check(csaidx_cuda_host_alloc(e, bytes, &p));
            } catch (...) {
                release(e);  // all or nothing
                throw;
            }
        }
        return static_cast<uint16_t*>(ptr[static_cast<size_t>(i)]);
    }
    void release(csaidx_engine* e) {
        for (void* p : ptr)
            if (p != nullptr) csaidx_cuda_host_free(e, p);
        ptr.clear();
        bytes = 0;
    }
};

PinnedSlabs& pinned_slabs() {
    thread_local PinnedSlabs s;  // per calling thread, like its engine
    return s;
}

PinnedSlabs& pinned_kc() {
    thread_local PinnedSlabs s;  // bf16 kc staging (the copy then runs async at full PCIe speed)
    return s;
}

PinnedSlabs& pinned_ring() {
    thread_local PinnedSlabs s;  // the ring pieces of CSAIDX_HOST_RING=1
    return s;
}

// State shared by the host-rounding producer thread and the thread that
// drives the lanes: the producer rounds chunk o's q rows into slab
// o % slabs once the copy of chunk o - slabs out of it has completed.
struct HostRounder {
    std::mutex mu;
    std::condition_variable cv;
    size_t converted = 0;  // chunks [0, converted) are in their slabs
    size_t enqueued = 0;   // ... and their copies are queued
    bool stop = false;
    bool inexact = false;  // a q row is not bf16-representable (non-strict): re-run on fp32
    std::string error;
    std::thread th;

    ~HostRounder() {
        {
            std::lock_guard<std::mutex> g(mu);
            stop = true;
        }
        cv.notify_all();
        if (th.joinable()) th.join();
    }
    void fail(const std::string& what) {
        {
            std::lock_guard<std::mutex> g(mu);
            error = what;
        }
        cv.notify_all();
    }
};

// CSAIDX_HOST_TRACE=1: per-chunk host timestamps of the pipelined entry
bool host_trace() {
    static const bool v = std::getenv("CSAIDX_HOST_TRACE") != nullptr;
    return v;
}
double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

Transfer& last_transfer() {
    thread_local Transfer t;
    return t;
}

namespace {

// The operands are not bf16-representable: ScoreKernel::auto_detect then
// re-runs on fp32 operands with the exact-order kernel (the reference's auto
// kernel is bit-identical to its scalar one on any fp32 input).
struct OperandsNotBf16 : std::exception {
    const char* what() const noexcept override { return "operands are not bf16-representable"; }
};

void run_chunked_rows_impl(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                           const std::vector<int64_t>* starts, int64_t* host_idx, float* host_val, int64_t out_rows,
                           MemoryLedger& ledger, RunStats* stats_out, int dtype);

}  // namespace

void run_chunked_rows_view(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                           const std::vector<int64_t>* starts, int64_t* host_idx, float* host_val, int64_t out_rows,
                           MemoryLedger& ledger, RunStats* stats_out) {
    const int dtype = operand_dtype(dims, mode_code(config.mode), kernel_code(config.kernel, config.mode));
    try {
        run_chunked_rows_impl(in, dims, config, starts, host_idx, host_val, out_rows, ledger, stats_out, dtype);
    } catch (const OperandsNotBf16&) {
        run_chunked_rows_impl(in, dims, config, starts, host_idx, host_val, out_rows, ledger, stats_out,
                              CSAIDX_DTYPE_F32);
    }
}

namespace {

void run_chunked_rows_impl(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                           const std::vector<int64_t>* starts, int64_t* host_idx, float* host_val, int64_t out_rows,
                           MemoryLedger& ledger, RunStats* stats_out, int dtype) {
    const ChunkPlan plan = plan_chunks(dims, config.tile, starts);
    int64_t need = 0;
    std::vector<std::pair<int64_t, int64_t>> ranges;
    for (size_t c = 0; c < plan.starts.size(); ++c) {
        const int64_t rows = std::min(plan.cs, dims.seq_len - plan.starts[c]);
        ranges.emplace_back(plan.starts[c], rows);
        need = plan.out_row0[c] + rows;
    }
    if (out_rows < need) throw std::invalid_argument("run_chunked: out_rows too small for the chunk list");
    const bool strict = gpu::options().strict_bf16;
    std::lock_guard<std::mutex> lock(engine_mutex());
    csaidx_engine* e = engine();

    // Three-lane pipeline: lane 1 copies chunk c+1's q / w rows in (and rounds
    // q to bf16) while lane 0 computes chunk c and lane 2 copies chunk c-1's
    // indices / values out. With pinned host buffers the PCIe traffic hides
    // behind the kernels; pageable buffers still work (copies then block).
    const int64_t B = dims.batch, k = dims.top_k, qrow = dims.heads * dims.head_dim;
    const size_t esz = dtype == CSAIDX_DTYPE_BF16 ? 2 : 4;
    // q / w on device hold only this call's chunks (rank-local stacks in plan
    // order, the same row layout as the outputs)
    DeviceBuffer q(e, static_cast<size_t>(B * out_rows * qrow) * esz), kc(e, static_cast<size_t>(dims.kc_elems()) * esz),
        w(e, static_cast<size_t>(B * out_rows * dims.heads) * sizeof(float));
    constexpr int kSlabs = 8, kConvDone = 128;  // staging slabs; event slots of their conversion
    // host_round: q rows are rounded to bf16 on the host cores into pinned
    // slabs by a producer thread running ahead of the copies, and cross PCIe
    // at 2 bytes per entry (PCIe bounds the end-to-end call); otherwise fp32
    // rows are copied into device slabs and rounded there.
    // (Measured: rounding only part of the chunks on the host, to balance
    // PCIe against host DRAM bandwidth, was slower than rounding all.)
    const size_t slab_elems = static_cast<size_t>(B * plan.cs * qrow);
    const int hslabs = host_slab_count();  // <= 32: the copy-done slots
    std::vector<uint16_t*> hslab(static_cast<size_t>(hslabs), nullptr);
    bool host_round = dtype == CSAIDX_DTYPE_BF16 && host_round_enabled();
    // ring mode: pieces of piece_elems bf16 through ring_n pinned buffers
    const bool ring = host_round && host_ring_enabled();
    const int ring_n = host_ring_pieces();
    const size_t piece_elems = static_cast<size_t>(host_piece_bytes()) / sizeof(uint16_t);
    constexpr int kRingSlot0 = 160;  // event slots 160.. belong to the rounding thread
    std::vector<uint16_t*> rslab(static_cast<size_t>(ring_n), nullptr);
    if (host_round) {
        try {
            if (ring) {
                for (int i = 0; i < ring_n; ++i)
                    rslab[static_cast<size_t>(i)] = pinned_ring().get(e, i, ring_n, piece_elems * sizeof(uint16_t));
                // the copy-in lane exists before the rounding thread enqueues on it
                check(csaidx_engine_use_lane(e, 1));
                check(csaidx_engine_use_lane(e, 0));
            } else {
                for (int i = 0; i < hslabs; ++i)
                    hslab[static_cast<size_t>(i)] = pinned_slabs().get(e, i, hslabs, slab_elems * sizeof(uint16_t));
            }
        } catch (const std::exception&) {
            host_round = false;  // no pinned staging available: round on the device
        }
    }
    // fp32 tail: the last chunks of the processing order (the lightest on
    // the GPU) cross PCIe as fp32 at the start of the call, beside the early
    // heavy chunks' bf16 pieces, and are rounded on the device when their
    // turn comes; the rounding thread then finishes that much earlier, which
    // is what bounds the end of the call on hosts with slower memory.
    // (pinned q only: pageable copies would block the calling thread)
    size_t ntail = 0;
    if (host_round) {
        int pinned = 0;
        check(csaidx_cuda_host_is_pinned(in.q, &pinned));
        if (pinned) ntail = std::min(plan.order.size(), host_fp32_tail(plan.order.size()));
    }
    const size_t tail0 = plan.order.size() - ntail;
    constexpr int kTailSlot0 = 164;  // event slots 164..191: one per tail chunk
    DeviceBuffer tailbuf;
    if (ntail > 0) tailbuf = DeviceBuffer(e, ntail * slab_elems * sizeof(float));
    DeviceBuffer slab[kSlabs];
    if (dtype == CSAIDX_DTYPE_BF16 && !host_round) {
        for (auto& sb : slab) sb = DeviceBuffer(e, slab_elems * sizeof(float));
    }
    const double t_start = now_ms();
    HostRounder rounder;
    if (host_round) {
        rounder.th = std::thread([&] {
            try {
                size_t rc = 0;  // ring pieces issued
                for (size_t o = 0; o < plan.order.size(); ++o) {
                    const double t0 = now_ms();
                    if (o >= tail0) {  // fp32 tail: rounded on the device
                        {
                            std::lock_guard<std::mutex> g(rounder.mu);
                            rounder.converted = o + 1;
                        }
                        rounder.cv.notify_all();
                        continue;
                    }
                    if (!ring && o >= static_cast<size_t>(hslabs)) {
                        {
                            std::unique_lock<std::mutex> g(rounder.mu);
                            rounder.cv.wait(g, [&] { return rounder.stop || rounder.enqueued > o - hslabs; });
                            if (rounder.stop) return;
                        }
                        // the copy out of this slab (chunk o - hslabs) has finished
                        check(csaidx_engine_sync_slot(e, static_cast<int>((o - hslabs) % 32)));
                    }
                    const double t1 = now_ms();
                    const size_t c = plan.order[o];
                    const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, dims.seq_len - s0);
                    Bf16Flags f;
                    for (int64_t b = 0; b < B; ++b) {
                        const int64_t hrow = in.local_rows ? b * out_rows + plan.out_row0[c] : b * dims.seq_len + s0;
                        if (ring) {
                            // piece by piece: round into the ring slot (regular
                            // stores, the lines stay cached) and copy it at once
                            const size_t n = static_cast<size_t>(rows * qrow);
                            const int64_t lrow = b * out_rows + plan.out_row0[c];
                            for (size_t off = 0; off < n; off += piece_elems, ++rc) {
                                const int slot = static_cast<int>(rc % static_cast<size_t>(ring_n));
                                if (rc >= static_cast<size_t>(ring_n)) check(csaidx_engine_sync_slot(e, kRingSlot0 + slot));
                                const size_t len = std::min(piece_elems, n - off);
                                const Bf16Flags fb = host_to_bf16(in.q + hrow * qrow + off, rslab[static_cast<size_t>(slot)],
                                                                  len, 0);
                                f.nonfinite = f.nonfinite || fb.nonfinite;
                                f.inexact = f.inexact || fb.inexact;
                                if (f.nonfinite || f.inexact) break;  // reported below; nothing more to send
                                check(csaidx_engine_copy_on_lane(e, 1, kRingSlot0 + slot, q.as<uint16_t>() + lrow * qrow + off,
                                                                 rslab[static_cast<size_t>(slot)], len * sizeof(uint16_t)));
                            }
                            continue;
                        }
                        const Bf16Flags fb = host_to_bf16(in.q + hrow * qrow, hslab[o % hslabs] + b * rows * qrow,
                                                          static_cast<size_t>(rows * qrow));
                        f.nonfinite = f.nonfinite || fb.nonfinite;
                        f.inexact = f.inexact || fb.inexact;
                    }
                    if (host_trace())
                        std::fprintf(stderr, "round %zu wait %.3f convert %.3f at %.3f\n", o, t1 - t0, now_ms() - t1,
                                     now_ms() - t_start);
                    if (f.nonfinite) return rounder.fail("IndexerInputs: non-finite entry in q/kc");
                    if (strict && f.inexact) return rounder.fail("operand is not bf16-representable (strict mode)");
                    if (f.inexact) {
                        rounder.inexact = true;
                        return rounder.fail("operands are not bf16-representable");
                    }
                    {
                        std::lock_guard<std::mutex> g(rounder.mu);
                        rounder.converted = o + 1;
                    }
                    rounder.cv.notify_all();
                }
            } catch (const std::exception& ex) {
                rounder.fail(ex.what());
            }
        });
    }
    const size_t n = static_cast<size_t>(B * out_rows * k);
    DeviceBuffer idx(e, n * sizeof(int64_t)), val(e, n * sizeof(float));
    const DeviceOps ops{q.as<void>(), kc.as<void>(), w.as<float>(), dtype, out_rows};
    constexpr int kMainLane = 0, kInLane = 1, kOutLane = 2;
    // Copy-in lane: raw fp32 rows only, so the DMA engine never waits for
    // SMs (a conversion kernel queued on the copy lane would sit behind the
    // persistent score kernel and stall the next copy). The bf16 rounding of
    // chunk o runs on the main lane right before chunk o's score; kSlabs
    // staging slabs let the copies run up to kSlabs chunks ahead.
    auto upload_rounded = [&](size_t o) {  // host_round: chunk o's bf16 slab and w rows, on the copy-in lane
        const size_t c = plan.order[o];
        const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, dims.seq_len - s0);
        const double t0 = now_ms();
        {
            std::unique_lock<std::mutex> g(rounder.mu);
            rounder.cv.wait(g, [&] { return rounder.converted > o || !rounder.error.empty(); });
            if (rounder.converted <= o) {
                if (rounder.inexact) throw OperandsNotBf16();
                throw std::invalid_argument(rounder.error);
            }
        }
        if (host_trace()) std::fprintf(stderr, "upload %zu waited %.3f at %.3f\n", o, now_ms() - t0, now_ms() - t_start);
        for (int64_t b = 0; b < B; ++b) {
            const int64_t lrow = b * out_rows + plan.out_row0[c];
            const int64_t hrow = in.local_rows ? lrow : b * dims.seq_len + s0;
            if (!ring && o < tail0)  // (ring: the rounding thread has enqueued the pieces on this lane; tail: fp32 below)
                check(csaidx_cuda_copy(e, q.as<uint16_t>() + lrow * qrow, hslab[o % hslabs] + b * rows * qrow,
                                       static_cast<size_t>(rows * qrow) * sizeof(uint16_t)));
            check(csaidx_cuda_copy(e, w.as<float>() + lrow * dims.heads, in.w + hrow * dims.heads,
                                   static_cast<size_t>(rows * dims.heads) * sizeof(float)));
        }
        check(csaidx_engine_signal(e, static_cast<int>(o % 32)));
        {
            std::lock_guard<std::mutex> g(rounder.mu);
            rounder.enqueued = o + 1;
        }
        rounder.cv.notify_all();
    };
    auto upload_raw = [&](size_t o) {  // o-th chunk in processing order, on the copy-in lane
        if (host_round) return upload_rounded(o);
        const size_t c = plan.order[o];
        const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, dims.seq_len - s0);
        if (dtype == CSAIDX_DTYPE_BF16 && o >= kSlabs)  // slab o % kSlabs: chunk o - kSlabs converted
            check(csaidx_engine_await(e, kConvDone + static_cast<int>((o - kSlabs) % 32)));
        for (int64_t b = 0; b < B; ++b) {
            const int64_t lrow = b * out_rows + plan.out_row0[c];  // operand row on device
            const int64_t hrow = in.local_rows ? lrow : b * dims.seq_len + s0;  // ... and on the host
            const int64_t qoff = hrow * qrow, woff = hrow * dims.heads;
            void* qdst = dtype == CSAIDX_DTYPE_BF16
                             ? static_cast<void*>(slab[o % kSlabs].as<float>() + b * rows * qrow)
                             : static_cast<void*>(q.as<float>() + lrow * qrow);
            check(csaidx_cuda_copy(e, qdst, in.q + qoff, static_cast<size_t>(rows * qrow) * sizeof(float)));
            check(csaidx_cuda_copy(e, w.as<float>() + lrow * dims.heads, in.w + woff,
                                   static_cast<size_t>(rows * dims.heads) * sizeof(float)));
        }
        check(csaidx_engine_signal(e, static_cast<int>(o % 32)));
    };
    auto convert = [&](size_t o) {  // on the main lane, after chunk o's copy
        if (host_round && o >= tail0) {  // fp32 tail chunk: its rows arrived early on lane 3
            const size_t t = o - tail0;
            const size_t c = plan.order[o];
            const int64_t rows = std::min(plan.cs, dims.seq_len - plan.starts[c]);
            check(csaidx_engine_await(e, kTailSlot0 + static_cast<int>(t)));
            for (int64_t b = 0; b < B; ++b) {
                const int64_t lrow = b * out_rows + plan.out_row0[c];
                check(csaidx_cuda_to_bf16(e, tailbuf.as<float>() + t * slab_elems + b * rows * qrow,
                                          q.as<uint16_t>() + lrow * qrow, rows * qrow, strict ? 1 : 0));
            }
            return;
        }
        if (dtype != CSAIDX_DTYPE_BF16 || host_round) return;
        const size_t c = plan.order[o];
        const int64_t rows = std::min(plan.cs, dims.seq_len - plan.starts[c]);
        for (int64_t b = 0; b < B; ++b) {
            const int64_t lrow = b * out_rows + plan.out_row0[c];
            check(csaidx_cuda_to_bf16(e, slab[o % kSlabs].as<float>() + b * rows * qrow,
                                      q.as<uint16_t>() + lrow * qrow, rows * qrow, strict ? 1 : 0));
        }
        check(csaidx_engine_signal(e, kConvDone + static_cast<int>(o % 32)));
    };
    ChunkHooks hooks;
    hooks.before = [&](size_t o) {
        check(csaidx_engine_use_lane(e, kInLane));
        if (o == 0) {
            if (dtype == CSAIDX_DTYPE_BF16) {
                // kc is small: rounded on the host (bit-identical to the
                // device rounding), which also tells representability up front
                const size_t kn = static_cast<size_t>(dims.kc_elems());
                uint16_t* kc16 = nullptr;
                std::vector<uint16_t> kc16v;  // pageable fallback when pinned staging is unavailable
                try {
                    kc16 = pinned_kc().get(e, 0, 1, kn * sizeof(uint16_t));
                } catch (const std::exception&) {
                    kc16v.resize(kn);
                    kc16 = kc16v.data();
                }
                const Bf16Flags f = host_to_bf16(in.kc, kc16, kn);
                if (f.nonfinite) throw std::invalid_argument("IndexerInputs: non-finite entry in q/kc");
                if (f.inexact && strict) throw std::invalid_argument("operand is not bf16-representable (strict mode)");
                if (f.inexact) throw OperandsNotBf16();
                kc.upload(kc16, kn * sizeof(uint16_t));
            } else {
                kc.upload(in.kc, static_cast<size_t>(dims.kc_elems()) * sizeof(float));
            }
            upload_raw(0);
            if (ntail > 0) {
                check(csaidx_engine_use_lane(e, 3));
                for (size_t t = 0; t < ntail; ++t) {
                    const size_t c = plan.order[tail0 + t];
                    const int64_t s0 = plan.starts[c], rows = std::min(plan.cs, dims.seq_len - s0);
                    for (int64_t b = 0; b < B; ++b) {
                        const int64_t hrow = in.local_rows ? b * out_rows + plan.out_row0[c] : b * dims.seq_len + s0;
                        check(csaidx_cuda_copy(e, tailbuf.as<float>() + t * slab_elems + b * rows * qrow,
                                               in.q + hrow * qrow, static_cast<size_t>(rows * qrow) * sizeof(float)));
                    }
                    check(csaidx_engine_signal(e, kTailSlot0 + static_cast<int>(t)));
                }
                check(csaidx_engine_use_lane(e, kInLane));
            }
        }
        if (o + 1 < plan.order.size()) upload_raw(o + 1);
        check(csaidx_engine_use_lane(e, kMainLane));
        check(csaidx_engine_await(e, static_cast<int>(o % 32)));
        convert(o);
    };
    hooks.after = [&](size_t o) {
        const size_t c = plan.order[o];
        check(csaidx_engine_signal(e, static_cast<int>(32 + o % 32)));
        check(csaidx_engine_use_lane(e, kOutLane));
        check(csaidx_engine_await(e, static_cast<int>(32 + o % 32)));
        const int64_t rows = std::min(plan.cs, dims.seq_len - plan.starts[c]);
        for (int64_t b = 0; b < B; ++b) {
            const int64_t off = (b * out_rows + plan.out_row0[c]) * k;
            check(csaidx_cuda_copy(e, host_idx + off, idx.as<int64_t>() + off, static_cast<size_t>(rows * k) * 8));
            check(csaidx_cuda_copy(e, host_val + off, val.as<float>() + off, static_cast<size_t>(rows * k) * 4));
        }
        check(csaidx_engine_use_lane(e, kMainLane));
    };
    RunStats stats;
    try {
        run_plan(e, ops, dims, config, plan, idx.as<int64_t>(), val.as<float>(), out_rows, ledger, stats, hooks);
    } catch (...) {
        csaidx_engine_use_lane(e, kMainLane);
        csaidx_engine_check(e);  // drain every lane before the buffers go away
        int seen = 0;
        csaidx_engine_take_inexact(e, &seen);
        throw;
    }
    if (dtype == CSAIDX_DTYPE_BF16 && (!host_round || ntail > 0) && !strict) {
        // the device rounding noted a q value bf16 cannot hold
        int seen = 0;
        check(csaidx_engine_take_inexact(e, &seen));
        if (seen) throw OperandsNotBf16();
    }
    // bytes this call moved over PCIe (csaidx_host_last_transfer)
    {
        const uint64_t qe = static_cast<uint64_t>(B * need) * static_cast<uint64_t>(qrow);
        const uint64_t q_bytes = qe * (dtype == CSAIDX_DTYPE_BF16 && host_round ? 2 : 4);
        last_transfer() = Transfer{q_bytes + static_cast<uint64_t>(dims.kc_elems()) * esz +
                                       static_cast<uint64_t>(B * need * dims.heads) * 4,
                                   static_cast<uint64_t>(B * need * k) * 12, host_round ? 0 : static_cast<int64_t>(plan.order.size()),
                                   static_cast<int64_t>(plan.order.size())};
    }
    if (stats_out != nullptr) *stats_out = stats;
}

}  // namespace

TopKResult run_chunked_view(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                            MemoryLedger& ledger, RunStats* stats_out) {
    TopKResult out = TopKResult::sized(dims);
    run_chunked_rows_view(in, dims, config, nullptr, out.indices.data(), out.values.data(), dims.seq_len, ledger,
                          stats_out);
    return out;
}

TopKResult run_materialize_view(const HostView& in, const ProblemDims& dims, AccumulationMode mode,
                                MemoryLedger& ledger, ScoreKernel kernel) {
    validate_dims(dims);
    TopKResult out = TopKResult::sized(dims);
    const int kcode = kernel_code(kernel, mode);
    const int mcode = mode_code(mode);
    std::lock_guard<std::mutex> lock(engine_mutex());
    csaidx_engine* e = engine();
    const StagedOperands ops(e, in, dims, operand_dtype(dims, mcode, kcode), gpu::options().strict_bf16);
    DeviceBuffer idx(e, out.indices.size() * sizeof(int64_t)), val(e, out.values.size() * sizeof(float));
    run_materialize_device(e, ops.ops(), dims, mcode, kcode, idx.as<int64_t>(), val.as<float>(), ledger);
    download_result(e, idx, val, out);
    return out;
}

}  // namespace detail

int64_t dispatch_count_model(const ProblemDims& dims, const TileConfig& tile) {
    tile.validate();
    const int64_t cs = std::min(tile.query_tile, dims.seq_len), ct = std::min(tile.key_tile, dims.key_blocks);
    return (dims.seq_len + cs - 1) / cs * ((dims.key_blocks + ct - 1) / ct);
}

TopKResult run_chunked(const IndexerInputs& inputs, const ProblemDims& dims, const DriverConfig& config,
                       MemoryLedger& ledger, RunStats* stats) {
    detail::check_extents(dims, inputs.q.size(), inputs.kc.size(), inputs.w.size());
    return detail::run_chunked_view({inputs.q.data(), inputs.kc.data(), inputs.w.data()}, dims, config, ledger,
                                    stats);
}

TopKResult run_materialize(const IndexerInputs& inputs, const ProblemDims& dims, AccumulationMode mode,
                           MemoryLedger& ledger, ScoreKernel kernel) {
    detail::check_extents(dims, inputs.q.size(), inputs.kc.size(), inputs.w.size());
    return detail::run_materialize_view({inputs.q.data(), inputs.kc.data(), inputs.w.data()}, dims, mode, ledger,
                                        kernel);
}

DispatchDecision choose_path(const ProblemDims& dims, uint64_t threshold_bytes) {
    const uint64_t predicted = materialize_bytes(dims);
    return {predicted <= threshold_bytes ? ExecutionPath::materialize : ExecutionPath::chunked, predicted};
}

TopKResult dispatch(const IndexerInputs& inputs, const ProblemDims& dims, const DriverConfig& config,
                    MemoryLedger& ledger, DispatchDecision* decision_out, RunStats* stats_out) {
    const DispatchDecision decision = choose_path(dims, config.auto_threshold_bytes);
    if (decision_out != nullptr) *decision_out = decision;
    if (decision.path == ExecutionPath::materialize) {
        if (stats_out != nullptr) *stats_out = RunStats{};
        return run_materialize(inputs, dims, config.mode, ledger, config.kernel);
    }
    return run_chunked(inputs, dims, config, ledger, stats_out);
}

namespace gpu {

void run_chunked_device(const DeviceOperands& ops, const ProblemDims& dims, const DriverConfig& config,
                        const std::vector<int64_t>* chunk_starts, int64_t* out_indices, float* out_values,
                        int64_t out_rows, MemoryLedger& ledger, RunStats* stats_out) {
    detail::validate_dims(dims);
    const detail::ChunkPlan plan = detail::plan_chunks(dims, config.tile, chunk_starts);
    int64_t need = 0;
    for (size_t c = 0; c < plan.starts.size(); ++c) need = plan.out_row0[c] + std::min(plan.cs, dims.seq_len - plan.starts[c]);
    if (out_rows < need) throw std::invalid_argument("run_chunked_device: out_rows too small for the chunk list");
    const int kcode = detail::kernel_code(config.kernel, config.mode);
    if (ops.dtype != detail::operand_dtype(dims, detail::mode_code(config.mode), kcode))
        throw std::invalid_argument("run_chunked_device: operand dtype does not match the selected score kernel");
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    csaidx_engine* e = detail::engine();
    // the operands were produced by the caller's (default-stream) work
    detail::check(csaidx_engine_await_stream(e, nullptr));
    RunStats stats;
    detail::run_plan(e, detail::DeviceOps{ops.q, ops.kc, ops.w, ops.dtype, ops.local_rows ? out_rows : 0}, dims,
                     config, plan, out_indices, out_values, out_rows, ledger, stats);
    if (stats_out != nullptr) *stats_out = stats;
}

}  // namespace gpu

}  // namespace csaidx
