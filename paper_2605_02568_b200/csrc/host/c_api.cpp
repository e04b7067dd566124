// C entry points of libcsaidx.so (include/csaidx_host.h): the reference
// driver API on raw host buffers (no IndexerInputs copy) and on device
// operands. Exceptions become status codes + a thread-local message.
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>

#include "csaidx/causal.hpp"
#include "csaidx/driver.hpp"
#include "csaidx/gpu.hpp"
#include "csaidx/tensor_io.hpp"
#include "csaidx_host.h"
#include "device.hpp"
#include "host_convert.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return CSAIDX_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return CSAIDX_INVALID_ARGUMENT;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return CSAIDX_OVERFLOW_ERROR;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return CSAIDX_LOGIC_ERROR;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return CSAIDX_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return CSAIDX_RUNTIME_ERROR;
    }
}

csaidx::ProblemDims from_c(const csaidx_dims* d) {
    if (d == nullptr) throw std::invalid_argument("null dims");
    csaidx::ProblemDims p{d->batch, d->seq_len, d->key_blocks, d->heads, d->head_dim, d->ratio, d->top_k};
    csaidx::detail::validate_dims(p);
    return p;
}

csaidx::DriverConfig from_c(const csaidx_run_config* c) {
    if (c == nullptr) throw std::invalid_argument("null config");
    csaidx::DriverConfig cfg;
    cfg.tile = csaidx::TileConfig{c->query_tile, c->key_tile};
    cfg.mode = c->mode == CSAIDX_MODE_FP16_EMULATED ? csaidx::AccumulationMode::fp16_emulated
                                                    : csaidx::AccumulationMode::fp32;
    switch (c->ablation) {
        case CSAIDX_ABLATION_NONE: cfg.ablation = csaidx::Ablation::none; break;
        case CSAIDX_ABLATION_A1_NO_MERGE: cfg.ablation = csaidx::Ablation::a1_no_merge; break;
        case CSAIDX_ABLATION_A2_SKIP_NARROW: cfg.ablation = csaidx::Ablation::a2_skip_narrow; break;
        default: throw std::invalid_argument("unknown ablation");
    }
    switch (c->kernel) {
        case CSAIDX_SCORE_AUTO: cfg.kernel = csaidx::ScoreKernel::auto_detect; break;
        case CSAIDX_SCORE_SCALAR: cfg.kernel = csaidx::ScoreKernel::scalar; break;
        case CSAIDX_SCORE_AVX2: cfg.kernel = csaidx::ScoreKernel::avx2; break;
        default: throw std::invalid_argument("unknown score kernel");
    }
    cfg.causal_early_exit = c->causal_early_exit != 0;
    cfg.bool_mask_tile = c->bool_mask_tile != 0;
    cfg.threads = c->threads;
    cfg.auto_threshold_bytes = c->auto_threshold_bytes;
    csaidx::gpu::Options o;
    o.device = c->device;
    o.strict_bf16 = c->strict_bf16 != 0;
    o.stream = c->stream;
    o.fp16_tensor_cores = c->fp16_tensor_cores != 0;
    csaidx::gpu::set_options(o);
    return cfg;
}

void copy_out(const csaidx::TopKResult& r, int64_t* idx, float* val) {
    std::memcpy(idx, r.indices.data(), r.indices.size() * sizeof(int64_t));
    std::memcpy(val, r.values.data(), r.values.size() * sizeof(float));
}

void fill_stats(csaidx_run_stats* st, const csaidx::RunStats& rs, const csaidx::MemoryLedger& ledger, int path) {
    if (st == nullptr) return;
    st->dispatch_count = rs.dispatch_count;
    st->tiles_skipped_masked = rs.tiles_skipped_masked;
    st->tiles_skipped_narrow = rs.tiles_skipped_narrow;
    st->ledger_peak_bytes = ledger.peak_bytes();
    st->device_peak_bytes = csaidx::gpu::device_memory().peak_bytes;
    st->path = path;
}

}  // namespace

extern "C" {

const char* csaidx_host_last_error(void) { return g_err.c_str(); }

void csaidx_host_default_config(csaidx_run_config* cfg) {
    if (cfg == nullptr) return;
    const csaidx::DriverConfig d;
    *cfg = csaidx_run_config{d.tile.query_tile, d.tile.key_tile, CSAIDX_MODE_FP32, CSAIDX_ABLATION_NONE,
                             CSAIDX_SCORE_AUTO, 1, 0, 1, d.auto_threshold_bytes, 0, 0, nullptr, 0};
}

int csaidx_host_engine(int device, csaidx_engine** out) {
    return guarded([&] {
        if (out == nullptr) throw std::invalid_argument("null out");
        csaidx::gpu::Options o = csaidx::gpu::options();
        o.device = device;
        csaidx::gpu::set_options(o);
        *out = csaidx::detail::engine();
    });
}

int csaidx_host_run_chunked(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                            const csaidx_run_config* cfg, int64_t* out_idx, float* out_val, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        const csaidx::TopKResult r = csaidx::detail::run_chunked_view({q, kc, w}, d, c, ledger, &rs);
        copy_out(r, out_idx, out_val);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_host_run_chunked_rows(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                 const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                                 int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        std::vector<int64_t> starts;
        if (chunk_starts != nullptr && n_chunks > 0) starts.assign(chunk_starts, chunk_starts + n_chunks);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        csaidx::detail::run_chunked_rows_view({q, kc, w}, d, c, starts.empty() ? nullptr : &starts, out_idx, out_val,
                                              out_rows, ledger, &rs);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_host_run_chunked_local(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                  const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                                  int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        std::vector<int64_t> starts;
        if (chunk_starts != nullptr && n_chunks > 0) starts.assign(chunk_starts, chunk_starts + n_chunks);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        csaidx::detail::run_chunked_rows_view({q, kc, w, true}, d, c, starts.empty() ? nullptr : &starts, out_idx, out_val,
                                              out_rows, ledger, &rs);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_host_run_materialize(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                                const csaidx_run_config* cfg, int64_t* out_idx, float* out_val,
                                csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        const csaidx::TopKResult r = csaidx::detail::run_materialize_view({q, kc, w}, d, c.mode, ledger, c.kernel);
        copy_out(r, out_idx, out_val);
        fill_stats(stats, csaidx::RunStats{}, ledger, 0);
    });
}

int csaidx_host_dispatch(const float* q, const float* kc, const float* w, const csaidx_dims* dims,
                         const csaidx_run_config* cfg, int64_t* out_idx, float* out_val, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        const csaidx::DispatchDecision dec = csaidx::choose_path(d, c.auto_threshold_bytes);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        const csaidx::TopKResult r =
            dec.path == csaidx::ExecutionPath::materialize
                ? csaidx::detail::run_materialize_view({q, kc, w}, d, c.mode, ledger, c.kernel)
                : csaidx::detail::run_chunked_view({q, kc, w}, d, c, ledger, &rs);
        copy_out(r, out_idx, out_val);
        fill_stats(stats, rs, ledger, dec.path == csaidx::ExecutionPath::materialize ? 0 : 1);
    });
}

int csaidx_device_run_chunked(const void* q, const void* kc, int dtype, const float* w, const csaidx_dims* dims,
                              const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                              int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        std::vector<int64_t> starts;
        if (chunk_starts != nullptr && n_chunks > 0) starts.assign(chunk_starts, chunk_starts + n_chunks);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        csaidx::gpu::run_chunked_device(csaidx::gpu::DeviceOperands{q, kc, w, dtype}, d, c,
                                        starts.empty() ? nullptr : &starts, out_idx, out_val, out_rows, ledger, &rs);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_device_run_chunked_local(const void* q, const void* kc, int dtype, const float* w, const csaidx_dims* dims,
                                    const csaidx_run_config* cfg, const int64_t* chunk_starts, int64_t n_chunks,
                                    int64_t* out_idx, float* out_val, int64_t out_rows, csaidx_run_stats* stats) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        std::vector<int64_t> starts;
        if (chunk_starts != nullptr && n_chunks > 0) starts.assign(chunk_starts, chunk_starts + n_chunks);
        csaidx::gpu::reset_device_peak();
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        csaidx::gpu::run_chunked_device(csaidx::gpu::DeviceOperands{q, kc, w, dtype, true}, d, c,
                                        starts.empty() ? nullptr : &starts, out_idx, out_val, out_rows, ledger, &rs);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_host_write_inputs_file(const char* path, const float* q, const float* kc, const float* w,
                                  const csaidx_dims* dims, uint64_t* bytes) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        csaidx::IndexerInputs in;
        in.q.assign(q, q + d.q_elems());
        in.kc.assign(kc, kc + d.kc_elems());
        in.w.assign(w, w + d.w_elems());
        const uint64_t n = csaidx::write_inputs_file(path, in, d);
        if (bytes != nullptr) *bytes = n;
    });
}

int csaidx_host_scan_sections(const char* path, csaidx_section_info* out, int max_sections, int* n_sections) {
    return guarded([&] {
        const auto secs = csaidx::detail::scan_sections_file(path);
        for (size_t i = 0; i < secs.size() && static_cast<int>(i) < max_sections; ++i) {
            out[i].tag = secs[i].tag;
            out[i].rank = secs[i].rank;
            for (int j = 0; j < 4; ++j) out[i].dims[j] = secs[i].dims[j];
            out[i].elems = secs[i].elems;
            out[i].offset = secs[i].offset;
        }
        *n_sections = static_cast<int>(secs.size());
    });
}

int csaidx_host_read_inputs(const char* path, const csaidx_dims* dims, float* q, float* kc, float* w) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        std::ifstream is(path, std::ios::binary);
        if (!is) throw std::runtime_error(std::string("read_sections: cannot open ") + path);
        const auto secs = csaidx::read_sections(is);
        const int64_t want[3] = {d.q_elems(), d.kc_elems(), d.w_elems()};
        float* dst[3] = {q, kc, w};
        if (secs.size() != 3) throw std::invalid_argument("read_inputs: expected 3 sections (q, kc, w)");
        for (int i = 0; i < 3; ++i) {
            if (secs[i].tag != i || static_cast<int64_t>(secs[i].data.size()) != want[i])
                throw std::invalid_argument("read_inputs: section " + std::to_string(i) + " does not match dims");
            std::memcpy(dst[i], secs[i].data.data(), secs[i].data.size() * sizeof(float));
        }
    });
}

int csaidx_host_load_inputs_device(const char* path, const csaidx_dims* dims, int64_t query_tile,
                                   const int64_t* chunk_starts, int64_t n_chunks, int dtype, int strict,
                                   int device, void* q, void* kc, float* w) {
    return guarded([&] {
        csaidx::gpu::Options o = csaidx::gpu::options();
        o.device = device;
        csaidx::gpu::set_options(o);
        std::vector<int64_t> starts;
        if (chunk_starts != nullptr && n_chunks > 0) starts.assign(chunk_starts, chunk_starts + n_chunks);
        const csaidx::ProblemDims d = from_c(dims);
        csaidx::gpu::load_inputs_device(path, d, csaidx::TileConfig{query_tile, d.key_blocks},
                                        starts.empty() ? nullptr : &starts, dtype, strict != 0, q, kc, w);
    });
}

int csaidx_host_problem_dims(int64_t batch, int64_t seq_len, int64_t ratio, int64_t heads, int64_t head_dim,
                             int64_t top_k, csaidx_dims* out) {
    return guarded([&] {
        const auto p = csaidx::ProblemDims::create(batch, seq_len, ratio, heads, head_dim, top_k);
        *out = csaidx::detail::to_c(p);
    });
}

int csaidx_host_dispatch_count_model(const csaidx_dims* dims, int64_t query_tile, int64_t key_tile, int64_t* out) {
    return guarded([&] { *out = csaidx::dispatch_count_model(from_c(dims), csaidx::TileConfig{query_tile, key_tile}); });
}

int csaidx_host_chunked_peak_model_bytes(int64_t batch, int64_t query_tile, int64_t key_tile, int64_t top_k,
                                         int bool_mask_tile, uint64_t* out) {
    return guarded([&] {
        *out = csaidx::chunked_peak_model_bytes(batch, csaidx::TileConfig{query_tile, key_tile}, top_k,
                                                bool_mask_tile != 0);
    });
}

int csaidx_host_materialize_bytes(const csaidx_dims* dims, uint64_t* out) {
    return guarded([&] {
        if (dims == nullptr) throw std::invalid_argument("null dims");
        csaidx::ProblemDims p{dims->batch, dims->seq_len, dims->key_blocks, dims->heads, dims->head_dim, dims->ratio,
                              dims->top_k};
        *out = csaidx::materialize_bytes(p);
    });
}

int csaidx_host_choose_path(const csaidx_dims* dims, uint64_t threshold, int* path, uint64_t* predicted) {
    return guarded([&] {
        const csaidx::DispatchDecision dd = csaidx::choose_path(from_c(dims), threshold);
        *path = dd.path == csaidx::ExecutionPath::materialize ? 0 : 1;
        *predicted = dd.predicted_bytes;
    });
}

int64_t csaidx_host_t_legal(int64_t t, int64_t ratio) {
    int64_t r = -1;
    guarded([&] { r = csaidx::t_legal(t, ratio); });
    return r;
}

int64_t csaidx_host_k_eff(int64_t t, int64_t ratio, int64_t top_k) {
    int64_t r = -1;
    guarded([&] { r = csaidx::k_eff(t, ratio, top_k); });
    return r;
}

int csaidx_host_round_bf16(const float* src, uint16_t* dst, uint64_t n, int* nonfinite, int* inexact) {
    return guarded([&] {
        if ((src == nullptr || dst == nullptr) && n > 0) throw std::invalid_argument("round_bf16: null buffer");
        const csaidx::detail::Bf16Flags f = csaidx::detail::host_to_bf16(src, dst, static_cast<size_t>(n));
        if (nonfinite != nullptr) *nonfinite = f.nonfinite ? 1 : 0;
        if (inexact != nullptr) *inexact = f.inexact ? 1 : 0;
    });
}

int csaidx_host_last_transfer(uint64_t* h2d_bytes, uint64_t* d2h_bytes, int64_t* fp32_chunks, int64_t* chunks) {
    return guarded([&] {
        const csaidx::detail::Transfer& t = csaidx::detail::last_transfer();
        if (h2d_bytes != nullptr) *h2d_bytes = t.h2d;
        if (d2h_bytes != nullptr) *d2h_bytes = t.d2h;
        if (fp32_chunks != nullptr) *fp32_chunks = t.fp32_chunks;
        if (chunks != nullptr) *chunks = t.chunks;
    });
}

int csaidx_host_plan_shards(const csaidx_dims* dims, int64_t query_tile, int world, int rank, int64_t* starts,
                            int64_t cap, int64_t* n_chunks, uint64_t* loads) {
    return guarded([&] {
        const csaidx::ProblemDims d = from_c(dims);
        if (n_chunks == nullptr) throw std::invalid_argument("plan_shards: null n_chunks");
        if (rank < 0 || rank >= world) throw std::invalid_argument("plan_shards: rank outside [0, world)");
        std::vector<uint64_t> ld;
        const auto plan = csaidx::gpu::plan_shards(d, query_tile, world, &ld);
        const auto& mine = plan[static_cast<size_t>(rank)];
        *n_chunks = static_cast<int64_t>(mine.size());
        if (starts != nullptr)
            for (size_t i = 0; i < mine.size() && static_cast<int64_t>(i) < cap; ++i) starts[i] = mine[i];
        if (loads != nullptr) std::memcpy(loads, ld.data(), ld.size() * sizeof(uint64_t));
    });
}

}  // extern "C"

struct csaidx_multi {
    csaidx_run_config cfg;
    csaidx::gpu::MultiRank* rank;
};

extern "C" {

int csaidx_multi_create(const csaidx_collectives* comm, const csaidx_dims* dims, const csaidx_run_config* cfg,
                        int gather_mode, int32_t* root_out, csaidx_multi** out) {
    return guarded([&] {
        if (comm == nullptr || out == nullptr) throw std::invalid_argument("multi_create: null argument");
        if (gather_mode != CSAIDX_GATHER_PEER && gather_mode != CSAIDX_GATHER_COLLECTIVE)
            throw std::invalid_argument("multi_create: unknown gather mode");
        const csaidx::ProblemDims d = from_c(dims);
        const csaidx::DriverConfig c = from_c(cfg);
        auto* m = new csaidx_multi{*cfg, nullptr};
        try {
            m->rank = new csaidx::gpu::MultiRank(*comm, d, c,
                                                 gather_mode == CSAIDX_GATHER_PEER ? csaidx::gpu::GatherMode::peer
                                                                                   : csaidx::gpu::GatherMode::collective,
                                                 root_out);
        } catch (...) {
            delete m;
            throw;
        }
        *out = m;
    });
}

int csaidx_multi_chunks(const csaidx_multi* m, const int64_t** starts, int64_t* n_chunks, int64_t* rows) {
    return guarded([&] {
        if (m == nullptr) throw std::invalid_argument("multi_chunks: null handle");
        if (starts != nullptr) *starts = m->rank->chunks().data();
        if (n_chunks != nullptr) *n_chunks = static_cast<int64_t>(m->rank->chunks().size());
        if (rows != nullptr) *rows = m->rank->rows();
    });
}

int csaidx_multi_run(csaidx_multi* m, const void* q, void* kc, int dtype, const float* w, int64_t* local_idx,
                     float* local_val, csaidx_run_stats* stats) {
    return guarded([&] {
        if (m == nullptr) throw std::invalid_argument("multi_run: null handle");
        (void)from_c(&m->cfg);  // this rank's device / stream options
        csaidx::MemoryLedger ledger;
        csaidx::RunStats rs;
        m->rank->run(q, kc, dtype, w, local_idx, local_val, ledger, &rs);
        fill_stats(stats, rs, ledger, 1);
    });
}

int csaidx_multi_destroy(csaidx_multi* m) {
    return guarded([&] {
        if (m == nullptr) return;
        delete m->rank;
        delete m;
    });
}

}  // extern "C"
