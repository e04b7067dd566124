// Query-sharded multi-GPU driver (include/csaidx/gpu.hpp MultiRank): the
// reference's threaded query-tile loop (driver.cpp:115-165) with GPUs as the
// workers. Per step: keys broadcast from rank 0 through the transport, this
// rank's chunks through the single-GPU driver (gpu::run_chunked_device), and
// the int32 index rows into rank 0's [B, S, k] buffer — stored there by the
// final select kernels over a CUDA IPC peer mapping (GatherMode::peer), or
// gathered after the compute (GatherMode::collective).
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "csaidx/gpu.hpp"
#include "device.hpp"

namespace csaidx::gpu {

namespace {

uint64_t chunk_cost(const ProblemDims& dims, int64_t cs, int64_t s0) {
    const int64_t T = dims.seq_len / dims.ratio;
    const int64_t end = std::min(s0 + cs, dims.seq_len);
    uint64_t c = 0;
    for (int64_t t = s0; t < end; ++t) c += static_cast<uint64_t>(std::min((t + 1) / dims.ratio, T));
    return c;
}

void comm_check(int rc, const char* what) {
    if (rc != CSAIDX_OK) {
        const char* msg = csaidx_cuda_last_error();
        detail::throw_status(rc, (std::string(what) + ": " + (msg != nullptr && *msg ? msg : "transport error")).c_str());
    }
}

}  // namespace

std::vector<std::vector<int64_t>> plan_shards(const ProblemDims& dims, int64_t query_tile, int world,
                                              std::vector<uint64_t>* loads) {
    if (world < 1) throw std::invalid_argument("plan_shards: world must be >= 1");
    if (query_tile < 1) throw std::invalid_argument("plan_shards: query_tile must be >= 1");
    const int64_t cs = std::min(query_tile, dims.seq_len);
    std::vector<std::pair<uint64_t, int64_t>> cost;
    for (int64_t s0 = 0; s0 < dims.seq_len; s0 += cs) cost.emplace_back(chunk_cost(dims, cs, s0), s0);
    std::sort(cost.begin(), cost.end(), [](const auto& a, const auto& b) { return a > b; });
    std::vector<uint64_t> load(static_cast<size_t>(world), 0);
    std::vector<std::vector<int64_t>> owned(static_cast<size_t>(world));
    for (const auto& [c, s0] : cost) {
        size_t r = 0;
        for (size_t i = 1; i < load.size(); ++i)
            if (load[i] < load[r]) r = i;
        load[r] += c;
        owned[r].push_back(s0);
    }
    for (auto& o : owned) std::sort(o.begin(), o.end());
    if (loads != nullptr) *loads = load;
    return owned;
}

struct MultiRank::Impl {
    csaidx_engine* e = nullptr;
    int32_t* root_out = nullptr;
    int32_t* peer = nullptr;  // rank 0's buffer as this rank sees it
    bool opened = false;      // peer came from csaidx_cuda_ipc_open
    uint64_t peer_off = 0;
    uint8_t handle[64] = {};
    detail::DeviceBuffer own_idx, own_val;  // outputs when the caller passes none
    detail::DeviceBuffer send32, recv32, row_map;  // collective gather
    std::vector<size_t> recv_bytes, recv_off;
};

MultiRank::MultiRank(const csaidx_collectives& comm, const ProblemDims& dims, const DriverConfig& config,
                     GatherMode mode, int32_t* root_out)
    : impl_(new Impl()), comm_(comm), dims_(dims), config_(config), mode_(mode), rank_(comm.rank),
      world_(comm.world) {
    try {
        detail::validate_dims(dims);
        if (world_ < 1 || rank_ < 0 || rank_ >= world_) throw std::invalid_argument("MultiRank: bad rank / world");
        if (comm.allgather_host == nullptr || comm.barrier == nullptr || comm.bcast == nullptr)
            throw std::invalid_argument("MultiRank: transport lacks bcast / allgather_host / barrier");
        if (mode == GatherMode::collective && comm.gatherv == nullptr)
            throw std::invalid_argument("MultiRank: collective gather needs the transport's gatherv");
        if (rank_ == 0 && root_out == nullptr) throw std::invalid_argument("MultiRank: rank 0 needs root_out");
        if (dims.key_blocks >= (int64_t{1} << 31)) throw std::invalid_argument("MultiRank: int32 index rows need T < 2^31");
        plan_ = plan_shards(dims, config.tile.query_tile, world_);
        const int64_t cs = std::min(config.tile.query_tile, dims.seq_len);
        for (const auto& sh : plan_) {
            int64_t r = 0;
            for (int64_t s0 : sh) r += std::min(cs, dims.seq_len - s0);
            rows_.push_back(r);
        }
        std::lock_guard<std::mutex> lock(detail::engine_mutex());
        Impl& m = *impl_;
        m.e = detail::engine();
        m.root_out = rank_ == 0 ? root_out : nullptr;
        const int64_t B = dims.batch, k = dims.top_k;
        if (mode == GatherMode::peer) {
            if (world_ == 1) {
                m.peer = root_out;
            } else {
                // rank 0's IPC handle to every rank (72-byte blobs)
                uint8_t blob[72] = {};
                if (rank_ == 0) {
                    uint64_t off = 0;
                    detail::check(csaidx_cuda_ipc_handle(m.e, root_out, blob, &off));
                    std::memcpy(blob + 64, &off, 8);
                }
                std::vector<uint8_t> all(72 * static_cast<size_t>(world_));
                comm_check(comm.allgather_host(comm.ctx, blob, all.data(), 72), "allgather (IPC handle)");
                if (rank_ == 0) {
                    m.peer = root_out;
                } else {
                    std::memcpy(m.handle, all.data(), 64);
                    std::memcpy(&m.peer_off, all.data() + 64, 8);
                    void* p = nullptr;
                    detail::check(csaidx_cuda_ipc_open(m.e, m.handle, m.peer_off, &p));
                    m.peer = static_cast<int32_t*>(p);
                    m.opened = true;
                }
            }
        } else {
            // packed [B, rows_r, k] int32 per rank, concatenated by rank on rank 0
            m.send32 = detail::DeviceBuffer(m.e, static_cast<size_t>(B * rows() * k) * sizeof(int32_t));
            size_t off = 0;
            for (int r = 0; r < world_; ++r) {
                const size_t bytes = static_cast<size_t>(B * rows_[static_cast<size_t>(r)] * k) * sizeof(int32_t);
                m.recv_bytes.push_back(bytes);
                m.recv_off.push_back(off);
                off += bytes;
            }
            if (rank_ == 0) {
                m.recv32 = detail::DeviceBuffer(m.e, off);
                std::vector<int64_t> map;  // packed row -> row of the [B, S] result
                for (int r = 0; r < world_; ++r)
                    for (int64_t b = 0; b < B; ++b)
                        for (int64_t s0 : plan_[static_cast<size_t>(r)])
                            for (int64_t t = s0; t < std::min(s0 + cs, dims.seq_len); ++t)
                                map.push_back(b * dims.seq_len + t);
                m.row_map = detail::DeviceBuffer(m.e, map.size() * sizeof(int64_t));
                m.row_map.upload(map.data(), map.size() * sizeof(int64_t));
            }
        }
    } catch (...) {
        if (impl_->opened) csaidx_cuda_ipc_close(impl_->e, impl_->peer, impl_->peer_off);
        delete impl_;
        throw;
    }
}

MultiRank::~MultiRank() {
    std::lock_guard<std::mutex> lock(detail::engine_mutex());
    if (impl_->opened) csaidx_cuda_ipc_close(impl_->e, impl_->peer, impl_->peer_off);
    delete impl_;
}

void MultiRank::run(const void* q, void* kc, int dtype, const float* w, int64_t* local_idx, float* local_val,
                    MemoryLedger& ledger, RunStats* stats) {
    Impl& m = *impl_;
    const int64_t B = dims_.batch, k = dims_.top_k, n_out = B * rows() * k;
    if (mode_ == GatherMode::peer && local_idx == nullptr && local_val == nullptr) {
        // the rows' only copy is the int32 one in rank 0's buffer: the final
        // kernels skip the local int64 / fp32 rows (less HBM, fewer writes)
    } else if (local_idx == nullptr || local_val == nullptr) {
        std::lock_guard<std::mutex> lock(detail::engine_mutex());
        if (m.own_idx.bytes() < static_cast<size_t>(n_out) * 8) {
            m.own_idx = detail::DeviceBuffer(m.e, static_cast<size_t>(n_out) * 8);
            m.own_val = detail::DeviceBuffer(m.e, static_cast<size_t>(n_out) * 4);
        }
        if (local_idx == nullptr) local_idx = m.own_idx.as<int64_t>();
        if (local_val == nullptr) local_val = m.own_val.as<float>();
    }
    void* stream = nullptr;
    detail::check(csaidx_engine_get_stream(m.e, &stream));
    // 1. the keys, once, from rank 0
    if (world_ > 1) {
        const size_t kbytes = static_cast<size_t>(dims_.kc_elems()) * (dtype == CSAIDX_DTYPE_BF16 ? 2 : 4);
        if (comm_.device_buffers) {
            std::lock_guard<std::mutex> lock(detail::engine_mutex());
            detail::check(csaidx_engine_await_stream(m.e, nullptr));  // kc produced on the default stream
            comm_check(comm_.bcast(comm_.ctx, kc, kbytes, 0, stream), "bcast (keys)");
        } else {
            std::vector<uint8_t> h(kbytes);
            {
                std::lock_guard<std::mutex> lock(detail::engine_mutex());
                detail::check(csaidx_engine_await_stream(m.e, nullptr));
                if (rank_ == 0) {
                    detail::check(csaidx_cuda_copy(m.e, h.data(), kc, kbytes));
                    detail::check(csaidx_engine_sync(m.e));
                }
            }
            comm_check(comm_.bcast(comm_.ctx, h.data(), kbytes, 0, nullptr), "bcast (keys)");
            if (rank_ != 0) {
                std::lock_guard<std::mutex> lock(detail::engine_mutex());
                detail::check(csaidx_cuda_copy(m.e, kc, h.data(), kbytes));
                detail::check(csaidx_engine_sync(m.e));
            }
        }
    }
    // 2. this rank's chunks; with the peer gather the final kernels also
    //    store each row's int32 indices at its sequence position in rank 0's
    //    buffer (the sink is set for this call only)
    struct SinkScope {
        csaidx_engine* e;
        bool on;
        ~SinkScope() {
            if (on) {
                std::lock_guard<std::mutex> lock(detail::engine_mutex());
                csaidx_engine_set_index_sink(e, nullptr, 0, 0, 0);
            }
        }
    } sink{m.e, false};
    if (mode_ == GatherMode::peer) {
        std::lock_guard<std::mutex> lock(detail::engine_mutex());
        detail::check(csaidx_engine_set_index_sink(m.e, m.peer, B, dims_.seq_len, k));
        sink.on = true;
    }
    DeviceOperands ops;
    ops.q = q;
    ops.kc = kc;
    ops.w = w;
    ops.dtype = dtype;
    ops.local_rows = true;
    run_chunked_device(ops, dims_, config_, &chunks(), local_idx, local_val, rows(), ledger, stats);
    // 3. the collective gather of the int32 rows
    if (mode_ == GatherMode::collective) {
        std::lock_guard<std::mutex> lock(detail::engine_mutex());
        detail::check(csaidx_cuda_narrow_indices(m.e, local_idx, m.send32.as<int32_t>(), n_out));
        const size_t send_bytes = static_cast<size_t>(n_out) * sizeof(int32_t);
        if (comm_.device_buffers) {
            comm_check(comm_.gatherv(comm_.ctx, m.send32.as<void>(), send_bytes, rank_ == 0 ? m.recv32.as<void>() : nullptr,
                                     m.recv_bytes.data(), m.recv_off.data(), 0, stream),
                       "gatherv (index rows)");
        } else {
            std::vector<uint8_t> hs(send_bytes), hr(rank_ == 0 ? m.recv32.bytes() : 0);
            detail::check(csaidx_cuda_copy(m.e, hs.data(), m.send32.as<void>(), send_bytes));
            detail::check(csaidx_engine_sync(m.e));
            comm_check(comm_.gatherv(comm_.ctx, hs.data(), send_bytes, rank_ == 0 ? hr.data() : nullptr,
                                     m.recv_bytes.data(), m.recv_off.data(), 0, nullptr),
                       "gatherv (index rows)");
            if (rank_ == 0) detail::check(csaidx_cuda_copy(m.e, m.recv32.as<void>(), hr.data(), hr.size()));
        }
        if (rank_ == 0) {
            int64_t total_rows = 0;
            for (int64_t r : rows_) total_rows += r;
            detail::check(csaidx_cuda_scatter_rows(m.e, m.recv32.as<int32_t>(), m.root_out, m.row_map.as<int64_t>(),
                                                   B * total_rows, k));
        }
    }
    // 4. every rank's rows are in rank 0's buffer once all ranks pass here
    comm_check(comm_.barrier(comm_.ctx, stream), "barrier");
}

}  // namespace csaidx::gpu
