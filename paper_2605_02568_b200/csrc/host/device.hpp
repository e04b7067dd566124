// Internal plumbing of libcsaidx.so: status -> exception mapping, the
// per-device engine registry, RAII device buffers, operand staging and the
// device-side chunk scheduler shared by every driver entry point. Every GPU
// action goes through the C-ABI in include/csaidx_cuda.h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <vector>

#include "csaidx/driver.hpp"
#include "csaidx/gpu.hpp"
#include "csaidx/types.hpp"
#include "csaidx_cuda.h"

namespace csaidx::detail {

// Throws the reference exception type for a C-ABI status (no-op on OK).
void check(int rc);
[[noreturn]] void throw_status(int rc, const char* what);

// The calling thread's engine for gpu::options().device, with the configured
// stream applied (one engine per thread and device: calls from different
// threads overlap); engine_mutex() guards it within the thread's own call.
csaidx_engine* engine();
std::mutex& engine_mutex();

class DeviceBuffer {
public:
    DeviceBuffer() = default;
    DeviceBuffer(csaidx_engine* e, size_t bytes);
    DeviceBuffer(DeviceBuffer&& o) noexcept;
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    ~DeviceBuffer();

    template <class T>
    T* as() const {
        return static_cast<T*>(ptr_);
    }
    [[nodiscard]] size_t bytes() const { return bytes_; }
    void upload(const void* host, size_t bytes);
    void download(void* host, size_t bytes) const;

private:
    void reset();
    csaidx_engine* e_ = nullptr;
    void* ptr_ = nullptr;
    size_t bytes_ = 0;
};

// Fused select pre-filter: off unless CSAIDX_SELECT_PREFILTER=1. Results are
// identical either way; measured at C3 it costs more in the score epilogue
// (+15 ms: one ballot + word store per score, plus the sample pass) than it
// saves in the select (-2 ms), so it stays an A/B option. The
// sample pass scores at most kPrefilterSampleTiles 128-key tiles per row.
bool prefilter_enabled();
// SMs given to the select while it runs beside the next chunk's score kernel
// (CSAIDX_SELECT_SMS; default 0 = no overlap: each select uses the GPU;
// -1 = overlap without a partition, the select lane at top priority).
int select_overlap_sms();
// Two-level select for long rows (CSAIDX_TWO_LEVEL=1; default off).
bool two_level_enabled();
// Device score-tile budget for widening the key tile (CSAIDX_KEY_TILE_BYTES,
// default 2 GiB; 0 keeps the requested c_T).
uint64_t key_tile_budget();
constexpr int64_t kPrefilterSampleTiles = 16;

int kernel_code(ScoreKernel kernel, AccumulationMode mode);  // throws like resolve_score_kernel for unavailable kernels
int mode_code(AccumulationMode mode);
csaidx_dims to_c(const ProblemDims& d);

struct HostView {
    const float* q;
    const float* kc;
    const float* w;
    // q / w hold only the call's chunks, stacked like the output rows
    // ([B, out_rows, ...]) instead of the full [B, S, ...] tensors.
    bool local_rows = false;
};

struct DeviceOps {
    const void* q;
    const void* kc;
    const float* w;
    int dtype;  // CSAIDX_DTYPE_*
    // 0: q / w are the full [B, S, ...] tensors. > 0: rank-local stacks of
    // the plan's chunks in plan order, op_rows rows per batch (chunk c at
    // operand row plan.out_row0[c]).
    int64_t op_rows = 0;
};

// Device copies of q / kc / w. dtype bf16 stages through a bounded fp32
// slab and rounds on device; fp32 copies straight. A non-strict bf16 request
// on operands bf16 cannot hold falls back to fp32 operands (ops().dtype
// tells which), so auto_detect scores them with the exact-order kernel.
class StagedOperands {
public:
    // row_ranges (s0, rows): only these query rows of q / w are staged (all
    // when null); the device arrays keep the full [B, S, ...] layout.
    StagedOperands(csaidx_engine* e, const HostView& host, const ProblemDims& dims, int dtype, bool strict,
                   const std::vector<std::pair<int64_t, int64_t>>* row_ranges = nullptr);
    [[nodiscard]] DeviceOps ops() const { return {q_.as<void>(), kc_.as<void>(), w_.as<float>(), dtype_}; }

private:
    void stage(csaidx_engine* e, const HostView& host, const ProblemDims& dims, bool strict,
               const std::vector<std::pair<int64_t, int64_t>>* row_ranges);
    DeviceBuffer q_, kc_, w_;
    int dtype_;
};

// Operand dtype the score kernel wants for this (dims, mode, kernel).
int operand_dtype(const ProblemDims& dims, int mode, int kernel);

struct ChunkPlan {
    int64_t cs = 0;  // clamped c_S
    int64_t ct = 0;  // clamped c_T
    std::vector<int64_t> starts;
    std::vector<int64_t> out_row0;
    // Processing order (indices into starts): latest chunk first. Causal
    // work grows with s0, so with host transfers the heavy chunks' kernels
    // run while the light chunks' rows are still crossing PCIe, and the
    // step ends on cheap chunks instead of a compute tail. Results and
    // RunStats do not depend on the order.
    std::vector<size_t> order;
};

ChunkPlan plan_chunks(const ProblemDims& dims, const TileConfig& tile, const std::vector<int64_t>* starts);

// Key tile the device runs for a plan (driver.cpp): the requested c_T, or a
// multiple of it (up to T) that fits key_tile_budget() bytes of fp32 scores
// when the results cannot depend on it. RunStats and ledger charges always
// follow the requested tiles.
int64_t physical_key_tile(const ProblemDims& dims, const DriverConfig& config, const ChunkPlan& plan);

// Per-chunk callbacks around run_plan's main-lane work (used to overlap host
// transfers of neighbouring chunks on the engine's copy lanes).
struct ChunkHooks {
    std::function<void(size_t)> before;  // before the o-th processed chunk's first kernel (plan.order[o])
    std::function<void(size_t)> after;   // after its finalize
};

// process_query_tile (driver.cpp:36-106) for every chunk of the plan, on
// device. Results land in device [B, out_rows, k] int64 / fp32.
void run_plan(csaidx_engine* e, const DeviceOps& ops, const ProblemDims& dims, const DriverConfig& config,
              const ChunkPlan& plan, int64_t* out_idx, float* out_val, int64_t out_rows, MemoryLedger& ledger,
              RunStats& stats, const ChunkHooks& hooks = {});

// Materialized path on device (driver.cpp:167-192).
void run_materialize_device(csaidx_engine* e, const DeviceOps& ops, const ProblemDims& dims, int mode, int kernel,
                            int64_t* out_idx, float* out_val, MemoryLedger& ledger);

TopKResult run_chunked_view(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                            MemoryLedger& ledger, RunStats* stats);
// Host-buffer Algorithm 2 over a chunk subset (all when starts is null);
// results into host [B, out_rows, k] with the plan's row packing.
void run_chunked_rows_view(const HostView& in, const ProblemDims& dims, const DriverConfig& config,
                           const std::vector<int64_t>* starts, int64_t* host_idx, float* host_val, int64_t out_rows,
                           MemoryLedger& ledger, RunStats* stats);
TopKResult run_materialize_view(const HostView& in, const ProblemDims& dims, AccumulationMode mode,
                                MemoryLedger& ledger, ScoreKernel kernel);

void validate_dims(const ProblemDims& d);

// Host <-> device bytes of the calling thread's last host-buffer chunked
// call, and how many of its chunks crossed PCIe as fp32 (all of them unless
// q was rounded to bf16 on the host).
struct Transfer {
    uint64_t h2d = 0, d2h = 0;
    int64_t fp32_chunks = 0, chunks = 0;
};
Transfer& last_transfer();

}  // namespace csaidx::detail
