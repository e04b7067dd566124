// GPU-only knobs and device-resident entry points of the B200 build. Not part
// of the reference API (the reference structs in driver.hpp / types.hpp are
// left untouched); everything here is additive.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "csaidx/driver.hpp"
#include "csaidx/memory_ledger.hpp"
#include "csaidx/types.hpp"
#include "csaidx_cuda.h"

namespace csaidx::gpu {

struct Options {
    int device = 0;            // CUDA ordinal used by the host-API entry points
    bool strict_bf16 = false;  // reject q / kc values that are not bf16-representable
    void* stream = nullptr;    // cudaStream_t to enqueue on; nullptr = engine's own stream
    // AccumulationMode::fp16_emulated with ScoreKernel::auto_detect on the V4
    // shape runs on the tensor cores (the reference's binary16 rounding points
    // applied to the MMA's dot products: agreement to binary16 rounding, not
    // bit for bit; the default keeps the bit-exact CUDA-core kernel)
    bool fp16_tensor_cores = false;
};

// Options of the calling thread (and the default of threads that never set
// their own). Each thread drives its own engine per device, so calls from
// several threads run concurrently on their own streams.
void set_options(const Options& options);
Options options();

// Device bytes held by the driver's allocations (live) and their high-water
// mark since the last reset, for the calling thread's device.
struct DeviceMemory {
    uint64_t live_bytes = 0;
    uint64_t peak_bytes = 0;
};
DeviceMemory device_memory();
void reset_device_peak();

// Operands already resident in HBM. dtype: 0 = bf16 (tensor-core path),
// 1 = fp32 (exact-order path).
struct DeviceOperands {
    const void* q = nullptr;   // [B, S, H_I, d_h]  (local_rows: [B, out_rows, H_I, d_h])
    const void* kc = nullptr;  // [B, T, d_h]
    const float* w = nullptr;  // [B, S, H_I]        (local_rows: [B, out_rows, H_I])
    int dtype = 0;
    // Query-sharded ranks: q / w hold only the listed chunks' rows, stacked
    // in list order exactly like the output rows (chunk c at row row0_c).
    bool local_rows = false;
};

// Device-resident Algorithm 2 over a subset of query chunks (all chunks when
// chunk_starts is null). Chunk starts must be multiples of the clamped c_S;
// chunk c of the list writes its rows to out rows [row0_c, row0_c + rows_c)
// where row0 accumulates over the list. Outputs are device [B, out_rows, k];
// both may be null while an index sink is set on the driver's engine
// (csaidx_engine_set_index_sink): the sink then receives the only copy.
void run_chunked_device(const DeviceOperands& ops, const ProblemDims& dims,
                        const DriverConfig& config, const std::vector<int64_t>* chunk_starts,
                        int64_t* out_indices, float* out_values, int64_t out_rows,
                        MemoryLedger& ledger, RunStats* stats = nullptr);

// Streams a CSAT input dump (tensor_io.hpp) into caller-owned device
// buffers: q / kc as dtype (CSAIDX_DTYPE_BF16: rounded to bf16 on device,
// strict rejects non-representable values; CSAIDX_DTYPE_F32: as stored),
// w as fp32. With chunk_starts only those query chunks' q / w rows are read,
// stacked like the output rows ([B, out_rows, ...], the local_rows layout);
// kc is always whole. Throws runtime_error on a malformed file (the
// reference's read_sections cases) and invalid_argument when the sections
// do not match dims.
void load_inputs_device(const std::string& path, const ProblemDims& dims, const TileConfig& tile,
                        const std::vector<int64_t>* chunk_starts, int dtype, bool strict, void* q, void* kc,
                        float* w);

// ------------------------------------------------------------ downstream
// The consumer of the index list (the attention step the
// reference leaves out): sparse MLA-style attention
// of `heads` (a multiple of 128) query heads over the rows indices[b, t, 0:k]
// of one shared latent KV head (576 dims, values = the first 512), on the
// calling thread's engine and stream. Device pointers: q bf16 [B, S, heads,
// 576], kv bf16 [B, kv_len, 576], indices int32 [B, S, idx_ld] (-1 / out of
// range = skipped), out bf16 [B, S, heads, 512], lse fp32 [B, S, heads] or
// null. Throws invalid_argument for other shapes (csaidx_cuda_sparse_attention).
void sparse_attention(const void* q, const void* kv, const int32_t* indices, int64_t batch, int64_t seq_len,
                      int64_t kv_len, int64_t heads, int64_t k, int64_t idx_ld, float sm_scale, void* out,
                      float* lse);

// ------------------------------------------------------------ multi-GPU
// Query-sharded driver, one process (rank) per GPU. The reference runs the
// same query-tile loop on `DriverConfig::threads` host workers over
// contiguous blocks of tiles (driver.cpp:115-165); here the workers are GPUs,
// the chunks are dealt by causal work (LPT), and the only exchanges are the
// ones north_star names: the keys are broadcast once from rank 0 and only
// the [B, S, k] int32 index rows travel back to rank 0.

// LPT assignment of the c_S query chunks by causal work (cost of a chunk =
// its legal (query, key) pairs, B-independent): chunks in decreasing cost
// (ties: later chunk first), each to the least-loaded rank (ties: lowest
// rank). Returns per-rank ascending chunk starts; loads = per-rank cost.
std::vector<std::vector<int64_t>> plan_shards(const ProblemDims& dims, int64_t query_tile, int world,
                                              std::vector<uint64_t>* loads = nullptr);

enum class GatherMode {
    peer = 0,        // final select/finalize kernels store rows into rank 0's buffer (CUDA IPC over NVLink)
    collective = 1,  // rows gathered after the compute through the transport's gatherv
};

// One rank of a query-sharded run: the plan, the peer mapping of rank 0's
// result buffer (set up once), and the per-step exchange. The transport
// (include/csaidx_cuda.h csaidx_collectives: NCCL, or a caller's own) must
// outlive the object.
class MultiRank {
public:
    // root_out: rank 0's device [B, S, k] int32 result (ignored elsewhere).
    MultiRank(const csaidx_collectives& comm, const ProblemDims& dims, const DriverConfig& config, GatherMode mode,
              int32_t* root_out);
    ~MultiRank();
    MultiRank(const MultiRank&) = delete;
    MultiRank& operator=(const MultiRank&) = delete;

    const std::vector<int64_t>& chunks() const { return plan_[static_cast<size_t>(rank_)]; }
    int64_t rows() const { return rows_[static_cast<size_t>(rank_)]; }  // this rank's rows per batch

    // One step. q / w: this rank's rows (DeviceOperands::local_rows layout,
    // chunks() order); kc: [B, T, d_h] on every rank, read on rank 0 and
    // overwritten by the broadcast elsewhere. local_idx / local_val: this
    // rank's [B, rows(), k] outputs; both null with the peer gather: rank
    // 0's int32 rows are the only output (the final kernels write nothing
    // else), with the collective gather: kept inside. On return the step is
    // complete on every rank and rank 0's root_out holds all rows.
    void run(const void* q, void* kc, int dtype, const float* w, int64_t* local_idx, float* local_val,
             MemoryLedger& ledger, RunStats* stats = nullptr);

private:
    struct Impl;
    Impl* impl_;
    csaidx_collectives comm_;
    ProblemDims dims_;
    DriverConfig config_;
    GatherMode mode_;
    int rank_, world_;
    std::vector<std::vector<int64_t>> plan_;
    std::vector<int64_t> rows_;
};

}  // namespace csaidx::gpu
