// Engine registry, error mapping, device buffers and operand staging.
#include "device.hpp"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>

namespace csaidx {
namespace gpu {

namespace {
// The process default (the last set_options of any thread) and the calling
// thread's own setting: C-ABI entry points set the options of the thread
// that calls them, so threads driving different devices / streams do not
// see each other's.
std::mutex g_opt_mu;
Options g_options;
thread_local bool t_opt_set = false;
thread_local Options t_options;
}  // namespace

void set_options(const Options& o) {
    {
        std::lock_guard<std::mutex> lock(g_opt_mu);
        g_options = o;
    }
    t_options = o;
    t_opt_set = true;
}

Options options() {
    if (t_opt_set) return t_options;
    std::lock_guard<std::mutex> lock(g_opt_mu);
    return g_options;
}

DeviceMemory device_memory() {
    DeviceMemory m;
    detail::check(csaidx_engine_mem_stats(detail::engine(), &m.live_bytes, &m.peak_bytes));
    return m;
}

void reset_device_peak() { detail::check(csaidx_engine_reset_peak(detail::engine())); }

void sparse_attention(const void* q, const void* kv, const int32_t* indices, int64_t batch, int64_t seq_len,
                      int64_t kv_len, int64_t heads, int64_t k, int64_t idx_ld, float sm_scale, void* out,
                      float* lse) {
    detail::check(csaidx_cuda_sparse_attention(detail::engine(), q, kv, indices, batch, seq_len, kv_len, heads, 576,
                                               512, k, idx_ld, sm_scale, out, 512, lse));
}

}  // namespace gpu

namespace detail {

void throw_status(int rc, const char* what) {
    switch (rc) {
        case CSAIDX_INVALID_ARGUMENT: throw std::invalid_argument(what);
        case CSAIDX_OVERFLOW_ERROR: throw std::overflow_error(what);
        case CSAIDX_LOGIC_ERROR: throw std::logic_error(what);
        case CSAIDX_RUNTIME_ERROR:
        case CSAIDX_CUDA_ERROR:
        default: throw std::runtime_error(what);
    }
}

void check(int rc) {
    if (rc != CSAIDX_OK) throw_status(rc, csaidx_cuda_last_error());
}

// One engine per (thread, device): its own stream, lanes, latched flags and
// scratch, so API calls from different threads run concurrently (each on its
// thread's stream) instead of serialising on one process-wide engine. The
// mutex guards a thread's engine against the helper threads of its own call.
std::mutex& engine_mutex() {
    thread_local std::mutex mu;
    return mu;
}

csaidx_engine* engine() {
    // intentionally never destroyed (CUDA teardown order at process exit)
    thread_local std::map<int, csaidx_engine*> engines;
    const gpu::Options o = gpu::options();
    auto it = engines.find(o.device);
    if (it == engines.end()) {
        csaidx_engine* e = nullptr;
        check(csaidx_engine_create(o.device, &e));
        it = engines.emplace(o.device, e).first;
    }
    if (o.stream != nullptr)
        check(csaidx_engine_set_stream(it->second, o.stream));
    else
        check(csaidx_engine_use_own_stream(it->second));
    return it->second;
}

DeviceBuffer::DeviceBuffer(csaidx_engine* e, size_t bytes) : e_(e), bytes_(bytes) {
    check(csaidx_cuda_alloc(e, bytes, &ptr_));
}

DeviceBuffer::DeviceBuffer(DeviceBuffer&& o) noexcept : e_(o.e_), ptr_(o.ptr_), bytes_(o.bytes_) {
    o.ptr_ = nullptr;
    o.bytes_ = 0;
}

DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
        reset();
        e_ = o.e_;
        ptr_ = o.ptr_;
        bytes_ = o.bytes_;
        o.ptr_ = nullptr;
        o.bytes_ = 0;
    }
    return *this;
}

DeviceBuffer::~DeviceBuffer() { reset(); }

void DeviceBuffer::reset() {
    if (ptr_ != nullptr) csaidx_cuda_free(e_, ptr_);
    ptr_ = nullptr;
    bytes_ = 0;
}

void DeviceBuffer::upload(const void* host, size_t bytes) { check(csaidx_cuda_copy(e_, ptr_, host, bytes)); }

void DeviceBuffer::download(void* host, size_t bytes) const { check(csaidx_cuda_copy(e_, host, ptr_, bytes)); }

bool two_level_enabled() {
    // Off by default (CSAIDX_TWO_LEVEL=1 enables): at C4 the select drops
    // 22.0 -> 14.9 ms but the group-max epilogue costs the score kernel
    // 206 -> 216.5 ms (profiles/r01_ncu_history.md).
    const char* v = std::getenv("CSAIDX_TWO_LEVEL");
    return v != nullptr && std::string(v) == "1";
}

int select_overlap_sms() {
    // Off by default: measured slower at C3 (profiles/r01_ncu_history.md) —
    // the score kernel loses more than the SMs it gives up once a select
    // runs beside it (shared power cap and HBM), and the select on a few
    // SMs does not get faster per SM.
    const char* v = std::getenv("CSAIDX_SELECT_SMS");
    return v != nullptr ? std::atoi(v) : 0;
}

uint64_t key_tile_budget() {
    const char* v = std::getenv("CSAIDX_KEY_TILE_BYTES");
    return v != nullptr ? std::strtoull(v, nullptr, 10) : (uint64_t{2} << 30);
}

bool prefilter_enabled() {
    const char* v = std::getenv("CSAIDX_SELECT_PREFILTER");
    return v != nullptr && std::string(v) == "1";
}

int kernel_code(ScoreKernel kernel, AccumulationMode mode) {
    switch (kernel) {
        case ScoreKernel::auto_detect:
            // fp16_emulated stays on the bit-exact kernel unless the caller
            // opts into the tensor-core form (gpu::Options::fp16_tensor_cores)
            return mode == AccumulationMode::fp16_emulated && gpu::options().fp16_tensor_cores ? CSAIDX_KERNEL_TENSOR
                                                                                                : CSAIDX_KERNEL_AUTO;
        case ScoreKernel::scalar: return CSAIDX_KERNEL_EXACT;
        case ScoreKernel::avx2:
            throw std::invalid_argument("avx2 kernel requested but this build has no AVX2 kernel (B200 path)");
    }
    throw std::invalid_argument("unknown score kernel");
}

int mode_code(AccumulationMode mode) {
    return mode == AccumulationMode::fp16_emulated ? CSAIDX_MODE_FP16_EMULATED : CSAIDX_MODE_FP32;
}

csaidx_dims to_c(const ProblemDims& d) {
    return csaidx_dims{d.batch, d.seq_len, d.key_blocks, d.heads, d.head_dim, d.ratio, d.top_k};
}

void validate_dims(const ProblemDims& d) {
    if (d.batch < 1 || d.seq_len < 1 || d.key_blocks < 1 || d.heads < 1 || d.head_dim < 1 || d.ratio < 1 ||
        d.top_k < 1)
        throw std::invalid_argument("ProblemDims: every extent must be >= 1");
}

int operand_dtype(const ProblemDims& dims, int mode, int kernel) {
    const csaidx_dims c = to_c(dims);
    return csaidx_cuda_score_uses_tensor_cores(&c, CSAIDX_DTYPE_BF16, mode, kernel) ? CSAIDX_DTYPE_BF16
                                                                                    : CSAIDX_DTYPE_F32;
}

namespace {

// fp32 host -> device, rounded to bf16 on device through a bounded slab.
void stage_bf16(csaidx_engine* e, DeviceBuffer& dst, int64_t dst_off, const float* host, int64_t n, bool strict) {
    constexpr int64_t kSlab = int64_t{1} << 26;  // 64 Mi elements (256 MiB fp32)
    if (n <= 0) return;
    DeviceBuffer slab(e, static_cast<size_t>(std::min(n, kSlab)) * sizeof(float));
    for (int64_t off = 0; off < n; off += kSlab) {
        const int64_t len = std::min(kSlab, n - off);
        check(csaidx_cuda_copy(e, slab.as<void>(), host + off, static_cast<size_t>(len) * sizeof(float)));
        check(csaidx_cuda_to_bf16(e, slab.as<float>(), dst.as<uint16_t>() + dst_off + off, len, strict ? 1 : 0));
    }
}

}  // namespace

StagedOperands::StagedOperands(csaidx_engine* e, const HostView& host, const ProblemDims& dims, int dtype,
                               bool strict, const std::vector<std::pair<int64_t, int64_t>>* row_ranges)
    : dtype_(dtype) {
    stage(e, host, dims, strict, row_ranges);
    if (dtype_ == CSAIDX_DTYPE_BF16 && !strict) {
        // auto_detect on operands bf16 cannot hold: the exact-order kernel on
        // fp32 operands (the reference's auto scores any fp32 input exactly)
        int seen = 0;
        check(csaidx_engine_take_inexact(e, &seen));
        if (seen) {
            dtype_ = CSAIDX_DTYPE_F32;
            stage(e, host, dims, strict, row_ranges);
        }
    }
}

void StagedOperands::stage(csaidx_engine* e, const HostView& host, const ProblemDims& dims, bool strict,
                           const std::vector<std::pair<int64_t, int64_t>>* row_ranges) {
    const int dtype = dtype_;
    const int64_t nq = dims.q_elems(), nk = dims.kc_elems(), nw = dims.w_elems();
    const size_t esz = dtype == CSAIDX_DTYPE_BF16 ? 2 : 4;
    q_ = DeviceBuffer(e, static_cast<size_t>(nq) * esz);
    kc_ = DeviceBuffer(e, static_cast<size_t>(nk) * esz);
    w_ = DeviceBuffer(e, static_cast<size_t>(nw) * sizeof(float));
    if (dtype == CSAIDX_DTYPE_BF16) {
        stage_bf16(e, kc_, 0, host.kc, nk, strict);
    } else {
        kc_.upload(host.kc, static_cast<size_t>(nk) * sizeof(float));
    }
    std::vector<std::pair<int64_t, int64_t>> all{{0, dims.seq_len}};
    const auto& ranges = row_ranges != nullptr ? *row_ranges : all;
    const int64_t qrow = dims.heads * dims.head_dim;
    for (int64_t b = 0; b < dims.batch; ++b) {
        for (const auto& [s0, rows] : ranges) {
            const int64_t qoff = (b * dims.seq_len + s0) * qrow, woff = (b * dims.seq_len + s0) * dims.heads;
            if (dtype == CSAIDX_DTYPE_BF16) {
                stage_bf16(e, q_, qoff, host.q + qoff, rows * qrow, strict);
            } else {
                check(csaidx_cuda_copy(e, q_.as<float>() + qoff, host.q + qoff,
                                       static_cast<size_t>(rows * qrow) * sizeof(float)));
            }
            check(csaidx_cuda_copy(e, w_.as<float>() + woff, host.w + woff,
                                   static_cast<size_t>(rows * dims.heads) * sizeof(float)));
        }
    }
}

}  // namespace detail
}  // namespace csaidx
