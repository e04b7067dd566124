// C-ABI implementation (include/csaidx_cuda.h). Argument validation mirrors
// the reference's checks so the C++ layer can rethrow the same exception
// types; kernels are enqueued on the engine stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "csaidx_cuda.h"
#include "kernels/kernels.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list args;
    va_start(args, fmt);
    vsnprintf(buf, sizeof(buf), fmt, args);
    va_end(args);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t err, const char* where) {
    return fail(CSAIDX_CUDA_ERROR, "%s: CUDA error %s (%s)", where, cudaGetErrorName(err),
                cudaGetErrorString(err));
}

#define CSAIDX_CUDA_TRY(expr, where)                 \
    do {                                             \
        cudaError_t _e = (expr);                     \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

// kInexactSeen: a non-strict bf16 staging met a value bf16 cannot hold (not
// an error: the host driver then re-runs on fp32 operands with the exact
// kernel, csaidx_engine_take_inexact)
enum Flag {
    kNonfiniteScore = 0,
    kInexact = 1,
    kNonfiniteInput = 2,
    kTrail = 3,
    kKeff = 4,
    kOverlap = 5,
    kInexactSeen = 6,
    kNumFlags = 8
};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
        }
    });
    return fn;
}

using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

// cuMemGetAddressRange: the base of the allocation holding a pointer (CUDA
// IPC maps whole allocations; a caching allocator's block may sit at an
// offset inside one).
AddressRangeFn get_range_fn() {
    static AddressRangeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) {
            fn = reinterpret_cast<AddressRangeFn>(ptr);
        }
    });
    return fn;
}

}  // namespace

struct csaidx_engine {
    int device = 0;
    int num_sms = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    int* flags = nullptr;  // device [kNumFlags]
    std::mutex mu;
    std::unordered_map<void*, size_t> sizes;
    uint64_t live = 0;
    uint64_t peak = 0;
    // per-kernel-class accounting (CSAIDX_KIND_*)
    int64_t launches[CSAIDX_NUM_KINDS] = {};
    double total_ms[CSAIDX_NUM_KINDS] = {};
    bool profiling = false;
    struct Pending {
        int kind;
        cudaEvent_t start, stop;
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    // copy lanes for overlapping host transfers with compute (created lazily)
    cudaStream_t lanes[4] = {nullptr, nullptr, nullptr, nullptr};  // [0] = main (== stream when lane 0 active)
    cudaStream_t main_stream = nullptr;
    int lane = 0;
    cudaEvent_t slots[192] = {};
    cudaEvent_t entry_event = nullptr;  // csaidx_engine_await_stream
    int32_t* sink = nullptr;            // csaidx_engine_set_index_sink
    int64_t sink_batch = 0, sink_seq = 0, sink_k = 0;
    // global scratch of the large-take select / merge (k > 4096), grown on
    // demand and counted in live / peak
    void* large = nullptr;
    size_t large_bytes = 0;
    // SM partition while a select runs beside the score kernel (0 = whole GPU)
    int score_sms = 0;
    int select_sms = 0;
    long long* select_probe = nullptr;  // optional per-row phase clocks (profiling)
    long long* score_probe = nullptr;   // optional per-CTA wait counters (profiling)
};

namespace {

int set_device(csaidx_engine* e) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    CSAIDX_CUDA_TRY(cudaSetDevice(e->device), "cudaSetDevice");
    return CSAIDX_OK;
}

cudaEvent_t take_event(csaidx_engine* e) {
    if (!e->event_pool.empty()) {
        cudaEvent_t ev = e->event_pool.back();
        e->event_pool.pop_back();
        return ev;
    }
    cudaEvent_t ev = nullptr;
    cudaEventCreate(&ev);
    return ev;
}

// Brackets one kernel launch: counts it and, when profiling, records CUDA
// events on the launching stream (resolved lazily by kernel_stats).
struct LaunchScope {
    csaidx_engine* e;
    int kind;
    cudaEvent_t start = nullptr;
    LaunchScope(csaidx_engine* e_, int kind_) : e(e_), kind(kind_) {
        ++e->launches[kind];
        if (e->profiling) {
            start = take_event(e);
            cudaEventRecord(start, e->stream);
        }
    }
    ~LaunchScope() {
        if (start != nullptr) {
            cudaEvent_t stop = take_event(e);
            cudaEventRecord(stop, e->stream);
            e->pending.push_back({kind, start, stop});
        }
    }
};

// 2D bf16 row-major [rows, 128] tensor map with a (64 x box_rows) SW128 box.
int make_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (enc == nullptr) return fail(CSAIDX_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {64, box_rows};
    const cuuint32_t estride[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estride,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CSAIDX_CUDA_ERROR, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return CSAIDX_OK;
}

int check_dims(const csaidx_dims* d) {
    if (d == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null dims");
    if (d->batch < 1 || d->seq_len < 1 || d->key_blocks < 1 || d->heads < 1 || d->head_dim < 1 || d->ratio < 1 ||
        d->top_k < 1)
        return fail(CSAIDX_INVALID_ARGUMENT, "dims: every extent must be >= 1");
    return CSAIDX_OK;
}

}  // namespace

extern "C" {

const char* csaidx_cuda_last_error(void) { return g_last_error.c_str(); }

int csaidx_cuda_abi_version(void) { return 1; }

int csaidx_cuda_device_count(int* count) {
    if (count == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null count");
    cudaError_t err = cudaGetDeviceCount(count);
    if (err != cudaSuccess) {
        *count = 0;
        cudaGetLastError();
    }
    return CSAIDX_OK;
}

int csaidx_engine_create(int device, csaidx_engine** out) {
    if (out == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null out");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(CSAIDX_CUDA_ERROR, "no CUDA device available (the B200 indexer has no CPU path)");
    }
    if (device < 0 || device >= count) return fail(CSAIDX_INVALID_ARGUMENT, "device ordinal %d out of range", device);
    auto* e = new csaidx_engine();
    e->device = device;
    CSAIDX_CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    CSAIDX_CUDA_TRY(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) {
        delete e;
        return fail(CSAIDX_CUDA_ERROR, "device %d is sm_%d%d; this build targets sm_100a only", device, prop.major,
                    prop.minor);
    }
    e->num_sms = prop.multiProcessorCount;
    CSAIDX_CUDA_TRY(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    e->stream = e->own_stream;
    e->main_stream = e->stream;
    // flags [0, kNumFlags) + the score kernel's self-resetting work counters
    CSAIDX_CUDA_TRY(cudaMalloc(&e->flags, 2 * kNumFlags * sizeof(int)), "cudaMalloc(flags)");
    CSAIDX_CUDA_TRY(cudaMemset(e->flags, 0, 2 * kNumFlags * sizeof(int)), "cudaMemset(flags)");
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thresh = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh);
    }
    *out = e;
    return CSAIDX_OK;
}

int csaidx_engine_destroy(csaidx_engine* e) {
    if (e == nullptr) return CSAIDX_OK;
    cudaSetDevice(e->device);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (auto& kv : e->sizes) cudaFree(kv.first);
    for (const auto& pd : e->pending) {
        cudaEventDestroy(pd.start);
        cudaEventDestroy(pd.stop);
    }
    for (cudaEvent_t ev : e->event_pool) cudaEventDestroy(ev);
    if (e->flags) cudaFree(e->flags);
    if (e->large) cudaFree(e->large);
    for (int i = 1; i < 4; ++i)
        if (e->lanes[i]) cudaStreamDestroy(e->lanes[i]);
    for (cudaEvent_t ev : e->slots)
        if (ev) cudaEventDestroy(ev);
    if (e->entry_event) cudaEventDestroy(e->entry_event);
    if (e->own_stream) cudaStreamDestroy(e->own_stream);
    delete e;
    return CSAIDX_OK;
}

int csaidx_engine_set_stream(csaidx_engine* e, void* stream) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    e->stream = static_cast<cudaStream_t>(stream);
    e->main_stream = e->stream;
    e->lane = 0;
    return CSAIDX_OK;
}

int csaidx_engine_use_lane(csaidx_engine* e, int lane) {
    if (int rc = set_device(e)) return rc;
    if (lane < 0 || lane > 3)
        return fail(CSAIDX_INVALID_ARGUMENT, "lane must be 0 (main), 1 (copy-in), 2 (copy-out) or 3 (side compute)");
    if (e->lane == 0) e->main_stream = e->stream;
    if (lane > 0 && e->lanes[lane] == nullptr) {
        // the side compute lane gets the highest stream priority: its CTAs
        // are dispatched first when SMs free up (a select beside a score)
        int least = 0, greatest = 0;
        CSAIDX_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&least, &greatest), "cudaDeviceGetStreamPriorityRange");
        CSAIDX_CUDA_TRY(cudaStreamCreateWithPriority(&e->lanes[lane], cudaStreamNonBlocking, lane == 3 ? greatest : least),
                        "cudaStreamCreate(lane)");
    }
    e->stream = lane == 0 ? e->main_stream : e->lanes[lane];
    e->lane = lane;
    return CSAIDX_OK;
}

int csaidx_engine_signal(csaidx_engine* e, int slot) {
    if (int rc = set_device(e)) return rc;
    if (slot < 0 || slot >= 192) return fail(CSAIDX_INVALID_ARGUMENT, "event slot out of range");
    if (e->slots[slot] == nullptr)
        CSAIDX_CUDA_TRY(cudaEventCreateWithFlags(&e->slots[slot], cudaEventDisableTiming), "cudaEventCreate");
    CSAIDX_CUDA_TRY(cudaEventRecord(e->slots[slot], e->stream), "cudaEventRecord");
    return CSAIDX_OK;
}

int csaidx_engine_await(csaidx_engine* e, int slot) {
    if (int rc = set_device(e)) return rc;
    if (slot < 0 || slot >= 192) return fail(CSAIDX_INVALID_ARGUMENT, "event slot out of range");
    if (e->slots[slot] == nullptr) return CSAIDX_OK;  // never signalled: nothing to wait for
    CSAIDX_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->slots[slot], 0), "cudaStreamWaitEvent");
    return CSAIDX_OK;
}

int csaidx_engine_sync_slot(csaidx_engine* e, int slot) {
    if (int rc = set_device(e)) return rc;
    if (slot < 0 || slot >= 192) return fail(CSAIDX_INVALID_ARGUMENT, "event slot out of range");
    if (e->slots[slot] == nullptr) return CSAIDX_OK;
    CSAIDX_CUDA_TRY(cudaEventSynchronize(e->slots[slot]), "cudaEventSynchronize");
    return CSAIDX_OK;
}

int csaidx_engine_copy_on_lane(csaidx_engine* e, int lane, int slot, void* dst, const void* src, size_t bytes) {
    if (int rc = set_device(e)) return rc;
    if (lane < 1 || lane > 3 || e->lanes[lane] == nullptr)
        return fail(CSAIDX_INVALID_ARGUMENT, "copy_on_lane: lane must be 1..3 and already in use");
    if (slot >= 192) return fail(CSAIDX_INVALID_ARGUMENT, "event slot out of range");
    if (bytes != 0) CSAIDX_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, e->lanes[lane]), "cudaMemcpyAsync");
    if (slot >= 0) {
        if (e->slots[slot] == nullptr)
            CSAIDX_CUDA_TRY(cudaEventCreateWithFlags(&e->slots[slot], cudaEventDisableTiming), "cudaEventCreate");
        CSAIDX_CUDA_TRY(cudaEventRecord(e->slots[slot], e->lanes[lane]), "cudaEventRecord");
    }
    return CSAIDX_OK;
}

int csaidx_engine_await_stream(csaidx_engine* e, void* stream) {
    if (int rc = set_device(e)) return rc;
    cudaStream_t src = stream == nullptr ? cudaStreamLegacy : static_cast<cudaStream_t>(stream);
    if (src == e->stream) return CSAIDX_OK;
    if (e->entry_event == nullptr)
        CSAIDX_CUDA_TRY(cudaEventCreateWithFlags(&e->entry_event, cudaEventDisableTiming), "cudaEventCreate");
    CSAIDX_CUDA_TRY(cudaEventRecord(e->entry_event, src), "cudaEventRecord(await_stream)");
    CSAIDX_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->entry_event, 0), "cudaStreamWaitEvent(await_stream)");
    return CSAIDX_OK;
}

int csaidx_engine_use_own_stream(csaidx_engine* e) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    e->stream = e->own_stream;
    e->main_stream = e->stream;
    e->lane = 0;
    return CSAIDX_OK;
}

int csaidx_engine_get_stream(csaidx_engine* e, void** stream) {
    if (e == nullptr || stream == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null argument");
    *stream = e->stream;
    return CSAIDX_OK;
}

int csaidx_engine_num_sms(csaidx_engine* e, int* num_sms) {
    if (e == nullptr || num_sms == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null argument");
    *num_sms = e->num_sms;
    return CSAIDX_OK;
}

int csaidx_engine_set_partition(csaidx_engine* e, int score_sms, int select_sms) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    if (score_sms < 0 || select_sms < 0 || score_sms + select_sms > e->num_sms)
        return fail(CSAIDX_INVALID_ARGUMENT, "partition exceeds the SM count");
    e->score_sms = score_sms;
    e->select_sms = select_sms;
    return CSAIDX_OK;
}

int csaidx_engine_check(csaidx_engine* e) {
    if (int rc = set_device(e)) return rc;
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(e->stream), "cudaStreamSynchronize");
    for (int i = 0; i < 4; ++i) {
        cudaStream_t s = i == 0 ? e->main_stream : e->lanes[i];
        if (s != nullptr && s != e->stream) CSAIDX_CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize(lane)");
    }
    int h[kNumFlags];
    CSAIDX_CUDA_TRY(cudaMemcpy(h, e->flags, sizeof(h), cudaMemcpyDeviceToHost), "flags D2H");
    bool any = false;
    for (int i = 0; i < kNumFlags; ++i) any = any || (i != kInexactSeen && h[i] != 0);
    if (!any) return CSAIDX_OK;
    // reset the error flags; kInexactSeen is consumed by csaidx_engine_take_inexact
    CSAIDX_CUDA_TRY(cudaMemset(e->flags, 0, kInexactSeen * sizeof(int)), "flags reset");
    CSAIDX_CUDA_TRY(cudaMemset(e->flags + kInexactSeen + 1, 0, (kNumFlags - kInexactSeen - 1) * sizeof(int)),
                    "flags reset");
    if (h[kNonfiniteInput]) return fail(CSAIDX_INVALID_ARGUMENT, "IndexerInputs: non-finite entry in q/kc");
    if (h[kInexact]) return fail(CSAIDX_INVALID_ARGUMENT, "operand is not bf16-representable (strict mode)");
    if (h[kOverlap]) return fail(CSAIDX_INVALID_ARGUMENT, "merge_topk: overlapping indices between buffer and tile");
    if (h[kNonfiniteScore]) return fail(CSAIDX_RUNTIME_ERROR, "score_tile: non-finite score in fp32 mode");
    if (h[kTrail]) return fail(CSAIDX_LOGIC_ERROR, "run_chunked: sentinel entries do not trail");
    if (h[kKeff]) return fail(CSAIDX_LOGIC_ERROR, "run_chunked: row valid count != k_eff");
    return fail(CSAIDX_LOGIC_ERROR, "unknown device flag");
}

int csaidx_engine_take_inexact(csaidx_engine* e, int* seen) {
    if (int rc = set_device(e)) return rc;
    if (seen == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "take_inexact: null out pointer");
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(e->stream), "cudaStreamSynchronize");
    for (int i = 0; i < 4; ++i) {
        cudaStream_t s = i == 0 ? e->main_stream : e->lanes[i];
        if (s != nullptr && s != e->stream) CSAIDX_CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize(lane)");
    }
    int h = 0;
    CSAIDX_CUDA_TRY(cudaMemcpy(&h, e->flags + kInexactSeen, sizeof(int), cudaMemcpyDeviceToHost), "flag D2H");
    if (h != 0) CSAIDX_CUDA_TRY(cudaMemset(e->flags + kInexactSeen, 0, sizeof(int)), "flag reset");
    *seen = h != 0;
    return CSAIDX_OK;
}

int csaidx_engine_mem_stats(csaidx_engine* e, uint64_t* live, uint64_t* peak) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    std::lock_guard<std::mutex> lock(e->mu);
    if (live) *live = e->live;
    if (peak) *peak = e->peak;
    return CSAIDX_OK;
}

int csaidx_engine_set_profiling(csaidx_engine* e, int enabled) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    e->profiling = enabled != 0;
    return CSAIDX_OK;
}

int csaidx_engine_kernel_stats(csaidx_engine* e, int kind, int64_t* launches, double* total_ms) {
    if (int rc = set_device(e)) return rc;
    if (kind < 0 || kind >= CSAIDX_NUM_KINDS) return fail(CSAIDX_INVALID_ARGUMENT, "unknown kernel kind");
    for (const auto& pd : e->pending) {
        float ms = 0.0f;
        CSAIDX_CUDA_TRY(cudaEventSynchronize(pd.stop), "cudaEventSynchronize");
        CSAIDX_CUDA_TRY(cudaEventElapsedTime(&ms, pd.start, pd.stop), "cudaEventElapsedTime");
        e->total_ms[pd.kind] += ms;
        e->event_pool.push_back(pd.start);
        e->event_pool.push_back(pd.stop);
    }
    e->pending.clear();
    if (launches) *launches = e->launches[kind];
    if (total_ms) *total_ms = e->total_ms[kind];
    return CSAIDX_OK;
}

int csaidx_engine_set_score_probe(csaidx_engine* e, long long* device_counters) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    e->score_probe = device_counters;
    return CSAIDX_OK;
}

int csaidx_engine_set_select_probe(csaidx_engine* e, long long* device_clocks) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    e->select_probe = device_clocks;
    return CSAIDX_OK;
}

int csaidx_engine_select_fallbacks(csaidx_engine* e, int64_t* rows, int reset) {
    if (int rc = set_device(e)) return rc;
    int h = 0;
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(e->stream), "cudaStreamSynchronize");
    CSAIDX_CUDA_TRY(cudaMemcpy(&h, e->flags + kNumFlags + 2, sizeof(int), cudaMemcpyDeviceToHost), "counter D2H");
    if (rows) *rows = h;
    if (reset) CSAIDX_CUDA_TRY(cudaMemset(e->flags + kNumFlags + 2, 0, sizeof(int)), "counter reset");
    return CSAIDX_OK;
}

int csaidx_engine_candidate_hits(csaidx_engine* e, int64_t* rows, int reset) {
    if (int rc = set_device(e)) return rc;
    int h = 0;
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(e->stream), "cudaStreamSynchronize");
    CSAIDX_CUDA_TRY(cudaMemcpy(&h, e->flags + kNumFlags + 3, sizeof(int), cudaMemcpyDeviceToHost), "counter D2H");
    if (rows) *rows = h;
    if (reset) CSAIDX_CUDA_TRY(cudaMemset(e->flags + kNumFlags + 3, 0, sizeof(int)), "counter reset");
    return CSAIDX_OK;
}

int csaidx_engine_reset_stats(csaidx_engine* e) {
    if (int rc = set_device(e)) return rc;
    for (const auto& pd : e->pending) {
        cudaEventSynchronize(pd.stop);
        e->event_pool.push_back(pd.start);
        e->event_pool.push_back(pd.stop);
    }
    e->pending.clear();
    for (int k = 0; k < CSAIDX_NUM_KINDS; ++k) {
        e->launches[k] = 0;
        e->total_ms[k] = 0.0;
    }
    return CSAIDX_OK;
}

int csaidx_engine_reset_peak(csaidx_engine* e) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    std::lock_guard<std::mutex> lock(e->mu);
    e->peak = e->live;
    return CSAIDX_OK;
}

int csaidx_cuda_alloc(csaidx_engine* e, size_t bytes, void** ptr) {
    if (int rc = set_device(e)) return rc;
    if (ptr == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null out pointer");
    *ptr = nullptr;
    if (bytes == 0) bytes = 16;
    CSAIDX_CUDA_TRY(cudaMallocAsync(ptr, bytes, e->stream), "cudaMallocAsync");
    std::lock_guard<std::mutex> lock(e->mu);
    e->sizes[*ptr] = bytes;
    e->live += bytes;
    if (e->live > e->peak) e->peak = e->live;
    return CSAIDX_OK;
}

int csaidx_cuda_free(csaidx_engine* e, void* ptr) {
    if (int rc = set_device(e)) return rc;
    if (ptr == nullptr) return CSAIDX_OK;
    {
        std::lock_guard<std::mutex> lock(e->mu);
        auto it = e->sizes.find(ptr);
        if (it == e->sizes.end()) return fail(CSAIDX_INVALID_ARGUMENT, "csaidx_cuda_free: unknown pointer");
        e->live -= it->second;
        e->sizes.erase(it);
    }
    CSAIDX_CUDA_TRY(cudaFreeAsync(ptr, e->stream), "cudaFreeAsync");
    return CSAIDX_OK;
}

int csaidx_cuda_copy(csaidx_engine* e, void* dst, const void* src, size_t bytes) {
    if (int rc = set_device(e)) return rc;
    if (bytes == 0) return CSAIDX_OK;
    CSAIDX_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, e->stream), "cudaMemcpyAsync");
    return CSAIDX_OK;
}

int csaidx_engine_set_index_sink(csaidx_engine* e, int32_t* dst, int64_t batch, int64_t seq_len, int64_t k) {
    if (e == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "null engine");
    if (dst != nullptr && (batch < 1 || seq_len < 1 || k < 1))
        return fail(CSAIDX_INVALID_ARGUMENT, "index sink: batch, seq_len and k must be >= 1");
    e->sink = dst;
    e->sink_batch = dst != nullptr ? batch : 0;
    e->sink_seq = dst != nullptr ? seq_len : 0;
    e->sink_k = dst != nullptr ? k : 0;
    return CSAIDX_OK;
}

int csaidx_cuda_ipc_handle(csaidx_engine* e, void* dev_ptr, void* handle, uint64_t* offset) {
    if (int rc = set_device(e)) return rc;
    if (dev_ptr == nullptr || handle == nullptr || offset == nullptr)
        return fail(CSAIDX_INVALID_ARGUMENT, "ipc_handle: null argument");
    AddressRangeFn range = get_range_fn();
    if (range == nullptr) return fail(CSAIDX_CUDA_ERROR, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
        return fail(CSAIDX_INVALID_ARGUMENT, "ipc_handle: not a device allocation");
    cudaIpcMemHandle_t h;
    CSAIDX_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
    std::memcpy(handle, &h, sizeof(h));
    *offset = reinterpret_cast<CUdeviceptr>(dev_ptr) - base;
    return CSAIDX_OK;
}

int csaidx_cuda_ipc_open(csaidx_engine* e, const void* handle, uint64_t offset, void** dev_ptr) {
    if (int rc = set_device(e)) return rc;
    if (dev_ptr == nullptr || handle == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "ipc_open: null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    CSAIDX_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    *dev_ptr = static_cast<char*>(base) + offset;
    return CSAIDX_OK;
}

int csaidx_cuda_ipc_close(csaidx_engine* e, void* dev_ptr, uint64_t offset) {
    if (int rc = set_device(e)) return rc;
    CSAIDX_CUDA_TRY(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset), "cudaIpcCloseMemHandle");
    return CSAIDX_OK;
}

int csaidx_cuda_host_alloc(csaidx_engine* e, size_t bytes, void** ptr) {
    if (int rc = set_device(e)) return rc;
    if (ptr == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "host_alloc: null out pointer");
    *ptr = nullptr;
    if (bytes == 0) return CSAIDX_OK;
    CSAIDX_CUDA_TRY(cudaHostAlloc(ptr, bytes, cudaHostAllocDefault), "cudaHostAlloc");
    return CSAIDX_OK;
}

int csaidx_cuda_host_is_pinned(const void* ptr, int* pinned) {
    if (pinned == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "host_is_pinned: null out pointer");
    *pinned = 0;
    cudaPointerAttributes a{};
    if (ptr != nullptr && cudaPointerGetAttributes(&a, ptr) == cudaSuccess)
        *pinned = (a.type == cudaMemoryTypeHost) ? 1 : 0;
    cudaGetLastError();  // a pageable pointer is not an error worth keeping
    return CSAIDX_OK;
}

int csaidx_cuda_host_free(csaidx_engine* e, void* ptr) {
    if (int rc = set_device(e)) return rc;
    if (ptr != nullptr) CSAIDX_CUDA_TRY(cudaFreeHost(ptr), "cudaFreeHost");
    return CSAIDX_OK;
}

int csaidx_cuda_memset(csaidx_engine* e, void* dst, int value, size_t bytes) {
    if (int rc = set_device(e)) return rc;
    if (bytes == 0) return CSAIDX_OK;
    CSAIDX_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, e->stream), "cudaMemsetAsync");
    return CSAIDX_OK;
}

int csaidx_cuda_to_bf16(csaidx_engine* e, const float* src, uint16_t* dst, int64_t n, int strict) {
    if (int rc = set_device(e)) return rc;
    if (n < 0) return fail(CSAIDX_INVALID_ARGUMENT, "to_bf16: negative length");
    ConvertParams p{src, reinterpret_cast<__nv_bfloat16*>(dst), n, e->flags + (strict ? kInexact : kInexactSeen),
                    e->flags + kNonfiniteInput};
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_convert_bf16(p, e->stream), "convert_bf16");
    return CSAIDX_OK;
}

int csaidx_cuda_score_uses_tensor_cores(const csaidx_dims* d, int dtype, int mode, int kernel) {
    if (d == nullptr) return 0;
    const bool mode_ok = (kernel == CSAIDX_KERNEL_AUTO && mode == CSAIDX_MODE_FP32) ||
                         (kernel == CSAIDX_KERNEL_TENSOR &&
                          (mode == CSAIDX_MODE_FP32 || mode == CSAIDX_MODE_FP16_EMULATED));
    return mode_ok && dtype == CSAIDX_DTYPE_BF16 && csaidx_kern::score_tc_supported(d->heads, d->head_dim);
}

}  // extern "C"

namespace {

// score_tc launch shared by the plain, sampled and filtered entry points.
int launch_tc(csaidx_engine* e, const void* q, const void* kc, const float* w, const csaidx_dims* d, int64_t s0,
              int64_t rows, int64_t t0, int64_t cols, int apply_mask, float* out, int64_t ld, int kt_stride,
              const float* tau, uint32_t* pass_bits, int64_t bits_ld, int64_t op_rows = -1, int64_t op_row0 = -1,
              float* gmax = nullptr, int64_t gmax_ld = 0, bool fp16 = false) {
    if (op_rows < 0) {
        op_rows = d->seq_len;
        op_row0 = s0;
    }
    CUtensorMap qmap, kmap;
    if (int rc = make_map(&qmap, q, static_cast<uint64_t>(d->batch * op_rows * d->heads), d->head_dim,
                          static_cast<uint32_t>(csaidx_kern::score_tc_q_box_rows())))
        return rc;
    if (int rc = make_map(&kmap, kc, static_cast<uint64_t>(d->batch * d->key_blocks), d->head_dim, 128)) return rc;
    ScoreTcParams p{};
    p.w = w;
    p.out = out;
    p.nonfinite = e->flags + kNonfiniteScore;
    p.sched = e->flags + kNumFlags;
    p.ld = ld;
    p.seq_len = d->seq_len;
    p.key_blocks = d->key_blocks;
    p.ratio = d->ratio;
    p.s0 = s0;
    p.rows = rows;
    p.t0 = t0;
    p.cols = cols;
    p.op_rows = op_rows;
    p.op_shift = op_row0 - s0;
    p.batch = static_cast<int>(d->batch);
    p.apply_mask = apply_mask;
    p.kt_stride = kt_stride;
    p.tau = tau;
    p.pass_bits = pass_bits;
    p.bits_ld = bits_ld;
    p.gmax = gmax;
    p.gmax_ld = gmax_ld;
    p.fp16 = fp16 ? 1 : 0;
    p.probe = e->score_probe;
    LaunchScope ls(e, CSAIDX_KIND_SCORE);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_score_tc(qmap, kmap, p, e->score_sms > 0 ? e->score_sms : e->num_sms,
                                                 e->stream),
                    "score_tc");
    return CSAIDX_OK;
}

int check_tile(const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols) {
    if (int rc = check_dims(d)) return rc;
    if (rows < 1 || cols < 1 || s0 < 0 || t0 < 0 || s0 + rows > d->seq_len || t0 + cols > d->key_blocks)
        return fail(CSAIDX_INVALID_ARGUMENT, "score_tile: tile out of range");
    return CSAIDX_OK;
}

}  // namespace

extern "C" {

int64_t csaidx_cuda_candidate_words(int64_t cols) { return cols < 1 ? 0 : (cols + 127) / 128 * 4; }

int csaidx_cuda_candidate_capacity(int64_t k) {
    return k < 1 || k > csaidx_kern::select_max_take() ? 0 : csaidx_kern::select_cand_capacity(static_cast<int>(k));
}

int csaidx_cuda_score_sampled(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                              const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, int kt_stride,
                              float* sample, int64_t lds) {
    if (int rc = set_device(e)) return rc;
    if (int rc = check_tile(d, s0, rows, t0, cols)) return rc;
    if (!csaidx_cuda_score_uses_tensor_cores(d, CSAIDX_DTYPE_BF16, CSAIDX_MODE_FP32, CSAIDX_KERNEL_AUTO))
        return fail(CSAIDX_INVALID_ARGUMENT, "score_sampled: tensor-core shape only");
    if (kt_stride < 1) return fail(CSAIDX_INVALID_ARGUMENT, "score_sampled: kt_stride must be >= 1");
    const int64_t vtiles = ((cols + 127) / 128 + kt_stride - 1) / kt_stride;
    if (lds < vtiles * 128 || (lds % 4) != 0) return fail(CSAIDX_INVALID_ARGUMENT, "score_sampled: lds too small");
    return launch_tc(e, q_bf16, kc_bf16, w, d, s0, rows, t0, cols, 1, sample, lds, kt_stride, nullptr, nullptr, 0);
}

int csaidx_cuda_row_threshold(csaidx_engine* e, const float* sample, int64_t lds, int64_t batch, int64_t rows,
                              int64_t cols, int64_t s0, int64_t t0, int64_t ratio, int kt_stride, int64_t k,
                              float* tau) {
    if (int rc = set_device(e)) return rc;
    const int cap = csaidx_cuda_candidate_capacity(k);
    if (cap == 0) return fail(CSAIDX_INVALID_ARGUMENT, "row_threshold: k outside the GPU selection capacity");
    TauParams p{};
    p.sample = sample;
    p.lds = lds;
    p.rows = rows;
    p.cols = cols;
    p.s0 = s0;
    p.t0 = t0;
    p.ratio = ratio;
    p.batch = static_cast<int>(batch);
    p.kt_stride = kt_stride < 1 ? 1 : kt_stride;
    p.k = static_cast<int>(k);
    p.cand_cap = cap;
    p.tau = tau;
    LaunchScope ls(e, CSAIDX_KIND_SELECT);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_tau(p, e->stream), "row_threshold");
    return CSAIDX_OK;
}

int csaidx_cuda_score_filtered(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                               const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, float* out,
                               int64_t ld, const float* tau, uint32_t* pass_bits, int64_t bits_ld) {
    if (int rc = set_device(e)) return rc;
    if (int rc = check_tile(d, s0, rows, t0, cols)) return rc;
    if (!csaidx_cuda_score_uses_tensor_cores(d, CSAIDX_DTYPE_BF16, CSAIDX_MODE_FP32, CSAIDX_KERNEL_AUTO))
        return fail(CSAIDX_INVALID_ARGUMENT, "score_filtered: tensor-core shape only");
    if (ld < cols || (ld % 4) != 0) return fail(CSAIDX_INVALID_ARGUMENT, "score: ld must be >= cols and a multiple of 4");
    if (tau == nullptr || pass_bits == nullptr)
        return fail(CSAIDX_INVALID_ARGUMENT, "score_filtered: missing tau / candidate bitmap");
    if (bits_ld < csaidx_cuda_candidate_words(cols))
        return fail(CSAIDX_INVALID_ARGUMENT, "score_filtered: bits_ld < csaidx_cuda_candidate_words(cols)");
    return launch_tc(e, q_bf16, kc_bf16, w, d, s0, rows, t0, cols, 1, out, ld, 1, tau, pass_bits, bits_ld);
}

int csaidx_cuda_score(csaidx_engine* e, const void* q, const void* kc, int dtype, const float* w,
                      const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, int mode, int kernel,
                      int apply_mask, float* out, int64_t ld) {
    if (int rc = check_dims(d)) return rc;
    return csaidx_cuda_score_rows(e, q, kc, dtype, w, d, s0, rows, t0, cols, mode, kernel, apply_mask, out, ld,
                                  d->seq_len, s0);
}

int csaidx_cuda_score_rows(csaidx_engine* e, const void* q, const void* kc, int dtype, const float* w,
                           const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, int mode,
                           int kernel, int apply_mask, float* out, int64_t ld, int64_t op_rows, int64_t op_row0) {
    if (int rc = set_device(e)) return rc;
    if (int rc = check_dims(d)) return rc;
    if (rows < 1 || cols < 1 || s0 < 0 || t0 < 0 || s0 + rows > d->seq_len || t0 + cols > d->key_blocks)
        return fail(CSAIDX_INVALID_ARGUMENT, "score_tile: tile out of range");
    if (op_rows < 1 || op_row0 < 0 || op_row0 + rows > op_rows)
        return fail(CSAIDX_INVALID_ARGUMENT, "score: operand rows [op_row0, op_row0 + rows) outside op_rows");
    if (ld < cols || (ld % 4) != 0) return fail(CSAIDX_INVALID_ARGUMENT, "score: ld must be >= cols and a multiple of 4");
    if (mode != CSAIDX_MODE_FP32 && mode != CSAIDX_MODE_FP16_EMULATED)
        return fail(CSAIDX_INVALID_ARGUMENT, "score: unknown accumulation mode");
    if (dtype != CSAIDX_DTYPE_BF16 && dtype != CSAIDX_DTYPE_F32)
        return fail(CSAIDX_INVALID_ARGUMENT, "score: unknown operand dtype");
    if (kernel != CSAIDX_KERNEL_AUTO && kernel != CSAIDX_KERNEL_EXACT && kernel != CSAIDX_KERNEL_TENSOR)
        return fail(CSAIDX_INVALID_ARGUMENT, "score: unknown kernel request");
    if (csaidx_cuda_score_uses_tensor_cores(d, dtype, mode, kernel)) {
        return launch_tc(e, q, kc, w, d, s0, rows, t0, cols, apply_mask, out, ld, 1, nullptr, nullptr, 0, op_rows,
                         op_row0, nullptr, 0, mode == CSAIDX_MODE_FP16_EMULATED);
    } else {
        ScoreExactParams p{};
        p.q = q;
        p.kc = kc;
        p.operand_f32 = dtype == CSAIDX_DTYPE_F32;
        p.w = w;
        p.out = out;
        p.nonfinite = e->flags + kNonfiniteScore;
        p.ld = ld;
        p.seq_len = d->seq_len;
        p.key_blocks = d->key_blocks;
        p.heads = d->heads;
        p.head_dim = d->head_dim;
        p.ratio = d->ratio;
        p.s0 = s0;
        p.rows = rows;
        p.t0 = t0;
        p.cols = cols;
        p.op_rows = op_rows;
        p.op_shift = op_row0 - s0;
        p.batch = static_cast<int>(d->batch);
        p.apply_mask = apply_mask;
        p.fp16 = mode == CSAIDX_MODE_FP16_EMULATED;
        LaunchScope ls(e, CSAIDX_KIND_SCORE);
        CSAIDX_CUDA_TRY(csaidx_kern::launch_score_exact(p, e->stream), "score_exact");
    }
    return CSAIDX_OK;
}

int csaidx_cuda_score_gmax(csaidx_engine* e, const void* q_bf16, const void* kc_bf16, const float* w,
                           const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, float* out,
                           int64_t ld, int64_t op_rows, int64_t op_row0, float* gmax, int64_t gmax_ld) {
    if (int rc = set_device(e)) return rc;
    if (int rc = check_tile(d, s0, rows, t0, cols)) return rc;
    if (!csaidx_cuda_score_uses_tensor_cores(d, CSAIDX_DTYPE_BF16, CSAIDX_MODE_FP32, CSAIDX_KERNEL_AUTO))
        return fail(CSAIDX_INVALID_ARGUMENT, "score_gmax: tensor-core shape only");
    if (ld < cols || (ld % 4) != 0) return fail(CSAIDX_INVALID_ARGUMENT, "score: ld must be >= cols and a multiple of 4");
    if (op_rows < 1 || op_row0 < 0 || op_row0 + rows > op_rows)
        return fail(CSAIDX_INVALID_ARGUMENT, "score: operand rows [op_row0, op_row0 + rows) outside op_rows");
    if (gmax == nullptr || gmax_ld < (cols + 31) / 32)
        return fail(CSAIDX_INVALID_ARGUMENT, "score_gmax: gmax_ld < ceil(cols / 32)");
    return launch_tc(e, q_bf16, kc_bf16, w, d, s0, rows, t0, cols, 1, out, ld, 1, nullptr, nullptr, 0, op_rows, op_row0,
                     gmax, gmax_ld);
}

int csaidx_cuda_bool_mask(csaidx_engine* e, uint8_t* keep, int64_t s0, int64_t t0, int64_t rows, int64_t cols,
                          int64_t ratio) {
    if (int rc = set_device(e)) return rc;
    if (rows < 1 || cols < 1 || s0 < 0 || t0 < 0 || ratio < 1)
        return fail(CSAIDX_INVALID_ARGUMENT, "build_mask_tile: bad tile extents");
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_bool_mask(keep, rows, cols, s0, t0, ratio, e->stream), "bool_mask");
    return CSAIDX_OK;
}

int csaidx_cuda_apply_bool_mask(csaidx_engine* e, float* scores, int64_t ld, const uint8_t* keep, int64_t batch,
                                int64_t rows, int64_t cols) {
    if (int rc = set_device(e)) return rc;
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_apply_bool_mask(scores, ld, keep, batch, rows, cols, e->stream),
                    "apply_bool_mask");
    return CSAIDX_OK;
}

int csaidx_cuda_select_capacity(void) { return csaidx_kern::select_max_take(); }

int csaidx_cuda_select_overlap_capable(int64_t k) {
    return k >= 1 && k <= csaidx_kern::select_max_take() && csaidx_kern::select_fat_fits(static_cast<int>(k)) ? 1 : 0;
}

}  // extern "C"

namespace {

// The engine's large-take scratch, at least `need` bytes (a growth waits for
// the queued work that may still use the old buffer).
int large_scratch(csaidx_engine* e, size_t need) {
    if (e->large_bytes >= need) return CSAIDX_OK;
    CSAIDX_CUDA_TRY(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    if (e->large != nullptr) {
        cudaFree(e->large);
        e->live -= e->large_bytes;
        e->large = nullptr;
        e->large_bytes = 0;
    }
    CSAIDX_CUDA_TRY(cudaMalloc(&e->large, need), "cudaMalloc(large-take scratch)");
    e->large_bytes = need;
    e->live += need;
    if (e->live > e->peak) e->peak = e->live;
    return CSAIDX_OK;
}

// The index sink holds [sink_batch, sink_seq, sink_k] int32: a final write
// of rows [s0, s0 + rows) of `batch` batches at row stride k must fit it.
int check_sink(const csaidx_engine* e, int64_t batch, int64_t s0, int64_t rows, int64_t k) {
    if (e->sink == nullptr) return CSAIDX_OK;
    if (batch != e->sink_batch || k != e->sink_k || s0 < 0 || s0 + rows > e->sink_seq)
        return fail(CSAIDX_INVALID_ARGUMENT,
                    "index sink [%lld, %lld, %lld] does not cover rows [%lld, %lld) of %lld batches at k = %lld",
                    static_cast<long long>(e->sink_batch), static_cast<long long>(e->sink_seq),
                    static_cast<long long>(e->sink_k), static_cast<long long>(s0), static_cast<long long>(s0 + rows),
                    static_cast<long long>(batch), static_cast<long long>(k));
    return CSAIDX_OK;
}

int select_impl(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows, int64_t ld, int64_t cols,
                int64_t s0, int64_t t0, int64_t ratio, int apply_mask, int64_t k, float* cand_val, int32_t* cand_idx,
                int64_t cand_ld, const uint32_t* pass_bits, int64_t bits_ld, int64_t* final_idx = nullptr,
                int64_t final_rows = 0, int64_t final_row0 = 0, const float* gmax = nullptr, int64_t gmax_ld = 0) {
    if (int rc = set_device(e)) return rc;
    if (k < 1) return fail(CSAIDX_INVALID_ARGUMENT, "tile_topk: top_k must be >= 1");
    if (rows < 1 || cols < 1 || batch < 1 || ratio < 1) return fail(CSAIDX_INVALID_ARGUMENT, "select: bad extents");
    if ((ld % 4) != 0 || ld < cols) return fail(CSAIDX_INVALID_ARGUMENT, "select: ld must be >= cols, multiple of 4");
    if ((reinterpret_cast<uintptr_t>(scores) & 15) != 0) return fail(CSAIDX_INVALID_ARGUMENT, "select: scores not 16B aligned");
    const int64_t width = final_rows > 0 ? k : (k < cols ? k : cols);
    if (k > (int64_t{1} << 30)) return fail(CSAIDX_INVALID_ARGUMENT, "tile_topk: top_k too large");
    if (cand_ld < width) return fail(CSAIDX_INVALID_ARGUMENT, "select: cand_ld < min(k, cols)");
    SelectParams p{};
    p.scores = scores;
    p.ld = ld;
    p.rows = rows;
    p.cols = cols;
    p.s0 = s0;
    p.t0 = t0;
    p.ratio = ratio;
    p.batch = static_cast<int>(batch);
    p.apply_mask = apply_mask;
    p.k = static_cast<int>(k);
    p.width = static_cast<int>(width);
    p.out_val = cand_val;
    p.out_idx = cand_idx;
    p.out_ld = cand_ld;
    p.fallbacks = e->flags + kNumFlags + 2;
    p.phase_clk = e->select_probe;
    p.pass_bits = pass_bits;
    p.bits_ld = bits_ld;
    p.cand_hits = e->flags + kNumFlags + 3;
    p.final_idx = final_idx;
    p.final_rows = final_rows;
    p.final_row0 = final_row0;
    if (final_rows > 0) {  // select_final
        if (int rc = check_sink(e, batch, s0, rows, cand_ld)) return rc;
        p.sink = e->sink;
        p.sink_seq = e->sink_seq;
        p.sink_only = final_idx == nullptr ? 1 : 0;
    }
    p.persistent_ctas = e->select_sms;
    p.gmax = gmax;
    p.gmax_ld = gmax_ld;
    if (k > csaidx_kern::select_max_take() || width > csaidx_kern::select_max_take()) {
        if (pass_bits != nullptr || gmax != nullptr)
            return fail(CSAIDX_INVALID_ARGUMENT, "select: candidate filters need k <= %d", csaidx_kern::select_max_take());
        const size_t need = csaidx_kern::select_large_scratch_bytes(static_cast<int>(k), cols, batch * rows);
        if (int rc = large_scratch(e, need)) return rc;
        p.scratch = e->large;
        p.scratch_bytes = e->large_bytes;
        p.persistent_ctas = 0;
    }
    LaunchScope ls(e, CSAIDX_KIND_SELECT);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_select(p, e->stream), "select");
    return CSAIDX_OK;
}

}  // namespace

extern "C" {

int csaidx_cuda_select(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows, int64_t ld, int64_t cols,
                       int64_t s0, int64_t t0, int64_t ratio, int apply_mask, int64_t k, float* cand_val,
                       int32_t* cand_idx, int64_t cand_ld) {
    return select_impl(e, scores, batch, rows, ld, cols, s0, t0, ratio, apply_mask, k, cand_val, cand_idx, cand_ld,
                       nullptr, 0);
}

int csaidx_cuda_select_from_candidates(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows,
                                       int64_t ld, int64_t cols, int64_t s0, int64_t t0, int64_t ratio, int64_t k,
                                       const uint32_t* pass_bits, int64_t bits_ld, float* out_val,
                                       int32_t* out_idx, int64_t out_ld) {
    if (pass_bits == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "select_from_candidates: missing candidate bitmap");
    if (bits_ld < csaidx_cuda_candidate_words(cols))
        return fail(CSAIDX_INVALID_ARGUMENT, "select_from_candidates: bits_ld < csaidx_cuda_candidate_words(cols)");
    return select_impl(e, scores, batch, rows, ld, cols, s0, t0, ratio, 1, k, out_val, out_idx, out_ld, pass_bits,
                       bits_ld);
}

int csaidx_cuda_select_final(csaidx_engine* e, const float* scores, int64_t batch, int64_t rows, int64_t ld,
                             int64_t cols, int64_t s0, int64_t t0, int64_t ratio, int64_t k, const uint32_t* pass_bits,
                             int64_t bits_ld, const float* gmax, int64_t gmax_ld, int64_t* out_idx, float* out_val,
                             int64_t out_rows, int64_t out_row0) {
    if ((out_idx == nullptr) != (out_val == nullptr) || (out_idx == nullptr && e != nullptr && e->sink == nullptr))
        return fail(CSAIDX_INVALID_ARGUMENT, "select_final: null output (allowed for both only with an index sink)");
    if (out_row0 < 0 || out_row0 + rows > out_rows)
        return fail(CSAIDX_INVALID_ARGUMENT, "select_final: rows out of range");
    if (pass_bits != nullptr && bits_ld < csaidx_cuda_candidate_words(cols))
        return fail(CSAIDX_INVALID_ARGUMENT, "select_final: bits_ld < csaidx_cuda_candidate_words(cols)");
    if (gmax != nullptr && gmax_ld < (cols + 31) / 32)
        return fail(CSAIDX_INVALID_ARGUMENT, "select_final: gmax_ld < ceil(cols / 32)");
    return select_impl(e, scores, batch, rows, ld, cols, s0, t0, ratio, 1, k, out_val, nullptr, k, pass_bits, bits_ld,
                       out_idx, out_rows, out_row0, gmax, gmax_ld);
}

int csaidx_cuda_merge(csaidx_engine* e, float* run_val, int32_t* run_idx, int64_t nrows, int64_t k,
                      const float* cand_val, const int32_t* cand_idx, int64_t cand_ld, int64_t width, int overwrite,
                      int check_overlap) {
    if (int rc = set_device(e)) return rc;
    if (k < 1 || k > (int64_t{1} << 30)) return fail(CSAIDX_INVALID_ARGUMENT, "merge: k must be >= 1");
    if (width < 0 || width > k || cand_ld < width) return fail(CSAIDX_INVALID_ARGUMENT, "merge: bad candidate width");
    MergeParams p{};
    p.run_val = run_val;
    p.run_idx = run_idx;
    p.cand_val = cand_val;
    p.cand_idx = cand_idx;
    p.cand_ld = cand_ld;
    p.nrows = nrows;
    p.k = static_cast<int>(k);
    p.width = static_cast<int>(width);
    p.overwrite = overwrite;
    p.check_overlap = check_overlap;
    p.overlap_flag = e->flags + kOverlap;
    if (k > csaidx_kern::select_max_take() && !overwrite) {
        const size_t row = static_cast<size_t>(k + width) * sizeof(uint64_t);
        if (int rc = large_scratch(e, csaidx_kern::merge_stage_bytes(static_cast<int>(k), static_cast<int>(width),
                                                                      nrows)))
            return rc;
        p.stage = static_cast<uint64_t*>(e->large);
        p.stage_rows = static_cast<int64_t>(e->large_bytes / row);
    }
    LaunchScope ls(e, CSAIDX_KIND_MERGE);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_merge(p, e->stream), "merge");
    return CSAIDX_OK;
}

int csaidx_cuda_sparse_attention(csaidx_engine* e, const void* q_bf16, const void* kv_bf16, const int32_t* indices,
                                 int64_t batch, int64_t seq_len, int64_t kv_len, int64_t heads, int64_t dqk,
                                 int64_t dv, int64_t k, int64_t idx_ld, float sm_scale, void* out_bf16,
                                 int64_t out_ld, float* lse) {
    if (int rc = set_device(e)) return rc;
    if (heads < 128 || heads % 128 != 0 || dqk != 576 || dv != 512)
        return fail(CSAIDX_INVALID_ARGUMENT,
                    "sparse_attention: compiled for heads = a multiple of 128, dqk = 576, dv = 512");
    if (batch < 1 || seq_len < 0 || kv_len < 1 || k < 1 || k > 4096 || idx_ld < k || out_ld < dv || (out_ld % 8) != 0)
        return fail(CSAIDX_INVALID_ARGUMENT,
                    "sparse_attention: bad extents (1 <= k <= 4096, idx_ld >= k, out_ld >= dv, out_ld %% 8 == 0)");
    if (q_bf16 == nullptr || kv_bf16 == nullptr || indices == nullptr || out_bf16 == nullptr)
        return fail(CSAIDX_INVALID_ARGUMENT, "sparse_attention: null operand");
    if (batch * kv_len > (int64_t{1} << 31) - 1 || batch * seq_len * heads > (int64_t{1} << 31) - 1 ||
        2 * seq_len > (int64_t{1} << 31) - 1 || batch > 65535)
        return fail(CSAIDX_INVALID_ARGUMENT, "sparse_attention: extents exceed the 32-bit TMA coordinates");
    if ((reinterpret_cast<uintptr_t>(q_bf16) & 15) != 0 || (reinterpret_cast<uintptr_t>(kv_bf16) & 15) != 0 ||
        (reinterpret_cast<uintptr_t>(out_bf16) & 15) != 0)
        return fail(CSAIDX_INVALID_ARGUMENT, "sparse_attention: operands must be 16-byte aligned");
    if (seq_len == 0) return CSAIDX_OK;
    CUtensorMap qmap;
    // q as [B*S*heads, dqk] rows (box 64 x 128: one panel of a query's heads)
    if (int rc = make_map(&qmap, q_bf16, static_cast<uint64_t>(batch * seq_len * heads), static_cast<uint64_t>(dqk), 128))
        return rc;
    SparseMlaParams p{};
    p.q = static_cast<const __nv_bfloat16*>(q_bf16);
    p.kv = static_cast<const __nv_bfloat16*>(kv_bf16);
    p.indices = indices;
    p.idx_ld = idx_ld;
    p.out = static_cast<__nv_bfloat16*>(out_bf16);
    p.out_ld = out_ld;
    p.lse = lse;
    p.seq_len = seq_len;
    p.kv_len = kv_len;
    p.batch = static_cast<int>(batch);
    p.k = static_cast<int>(k);
    p.head_groups = static_cast<int>(heads / 128);
    p.sm_scale = sm_scale;
    LaunchScope ls(e, CSAIDX_KIND_ATTENTION);
    // Single-CTA kernel by default; CSAIDX_ATTN_PAIR=1 runs the CTA-pair form
    // (Dqk split across a cluster of 2, partial scores swapped through DSMEM):
    // same results within the tolerance, measured no faster
    // (profiles/r02_attention.md)
    const char* pv = getenv("CSAIDX_ATTN_PAIR");
    const bool pair = pv != nullptr && pv[0] == '1';
    if (pair)
        CSAIDX_CUDA_TRY(csaidx_kern::launch_sparse_mla_pair(qmap, p, e->stream), "sparse_attention");
    else
        CSAIDX_CUDA_TRY(csaidx_kern::launch_sparse_mla(qmap, p, e->stream), "sparse_attention");
    return CSAIDX_OK;
}

int csaidx_cuda_fill_sentinel(csaidx_engine* e, float* val, int32_t* idx, int64_t n) {
    if (int rc = set_device(e)) return rc;
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_fill_sentinel(val, idx, n, e->stream), "fill_sentinel");
    return CSAIDX_OK;
}

int csaidx_cuda_narrow_indices(csaidx_engine* e, const int64_t* src, int32_t* dst, int64_t n) {
    if (int rc = set_device(e)) return rc;
    if (n < 0) return fail(CSAIDX_INVALID_ARGUMENT, "narrow_indices: negative length");
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_narrow(src, dst, n, e->stream), "narrow_indices");
    return CSAIDX_OK;
}

int csaidx_cuda_scatter_rows(csaidx_engine* e, const int32_t* src, int32_t* dst, const int64_t* dst_row,
                             int64_t nrows, int64_t row_elems) {
    if (int rc = set_device(e)) return rc;
    if (nrows < 0 || row_elems < 1) return fail(CSAIDX_INVALID_ARGUMENT, "scatter_rows: bad extents");
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_scatter_rows(src, dst, dst_row, nrows, row_elems, e->stream), "scatter_rows");
    return CSAIDX_OK;
}

int csaidx_engine_sync(csaidx_engine* e) {
    if (int rc = set_device(e)) return rc;
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(e->stream), "cudaStreamSynchronize");
    return CSAIDX_OK;
}

int csaidx_cuda_finalize(csaidx_engine* e, const float* run_val, const int32_t* run_idx, int64_t batch, int64_t rows,
                         int64_t s0, int64_t ratio, int64_t k, int check_keff, int64_t* out_idx, float* out_val,
                         int64_t out_rows, int64_t out_row0) {
    if (int rc = set_device(e)) return rc;
    if (out_row0 < 0 || out_row0 + rows > out_rows) return fail(CSAIDX_INVALID_ARGUMENT, "finalize: rows out of range");
    if ((out_idx == nullptr) != (out_val == nullptr) || (out_idx == nullptr && e->sink == nullptr))
        return fail(CSAIDX_INVALID_ARGUMENT, "finalize: null output (allowed for both only with an index sink)");
    FinalizeParams p{};
    p.run_val = run_val;
    p.run_idx = run_idx;
    p.rows = rows;
    p.s0 = s0;
    p.ratio = ratio;
    p.batch = static_cast<int>(batch);
    p.k = static_cast<int>(k);
    p.check_keff = check_keff;
    p.out_idx = out_idx;
    p.out_val = out_val;
    p.out_rows = out_rows;
    p.out_row0 = out_row0;
    p.trail_flag = e->flags + kTrail;
    p.keff_flag = e->flags + kKeff;
    if (int rc = check_sink(e, batch, s0, rows, k)) return rc;
    p.sink = e->sink;
    p.sink_seq = e->sink_seq;
    LaunchScope ls(e, CSAIDX_KIND_FINALIZE);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_finalize(p, e->stream), "finalize");
    return CSAIDX_OK;
}

int csaidx_cuda_chunk_step(csaidx_engine* e, const void* q, const void* kc, int dtype, const float* w,
                           const csaidx_dims* d, int64_t s0, int64_t rows, int64_t t0, int64_t cols, int mode,
                           int kernel, float* score_buf, int64_t ld, float* cand_val, int32_t* cand_idx, float* run_val,
                           int32_t* run_idx, int first_tile, int overwrite) {
    if (int rc = csaidx_cuda_score(e, q, kc, dtype, w, d, s0, rows, t0, cols, mode, kernel, 1, score_buf, ld))
        return rc;
    const int64_t k = d->top_k;
    const int64_t width = k < cols ? k : cols;
    if (first_tile && width == k) {
        // Merging into an all-sentinel buffer is a copy (and so is A1's
        // overwrite): select straight into the running rows.
        return csaidx_cuda_select(e, score_buf, d->batch, rows, ld, cols, s0, t0, d->ratio, 1, k, run_val, run_idx, k);
    }
    if (int rc = csaidx_cuda_select(e, score_buf, d->batch, rows, ld, cols, s0, t0, d->ratio, 1, k, cand_val, cand_idx,
                                    width))
        return rc;
    return csaidx_cuda_merge(e, run_val, run_idx, d->batch * rows, k, cand_val, cand_idx, width, width, overwrite, 0);
}

int csaidx_cuda_gen_normal_bf16(csaidx_engine* e, uint16_t* dst, int64_t n, double stddev, uint64_t seed,
                                uint64_t stream_id, int64_t offset) {
    if (int rc = set_device(e)) return rc;
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_gen_normal_bf16(reinterpret_cast<__nv_bfloat16*>(dst), n, stddev, seed,
                                                        stream_id, offset, e->stream),
                    "gen_bf16");
    return CSAIDX_OK;
}

int csaidx_cuda_gen_normal_f32(csaidx_engine* e, float* dst, int64_t n, double stddev, uint64_t seed,
                               uint64_t stream_id, int64_t offset) {
    if (int rc = set_device(e)) return rc;
    LaunchScope ls(e, CSAIDX_KIND_PREP);
    CSAIDX_CUDA_TRY(csaidx_kern::launch_gen_normal_f32(dst, n, stddev, seed, stream_id, offset, e->stream), "gen_f32");
    return CSAIDX_OK;
}

}  // extern "C"

// ------------------------------------------------------------ NCCL transport
// libnccl.so.2 is resolved with dlopen at first use (the copy the process
// already loaded, e.g. PyTorch's, or the system library), so the C-ABI
// library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            a.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (fn == nullptr && a.why.empty()) a.why = std::string("libnccl lacks ") + name;
        };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.broadcast, "ncclBroadcast");
        sym(a.all_gather, "ncclAllGather");
        sym(a.all_reduce, "ncclAllReduce");
        sym(a.send, "ncclSend");
        sym(a.recv, "ncclRecv");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.error_string, "ncclGetErrorString");
        a.ok = a.why.empty();
        return a;
    }();
    return api;
}

#define CSAIDX_NCCL_TRY(expr, where)                                                                  \
    do {                                                                                              \
        ncclResult_t _r = (expr);                                                                     \
        if (_r != ncclSuccess) return fail(CSAIDX_RUNTIME_ERROR, "%s: NCCL error %s", where,          \
                                           nccl().error_string != nullptr ? nccl().error_string(_r) : "?"); \
    } while (0)

struct NcclCtx {
    csaidx_collectives pub{};
    ncclComm_t comm = nullptr;
    int device = 0;
    void* scratch = nullptr;  // device bytes for blobs / the barrier word
    size_t scratch_bytes = 0;
    cudaStream_t own = nullptr;
};

int nccl_bcast(void* ctx, void* buf, size_t bytes, int root, void* stream) {
    auto* c = static_cast<NcclCtx*>(ctx);
    CSAIDX_CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    CSAIDX_NCCL_TRY(nccl().broadcast(buf, buf, bytes, ncclUint8, root, c->comm, static_cast<cudaStream_t>(stream)),
                    "ncclBroadcast");
    return CSAIDX_OK;
}

int nccl_scratch(NcclCtx* c, size_t bytes) {
    if (c->scratch_bytes >= bytes) return CSAIDX_OK;
    if (c->scratch != nullptr) cudaFree(c->scratch);
    c->scratch = nullptr;
    c->scratch_bytes = 0;
    CSAIDX_CUDA_TRY(cudaMalloc(&c->scratch, bytes), "cudaMalloc(nccl scratch)");
    c->scratch_bytes = bytes;
    return CSAIDX_OK;
}

int nccl_allgather_host(void* ctx, const void* in, void* out, size_t bytes) {
    auto* c = static_cast<NcclCtx*>(ctx);
    CSAIDX_CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    const size_t all = bytes * static_cast<size_t>(c->pub.world);
    if (int rc = nccl_scratch(c, bytes + all)) return rc;
    char* d = static_cast<char*>(c->scratch);
    CSAIDX_CUDA_TRY(cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, c->own), "allgather H2D");
    CSAIDX_NCCL_TRY(nccl().all_gather(d, d + bytes, bytes, ncclUint8, c->comm, c->own), "ncclAllGather");
    CSAIDX_CUDA_TRY(cudaMemcpyAsync(out, d + bytes, all, cudaMemcpyDeviceToHost, c->own), "allgather D2H");
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(c->own), "cudaStreamSynchronize");
    return CSAIDX_OK;
}

int nccl_barrier(void* ctx, void* stream) {
    auto* c = static_cast<NcclCtx*>(ctx);
    CSAIDX_CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    if (int rc = nccl_scratch(c, 64)) return rc;
    auto s = static_cast<cudaStream_t>(stream);
    CSAIDX_NCCL_TRY(nccl().all_reduce(c->scratch, c->scratch, 1, ncclInt32, ncclSum, c->comm, s), "ncclAllReduce");
    CSAIDX_CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    return CSAIDX_OK;
}

int nccl_gatherv(void* ctx, const void* send, size_t send_bytes, void* recv, const size_t* recv_bytes,
                 const size_t* recv_off, int root, void* stream) {
    auto* c = static_cast<NcclCtx*>(ctx);
    CSAIDX_CUDA_TRY(cudaSetDevice(c->device), "cudaSetDevice");
    auto s = static_cast<cudaStream_t>(stream);
    CSAIDX_NCCL_TRY(nccl().group_start(), "ncclGroupStart");
    if (c->pub.rank == root) {
        for (int r = 0; r < c->pub.world; ++r) {
            char* dst = static_cast<char*>(recv) + recv_off[r];
            if (r == root) {
                if (recv_bytes[r] > 0)
                    CSAIDX_CUDA_TRY(cudaMemcpyAsync(dst, send, recv_bytes[r], cudaMemcpyDeviceToDevice, s),
                                    "gatherv self copy");
            } else if (recv_bytes[r] > 0) {
                CSAIDX_NCCL_TRY(nccl().recv(dst, recv_bytes[r], ncclUint8, r, c->comm, s), "ncclRecv");
            }
        }
    } else if (send_bytes > 0) {
        CSAIDX_NCCL_TRY(nccl().send(send, send_bytes, ncclUint8, root, c->comm, s), "ncclSend");
    }
    CSAIDX_NCCL_TRY(nccl().group_end(), "ncclGroupEnd");
    return CSAIDX_OK;
}

}  // namespace

extern "C" {

int csaidx_nccl_unique_id(uint8_t id[128]) {
    if (id == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "nccl_unique_id: null out");
    if (!nccl().ok) return fail(CSAIDX_RUNTIME_ERROR, "NCCL unavailable: %s", nccl().why.c_str());
    ncclUniqueId u;
    CSAIDX_NCCL_TRY(nccl().get_unique_id(&u), "ncclGetUniqueId");
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return CSAIDX_OK;
}

int csaidx_nccl_collectives_create(int rank, int world, const uint8_t id[128], int device,
                                   csaidx_collectives** out) {
    if (out == nullptr || id == nullptr) return fail(CSAIDX_INVALID_ARGUMENT, "nccl_collectives: null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(CSAIDX_INVALID_ARGUMENT, "nccl_collectives: bad rank");
    if (!nccl().ok) return fail(CSAIDX_RUNTIME_ERROR, "NCCL unavailable: %s", nccl().why.c_str());
    CSAIDX_CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
    auto* c = new NcclCtx();
    c->device = device;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    ncclResult_t r = nccl().comm_init_rank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(CSAIDX_RUNTIME_ERROR, "ncclCommInitRank: %s", nccl().error_string(r));
    }
    if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
        nccl().comm_destroy(c->comm);
        delete c;
        return fail(CSAIDX_CUDA_ERROR, "cudaStreamCreate failed");
    }
    c->pub.ctx = c;
    c->pub.rank = rank;
    c->pub.world = world;
    c->pub.device_buffers = 1;
    c->pub.bcast = nccl_bcast;
    c->pub.allgather_host = nccl_allgather_host;
    c->pub.barrier = nccl_barrier;
    c->pub.gatherv = nccl_gatherv;
    *out = &c->pub;
    return CSAIDX_OK;
}

int csaidx_nccl_collectives_destroy(csaidx_collectives* pub) {
    if (pub == nullptr) return CSAIDX_OK;
    auto* c = static_cast<NcclCtx*>(pub->ctx);
    cudaSetDevice(c->device);
    if (c->own) cudaStreamSynchronize(c->own);
    if (c->comm) nccl().comm_destroy(c->comm);
    if (c->scratch) cudaFree(c->scratch);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
    return CSAIDX_OK;
}

}  // extern "C"
