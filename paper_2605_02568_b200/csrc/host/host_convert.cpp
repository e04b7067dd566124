// Host fp32 -> bf16 rounding on a small persistent worker pool (see
// host_convert.hpp).
#include "host_convert.hpp"

#include <immintrin.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace csaidx::detail {

namespace {

// One element: the device's __float2bfloat16_rn for finite x (round to
// nearest, ties to even, carrying into the exponent).
inline uint16_t rne(uint32_t u) { return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16); }

inline void scalar_range(const float* src, uint16_t* dst, size_t n, uint32_t& bad_exp, uint32_t& low_bits) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t u;
        std::memcpy(&u, src + i, 4);
        if ((u & 0x7f800000u) == 0x7f800000u) bad_exp = 1;
        low_bits |= u & 0xffffu;
        dst[i] = rne(u);
    }
}

bool nt_stores() {
    static const bool v = [] {
        const char* e = std::getenv("CSAIDX_HOST_NT");
        return e == nullptr || std::string(e) != "0";
    }();
    return v;
}

// bytes ahead of the load the source is prefetched (CSAIDX_HOST_PREFETCH,
// default one 4 KiB page)
int prefetch_distance() {
    static const int v = [] {
        const char* e = std::getenv("CSAIDX_HOST_PREFETCH");
        return e != nullptr ? std::clamp(std::atoi(e), 0, 1 << 16) : 4096;
    }();
    return v;
}

__attribute__((target("avx512f,avx512bw"))) void avx512_range(const float* src, uint16_t* dst, size_t n,
                                                               uint32_t& bad_exp, uint32_t& low_bits, bool nt) {
    const __m512i bias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1);
    const __m512i expm = _mm512_set1_epi32(0x7f800000), lowm = _mm512_set1_epi32(0xffff);
    __mmask16 nonfin = 0, inexact = 0;
    size_t i = 0;
    // head: scalar until dst is 32-byte aligned (non-temporal 256-bit stores)
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31u) != 0) {
        scalar_range(src + i, dst + i, 1, bad_exp, low_bits);
        ++i;
    }
    for (; i + 16 <= n; i += 16) {
        // one page ahead: the hardware prefetcher stops at 4 KiB boundaries
        // (pinned caller buffers are 4 KiB pages); +40% measured on the box
        _mm_prefetch(reinterpret_cast<const char*>(src + i) + prefetch_distance(), _MM_HINT_T0);
        const __m512i u = _mm512_loadu_si512(reinterpret_cast<const void*>(src + i));
        const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(u, 16), one);
        const __m512i r = _mm512_srli_epi32(_mm512_add_epi32(u, _mm512_add_epi32(bias, lsb)), 16);
        nonfin |= _mm512_cmpeq_epi32_mask(_mm512_and_si512(u, expm), expm);
        inexact |= _mm512_test_epi32_mask(u, lowm);
        if (nt)
            _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm512_cvtepi32_epi16(r));
        else
            _mm256_store_si256(reinterpret_cast<__m256i*>(dst + i), _mm512_cvtepi32_epi16(r));
    }
    _mm_sfence();
    if (nonfin) bad_exp = 1;
    if (inexact) low_bits |= 1u;
    scalar_range(src + i, dst + i, n - i, bad_exp, low_bits);
}

bool have_avx512() {
    static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
    return v;
}

class Pool {
public:
    explicit Pool(int workers) {
        for (int t = 0; t < workers; ++t) threads_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        start_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return static_cast<int>(threads_.size()); }

    void run(int parts, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> serial(run_mu_);  // one parallel region at a time
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            parts_ = parts;
            next_.store(0);
            finished_ = 0;
            ++gen_;
        }
        start_.notify_all();
        work();
        std::unique_lock<std::mutex> g(mu_);
        done_.wait(g, [this] { return finished_ == size(); });
        fn_ = nullptr;
    }

private:
    void work() {
        for (int p = next_.fetch_add(1); p < parts_; p = next_.fetch_add(1)) (*fn_)(p);
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu_);
                start_.wait(g, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
            {
                std::lock_guard<std::mutex> g(mu_);
                ++finished_;
            }
            done_.notify_one();
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_, run_mu_;
    std::condition_variable start_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int parts_ = 0;
    std::atomic<int> next_{0};
    int finished_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p(host_threads() - 1);  // + the calling thread
    return p;
}

}  // namespace

int host_threads() {
    static const int n = [] {
        if (const char* v = std::getenv("CSAIDX_HOST_THREADS")) return std::clamp(std::atoi(v), 1, 64);
        // the cores this process may run on, shared with the other ranks of
        // this node (torchrun's LOCAL_WORLD_SIZE), less one for the thread
        // issuing the CUDA calls
        cpu_set_t set;
        int cores = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set)
                                                                 : static_cast<int>(std::thread::hardware_concurrency());
        const char* lws = std::getenv("LOCAL_WORLD_SIZE");
        const int ranks = lws != nullptr ? std::max(1, std::atoi(lws)) : 1;
        return std::clamp(cores / ranks - 1, 1, 64);
    }();
    return n;
}

bool host_round_enabled() {
    if (const char* v = std::getenv("CSAIDX_HOST_ROUND")) return std::string(v) != "0";
    // Default: on for one rank per node. Host rounding moves more bytes
    // through host DRAM (fp32 read + bf16 write + its DMA re-read, ~1.7x the
    // fp32 path's) to halve the PCIe bytes; with several ranks sharing the
    // node's memory system the fp32 path's lower DRAM traffic is the safer
    // choice.
    const char* lws = std::getenv("LOCAL_WORLD_SIZE");
    return lws == nullptr || std::atoi(lws) <= 1;
}

int host_slab_count() {
    const char* v = std::getenv("CSAIDX_HOST_SLABS");
    return std::clamp(v != nullptr ? std::atoi(v) : 8, 2, 32);
}

int64_t host_piece_bytes() {
    const char* v = std::getenv("CSAIDX_HOST_PIECE_KB");
    return int64_t{1024} * std::clamp<int64_t>(v != nullptr ? std::atoll(v) : 8192, 64, 1 << 20);
}

bool host_ring_enabled() {
    // Default on (CSAIDX_HOST_RING=0: whole-chunk slabs with non-temporal
    // stores). C3 end to end on three boxes: 130.2-131.9 ms vs 132.3-138.5 ms
    // with 8 MiB pieces through a 4-piece ring; 2 MiB pieces lose to the
    // per-piece overhead (162-165 ms).
    const char* v = std::getenv("CSAIDX_HOST_RING");
    return v == nullptr || std::string(v) != "0";
}

int host_ring_pieces() {
    const char* v = std::getenv("CSAIDX_HOST_RING_PIECES");
    return std::clamp(v != nullptr ? std::atoi(v) : 4, 2, 32);
}

size_t host_fp32_tail(size_t chunks) {
    // Off by default: C3 e2e 125 ms with no tail, 133 ms with chunks / 8 and
    // 150 ms with 24 fp32 chunks on the same box (profiles/r02_host_ring.md):
    // the extra PCIe bytes beside the first chunks cost more than the
    // rounding thread saves.
    (void)chunks;
    const char* v = std::getenv("CSAIDX_HOST_FP32_TAIL");
    const long long n = v != nullptr ? std::atoll(v) : 0;
    return static_cast<size_t>(std::clamp<long long>(n, 0, 27));
}

uint16_t host_bf16_rne(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    return rne(u);
}

void host_parallel_for(int parts, const std::function<void(int)>& fn) {
    if (parts <= 1 || host_threads() == 1) {
        for (int p = 0; p < parts; ++p) fn(p);
        return;
    }
    pool().run(parts, fn);
}

Bf16Flags host_to_bf16(const float* src, uint16_t* dst, size_t n, int nt_mode) {
    const bool nt = nt_mode < 0 ? nt_stores() : nt_mode != 0;
    // parts of >= 256 KiB of source, 16-element aligned, a few per thread
    constexpr size_t kMinPart = size_t{1} << 16;
    const size_t want = static_cast<size_t>(host_threads()) * 4;
    const size_t parts = std::max<size_t>(1, std::min(want, n / kMinPart));
    const size_t per = (n / parts + 15) & ~size_t{15};
    std::vector<uint32_t> bad(parts, 0), low(parts, 0);
    const bool vec = have_avx512();
    host_parallel_for(static_cast<int>(parts), [&](int p) {
        const size_t a = std::min(n, per * static_cast<size_t>(p));
        const size_t b = p + 1 == static_cast<int>(parts) ? n : std::min(n, a + per);
        if (vec)
            avx512_range(src + a, dst + a, b - a, bad[p], low[p], nt);
        else
            scalar_range(src + a, dst + a, b - a, bad[p], low[p]);
    });
    Bf16Flags f;
    for (size_t p = 0; p < parts; ++p) {
        f.nonfinite = f.nonfinite || bad[p] != 0;
        f.inexact = f.inexact || low[p] != 0;
    }
    return f;
}

}  // namespace csaidx::detail
