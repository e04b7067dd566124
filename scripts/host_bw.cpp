// Host memory bandwidth probe for the e2e entry's host rounding: fp32 ->
// bf16 (RNE, integer AVX-512 like host_convert.cpp) on N threads, over
// buffers backed by huge pages or by 4 KiB pages (as cudaHostAlloc gives),
// with and without software prefetch. Build:
//   g++ -O3 -march=sapphirerapids -pthread scripts/host_bw.cpp -o build_tmp/host_bw
#include <immintrin.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

template <int kPf>
static void convert(const float* src, uint16_t* dst, size_t n) {
    const __m512i bias = _mm512_set1_epi32(0x7fff), one = _mm512_set1_epi32(1);
    for (size_t i = 0; i + 16 <= n; i += 16) {
        if (kPf > 0 && (i & 15) == 0) _mm_prefetch(reinterpret_cast<const char*>(src + i) + kPf, _MM_HINT_T0);
        const __m512i u = _mm512_loadu_si512(src + i);
        const __m512i lsb = _mm512_and_si512(_mm512_srli_epi32(u, 16), one);
        const __m512i r = _mm512_srli_epi32(_mm512_add_epi32(u, _mm512_add_epi32(bias, lsb)), 16);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), _mm512_cvtepi32_epi16(r));
    }
    _mm_sfence();
}

static void* alloc(size_t bytes, bool huge) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p, bytes, huge ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
    std::memset(p, 0, bytes);
    return p;
}

int main(int argc, char** argv) {
    const size_t n = (argc > 1 ? std::atol(argv[1]) : 1024) * (size_t{1} << 20);
    for (int huge = 1; huge >= 0; --huge) {
        float* src = static_cast<float*>(alloc(n * 4, huge));
        uint16_t* dst = static_cast<uint16_t*>(alloc(n * 2, huge));
        for (size_t i = 0; i < n; ++i) src[i] = static_cast<float>(i % 1000) * 0.001f;
        for (int pf : {0, 1024, 4096}) {
            for (int nt : {8, 15}) {
                double best = 1e30;
                for (int rep = 0; rep < 3; ++rep) {
                    auto t0 = std::chrono::steady_clock::now();
                    std::vector<std::thread> th;
                    for (int t = 0; t < nt; ++t)
                        th.emplace_back([&, t] {
                            const size_t a = (n * t / nt) & ~size_t{31};
                            const size_t b = t + 1 == nt ? n : (n * (t + 1) / nt) & ~size_t{31};
                            if (pf == 0) convert<0>(src + a, dst + a, b - a);
                            else if (pf == 1024) convert<1024>(src + a, dst + a, b - a);
                            else convert<4096>(src + a, dst + a, b - a);
                        });
                    for (auto& x : th) x.join();
                    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                    if (s < best) best = s;
                }
                std::printf("%s pages, prefetch %4d B, %2d threads: src %.1f GB/s\n", huge ? "huge" : "4KiB", pf, nt,
                            n * 4.0 / best / 1e9);
            }
        }
        munmap(src, n * 4);
        munmap(dst, n * 2);
    }
    return 0;
}
