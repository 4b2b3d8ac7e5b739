// host_scan_probe.cpp -- read bandwidth of the ingest's finiteness scan on
// the host: the current integer loop, the same with software prefetch, and
// an AVX2 version, at 1 and all threads, over 8 GiB of page-locked-like
// (touched) memory.   g++ -O3 -std=c++17 -pthread host_scan_probe.cpp
#include <immintrin.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static bool scan_plain(const uint32_t* p, int64_t count) {
    uint32_t acc = 0;
    for (int64_t i = 0; i < count; ++i) acc |= ((p[i] & 0x7f800000u) + 0x00800000u) >> 31;
    return acc != 0;
}

static bool scan_prefetch(const uint32_t* p, int64_t count) {
    uint32_t acc = 0;
    constexpr int64_t kAhead = 1024;  // 4 KiB ahead
    for (int64_t i = 0; i < count; i += 16) {
        __builtin_prefetch(p + i + kAhead);
        for (int j = 0; j < 16 && i + j < count; ++j) acc |= ((p[i + j] & 0x7f800000u) + 0x00800000u) >> 31;
    }
    return acc != 0;
}

__attribute__((target("avx2"))) static bool scan_avx2(const uint32_t* p, int64_t count) {
    const __m256i e = _mm256_set1_epi32(0x7f800000), one = _mm256_set1_epi32(0x00800000);
    __m256i acc = _mm256_setzero_si256();
    int64_t i = 0;
    for (; i + 32 <= count; i += 32) {
        for (int k = 0; k < 4; ++k) {
            const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 8 * k));
            acc = _mm256_or_si256(acc, _mm256_add_epi32(_mm256_and_si256(v, e), one));
        }
    }
    uint32_t r = 0;
    for (; i < count; ++i) r |= ((p[i] & 0x7f800000u) + 0x00800000u) >> 31;
    return r != 0 || _mm256_movemask_ps(_mm256_castsi256_ps(acc)) != 0;
}

__attribute__((target("avx512f,avx512dq"))) static bool scan_avx512(const uint32_t* p, int64_t count) {
    const __m512i e = _mm512_set1_epi32(0x7f800000), one = _mm512_set1_epi32(0x00800000);
    __m512i acc = _mm512_setzero_si512();
    int64_t i = 0;
    for (; i + 64 <= count; i += 64)
        for (int k = 0; k < 4; ++k) {
            const __m512i v = _mm512_loadu_si512(p + i + 16 * k);
            acc = _mm512_or_si512(acc, _mm512_add_epi32(_mm512_and_si512(v, e), one));
        }
    uint32_t r = 0;
    for (; i < count; ++i) r |= ((p[i] & 0x7f800000u) + 0x00800000u) >> 31;
    return r != 0 || _mm512_movepi32_mask(acc) != 0;
}

__attribute__((target("avx2"))) static bool scan_avx2_pf(const uint32_t* p, int64_t count) {
    const __m256i e = _mm256_set1_epi32(0x7f800000), one = _mm256_set1_epi32(0x00800000);
    __m256i acc = _mm256_setzero_si256();
    int64_t i = 0;
    for (; i + 32 <= count; i += 32) {
        __builtin_prefetch(p + i + 1024);
        __builtin_prefetch(p + i + 1024 + 16);
        for (int k = 0; k < 4; ++k) {
            const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 8 * k));
            acc = _mm256_or_si256(acc, _mm256_add_epi32(_mm256_and_si256(v, e), one));
        }
    }
    uint32_t r = 0;
    for (; i < count; ++i) r |= ((p[i] & 0x7f800000u) + 0x00800000u) >> 31;
    return r != 0 || _mm256_movemask_ps(_mm256_castsi256_ps(acc)) != 0;
}

int main() {
    const int64_t bytes = int64_t{8} << 30;
    const int64_t words = bytes / 4;
    uint32_t* buf = static_cast<uint32_t*>(std::aligned_alloc(4096, bytes));
    std::memset(buf, 0, bytes);
    const int hw = static_cast<int>(std::thread::hardware_concurrency());
    using Fn = bool (*)(const uint32_t*, int64_t);
    const bool v512 = __builtin_cpu_supports("avx512f");
    const Fn fns[] = {scan_plain, scan_prefetch, scan_avx2, scan_avx2_pf, scan_avx512};
    const char* names[] = {"plain", "prefetch", "avx2", "avx2+pf", "avx512"};
    for (int f = 0; f < (v512 ? 5 : 4); ++f) {
        for (int threads : {1, hw}) {
            std::atomic<int> bad{0};
            const int64_t per = words / threads;
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> ts;
            for (int t = 0; t < threads; ++t)
                ts.emplace_back([&, t] {
                    const int64_t lo = t * per;
                    const int64_t len = threads == 1 ? words / 4 : per;  // 1 thread: 2 GiB
                    if (fns[f](buf + lo, len)) bad = 1;
                });
            for (auto& th : ts) th.join();
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            const double gb = (threads == 1 ? bytes / 4.0 : static_cast<double>(per) * threads * 4) / 1e9;
            std::printf("%-9s threads %3d  %7.1f GB/s%s\n", names[f], threads, gb / s, bad ? " (bad)" : "");
        }
    }
    return 0;
}
