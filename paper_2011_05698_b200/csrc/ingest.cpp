// ingest.cpp -- see ingest.hpp.
#include "ingest.hpp"

#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

namespace msfft_b200 {

int64_t IngestMap::position(int m, int64_t t) const {
    const auto& u = uni[m];
    // last interval with lo <= t
    auto it = std::upper_bound(u.begin(), u.end(), t,
                               [](int64_t v, const std::pair<int64_t, int64_t>& p) {
                                   return v < p.first;
                               });
    if (it == u.begin()) throw std::logic_error("IngestMap: t' below the union");
    --it;
    if (t > it->second) throw std::logic_error("IngestMap: t' outside the union");
    return pos[m][it - u.begin()] + (t - it->first);
}

IngestMap make_ingest_map(const SchedulePlan& plan) {
    IngestMap mp;
    int64_t off = 0;
    for (int m = 0; m < plan.iterations; ++m) {
        mp.uni.push_back(iteration_union(plan.iters[m]));
        std::vector<int64_t> p;
        for (const auto& iv : mp.uni.back()) {
            p.push_back(off);
            off += iv.second - iv.first + 1;
        }
        mp.pos.push_back(std::move(p));
    }
    mp.per_signal = off;
    return mp;
}

HostPool::HostPool(int threads) {
    for (int i = 1; i < std::max(1, threads); ++i) workers_.emplace_back([this] { work(); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void HostPool::drain() {
    for (;;) {
        const int64_t i = next_.fetch_add(1, std::memory_order_acq_rel);
        if (i >= items_.load(std::memory_order_acquire)) break;
        (*fn_.load(std::memory_order_acquire))(i);
    }
}

void HostPool::work() {
    uint64_t seen = 0;
    for (;;) {
        {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            ++active_;
        }
        drain();
        {
            std::lock_guard<std::mutex> lk(mu_);
            if (--active_ == 0) done_cv_.notify_all();
        }
    }
}

void HostPool::run(int64_t items, const std::function<void(int64_t)>& fn) {
    {
        std::lock_guard<std::mutex> lk(mu_);
        fn_.store(&fn);
        items_.store(items);
        next_.store(0);
        ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0 && next_.load() >= items_.load(); });
}

int ingest_threads() {
    if (const char* e = std::getenv("MSFFT_INGEST_THREADS")) {
        const int v = std::atoi(e);
        if (v > 0) return v;
    }
    const unsigned hc = std::thread::hardware_concurrency();
    int threads = hc ? static_cast<int>(hc) : 8;
    // one process per GPU (torchrun): the local ranks share the host cores
    if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
        const int ranks = std::atoi(e);
        if (ranks > 1) threads = std::max(1, threads / ranks);
    }
    return threads;
}

namespace {

// x[(sg * t) mod n] for t in [lo, hi], software-prefetched kDist ahead.
template <class E>
void gather_interval(const E* __restrict__ xs, uint64_t mask, uint64_t sg, int64_t lo, int64_t hi,
                     E* __restrict__ o) {
    constexpr int64_t kDist = 24;
    uint64_t idx = (sg * static_cast<uint64_t>(lo)) & mask;
    uint64_t pf = (idx + static_cast<uint64_t>(kDist) * sg) & mask;
    const int64_t len = hi - lo + 1;
    for (int64_t j = 0; j < len; ++j) {
        __builtin_prefetch(xs + pf);
        o[j] = xs[idx];
        idx = (idx + sg) & mask;
        pf = (pf + sg) & mask;
    }
}

struct C64 {
    float re, im;
};
struct C128 {
    double re, im;
};

// true iff one of the `count` IEEE values has an all-ones exponent (inf or
// NaN); integer-only so the pass vectorizes
template <class U>
bool block_non_finite_scalar(const U* p, int64_t count) {
    constexpr int kBits = 8 * sizeof(U);
    constexpr U kExp = sizeof(U) == 4 ? U(0x7f800000u) : U(0x7ff0000000000000ull);
    constexpr U kOne = sizeof(U) == 4 ? U(0x00800000u) : U(0x0010000000000000ull);
    U acc = 0;
    for (int64_t i = 0; i < count; ++i) acc |= ((p[i] & kExp) + kOne) >> (kBits - 1);
    return acc != 0;
}

// AVX2 version with a 4 KiB software prefetch (measured on the GPU box over
// 16 threads, tools/host_scan_probe.cpp: 131 GB/s vs 121 without the
// prefetch and 100-118 for the scalar loop): exponent field + 1 overflows
// into the sign bit.
__attribute__((target("avx2"))) bool non_finite_avx2_32(const uint32_t* p, int64_t count) {
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
    return _mm256_movemask_ps(_mm256_castsi256_ps(acc)) != 0 ||
           block_non_finite_scalar(p + i, count - i);
}

__attribute__((target("avx2"))) bool non_finite_avx2_64(const uint64_t* p, int64_t count) {
    const __m256i e = _mm256_set1_epi64x(0x7ff0000000000000ll);
    const __m256i one = _mm256_set1_epi64x(0x0010000000000000ll);
    __m256i acc = _mm256_setzero_si256();
    int64_t i = 0;
    for (; i + 16 <= count; i += 16) {
        __builtin_prefetch(p + i + 512);
        __builtin_prefetch(p + i + 512 + 8);
        for (int k = 0; k < 4; ++k) {
            const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(p + i + 4 * k));
            acc = _mm256_or_si256(acc, _mm256_add_epi64(_mm256_and_si256(v, e), one));
        }
    }
    return _mm256_movemask_pd(_mm256_castsi256_pd(acc)) != 0 ||
           block_non_finite_scalar(p + i, count - i);
}

bool has_avx2() {
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}

bool block_non_finite(const uint32_t* p, int64_t count) {
    return has_avx2() ? non_finite_avx2_32(p, count) : block_non_finite_scalar(p, count);
}

bool block_non_finite(const uint64_t* p, int64_t count) {
    return has_avx2() ? non_finite_avx2_64(p, count) : block_non_finite_scalar(p, count);
}

// Compact samples of row s, iteration m (random reads with prefetch).
template <class E>
void gather_row_iteration(const IngestMap& map, int64_t n, int iterations, const void* x,
                          int64_t x_stride, int64_t s, int m, const int64_t* sigma, void* out) {
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const uint64_t sg = static_cast<uint64_t>(sigma[s * iterations + m]);
    const auto& u = map.uni[m];
    const auto& ps = map.pos[m];
    const E* xs = static_cast<const E*>(x) + s * x_stride;
    E* o = static_cast<E*>(out) + s * map.per_signal;
    for (size_t i = 0; i < u.size(); ++i)
        gather_interval(xs, mask, sg, u[i].first, u[i].second, o + ps[i]);
}

constexpr int kFuseShift = 17;  // 2^17-sample blocks: 1 MiB (c64) / 2 MiB (c128)

// Validation scan of row s fused with its gather: the row's compact entries
// are bucketed by source block once, then each block is scanned and its
// entries copied while it is cache-resident.  Returns true on a non-finite
// sample.
template <class E, class U>
bool scan_gather_row(const IngestMap& map, int64_t n, int iterations, const void* x,
                     int64_t x_stride, int64_t s, const int64_t* sigma, void* out) {
    thread_local std::vector<uint32_t> src, dst;
    thread_local std::vector<int64_t> start;
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const int64_t C = map.per_signal;
    int shift = 0;
    while ((int64_t{1} << (shift + 1)) <= n && shift < kFuseShift) ++shift;
    const int64_t nblk = n >> shift;
    src.resize(static_cast<size_t>(C));
    dst.resize(static_cast<size_t>(C));
    start.assign(static_cast<size_t>(nblk + 1), 0);
    // counting sort of (source index, compact position) by source block
    for (int pass = 0; pass < 2; ++pass) {
        for (int m = 0; m < iterations; ++m) {
            const uint64_t sg = static_cast<uint64_t>(sigma[s * iterations + m]);
            const auto& u = map.uni[m];
            const auto& ps = map.pos[m];
            for (size_t i = 0; i < u.size(); ++i) {
                uint64_t idx = (sg * static_cast<uint64_t>(u[i].first)) & mask;
                const int64_t len = u[i].second - u[i].first + 1;
                for (int64_t j = 0; j < len; ++j) {
                    const int64_t bk = static_cast<int64_t>(idx >> shift);
                    if (pass == 0) {
                        ++start[bk + 1];
                    } else {
                        const int64_t at = start[bk]++;
                        src[at] = static_cast<uint32_t>(idx);
                        dst[at] = static_cast<uint32_t>(ps[i] + j);
                    }
                    idx = (idx + sg) & mask;
                }
            }
        }
        if (pass == 0) {
            for (int64_t b = 0; b < nblk; ++b) start[b + 1] += start[b];
        } else {  // the fill advanced start[b] to the end of block b: shift back
            for (int64_t b = nblk; b > 0; --b) start[b] = start[b - 1];
            start[0] = 0;
        }
    }
    const E* xs = static_cast<const E*>(x) + s * x_stride;
    E* o = static_cast<E*>(out) + s * C;
    const int64_t bl = int64_t{1} << shift;
    bool nf = false;
    for (int64_t b = 0; b < nblk; ++b) {
        nf |= block_non_finite(reinterpret_cast<const U*>(xs + b * bl), 2 * bl);
        for (int64_t e = start[b]; e < start[b + 1]; ++e) o[dst[e]] = xs[src[e]];
    }
    return nf;
}

}  // namespace

bool gather_compact(HostPool& pool, const IngestMap& map, int64_t n, int iterations,
                    const void* x, int64_t x_stride, int elem_bytes, int64_t count,
                    const int64_t* sigma, void* out, bool validate, int64_t scan_from) {
    scan_from = validate ? std::min(std::max<int64_t>(scan_from, 0), count) : count;
    static const bool fused = [] {
        const char* e = std::getenv("MSFFT_INGEST_FUSED");
        return !e || std::atoi(e) != 0;
    }();
    // Rows [0, scan_from) need only their samples: one item per (row,
    // iteration), random reads with prefetch.  Rows [scan_from, count) are
    // also scanned for non-finite values: fused, one item per row scans it in
    // cache-sized blocks and copies each block's samples while it is hot;
    // otherwise (MSFFT_INGEST_FUSED=0) gather items for every row plus
    // separate scan items per 2^20-sample block.
    constexpr int64_t kScanBlock = int64_t{1} << 20;
    const int64_t blocks_per_row = (n + kScanBlock - 1) / kScanBlock;
    const int64_t gather_rows = fused ? scan_from : count;
    const int64_t gather_items = gather_rows * iterations;
    const int64_t scan_items = fused ? (count - scan_from) : (count - scan_from) * blocks_per_row;
    std::atomic<int> bad{0};
    const std::function<void(int64_t)> fn = [&](int64_t item) {
        if (item < gather_items) {
            const int64_t s = item / iterations;
            const int m = static_cast<int>(item - s * iterations);
            if (elem_bytes == 8)
                gather_row_iteration<C64>(map, n, iterations, x, x_stride, s, m, sigma, out);
            else
                gather_row_iteration<C128>(map, n, iterations, x, x_stride, s, m, sigma, out);
            return;
        }
        const int64_t v = item - gather_items;
        bool nf;
        if (fused) {
            const int64_t s = scan_from + v;
            nf = elem_bytes == 8 ? scan_gather_row<C64, uint32_t>(map, n, iterations, x, x_stride,
                                                                 s, sigma, out)
                                 : scan_gather_row<C128, uint64_t>(map, n, iterations, x, x_stride,
                                                                  s, sigma, out);
        } else {
            const int64_t r = v / blocks_per_row;
            const int64_t s = scan_from + r;
            const int64_t b0 = (v - r * blocks_per_row) * kScanBlock;
            const int64_t len = std::min(kScanBlock, n - b0);
            nf = elem_bytes == 8
                     ? block_non_finite(static_cast<const uint32_t*>(x) + 2 * (s * x_stride + b0), 2 * len)
                     : block_non_finite(static_cast<const uint64_t*>(x) + 2 * (s * x_stride + b0), 2 * len);
        }
        if (nf) bad.store(1, std::memory_order_relaxed);
    };
    pool.run(gather_items + scan_items, fn);
    return bad.load() != 0;
}

}  // namespace msfft_b200
