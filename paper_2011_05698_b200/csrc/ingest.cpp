// ingest.cpp -- see ingest.hpp.
#include "ingest.hpp"

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
    return hc ? static_cast<int>(hc) : 8;
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
bool block_non_finite(const U* p, int64_t count) {
    constexpr int kBits = 8 * sizeof(U);
    constexpr U kExp = sizeof(U) == 4 ? U(0x7f800000u) : U(0x7ff0000000000000ull);
    constexpr U kOne = sizeof(U) == 4 ? U(0x00800000u) : U(0x0010000000000000ull);
    U acc = 0;
    for (int64_t i = 0; i < count; ++i) acc |= ((p[i] & kExp) + kOne) >> (kBits - 1);
    return acc != 0;
}

}  // namespace

bool gather_compact(HostPool& pool, const IngestMap& map, int64_t n, int iterations,
                    const void* x, int64_t x_stride, int elem_bytes, int64_t count,
                    const int64_t* sigma, void* out, bool validate, int64_t scan_from) {
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const int64_t C = map.per_signal;
    // work items: (signal, iteration) gathers, then validation blocks
    constexpr int64_t kScanBlock = int64_t{1} << 20;  // samples per scan item
    scan_from = std::min(std::max<int64_t>(scan_from, 0), count);
    const int64_t blocks_per_sig = validate ? (n + kScanBlock - 1) / kScanBlock : 0;
    const int64_t gather_items = count * iterations;
    std::atomic<int> bad{0};
    const std::function<void(int64_t)> fn = [&](int64_t item) {
        if (item < gather_items) {
            const int64_t s = item / iterations;
            const int m = static_cast<int>(item - s * iterations);
            const uint64_t sg = static_cast<uint64_t>(sigma[s * iterations + m]);
            const auto& u = map.uni[m];
            const auto& ps = map.pos[m];
            if (elem_bytes == 8) {
                const C64* xs = static_cast<const C64*>(x) + s * x_stride;
                C64* o = static_cast<C64*>(out) + s * C;
                for (size_t i = 0; i < u.size(); ++i)
                    gather_interval(xs, mask, sg, u[i].first, u[i].second, o + ps[i]);
            } else {
                const C128* xs = static_cast<const C128*>(x) + s * x_stride;
                C128* o = static_cast<C128*>(out) + s * C;
                for (size_t i = 0; i < u.size(); ++i)
                    gather_interval(xs, mask, sg, u[i].first, u[i].second, o + ps[i]);
            }
            return;
        }
        const int64_t v = item - gather_items;
        const int64_t s = scan_from + v / blocks_per_sig;
        const int64_t b0 = (v - s * blocks_per_sig) * kScanBlock;
        const int64_t len = std::min(kScanBlock, n - b0);
        bool nf;
        if (elem_bytes == 8)
            nf = block_non_finite(static_cast<const uint32_t*>(x) + 2 * (s * x_stride + b0), 2 * len);
        else
            nf = block_non_finite(static_cast<const uint64_t*>(x) + 2 * (s * x_stride + b0), 2 * len);
        if (nf) bad.store(1, std::memory_order_relaxed);
    };
    pool.run(gather_items + (count - scan_from) * blocks_per_sig, fn);
    return bad.load() != 0;
}

}  // namespace msfft_b200
