// host_plan.cpp -- see host_plan.hpp.
#include "host_plan.hpp"

#include <cmath>

namespace msfft_b200 {

int64_t mod_inverse(int64_t sigma, int64_t n) {
    if (n < 2 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("mod_inverse: n must be a power of two");
    if (sigma % 2 == 0) throw std::invalid_argument("mod_inverse: sigma must be odd");
    // For odd sigma mod 2^k the inverse also follows from Newton's iteration
    // x <- x(2 - sigma x), which doubles the correct low bits each step.
    const uint64_t s = static_cast<uint64_t>(((sigma % n) + n) % n);
    uint64_t x = s;  // correct to 3 bits for odd s
    for (int i = 0; i < 6; ++i) x *= 2 - s * x;
    return static_cast<int64_t>(x & static_cast<uint64_t>(n - 1));
}

void validate_cfg(int64_t l, double q) {
    if (l < 2) throw std::invalid_argument("MultiscaleConfig: l must be >= 2");
    if (q < 0.0) throw std::invalid_argument("MultiscaleConfig: q must be >= 0");
    if (!(static_cast<double>(l) / (q + 1.0) > 1.0))
        throw std::invalid_argument("MultiscaleConfig: l/(q+1) must exceed 1");
}

int64_t tau_schedule(double region_length, int64_t n) {
    const int64_t tau = std::llround(static_cast<double>(n) / region_length);
    return std::clamp<int64_t>(tau, 1, n - 1);
}

int stage_count(double region_length, int64_t l, double q) {
    const double s = static_cast<double>(l) / (q + 1.0);
    int r = 0;
    double acc = 1.0;
    while (acc * (1.0 + 1e-12) < region_length) {
        acc *= s;
        ++r;
    }
    return r;
}

int64_t bucket_of(int64_t u, int64_t l_width, int64_t b) {
    const int64_t i = static_cast<int64_t>(
        std::floor(static_cast<double>(u) / static_cast<double>(l_width) + 0.5));
    return ((i % b) + b) % b;
}

void check_parameter_bounds(double max_dphi, int64_t l, bool* l_ok, double* q_min) {
    if (!(max_dphi > 0.0))
        throw std::invalid_argument("check_parameter_bounds: max_dphi must be positive");
    constexpr double kPi = 3.141592653589793238462643383279502884;
    *l_ok = static_cast<double>(l) <= kPi / max_dphi;
    *q_min = max_dphi * static_cast<double>(l) / kPi;
}

int64_t ceil_log2(int64_t k) {
    int64_t r = 0;
    while ((int64_t{1} << r) < k) ++r;
    return r;
}

void draw_sigmas(uint64_t seed, int64_t n, int iterations, int64_t* sigma, int64_t* sigma_inv) {
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("random_params: bad n");
    HostRng rng(seed);
    for (int m = 0; m < iterations; ++m) {
        sigma[m] = 2 * static_cast<int64_t>(rng.below(static_cast<uint64_t>(n / 2))) + 1;
        sigma_inv[m] = mod_inverse(sigma[m], n);
    }
}

int64_t count_samples_used(const SchedulePlan& plan, const int64_t* sigma) {
    const int64_t n = plan.n;
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    std::vector<uint64_t> seen(static_cast<size_t>((n + 63) / 64), 0);
    int64_t distinct = 0;
    for (int m = 0; m < plan.iterations; ++m) {
        const IterationPlan& it = plan.iters[m];
        const int64_t h = (it.w - 1) / 2;
        // Union of the rounds' shifted intervals t' in [-h - tau, h - tau].
        std::vector<std::pair<int64_t, int64_t>> iv;
        for (int64_t tau : it.taus) iv.emplace_back(-h - tau, h - tau);
        std::sort(iv.begin(), iv.end());
        std::vector<std::pair<int64_t, int64_t>> merged;
        for (const auto& seg : iv) {
            if (!merged.empty() && seg.first <= merged.back().second + 1)
                merged.back().second = std::max(merged.back().second, seg.second);
            else
                merged.push_back(seg);
        }
        const uint64_t s = static_cast<uint64_t>(sigma[m]);
        for (const auto& seg : merged) {
            for (int64_t t = seg.first; t <= seg.second; ++t) {
                const uint64_t src = (s * static_cast<uint64_t>(t)) & mask;
                uint64_t& word = seen[src >> 6];
                const uint64_t bit = uint64_t{1} << (src & 63);
                if (!(word & bit)) {
                    word |= bit;
                    ++distinct;
                }
            }
        }
    }
    return distinct;
}

std::vector<std::pair<int64_t, int64_t>> iteration_union(const IterationPlan& it) {
    const int64_t h = (it.w - 1) / 2;
    std::vector<std::pair<int64_t, int64_t>> iv;
    for (int64_t tau : it.taus) iv.emplace_back(-h - tau, h - tau);
    std::sort(iv.begin(), iv.end());
    std::vector<std::pair<int64_t, int64_t>> merged;
    for (const auto& seg : iv) {
        if (!merged.empty() && seg.first <= merged.back().second + 1)
            merged.back().second = std::max(merged.back().second, seg.second);
        else
            merged.push_back(seg);
    }
    return merged;
}

void gather_traffic(const SchedulePlan& plan, const int64_t* sigma, int elem_bytes,
                    int64_t* loads, int64_t* sectors) {
    const uint64_t mask = static_cast<uint64_t>(plan.n - 1);
    std::vector<uint64_t> sec;
    for (int m = 0; m < plan.iterations; ++m) {
        const auto merged = iteration_union(plan.iters[m]);
        sec.clear();
        const uint64_t s = static_cast<uint64_t>(sigma[m]);
        for (const auto& seg : merged)
            for (int64_t t = seg.first; t <= seg.second; ++t)
                sec.push_back((((s * static_cast<uint64_t>(t)) & mask) * elem_bytes) >> 5);
        *loads += static_cast<int64_t>(sec.size());
        std::sort(sec.begin(), sec.end());
        *sectors += static_cast<int64_t>(std::unique(sec.begin(), sec.end()) - sec.begin());
    }
}

}  // namespace msfft_b200
