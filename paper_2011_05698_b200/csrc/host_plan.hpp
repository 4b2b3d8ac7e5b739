// host_plan.hpp -- the data-independent part of sfft4: parameter checks,
// the sigma draws, the bucket-count halving schedule, stage counts and the
// tau plans.  All of it is a pure function of (n, k, l, q, seed, delta) and
// must be bit-identical to the reference, so it is restated here on the host
// (the GPU never makes these decisions).
#pragma once

#include <algorithm>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace msfft_b200 {

// Rng::below of proj/include/msfft/rng.hpp:34-37: mt19937_64 (sequence pinned
// by the C++ standard) and a 128-bit multiply-shift.
class HostRng {
public:
    explicit HostRng(uint64_t seed) : eng_(seed) {}
    uint64_t u64() { return eng_(); }
    uint64_t below(uint64_t bound) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(u64()) * bound) >> 64);
    }

private:
    std::mt19937_64 eng_;
};

inline bool is_pow2_u(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }

// proj/src/bucketize.cpp:21-37 (extended Euclid mod a power of two).
int64_t mod_inverse(int64_t sigma, int64_t n);

// proj/src/locate.cpp:25-30 (MultiscaleConfig::validate).
void validate_cfg(int64_t l, double q);

// proj/src/locate.cpp:39-42.
int64_t tau_schedule(double region_length, int64_t n);

// proj/src/locate.cpp:44-53.
int stage_count(double region_length, int64_t l, double q);

// proj/src/bucketize.cpp:63-68: round(u/L) mod b, ties away from zero.
int64_t bucket_of(int64_t u, int64_t l_width, int64_t b);

// proj/src/locate.cpp:125-132.  Throws std::invalid_argument for max_dphi <= 0.
void check_parameter_bounds(double max_dphi, int64_t l, bool* l_ok, double* q_min);

// proj/src/sfft4.cpp:14-18, 20-23.
int64_t ceil_log2(int64_t k);
inline int64_t next_bucket_count(int64_t b) { return b > 32 ? b / 2 : b; }

struct IterationPlan {
    int64_t b = 0;          // bucket count b_m
    int64_t l_width = 0;    // L = n / b
    int64_t w = 0;          // window support (odd)
    int64_t k_m = 0;        // expected residual sparsity
    int64_t budget = 0;     // min(k_m, b_m)   (proj/src/sfft4.cpp:77)
    int stages = 0;         // R_m = stage_count(L)
    std::vector<int64_t> taus;  // {0, tau_1..tau_R}   (proj/src/sfft4.cpp:49-55)
};

// Everything of one sfft4 call that does not depend on the signal or the
// seed.  Windows are resolved by the caller-supplied designer (GPU).
struct SchedulePlan {
    int64_t n = 0, k = 0, l = 16;
    double q = 1.0, delta = 1e-8;
    int iterations = 0;
    int64_t b_first = 0;
    std::vector<IterationPlan> iters;
    int64_t values_per_signal = 0;  // sum_m rounds_m * b_m
    int64_t acc_cap = 0;            // sum_m budget_m: bound on |accumulated|
    int64_t samples_round_sum = 0;  // sum_m rounds_m * w_m (TransformStats)
};

// Validates (x length/pow2 is checked by the caller), then builds the
// schedule.  `window_w(n, b, delta)` must return w or throw
// std::invalid_argument exactly like get_flat_window.
template <class WindowW>
SchedulePlan build_schedule(int64_t n, int64_t k, int64_t l, double q, double delta,
                            WindowW&& window_w);

// sigma_m, sigma_inv_m for m < iterations from Rng(seed): random_params(n,
// rng, 0) once per iteration (proj/src/sfft4.cpp:48, bucketize.cpp:39-48).
void draw_sigmas(uint64_t seed, int64_t n, int iterations, int64_t* sigma, int64_t* sigma_inv);

// Distinct sample indices touched by all rounds of one transform
// (SampleTracker, proj/include/msfft/bucketize.hpp:33-44).  It depends only
// on the plan, never on the data.
int64_t count_samples_used(const SchedulePlan& plan, const int64_t* sigma);

// The t' intervals [-h - tau_r, h - tau_r] of all rounds of iteration `it`,
// merged and ascending: the samples x[sigma * t' mod n] one iteration reads.
std::vector<std::pair<int64_t, int64_t>> iteration_union(const IterationPlan& it);

// Algorithmic traffic of the fused gather for one signal: per iteration the
// kernel loads every distinct t' of the union of the rounds' tap intervals
// once.  Adds to *loads the number of such samples and to *sectors the
// number of distinct 32-byte sectors they fall in (elem_bytes per sample).
void gather_traffic(const SchedulePlan& plan, const int64_t* sigma, int elem_bytes,
                    int64_t* loads, int64_t* sectors);

// ---- template definition ----
template <class WindowW>
SchedulePlan build_schedule(int64_t n, int64_t k, int64_t l, double q, double delta,
                            WindowW&& window_w) {
    validate_cfg(l, q);
    if (k < 1 || k > n / 8) throw std::invalid_argument("sfft4: need 1 <= K <= n/8");
    SchedulePlan p;
    p.n = n;
    p.k = k;
    p.l = l;
    p.q = q;
    p.delta = delta;
    p.iterations = static_cast<int>(ceil_log2(k)) + 2;
    // initial_bucket_count (proj/src/sfft4.cpp:115-129).
    int64_t b = 4;
    while (b < 4 * k) b *= 2;
    b = std::min(b, n / 4);
    b = std::max<int64_t>(b, 4);
    int64_t w0 = 0;
    for (;;) {
        try {
            w0 = window_w(n, b, delta);
            break;
        } catch (const std::invalid_argument&) {
            if (b <= 4) throw;
            b /= 2;
        }
    }
    p.b_first = b;
    int64_t k_m = k;
    for (int m = 0; m < p.iterations; ++m) {
        IterationPlan it;
        it.b = b;
        it.l_width = n / b;
        it.w = (m == 0) ? w0 : window_w(n, b, delta);
        it.k_m = k_m;
        it.budget = std::min(k_m, b);
        it.stages = stage_count(static_cast<double>(it.l_width), l, q);
        it.taus.push_back(0);
        double len = static_cast<double>(it.l_width);
        for (int s = 0; s < it.stages; ++s) {
            it.taus.push_back(tau_schedule(len, n));
            len *= (q + 1.0) / static_cast<double>(l);
        }
        const int64_t rounds = static_cast<int64_t>(it.taus.size());
        p.values_per_signal += rounds * b;
        p.acc_cap += it.budget;
        p.samples_round_sum += rounds * it.w;
        p.iters.push_back(std::move(it));
        k_m = (k_m + 1) / 2;
        b = next_bucket_count(b);
    }
    return p;
}

}  // namespace msfft_b200
