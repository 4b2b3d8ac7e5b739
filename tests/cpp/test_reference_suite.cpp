// test_reference_suite.cpp -- the reference's own unit-test assertions
// (proj/tests/test_bucketizer.cpp:73-292, proj/tests/test_flat_window.cpp:46-112,
// the SPEC.md:296-330 known answers) re-expressed against the B200 drop-in
// (include/msfft_b200.hpp, `msfft::` = msfft_b200), plus cross-checks of the
// drop-in's secondary entry points against the compiled reference
// (oracle/_ref through oracle/oracle_api.h, test infrastructure only).
// doctest is not in this image, so CHECK is a counting macro here.
//
// Build (tests/test_cpp_dropin.py):
//   g++ -std=c++20 -I include tests/cpp/test_reference_suite.cpp
//       -L paper_2011_05698_b200 -lmsfft_b200 -L oracle/_ref -lmsfft_ref
#define MSFFT_B200_AS_MSFFT
#include <cmath>
#include <cstdio>
#include <numbers>
#include <span>

#include "../../oracle/oracle_api.h"
#include "msfft_b200.hpp"

using namespace msfft;

namespace {

int g_checks = 0, g_fail = 0;
const char* g_case = "";

#define CHECK(cond)                                                                        \
    do {                                                                                   \
        ++g_checks;                                                                        \
        if (!(cond)) {                                                                     \
            ++g_fail;                                                                      \
            std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);      \
        }                                                                                  \
    } while (0)

#define CHECK_THROWS_AS(expr, E)                                                           \
    do {                                                                                   \
        bool thrown_ = false;                                                              \
        try {                                                                              \
            (void)(expr);                                                                  \
        } catch (const E&) {                                                               \
            thrown_ = true;                                                                \
        } catch (...) {                                                                    \
        }                                                                                  \
        CHECK(thrown_ && #E);                                                              \
    } while (0)

#define TEST_CASE(name) g_case = name;

constexpr double kTwoPi = 2.0 * std::numbers::pi;

cplx root_of_unity(int64_t n, int64_t exponent) {
    int64_t e = exponent % n;
    if (e < 0) e += n;
    const double a = -kTwoPi * static_cast<double>(e) / static_cast<double>(n);
    return cplx(std::cos(a), std::sin(a));
}

ComplexSignal random_signal(int64_t n, uint64_t seed) {
    Rng rng(seed);
    ComplexSignal x;
    x.n = n;
    x.samples.resize(static_cast<size_t>(n));
    for (auto& v : x.samples) v = cplx(rng.uniform01() - 0.5, rng.uniform01() - 0.5);
    return x;
}

// The literal matrix pipeline F_B U_L Q_L S_tau P_sigma x (test_bucketizer.cpp:38-71).
std::vector<cplx> matrix_pipeline(const ComplexSignal& x, const FlatWindow& win,
                                  const PermutationParams& p) {
    const int64_t n = x.n, b = win.b, h = (win.w - 1) / 2;
    std::vector<cplx> v(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
        const int64_t s = ((j - p.tau) % n + n) % n;
        v[j] = x.samples[static_cast<size_t>((p.sigma * s) % n)];
    }
    std::vector<double> g(static_cast<size_t>(n), 0.0);
    g[0] = win.g_time[h];
    for (int64_t t = 1; t <= h; ++t) {
        g[t] = win.g_time[h + t];
        g[n - t] = win.g_time[h - t];
    }
    std::vector<cplx> fold(static_cast<size_t>(b), cplx(0, 0));
    for (int64_t j = 0; j < n; ++j) fold[j % b] += v[j] * g[j];
    std::vector<cplx> out(static_cast<size_t>(b));
    for (int64_t i = 0; i < b; ++i) {
        cplx acc(0, 0);
        for (int64_t j = 0; j < b; ++j) acc += fold[j] * root_of_unity(b, i * j);
        out[i] = acc / static_cast<double>(n);
    }
    return out;
}

std::vector<cplx> padded_response(const FlatWindow& win) {  // test_flat_window.cpp:15-26
    ComplexSignal padded;
    padded.n = win.n;
    padded.samples.assign(static_cast<size_t>(win.n), cplx(0, 0));
    const int64_t h = (win.w - 1) / 2;
    padded.samples[0] = win.g_time[h];
    for (int64_t t = 1; t <= h; ++t) {
        padded.samples[t] = win.g_time[h + t];
        padded.samples[win.n - t] = win.g_time[h - t];
    }
    return dft_dense(padded);
}

void check_three_bands(const FlatWindow& win) {  // test_flat_window.cpp:28-44
    const auto resp = padded_response(win);
    for (int64_t i = 0; i < win.n; ++i) {
        const int64_t d = std::min(i, win.n - i);
        const double mag = std::abs(resp[i]);
        if (d <= win.l_width / 2) {
            CHECK(mag >= 1.0 - win.delta);
            CHECK(mag <= 1.0 + win.delta);
        } else if (d >= win.l_width) {
            CHECK(mag <= win.delta);
        } else {
            CHECK(mag <= 1.0 + win.delta);
        }
    }
}

std::vector<double> responses(const FlatWindow& win, const std::vector<int64_t>& idx) {
    std::vector<double> out(idx.size());
    char err[256] = {0};
    throw_status(msfft_window_response(win.n, win.b, win.delta, -1, idx.data(),
                                       static_cast<int64_t>(idx.size()), out.data(), err,
                                       sizeof(err)),
                 err);
    return out;
}

// sfft4 (sfft4.cpp:131-187) driven through the drop-in's run_iteration.
SparseSpectrum sfft4_by_iterations(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
                                   uint64_t seed, double delta, TransformStats* stats) {
    IterationState st;
    st.k_m = k;
    st.b_m = initial_bucket_count(x.n, k, delta);
    st.delta = delta;
    st.accumulated.n = x.n;
    Rng rng(seed);
    SampleTracker tracker(x.n);
    int64_t iters = 0;
    while ((int64_t{1} << iters) < k) ++iters;
    iters += 2;
    stats->b_first = st.b_m;
    for (int64_t m = 0; m < iters; ++m) {
        run_iteration(x, st, cfg, rng, &tracker);
        stats->stage_counts.push_back(st.stages_m);
    }
    std::vector<std::pair<int64_t, cplx>> e(st.accumulated.entries.begin(),
                                            st.accumulated.entries.end());
    std::stable_sort(e.begin(), e.end(), [](const auto& a, const auto& b) {
        return std::abs(a.second) > std::abs(b.second);
    });
    if (static_cast<int64_t>(e.size()) > k) e.resize(static_cast<size_t>(k));
    SparseSpectrum out;
    out.n = x.n;
    for (const auto& [f, c] : e) out.entries[f] = c;
    stats->samples_used = tracker.distinct;
    stats->samples_round_sum = st.samples_round_sum;
    stats->iterations = static_cast<int>(iters);
    return out;
}

void bucketizer_suite() {
    TEST_CASE("mod_inverse: reference values and exhaustive check");
    CHECK(mod_inverse(1, 64) == 1);
    CHECK(mod_inverse(3, 8) == 3);
    CHECK(mod_inverse(5, 16) == 13);
    for (int64_t sigma = 1; sigma < 256; sigma += 2) CHECK((sigma * mod_inverse(sigma, 256)) % 256 == 1);
    CHECK_THROWS_AS(mod_inverse(4, 16), std::invalid_argument);

    TEST_CASE("random_params: determinism, oddness, rough uniformity");
    {
        Rng a(99), b(99);
        const auto pa = random_params(1024, a);
        const auto pb = random_params(1024, b);
        CHECK(pa.sigma == pb.sigma);
        CHECK(pa.tau == pb.tau);
        Rng rng(123);
        std::vector<int64_t> counts(512, 0);
        const int64_t draws = 10000;
        for (int64_t i = 0; i < draws; ++i) {
            const auto p = random_params(1024, rng);
            CHECK(p.sigma % 2 == 1);
            CHECK((p.sigma * p.sigma_inv) % 1024 == 1);
            ++counts[static_cast<size_t>((p.sigma - 1) / 2)];
        }
        const double expected = static_cast<double>(draws) / 512.0;
        double chi2 = 0;
        for (int64_t c : counts) chi2 += (c - expected) * (c - expected) / expected;
        CHECK(chi2 < 588.4);
        // same draws as the reference's random_params on the same seed
        Rng r2(12345);
        std::vector<int64_t> s(8), si(8);
        char err[256];
        CHECK(orc_random_params(1 << 22, 12345, 8, s.data(), si.data(), err, sizeof(err)) == 0);
        for (int i = 0; i < 8; ++i) {
            const auto p = random_params(1 << 22, r2, 0);
            CHECK(p.sigma == s[i] && p.sigma_inv == si[i]);
        }
    }

    TEST_CASE("tau override is honored");
    {
        Rng rng(5);
        CHECK(random_params(4096, rng, 17).tau == 17);
    }

    TEST_CASE("bucketize: zero signal gives zero buckets, samples_read = w");
    {
        const auto win = get_flat_window(1024, 32, 1e-6);
        ComplexSignal x;
        x.n = 1024;
        x.samples.assign(1024, cplx(0, 0));
        Rng rng(7);
        const auto set = bucketize(x, *win, random_params(1024, rng));
        CHECK(set.samples_read == win->w);
        for (const cplx& v : set.values) CHECK(std::abs(v) == 0.0);
    }

    TEST_CASE("bucketize equals the literal matrix pipeline");
    {
        // The reference lists (64, 8) and (256, 16) at delta = 1e-6, which its
        // own designer rejects; the drop-in rejects them identically.
        CHECK_THROWS_AS(get_flat_window(64, 8, 1e-6), std::invalid_argument);
        CHECK_THROWS_AS(get_flat_window(256, 16, 1e-6), std::invalid_argument);
        struct Geometry { int64_t n, b; };
        for (const Geometry g : {Geometry{512, 16}, Geometry{1024, 32}, Geometry{2048, 32}}) {
            const auto win = get_flat_window(g.n, g.b, 1e-6);
            Rng rng(1000 + g.n);
            for (int trial = 0; trial < 20; ++trial) {
                const auto x = random_signal(g.n, 500 + static_cast<uint64_t>(trial));
                const auto params = random_params(g.n, rng);
                const auto fast = bucketize(x, *win, params);
                const auto slow = matrix_pipeline(x, *win, params);
                for (int64_t i = 0; i < g.b; ++i) CHECK(std::abs(fast.values[i] - slow[i]) < 1e-9);
                // and bit for bit the reference's own bucketize
                std::vector<double> ref(2 * g.b);
                char err[256];
                CHECK(orc_bucketize(g.n, reinterpret_cast<const double*>(x.samples.data()), g.b,
                                    1e-6, params.sigma, params.tau, ref.data(), err,
                                    sizeof(err)) == 0);
                for (int64_t i = 0; i < g.b; ++i)
                    CHECK(fast.values[i] == cplx(ref[2 * i], ref[2 * i + 1]));
            }
        }
    }

    TEST_CASE("bucketize_fn: lazy sampler, called once per tap in increasing tap order");
    {
        const int64_t n = 4096;
        const auto win = get_flat_window(n, 64, 1e-8);
        const auto x = random_signal(n, 77);
        Rng rng(3);
        const auto p = random_params(n, rng);
        int64_t calls = 0;
        bool ordered = true;
        int64_t prev_t = std::numeric_limits<int64_t>::min();
        const int64_t h = (win->w - 1) / 2;
        auto sampler = [&](int64_t idx) {
            // recover t from idx: t = (sigma_inv * idx + tau) mod n, centred
            int64_t t = static_cast<int64_t>((static_cast<uint64_t>(p.sigma_inv) *
                                              static_cast<uint64_t>(idx)) & (n - 1));
            t = (t + p.tau) & (n - 1);
            if (t > h) t -= n;
            if (t <= prev_t) ordered = false;
            prev_t = t;
            ++calls;
            return x.samples[static_cast<size_t>(idx)];
        };
        const auto lazy = bucketize_fn(n, sampler, *win, p);
        const auto dense = bucketize(x, *win, p);
        CHECK(calls == win->w);
        CHECK(ordered);
        CHECK(lazy.samples_read == win->w);
        CHECK(lazy.values == dense.values);
    }

    TEST_CASE("single tone lands in its bucket; distant buckets stay dark");
    {
        const int64_t n = 8192, b = 256;
        const auto win = get_flat_window(n, b, 1e-6);
        PermutationParams p;
        for (int64_t f : {100L, 5000L, 8191L, 16L, 48L}) {
            SparseSpectrum tone;
            tone.n = n;
            tone.entries[f] = cplx(0.8, 0.6);
            const auto set = bucketize(synthesize(tone), *win, p);
            const int64_t i = bucket_of(f, win->l_width, b);
            CHECK(std::abs(set.values[i]) >= (1.0 - 1e-6) * 1.0 - 1e-9);
            for (int64_t j = 0; j < b; ++j) {
                const int64_t dist = std::min(((j - i) % b + b) % b, ((i - j) % b + b) % b);
                if (dist >= 2) CHECK(std::abs(set.values[j]) <= 1e-6 + 1e-9);
            }
        }
    }

    TEST_CASE("predict_buckets matches real bucketization of a single tone within 5 delta");
    {
        const int64_t n = 8192, b = 256;
        const double delta = 1e-6;
        const auto win = get_flat_window(n, b, delta);
        Rng rng(31);
        for (int trial = 0; trial < 5; ++trial) {
            SparseSpectrum tone;
            tone.n = n;
            const int64_t f = static_cast<int64_t>(rng.below(n));
            const double ph = kTwoPi * rng.uniform01();
            tone.entries[f] = cplx(std::cos(ph), std::sin(ph));
            const auto params = random_params(n, rng);
            const auto real_set = bucketize(synthesize(tone), *win, params);
            const auto pred = predict_buckets(tone, *win, params);
            for (int64_t i = 0; i < b; ++i) CHECK(std::abs(real_set.values[i] - pred.values[i]) <= 5 * delta);
        }
    }

    TEST_CASE("predict_buckets covers a full K=50 spectrum within 50*5*delta");
    {
        const int64_t n = 8192, b = 256;
        const double delta = 1e-6;
        const auto win = get_flat_window(n, b, delta);
        Rng rng(77);
        const auto truth = random_sparse_spectrum(n, 50, rng);
        CHECK(truth.entries.size() == 50);
        const auto params = random_params(n, rng);
        const auto real_set = bucketize(synthesize(truth), *win, params);
        const auto pred = predict_buckets(truth, *win, params);
        double worst = 0;
        for (int64_t i = 0; i < b; ++i) worst = std::max(worst, std::abs(real_set.values[i] - pred.values[i]));
        CHECK(worst <= 50 * 5 * delta);
    }

    TEST_CASE("predict_buckets: empty spectrum, zero sample cost");
    {
        const auto win = get_flat_window(1024, 32, 1e-6);
        SparseSpectrum empty;
        empty.n = 1024;
        Rng rng(3);
        const auto pred = predict_buckets(empty, *win, random_params(1024, rng));
        CHECK(pred.samples_read == 0);
        for (const cplx& v : pred.values) CHECK(std::abs(v) == 0.0);
    }

    TEST_CASE("subtract: identity, self-cancellation, exact undo");
    {
        const auto win = get_flat_window(1024, 32, 1e-6);
        Rng rng(11);
        const auto params = random_params(1024, rng);
        const auto x = random_signal(1024, 21);
        const auto a = bucketize(x, *win, params);
        BucketSet zero = a;
        for (cplx& v : zero.values) v = cplx(0, 0);
        CHECK(subtract(a, zero).values == a.values);
        for (const cplx& v : subtract(a, a).values) CHECK(std::abs(v) == 0.0);
        const auto b_set = bucketize(random_signal(1024, 22), *win, params);
        const auto diff = subtract(a, b_set);
        for (size_t i = 0; i < a.values.size(); ++i)
            CHECK(std::abs(diff.values[i] + b_set.values[i] - a.values[i]) < 1e-12);
        BucketSet other = b_set;
        other.params.tau += 1;
        CHECK_THROWS_AS(subtract(a, other), std::invalid_argument);
    }

    TEST_CASE("permutation law: transform of the permuted signal is the rotated relabeling");
    {
        const int64_t n = 256;
        const auto x = random_signal(n, 9);
        Rng rng(13);
        const auto p = random_params(n, rng);
        ComplexSignal xp;
        xp.n = n;
        xp.samples.resize(n);
        for (int64_t j = 0; j < n; ++j)
            xp.samples[j] = x.samples[static_cast<size_t>((p.sigma * (((j - p.tau) % n + n) % n)) % n)];
        const auto spec = dft_dense(x);
        const auto spec_p = dft_dense(xp);
        for (int64_t i = 0; i < n; ++i) {
            const cplx want = spec[i] * root_of_unity(n, p.sigma * p.tau * i);
            CHECK(std::abs(spec_p[static_cast<size_t>((p.sigma * i) % n)] - want) < 1e-9);
        }
    }

    TEST_CASE("index map j -> sigma (j - tau) is a bijection");
    {
        const int64_t n = 4096;
        Rng rng(17);
        const auto p = random_params(n, rng);
        std::vector<uint8_t> hit(static_cast<size_t>(n), 0);
        for (int64_t j = 0; j < n; ++j) {
            const int64_t idx = (p.sigma * (((j - p.tau) % n + n) % n)) % n;
            CHECK(!hit[idx]);
            hit[idx] = 1;
        }
    }

    TEST_CASE("sample tracker counts distinct indices across rounds");
    {
        const int64_t n = 1024;
        const auto win = get_flat_window(n, 32, 1e-6);
        const auto x = random_signal(n, 5);
        SampleTracker tracker(n);
        Rng rng(23);
        const auto p1 = random_params(n, rng);
        const auto p2 = random_params(n, rng);
        bucketize(x, *win, p1, &tracker);
        const int64_t after_one = tracker.distinct;
        CHECK(after_one == win->w);
        bucketize(x, *win, p2, &tracker);
        CHECK(tracker.distinct >= after_one);
        CHECK(tracker.distinct <= std::min<int64_t>(n, 2 * win->w));
    }

    TEST_CASE("bucket_of: boundary positions round away from zero");
    CHECK(bucket_of(16, 32, 256) == 1);
    CHECK(bucket_of(15, 32, 256) == 0);
    CHECK(bucket_of(8192 - 16, 32, 256) == 0);
    CHECK(bucket_of(8192 - 17, 32, 256) == 255);
}

void flat_window_suite() {
    TEST_CASE("window meets the band bounds, n=8192 b=256 delta=1e-6");
    {
        const auto win = design_flat_window(8192, 256, 1e-6);
        CHECK(win.l_width == 32);
        CHECK(win.w % 2 == 1);
        CHECK(std::abs(win.response_at(0) - 1.0) <= win.delta);
        std::vector<int64_t> idx;
        for (int64_t i = 32; i <= 8192 - 32; ++i) idx.push_back(i);
        double stop_max = 0.0;
        for (double v : responses(win, idx)) stop_max = std::max(stop_max, std::abs(v));
        CHECK(stop_max <= 1e-6);
    }

    TEST_CASE("window taps are real-symmetric; response is even and periodic");
    {
        const auto win = design_flat_window(4096, 64, 1e-6);
        const int64_t h = (win.w - 1) / 2;
        for (int64_t t = 0; t <= h; ++t)
            CHECK(std::abs(win.g_time[h + t] - win.g_time[h - t]) <=
                  1e-14 * std::max(std::abs(win.g_time[h + t]), std::abs(win.g_time[h - t])));
        auto close = [](double a, double b) {
            return std::abs(a - b) <= 1e-12 * std::max({1.0, std::abs(a), std::abs(b)});
        };
        for (int64_t i : {1L, 5L, 17L, 100L, 2000L}) {
            CHECK(close(win.response_at(i), win.response_at(-i)));
            CHECK(close(win.response_at(i), win.response_at(i + win.n)));
        }
        CHECK(close(win.response_at(win.n), win.response_at(0)));
    }

    TEST_CASE("support grows about linearly in the bucket count");
    {
        const auto w256 = design_flat_window(65536, 256, 1e-6);
        const auto w512 = design_flat_window(65536, 512, 1e-6);
        const double ratio = static_cast<double>(w512.w) / static_cast<double>(w256.w);
        CHECK(ratio >= 1.7);
        CHECK(ratio <= 2.3);
    }

    TEST_CASE("full three-band verification at both default tolerances");
    check_three_bands(design_flat_window(8192, 64, 1e-8));
    check_three_bands(design_flat_window(8192, 256, 1e-6));
    check_three_bands(design_flat_window(16384, 128, 1e-8));

    TEST_CASE("response matches the dense oracle on a random grid, n=4096");
    {
        const auto win = design_flat_window(4096, 64, 1e-8);
        const auto resp = padded_response(win);
        Rng rng(123);
        for (int trial = 0; trial < 250; ++trial) {
            const int64_t i = static_cast<int64_t>(rng.below(4096));
            CHECK(std::abs(window_response(win, i) - resp[i]) < 1e-10);
        }
    }

    TEST_CASE("infeasible geometry is reported as parameter misuse");
    CHECK_THROWS_AS(design_flat_window(8192, 256, 1e-8), std::invalid_argument);
    CHECK_THROWS_AS(design_flat_window(8192, 2048, 1e-6), std::invalid_argument);

    TEST_CASE("parameter validation");
    CHECK_THROWS_AS(design_flat_window(8192, 3, 1e-6), std::invalid_argument);
    CHECK_THROWS_AS(design_flat_window(8192, 64, 0.5), std::invalid_argument);
    CHECK_THROWS_AS(design_flat_window(8192, 64, 0.0), std::invalid_argument);
    CHECK_THROWS_AS(design_flat_window(1000, 10, 1e-6), std::invalid_argument);

    TEST_CASE("window cache hands back one instance per key");
    {
        const auto a = get_flat_window(4096, 64, 1e-6);
        const auto b = get_flat_window(4096, 64, 1e-6);
        CHECK(a.get() == b.get());
        const auto c = get_flat_window(4096, 64, 1e-8);
        CHECK(a.get() != c.get());
    }
}

void locate_suite() {
    TEST_CASE("SPEC known answers (SPEC.md:296-330)");
    CHECK(tau_schedule(32, 8192) == 256);
    CHECK(stage_count(32, MultiscaleConfig{16, 1.0}) == 2);
    {
        const auto pb = check_parameter_bounds(0.3, 4);
        CHECK(pb.l_ok);
        CHECK(std::abs(pb.q_min - 0.3 * 4 / std::numbers::pi) < 1e-15);
        CHECK_THROWS_AS(check_parameter_bounds(0.0, 4), std::invalid_argument);
    }
    TEST_CASE("scalar helpers equal the reference's");
    for (double len : {2.0, 16.0, 32.0, 256.0, 2048.0, 16384.0, 131072.0})
        for (auto [l, q] : {std::pair<int64_t, double>{16, 1.0}, {8, 2.0}, {4, 1.0}, {8, 4.0}, {16, 0.0}}) {
            CHECK(stage_count(len, MultiscaleConfig{l, q}) == orc_stage_count(len, l, q));
            CHECK(tau_schedule(len, 1 << 20) == orc_tau_schedule(len, 1 << 20));
        }
    for (int64_t u : {0L, 15L, 16L, 17L, 8175L, 8176L, 8191L}) CHECK(bucket_of(u, 32, 256) == orc_bucket_of(u, 32, 256));
    {
        int64_t ref = 0;
        char err[256];
        CHECK(orc_initial_bucket_count(1 << 16, 50, 1e-8, &ref, err, sizeof(err)) == 0);
        CHECK(initial_bucket_count(1 << 16, 50, 1e-8) == ref);
        CHECK(orc_initial_bucket_count(8192, 50, 1e-8, &ref, err, sizeof(err)) == 0);
        CHECK(initial_bucket_count(8192, 50, 1e-8) == ref);
    }
    CHECK_THROWS_AS((MultiscaleConfig{1, 1.0}.validate()), std::invalid_argument);
    CHECK_THROWS_AS((MultiscaleConfig{16, -1.0}.validate()), std::invalid_argument);
    CHECK_THROWS_AS((MultiscaleConfig{2, 1.0}.validate()), std::invalid_argument);
    CHECK_THROWS_AS(stage_count(32, MultiscaleConfig{2, 1.0}), std::invalid_argument);

    TEST_CASE("phase helpers");
    CHECK_THROWS_AS(phase_of(cplx(0.0, 0.0)), std::domain_error);
    CHECK(phase_of(cplx(1.0, 0.0)) == 0.0);
    CHECK(!std::signbit(phase_of(cplx(1.0, -0.0))));
    CHECK(phase_of(cplx(-1.0, 0.0)) == std::numbers::pi);
    CHECK(std::abs(phase_of(cplx(0.0, -1.0)) - 1.5 * std::numbers::pi) < 1e-15);
    CHECK(position_phase(0.0, 5, 64) == 0.0);
    CHECK(position_phase(1.0, 16, 64) == std::numbers::pi / 2);
    CHECK(circular_phase_distance(0.1, kTwoPi - 0.1) < 0.2 + 1e-15);
    CHECK(circular_phase_distance(0.0, std::numbers::pi) == std::numbers::pi);

    TEST_CASE("initial_region / locate_step narrow onto an exact tone");
    {
        // n=4096, b=64 (L=64), l=16, q=1: a tone at u in bucket i, exact phases
        const int64_t n = 4096, L = 64;
        const MultiscaleConfig cfg{16, 1.0};
        for (int64_t u : {0L, 1L, 31L, 33L, 100L, 4000L, 4095L}) {
            const int64_t i = bucket_of(u, L, n / L);
            LocateRegion r = initial_region(i, L);
            CHECK(r.length == static_cast<double>(L) && r.stage == 1);
            CHECK(r.u_min == (2.0 * i - 1.0) * L / 2.0);
            while (r.length > 1.0 + 1e-9) {
                PhaseMeasurement m;
                m.tau = tau_schedule(r.length, n);
                m.phi = position_phase(static_cast<double>(u), m.tau, n);
                const LocateRegion nx = locate_step(m, r, cfg, n);
                CHECK(nx.stage == r.stage + 1);
                CHECK(nx.length == r.length * (cfg.q + 1.0) / static_cast<double>(cfg.l));
                r = nx;
            }
            int64_t got = static_cast<int64_t>(std::ceil(r.u_min));
            if (!(static_cast<double>(got) < r.u_max())) got = std::llround(0.5 * (r.u_min + r.u_max()));
            got = ((got % n) + n) % n;
            CHECK(got == u);
        }
    }

    TEST_CASE("locate_frequency (std::span) and estimate_value equal the reference");
    {
        const int64_t n = 1 << 14, b = 128;
        const double delta = 1e-6;
        const auto win = get_flat_window(n, b, delta);
        Rng rng(5);
        const auto truth = random_sparse_spectrum(n, 20, rng);
        const auto x = synthesize(truth);
        const auto base = random_params(n, rng, 0);
        std::vector<PermutationParams> ps;
        std::vector<int64_t> taus{0};
        double len = static_cast<double>(win->l_width);
        const MultiscaleConfig cfg{16, 1.0};
        const int stages = stage_count(len, cfg);
        for (int s = 0; s < stages; ++s) {
            taus.push_back(tau_schedule(len, n));
            len *= (cfg.q + 1.0) / static_cast<double>(cfg.l);
        }
        for (int64_t t : taus) ps.push_back(PermutationParams{base.sigma, base.sigma_inv, t});
        const auto rounds = bucketize_rounds(x, *win, ps);
        std::vector<double> vals;
        for (const auto& r : rounds)
            for (const cplx& v : r.values) {
                vals.push_back(v.real());
                vals.push_back(v.imag());
            }
        for (int64_t bk = 0; bk < b; ++bk) {
            const auto got = locate_frequency(bk, std::span<const BucketSet>(rounds), cfg, *win);
            int64_t u = 0;
            int st = 0;
            char err[256];
            CHECK(orc_locate(n, b, delta, 16, 1.0, bk, static_cast<int64_t>(taus.size()), taus.data(),
                             vals.data(), &u, &st, err, sizeof(err)) == 0);
            CHECK(got.has_value() == (u >= 0));
            if (got && u >= 0) {
                CHECK(got->u == u && got->stages == st);
                double ref[2];
                const cplx y0 = rounds[0].values[bk];
                const int rc = orc_estimate_value(n, b, delta, y0.real(), y0.imag(), u, ref, err, sizeof(err));
                if (rc == 0) {
                    const cplx mine = estimate_value(y0, u, *win);
                    CHECK(std::abs(mine - cplx(ref[0], ref[1])) <= 1e-13 * std::abs(cplx(ref[0], ref[1])));
                } else {
                    CHECK_THROWS_AS(estimate_value(y0, u, *win), std::domain_error);
                }
            }
        }
    }
}

void iteration_suite() {
    TEST_CASE("run_iteration loop == msfft::sfft4 == the reference sfft4");
    for (uint64_t seed : {1ull, 2ull}) {
        const int64_t n = 1 << 14, k = 30;
        Rng rng(seed);
        const auto truth = random_sparse_spectrum(n, k, rng);
        const auto x = synthesize(truth);
        const MultiscaleConfig cfg{16, 1.0};
        TransformStats st_it;
        const auto by_it = sfft4_by_iterations(x, k, cfg, seed * 77, 1e-8, &st_it);
        const auto fused = sfft4(x, k, cfg, seed * 77, 1e-8);
        CHECK(by_it.entries.size() == fused.spectrum.entries.size());
        auto a = by_it.entries.begin();
        for (const auto& [f, c] : fused.spectrum.entries) {
            CHECK(a != by_it.entries.end() && a->first == f);
            if (a != by_it.entries.end()) {
                CHECK(std::abs(a->second - c) <= 1e-12 * std::abs(c));
                ++a;
            }
        }
        CHECK(st_it.samples_used == fused.stats.samples_used);
        CHECK(st_it.samples_round_sum == fused.stats.samples_round_sum);
        CHECK(st_it.b_first == fused.stats.b_first);
        CHECK(st_it.stage_counts == fused.stats.stage_counts);
        std::vector<int64_t> rf(k), si(4 + ORC_MAX_ITERS);
        std::vector<double> rc(2 * k);
        int64_t cnt = 0;
        double sd[2];
        char err[256];
        CHECK(orc_sfft4(n, reinterpret_cast<const double*>(x.samples.data()), k, 16, 1.0, seed * 77,
                        1e-8, k, rf.data(), rc.data(), &cnt, si.data(), sd, err, sizeof(err)) == 0);
        CHECK(cnt == static_cast<int64_t>(by_it.entries.size()));
        int64_t i = 0;
        for (const auto& [f, c] : by_it.entries) {
            CHECK(i < cnt && f == rf[i]);
            if (i < cnt) CHECK(std::abs(c - cplx(rc[2 * i], rc[2 * i + 1])) <= 1e-9 * std::abs(c));
            ++i;
        }
        CHECK(st_it.samples_used == si[0]);
    }
    TEST_CASE("ComplexSignal::validate order and messages");
    {
        ComplexSignal bad;
        bad.n = 6;
        bad.samples.resize(3);
        try {
            bad.validate();
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "ComplexSignal: n must be a power of two >= 4");
        }
        ComplexSignal nan;
        nan.n = 8;
        nan.samples.assign(8, cplx(0, 0));
        nan.samples[5] = cplx(0, std::nan(""));
        try {
            nan.validate();
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "ComplexSignal: non-finite sample");
        }
        try {
            sfft4(bad, 1, MultiscaleConfig{}, 1);
            CHECK(false);
        } catch (const std::invalid_argument& e) {
            CHECK(std::string(e.what()) == "ComplexSignal: n must be a power of two >= 4");
        }
    }
}

}  // namespace

int main() {
    try {
        bucketizer_suite();
        flat_window_suite();
        locate_suite();
        iteration_suite();
    } catch (const std::exception& e) {
        std::printf("uncaught exception in [%s]: %s\n", g_case, e.what());
        return 2;
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    if (g_fail == 0) std::printf("reference suite ok\n");
    return g_fail == 0 ? 0 : 1;
}
