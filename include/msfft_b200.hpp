// msfft_b200.hpp -- header-only C++ drop-in over the C ABI (msfft_b200.h).
//
// Mirrors the reference's public types and entry point
//   SfftResult sfft4(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
//                    uint64_t seed, double delta = 1e-8);
// (proj/include/msfft/sfft4.hpp:32-45, 64-65; signal.hpp:13-28;
// locate.hpp:13-19) with the same field names, the same ascending std::map
// result and the same exception classes/messages -- and the functions its
// callers use around the transform: signal.hpp:31-70 (dft_dense,
// idft_dense, synthesize, generate_test_signal, add_awgn, error_metrics),
// io.hpp:11-17 (signal files, truth CSV), phase_mc.hpp:19-56
// (run_phase_experiment) and bench.cpp:33-46 (top_k_spectrum) -- and the
// component API on the path (get_flat_window, bucketize, predict_buckets,
// subtract, locate_frequency, estimate_value).  A caller of the reference
// switches by including this header and linking libmsfft_b200.so; defining
// MSFFT_B200_AS_MSFFT before the include also makes `msfft::` name these
// types (only when the reference headers are not included in the same TU).
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <optional>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>
#include <vector>
#if __cplusplus >= 202002L
#include <span>
#endif

#include "msfft_b200.h"

namespace msfft_b200 {

using cplx = std::complex<double>;

inline bool is_pow2(uint64_t n) { return n != 0 && (n & (n - 1)) == 0; }  // fft.hpp

// Thrown for device / CUDA failures (no CPU fallback exists).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void throw_status(int status, const char* msg) {
    switch (status) {
        case MSFFT_OK: return;
        case MSFFT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MSFFT_ERR_DOMAIN: throw std::domain_error(msg);
        case MSFFT_ERR_CUDA: throw DeviceError(msg);
        default: throw std::runtime_error(msg);
    }
}

// ---- seeded randomness (proj/include/msfft/rng.hpp:9-59) --------------------
// Host-side like the reference: every draw a caller's code makes from its Rng
// (random_params, random_sparse_spectrum, its own test signals) must consume
// the same mt19937_64 stream (sequence fixed by the C++ standard).
inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

class Rng {
public:
    explicit Rng(uint64_t seed) : eng_(seed) {}
    static Rng stream(uint64_t master, uint64_t tag) { return Rng(splitmix64(master ^ splitmix64(tag))); }
    uint64_t u64() { return eng_(); }
    double uniform01() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t bound) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(u64()) * bound) >> 64);
    }
    double gaussian() {  // Box-Muller, second variate cached
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        double u1 = uniform01();
        const double u2 = uniform01();
        while (u1 == 0.0) u1 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare_ = r * std::sin(a);
        spare_ok_ = true;
        return r * std::cos(a);
    }

private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool spare_ok_ = false;
};

struct ComplexSignal {  // signal.hpp:13-18
    int64_t n = 0;
    std::vector<cplx> samples;
    // ComplexSignal::validate (signal.cpp:18-26): pow2 n >= 4, size == n,
    // every sample finite -- in that order, the reference's messages.
    void validate() const {
        char err[256] = {0};
        throw_status(msfft_validate_signal(samples.data(), n, static_cast<int64_t>(samples.size()),
                                           1, n, MSFFT_C128, MSFFT_HOST, nullptr, nullptr, err,
                                           sizeof(err)),
                     err);
    }
};

struct SparseSpectrum {  // signal.hpp:23-28
    int64_t n = 0;
    std::map<int64_t, cplx> entries;
    void validate() const {  // signal.cpp:28-39
        if (n < 4 || !is_pow2(static_cast<uint64_t>(n)))
            throw std::invalid_argument("SparseSpectrum: n must be a power of two >= 4");
        if (static_cast<int64_t>(entries.size()) > n)
            throw std::invalid_argument("SparseSpectrum: more entries than n");
        for (const auto& [f, c] : entries) {
            if (f < 0 || f >= n) throw std::invalid_argument("SparseSpectrum: position out of range");
            if (!std::isfinite(c.real()) || !std::isfinite(c.imag()))
                throw std::invalid_argument("SparseSpectrum: non-finite coefficient");
        }
    }
};

struct MultiscaleConfig {  // locate.hpp:13-19
    int64_t l = 16;
    double q = 1.0;
    double shrink() const { return static_cast<double>(l) / (q + 1.0); }
    void validate() const {  // locate.cpp:25-30
        char err[256] = {0};
        throw_status(msfft_config_validate(l, q, err, sizeof(err)), err);
    }
};

struct TransformStats {
    int64_t samples_used = 0;
    int64_t samples_round_sum = 0;
    double sample_fraction = 0.0;
    double runtime_ms = 0.0;  // device time of the transform
    int iterations = 0;
    int64_t b_first = 0;
    std::vector<int> stage_counts;
};

struct SfftResult {
    SparseSpectrum spectrum;
    TransformStats stats;
};

inline SfftResult sfft4(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
                        uint64_t seed, double delta = 1e-8) {
    // ComplexSignal::validate's first two checks, in its order (signal.cpp:19-22);
    // finiteness is scanned by the library
    if (x.n < 4 || !is_pow2(static_cast<uint64_t>(x.n)))
        throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
    if (static_cast<int64_t>(x.samples.size()) != x.n)
        throw std::invalid_argument("ComplexSignal: sample count != n");
    const int64_t cap = k > 0 ? k : 1;
    std::vector<int64_t> f(static_cast<size_t>(cap));
    std::vector<double> c(static_cast<size_t>(2 * cap));
    int64_t count = 0;
    msfft_stats st{};
    char err[1024] = {0};
    const int rc = msfft_sfft4(x.samples.data(), x.n, MSFFT_C128, MSFFT_HOST, k, cfg.l, cfg.q,
                               seed, delta, cap, f.data(), c.data(), &count, &st, err,
                               sizeof(err));
    throw_status(rc, err);
    SfftResult r;
    r.spectrum.n = x.n;
    for (int64_t i = 0; i < count; ++i) r.spectrum.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    r.stats.samples_used = st.samples_used;
    r.stats.samples_round_sum = st.samples_round_sum;
    r.stats.sample_fraction = st.sample_fraction;
    r.stats.runtime_ms = st.runtime_ms;
    r.stats.iterations = st.iterations;
    r.stats.b_first = st.b_first;
    r.stats.stage_counts.assign(st.stage_counts, st.stage_counts + st.iterations);
    return r;
}

// ---- around the transform ----------------------------------------------------

struct EvalMetrics {  // signal.hpp:31-38
    int64_t l0_err = 0;
    double l1_err = 0.0;
    double l2_err = 0.0;
    double runtime_ms = 0.0;
    int64_t samples_used = 0;
    double sample_fraction = 0.0;
};

namespace detail {
inline void spectrum_arrays(const SparseSpectrum& s, std::vector<int64_t>& f,
                            std::vector<double>& c) {
    f.clear();
    c.clear();
    for (const auto& [pos, v] : s.entries) {
        f.push_back(pos);
        c.push_back(v.real());
        c.push_back(v.imag());
    }
}
inline ComplexSignal signal_of(std::vector<double>& xi, int64_t n) {
    ComplexSignal x;
    x.n = n;
    x.samples.resize(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) x.samples[j] = cplx(xi[2 * j], xi[2 * j + 1]);
    return x;
}
}  // namespace detail

// Forward transform with the 1/n factor (bit-identical to the reference).
inline std::vector<cplx> dft_dense(const ComplexSignal& x) {
    if (static_cast<int64_t>(x.samples.size()) != x.n)
        throw std::invalid_argument("ComplexSignal: sample count != n");
    std::vector<cplx> out(x.samples.size());
    char err[1024] = {0};
    throw_status(msfft_dft_dense(x.samples.data(), x.n, 1, MSFFT_C128, MSFFT_HOST,
                                 reinterpret_cast<double*>(out.data()), err, sizeof(err)),
                 err);
    return out;
}

inline ComplexSignal idft_dense(const std::vector<cplx>& spectrum) {
    ComplexSignal x;
    x.n = static_cast<int64_t>(spectrum.size());
    x.samples.resize(spectrum.size());
    char err[1024] = {0};
    throw_status(msfft_idft_dense(reinterpret_cast<const double*>(spectrum.data()), x.n, 1,
                                  MSFFT_HOST, reinterpret_cast<double*>(x.samples.data()), err,
                                  sizeof(err)),
                 err);
    return x;
}

inline ComplexSignal synthesize(const SparseSpectrum& spec) {
    std::vector<int64_t> f;
    std::vector<double> c;
    detail::spectrum_arrays(spec, f, c);
    ComplexSignal x;
    x.n = spec.n;
    x.samples.resize(static_cast<size_t>(spec.n > 0 ? spec.n : 0));
    char err[1024] = {0};
    throw_status(msfft_synthesize(spec.n, f.data(), c.data(), static_cast<int64_t>(f.size()),
                                  MSFFT_C128, MSFFT_HOST, x.samples.data(), nullptr, err,
                                  sizeof(err)),
                 err);
    return x;
}

// random_sparse_spectrum (signal.cpp:100-121): Floyd's sampling of k distinct
// positions then a uniform phase per position (ascending), drawn from the
// caller's Rng -- host-side, since the caller's stream must advance exactly
// as the reference's does.
inline SparseSpectrum random_sparse_spectrum(int64_t n, int64_t k, Rng& rng) {
    if (n < 4 || !is_pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("random_sparse_spectrum: bad n");
    if (k < 0 || k > n) throw std::invalid_argument("random_sparse_spectrum: k out of range");
    std::set<int64_t> pos;
    for (int64_t j = n - k; j < n; ++j) {
        const int64_t t = static_cast<int64_t>(rng.below(static_cast<uint64_t>(j) + 1));
        if (!pos.insert(t).second) pos.insert(j);
    }
    SparseSpectrum s;
    s.n = n;
    for (int64_t f : pos) {
        const double ph = 6.283185307179586476925286766559 * rng.uniform01();
        s.entries[f] = cplx(std::cos(ph), std::sin(ph));
    }
    return s;
}

// Same truth (positions, coefficients) as the reference; samples bit-identical
// while k * ceil(n/1024) <= 2^23.
inline std::pair<ComplexSignal, SparseSpectrum> generate_test_signal(int64_t n, int64_t k,
                                                                     uint64_t seed) {
    std::vector<cplx> xs(static_cast<size_t>(n > 0 ? n : 0));
    std::vector<int64_t> f(static_cast<size_t>(k > 0 ? k : 1));
    std::vector<double> c(2 * f.size());
    char err[1024] = {0};
    throw_status(msfft_generate_test_signal(n, k, seed, MSFFT_C128, MSFFT_HOST, xs.data(),
                                            f.data(), c.data(), nullptr, err, sizeof(err)),
                 err);
    std::pair<ComplexSignal, SparseSpectrum> out;
    out.first.n = n;
    out.first.samples = std::move(xs);
    out.second.n = n;
    for (int64_t i = 0; i < k; ++i) out.second.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    return out;
}

// Same validation, sentinel and realised-power scaling as the reference; the
// Gaussian noise comes from a counter-based generator (same law, not the
// same samples as the reference's mt19937_64 stream).
inline ComplexSignal add_awgn(const ComplexSignal& x, double snr_db, uint64_t seed) {
    ComplexSignal y = x;
    char err[1024] = {0};
    throw_status(msfft_add_awgn(y.samples.data(), y.n, MSFFT_C128, MSFFT_HOST, snr_db, seed, err,
                                sizeof(err)),
                 err);
    return y;
}

inline EvalMetrics error_metrics(const SparseSpectrum& truth, const SparseSpectrum& estimate,
                                 int64_t k) {
    std::vector<int64_t> tf, ef;
    std::vector<double> tc, ec;
    detail::spectrum_arrays(truth, tf, tc);
    detail::spectrum_arrays(estimate, ef, ec);
    msfft_eval_metrics m{};
    char err[1024] = {0};
    throw_status(msfft_error_metrics(truth.n, tf.data(), tc.data(), static_cast<int64_t>(tf.size()),
                                     estimate.n, ef.data(), ec.data(),
                                     static_cast<int64_t>(ef.size()), k, &m, err, sizeof(err)),
                 err);
    EvalMetrics r;
    r.l0_err = m.l0_err;
    r.l1_err = m.l1_err;
    r.l2_err = m.l2_err;
    return r;
}

// Top-k magnitudes of a dense spectrum as a sparse estimate (bench.cpp:33-46).
inline SparseSpectrum top_k_spectrum(const std::vector<cplx>& spectrum, int64_t n, int64_t k) {
    const int64_t cap = k > 0 ? k : 1;
    std::vector<int64_t> f(static_cast<size_t>(cap));
    std::vector<double> c(static_cast<size_t>(2 * cap));
    int64_t count = 0;
    char err[1024] = {0};
    throw_status(msfft_top_k_spectrum(reinterpret_cast<const double*>(spectrum.data()),
                                      static_cast<int64_t>(spectrum.size()), k, MSFFT_HOST,
                                      f.data(), c.data(), &count, err, sizeof(err)),
                 err);
    SparseSpectrum out;
    out.n = n;
    for (int64_t i = 0; i < count; ++i) out.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    return out;
}

inline void write_signal_file(const std::string& path, const ComplexSignal& x) {
    char err[1024] = {0};
    throw_status(msfft_write_signal_file(path.c_str(), x.samples.data(), x.n, MSFFT_C128,
                                         MSFFT_HOST, err, sizeof(err)),
                 err);
}

inline ComplexSignal read_signal_file(const std::string& path) {
    char err[1024] = {0};
    int64_t n = 0;
    throw_status(msfft_signal_file_length(path.c_str(), &n, err, sizeof(err)), err);
    ComplexSignal x;
    x.n = n;
    x.samples.resize(static_cast<size_t>(n));
    int64_t got = 0;
    throw_status(msfft_read_signal_file(path.c_str(), MSFFT_C128, MSFFT_HOST, x.samples.data(), n,
                                        &got, err, sizeof(err)),
                 err);
    return x;
}

inline void write_truth_csv(const std::string& path, const SparseSpectrum& truth) {
    std::vector<int64_t> f;
    std::vector<double> c;
    detail::spectrum_arrays(truth, f, c);
    char err[1024] = {0};
    throw_status(msfft_write_truth_csv(path.c_str(), f.data(), c.data(),
                                       static_cast<int64_t>(f.size()), err, sizeof(err)),
                 err);
}

inline SparseSpectrum read_truth_csv(const std::string& path, int64_t n) {
    char err[1024] = {0};
    int64_t count = 0;
    std::vector<int64_t> f(1);
    std::vector<double> c(2);
    throw_status(msfft_read_truth_csv(path.c_str(), n, f.data(), c.data(), 0, &count, err,
                                      sizeof(err)),
                 err);
    f.resize(static_cast<size_t>(count > 0 ? count : 1));
    c.resize(2 * f.size());
    throw_status(msfft_read_truth_csv(path.c_str(), n, f.data(), c.data(), count, &count, err,
                                      sizeof(err)),
                 err);
    SparseSpectrum s;
    s.n = n;
    for (int64_t i = 0; i < count; ++i) s.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    return s;
}

struct PhaseErrorHistogram {  // phase_mc.hpp:19-30
    double snr_db = 0.0;
    int64_t n = 0, k = 0, l_width = 0;
    int64_t trials = 0;
    std::vector<double> bin_mass;
    double p50 = 0.0, p99 = 0.0, max = 0.0;
    static constexpr double kBinLo = -6.0;
    static constexpr double kBinWidth = 0.1;
    static constexpr int kBinCount = MSFFT_PHASE_BINS;
    static double bin_center(int i) { return kBinLo + kBinWidth * (i + 0.5); }
};

inline std::vector<PhaseErrorHistogram> run_phase_experiment(int64_t n, int64_t k, int64_t b,
                                                             const std::vector<double>& snr_list,
                                                             int64_t trials, uint64_t seed) {
    std::vector<msfft_phase_histogram> hs(snr_list.size() ? snr_list.size() : 1);
    char err[1024] = {0};
    throw_status(msfft_phase_experiment(n, k, b, snr_list.data(),
                                        static_cast<int64_t>(snr_list.size()), trials, seed,
                                        hs.data(), nullptr, err, sizeof(err)),
                 err);
    std::vector<PhaseErrorHistogram> out;
    for (size_t i = 0; i < snr_list.size(); ++i) {
        PhaseErrorHistogram h;
        h.snr_db = hs[i].snr_db;
        h.n = hs[i].n;
        h.k = hs[i].k;
        h.l_width = hs[i].l_width;
        h.trials = hs[i].trials;
        h.bin_mass.assign(hs[i].bin_mass, hs[i].bin_mass + MSFFT_PHASE_BINS);
        h.p50 = hs[i].p50;
        h.p99 = hs[i].p99;
        h.max = hs[i].max;
        out.push_back(std::move(h));
    }
    return out;
}

// ---- component API on the path (bucketize.hpp:56-95, locate.hpp:75-78,
// sfft4.hpp:50): the functions the reference's own tests call directly ------

struct FlatWindow {  // window.hpp:16-30 (taps as designed; G_d lives on the device)
    int64_t n = 0, b = 0, l_width = 0, w = 0;
    double delta = 0.0;
    double eps = 0.0;        // L/n
    double eps_prime = 0.0;  // L/(2n)
    std::vector<double> g_time;
    // window.cpp:89-99, evaluated on the GPU (the series the decode's table uses)
    double response_at(int64_t i) const {
        double out = 0.0;
        char err[512] = {0};
        throw_status(msfft_window_response(n, b, delta, -1, &i, 1, &out, err, sizeof(err)), err);
        return out;
    }
};

// design_flat_window (window.cpp:105-177): designed on the GPU, taps
// bit-identical to the reference's; the same std::invalid_argument messages.
inline FlatWindow design_flat_window(int64_t n, int64_t b, double delta) {
    FlatWindow win;
    char err[1024] = {0};
    int64_t w = 0;
    throw_status(msfft_window(n, b, delta, -1, &w, nullptr, 0, err, sizeof(err)), err);
    win.g_time.resize(static_cast<size_t>(w));
    throw_status(msfft_window(n, b, delta, -1, &w, win.g_time.data(), w, err, sizeof(err)), err);
    win.n = n;
    win.b = b;
    win.l_width = n / b;
    win.w = w;
    win.delta = delta;
    win.eps = static_cast<double>(win.l_width) / static_cast<double>(n);
    win.eps_prime = win.eps / 2.0;
    return win;
}

inline cplx window_response(const FlatWindow& win, int64_t i) {  // window.cpp:100-102
    return cplx(win.response_at(i), 0.0);
}

// get_flat_window (window.cpp:179-193): one instance per (n, b, delta) for the
// process; construction outside the lock, lookups synchronized.
inline std::shared_ptr<const FlatWindow> get_flat_window(int64_t n, int64_t b, double delta) {
    using Key = std::tuple<int64_t, int64_t, double>;
    static std::mutex mu;
    static std::map<Key, std::shared_ptr<const FlatWindow>> cache;
    const Key key{n, b, delta};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    auto win = std::make_shared<const FlatWindow>(design_flat_window(n, b, delta));
    std::lock_guard<std::mutex> lock(mu);
    return cache.emplace(key, win).first->second;
}

struct PermutationParams {  // bucketize.hpp:16-20
    int64_t sigma = 1, sigma_inv = 1, tau = 0;
};

struct BucketSet {  // bucketize.hpp:24-30
    int64_t n = 0, b = 0;
    std::vector<cplx> values;
    PermutationParams params;
    int64_t samples_read = 0;
};

struct SampleTracker {  // bucketize.hpp:33-44
    std::vector<uint8_t> seen;
    int64_t distinct = 0;
    explicit SampleTracker(int64_t n) : seen(static_cast<size_t>(n), 0) {}
    void touch(int64_t idx) {
        if (!seen[static_cast<size_t>(idx)]) {
            seen[static_cast<size_t>(idx)] = 1;
            ++distinct;
        }
    }
};

// mod_inverse (bucketize.cpp:21-37): the library's own (plan) implementation.
inline int64_t mod_inverse(int64_t sigma, int64_t n) {
    int64_t out = 0;
    char err[256] = {0};
    throw_status(msfft_mod_inverse(sigma, n, &out, err, sizeof(err)), err);
    return out;
}

// random_params (bucketize.cpp:39-48): one below(n/2) draw for sigma, one
// below(n) for tau unless overridden -- from the caller's Rng.
inline PermutationParams random_params(int64_t n, Rng& rng,
                                       std::optional<int64_t> tau_override = std::nullopt) {
    if (n < 4 || !is_pow2(static_cast<uint64_t>(n))) throw std::invalid_argument("random_params: bad n");
    PermutationParams p;
    p.sigma = 2 * static_cast<int64_t>(rng.below(static_cast<uint64_t>(n / 2))) + 1;
    p.sigma_inv = mod_inverse(p.sigma, n);
    p.tau = tau_override ? *tau_override : static_cast<int64_t>(rng.below(static_cast<uint64_t>(n)));
    return p;
}

// bucket_of (bucketize.cpp:63-68): round(u/L) mod b, ties away from zero.
inline int64_t bucket_of(int64_t u, int64_t l_width, int64_t b) {
    return msfft_bucket_of(u, l_width, b);
}

namespace detail {
// The source index of tap t: sigma * ((t - tau) mod n) mod n (bucketize.hpp:70-71).
inline int64_t tap_source(int64_t t, const PermutationParams& p, int64_t n) {
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const uint64_t s = static_cast<uint64_t>(t - p.tau) & mask;
    return static_cast<int64_t>((static_cast<uint64_t>(p.sigma) * s) & mask);
}
inline BucketSet bucket_set(int64_t n, int64_t b, const cplx* vals, const PermutationParams& p,
                            int64_t samples_read) {
    BucketSet out;
    out.n = n;
    out.b = b;
    out.values.assign(vals, vals + b);
    out.params = p;
    out.samples_read = samples_read;
    return out;
}
}  // namespace detail

// bucketize of one signal under several permutations in one launch.
inline std::vector<BucketSet> bucketize_rounds(const ComplexSignal& x, const FlatWindow& win,
                                               const std::vector<PermutationParams>& params,
                                               SampleTracker* tracker = nullptr) {
    if (x.n != win.n) throw std::invalid_argument("bucketize: signal/window size mismatch");
    std::vector<int64_t> sg, tu;
    for (const auto& p : params) {
        sg.push_back(p.sigma);
        tu.push_back(p.tau);
    }
    std::vector<cplx> vals(params.size() * static_cast<size_t>(win.b));
    int64_t w = 0;
    char err[1024] = {0};
    throw_status(msfft_bucketize(x.samples.data(), x.n, MSFFT_C128, MSFFT_HOST, win.b, win.delta,
                                 sg.data(), tu.data(), static_cast<int64_t>(params.size()),
                                 reinterpret_cast<double*>(vals.data()), MSFFT_HOST, &w, err,
                                 sizeof(err)),
                 err);
    if (tracker) {  // SampleTracker::touch per tap (bucketize.cpp:55-58): plan-only bookkeeping
        const int64_t h = (win.w - 1) / 2;
        for (const auto& p : params)
            for (int64_t t = -h; t <= h; ++t) tracker->touch(detail::tap_source(t, p, x.n));
    }
    std::vector<BucketSet> out;
    for (size_t r = 0; r < params.size(); ++r)
        out.push_back(detail::bucket_set(x.n, win.b, vals.data() + r * win.b, params[r], w));
    return out;
}

// bucketize (bucketize.hpp:56-57, bucketize.cpp:50-61).
inline BucketSet bucketize(const ComplexSignal& x, const FlatWindow& win,
                           const PermutationParams& params, SampleTracker* tracker = nullptr) {
    return bucketize_rounds(x, win, {params}, tracker)[0];
}

// bucketize_fn<Sampler> (bucketize.hpp:63-86): the sampler is invoked exactly
// once per filter tap, in increasing tap order, on the calling thread (so
// stateful samplers behave as with the reference); the fold, the b-point DIT
// and the 1/n scale run on the GPU, bit-identical to the reference's loop.
template <class Sampler>
BucketSet bucketize_fn(int64_t n, Sampler&& sample, const FlatWindow& win,
                       const PermutationParams& params) {
    const int64_t h = (win.w - 1) / 2;
    std::vector<cplx> v(static_cast<size_t>(win.w));
    for (int64_t t = -h; t <= h; ++t) v[static_cast<size_t>(h + t)] = sample(detail::tap_source(t, params, n));
    std::vector<cplx> out(static_cast<size_t>(win.b));
    int64_t w = 0;
    char err[1024] = {0};
    throw_status(msfft_bucketize_taps(n, win.b, win.delta, reinterpret_cast<const double*>(v.data()),
                                      1, reinterpret_cast<double*>(out.data()), &w, err, sizeof(err)),
                 err);
    return detail::bucket_set(n, win.b, out.data(), params, w);
}

// predict_buckets (bucketize.cpp:70-95) for several permutations in one launch;
// samples_read stays 0 (no signal samples are read).
inline std::vector<BucketSet> predict_buckets_rounds(const SparseSpectrum& known,
                                                     const FlatWindow& win,
                                                     const std::vector<PermutationParams>& params) {
    if (known.n != win.n) throw std::invalid_argument("predict_buckets: size mismatch");
    std::vector<int64_t> f, sg, tu;
    std::vector<double> c;
    detail::spectrum_arrays(known, f, c);
    for (const auto& p : params) {
        sg.push_back(p.sigma);
        tu.push_back(p.tau);
    }
    std::vector<cplx> vals(params.size() * static_cast<size_t>(win.b));
    char err[1024] = {0};
    throw_status(msfft_predict_buckets(win.n, win.b, win.delta, f.data(), c.data(),
                                       static_cast<int64_t>(f.size()), sg.data(), tu.data(),
                                       static_cast<int64_t>(params.size()),
                                       reinterpret_cast<double*>(vals.data()), MSFFT_HOST, err,
                                       sizeof(err)),
                 err);
    std::vector<BucketSet> out;
    for (size_t r = 0; r < params.size(); ++r)
        out.push_back(detail::bucket_set(win.n, win.b, vals.data() + r * win.b, params[r], 0));
    return out;
}

inline BucketSet predict_buckets(const SparseSpectrum& known, const FlatWindow& win,
                                 const PermutationParams& params) {
    return predict_buckets_rounds(known, win, {params})[0];
}

inline BucketSet subtract(const BucketSet& a, const BucketSet& b_set) {  // bucketize.cpp:97-104
    if (a.b != b_set.b || a.n != b_set.n || a.params.sigma != b_set.params.sigma ||
        a.params.tau != b_set.params.tau)
        throw std::invalid_argument("subtract: bucket sets are not from the same round");
    BucketSet out = a;
    for (size_t i = 0; i < out.values.size(); ++i) out.values[i] -= b_set.values[i];
    return out;
}

// ---- locate (locate.hpp:21-87) ------------------------------------------------

struct LocateRegion {  // locate.hpp:23-32
    double u_min = 0.0;
    double length = 0.0;
    int stage = 1;
    double u_max() const { return u_min + length; }
    double block(const MultiscaleConfig& cfg) const { return length / static_cast<double>(cfg.l); }
};

struct PhaseMeasurement {  // locate.hpp:35-40
    cplx y0;
    cplx y_tau;
    int64_t tau = 0;
    double phi = 0.0;
};

struct LocateOutcome {  // locate.hpp:42-45
    int64_t u = 0;
    int stages = 0;
};

struct ParameterBounds {  // locate.hpp:82-85
    bool l_ok = false;
    double q_min = 0.0;
};

// phase_of / position_phase / circular_phase_distance / locate_step run on
// the GPU: the same device functions the transform's decode uses.
inline double phase_of(cplx z) {  // locate.cpp:32-37
    double out = 0.0;
    int32_t status = 0;
    char err[256] = {0};
    throw_status(msfft_phase_of(reinterpret_cast<const double*>(&z), 1, &out, &status, err,
                                sizeof(err)),
                 err);
    if (status != 0) throw std::domain_error("phase_of: zero value");
    return out;
}

inline double position_phase(double u, int64_t tau, int64_t n) {  // locate.cpp:19-23
    double out = 0.0;
    char err[256] = {0};
    throw_status(msfft_position_phase(&u, &tau, 1, n, &out, err, sizeof(err)), err);
    return out;
}

inline double circular_phase_distance(double a, double b) {  // locate.cpp:14-17
    double out = 0.0;
    char err[256] = {0};
    throw_status(msfft_circular_phase_distance(&a, &b, 1, &out, err, sizeof(err)), err);
    return out;
}

inline int64_t tau_schedule(double region_length, int64_t n) {  // locate.cpp:39-42
    int64_t out = 0;
    char err[256] = {0};
    throw_status(msfft_tau_schedule(region_length, n, &out, err, sizeof(err)), err);
    return out;
}

inline int stage_count(double region_length, const MultiscaleConfig& cfg) {  // locate.cpp:44-53
    int32_t out = 0;
    char err[256] = {0};
    throw_status(msfft_stage_count(region_length, cfg.l, cfg.q, &out, err, sizeof(err)), err);
    return out;
}

inline LocateRegion initial_region(int64_t bucket, int64_t l_width) {  // locate.cpp:55-61
    LocateRegion r;
    r.u_min = (2.0 * static_cast<double>(bucket) - 1.0) * static_cast<double>(l_width) / 2.0;
    r.length = static_cast<double>(l_width);
    r.stage = 1;
    return r;
}

inline LocateRegion locate_step(const PhaseMeasurement& meas, const LocateRegion& region,
                                const MultiscaleConfig& cfg, int64_t n) {  // locate.cpp:63-81
    msfft_locate_region in{region.u_min, region.length, region.stage, 0}, out{};
    char err[256] = {0};
    throw_status(msfft_locate_step(&meas.phi, &meas.tau, &in, 1, cfg.l, cfg.q, n, &out, err,
                                   sizeof(err)),
                 err);
    LocateRegion r;
    r.u_min = out.u_min;
    r.length = out.length;
    r.stage = out.stage;
    return r;
}

inline ParameterBounds check_parameter_bounds(double max_dphi, int64_t l, double q = 0.0) {
    int32_t ok = 0;
    ParameterBounds b;
    char err[256] = {0};
    throw_status(msfft_check_parameter_bounds(max_dphi, l, q, &ok, &b.q_min, err, sizeof(err)), err);
    b.l_ok = ok != 0;
    return b;
}

// locate_frequency for many buckets against one round set (one launch).
inline std::vector<std::optional<LocateOutcome>> locate_frequencies(
    const std::vector<int64_t>& buckets, const BucketSet* rounds, size_t nrounds,
    const MultiscaleConfig& cfg, const FlatWindow& win) {
    if (nrounds == 0) throw std::invalid_argument("locate_frequency: no rounds");
    std::vector<cplx> vals;
    std::vector<int64_t> tau;
    for (size_t r = 0; r < nrounds; ++r) {
        vals.insert(vals.end(), rounds[r].values.begin(), rounds[r].values.end());
        tau.push_back(rounds[r].params.tau);
    }
    std::vector<int64_t> u(buckets.size());
    std::vector<int32_t> st(buckets.size()), status(buckets.size());
    char err[1024] = {0};
    throw_status(msfft_locate_frequency(win.n, win.b, cfg.l, cfg.q, buckets.data(),
                                        static_cast<int64_t>(buckets.size()),
                                        reinterpret_cast<const double*>(vals.data()), tau.data(),
                                        static_cast<int64_t>(nrounds), u.data(), st.data(),
                                        status.data(), MSFFT_HOST, err, sizeof(err)),
                 err);
    std::vector<std::optional<LocateOutcome>> out(buckets.size());
    for (size_t i = 0; i < buckets.size(); ++i)
        if (status[i] == 0) out[i] = LocateOutcome{u[i], st[i]};
    return out;
}

inline std::vector<std::optional<LocateOutcome>> locate_frequencies(
    const std::vector<int64_t>& buckets, const std::vector<BucketSet>& rounds,
    const MultiscaleConfig& cfg, const FlatWindow& win) {
    return locate_frequencies(buckets, rounds.data(), rounds.size(), cfg, win);
}

inline std::optional<LocateOutcome> locate_frequency(int64_t bucket,
                                                     const std::vector<BucketSet>& rounds,
                                                     const MultiscaleConfig& cfg,
                                                     const FlatWindow& win) {
    return locate_frequencies({bucket}, rounds.data(), rounds.size(), cfg, win)[0];
}

#if __cplusplus >= 202002L
// The reference's exact signature (locate.hpp:75-78).
inline std::optional<LocateOutcome> locate_frequency(int64_t bucket,
                                                     std::span<const BucketSet> rounds,
                                                     const MultiscaleConfig& cfg,
                                                     const FlatWindow& win) {
    return locate_frequencies({bucket}, rounds.data(), rounds.size(), cfg, win)[0];
}
#endif

inline cplx estimate_value(cplx y0_bucket, int64_t u, const FlatWindow& win) {
    double out[2] = {0.0, 0.0};
    int32_t status = 0;
    char err[1024] = {0};
    throw_status(msfft_estimate_values(win.n, win.b, win.delta,
                                       reinterpret_cast<const double*>(&y0_bucket), &u, 1, out,
                                       &status, MSFFT_HOST, err, sizeof(err)),
                 err);
    if (status != 0)
        throw std::domain_error("estimate_value: located position outside the pass region");
    return cplx(out[0], out[1]);
}

// ---- one iteration and the schedule (sfft4.hpp:14-30, 54-60) ------------------

struct IterationState {  // sfft4.hpp:14-30
    int m = 1;
    int64_t k_m = 0;
    int64_t b_m = 0;
    double delta = 1e-8;
    SparseSpectrum accumulated;
    int64_t sigma_m = 1;
    std::vector<int64_t> tau_plan;
    int64_t w_m = 0;
    int stages_m = 0;
    int64_t samples_round_sum = 0;
    double runtime_ms = 0.0;
};

// initial_bucket_count (sfft4.cpp:115-129), windows designed on the GPU.
inline int64_t initial_bucket_count(int64_t n, int64_t k, double delta) {
    int64_t out = 0;
    char err[1024] = {0};
    throw_status(msfft_initial_bucket_count(n, k, delta, &out, err, sizeof(err)), err);
    return out;
}

// run_iteration (sfft4.cpp:38-113) composed from the GPU components in the
// reference's order: all rounds encoded in one launch, the accumulated
// tones predicted for all rounds in one launch and subtracted, the stable
// |y0| ranking and threshold (std::abs = glibc hypot, as the reference), the
// candidate buckets located and estimated in one launch each, the found
// tones summed in rank order into the ascending map.  The fused msfft_sfft4
// never calls this; it equals it (tests/cpp/test_reference_suite.cpp).
inline SparseSpectrum run_iteration(const ComplexSignal& x, IterationState& state,
                                    const MultiscaleConfig& cfg, Rng& rng,
                                    SampleTracker* tracker = nullptr) {
    cfg.validate();
    x.validate();
    const int64_t n = x.n;
    const auto win = get_flat_window(n, state.b_m, state.delta);
    const PermutationParams base = random_params(n, rng, 0);
    const int stages = stage_count(static_cast<double>(win->l_width), cfg);
    std::vector<int64_t> taus{0};
    double len = static_cast<double>(win->l_width);
    for (int s = 0; s < stages; ++s) {
        taus.push_back(tau_schedule(len, n));
        len *= (cfg.q + 1.0) / static_cast<double>(cfg.l);
    }
    state.sigma_m = base.sigma;
    state.tau_plan = taus;
    state.w_m = win->w;
    state.stages_m = stages;
    std::vector<PermutationParams> params;
    for (int64_t t : taus) params.push_back(PermutationParams{base.sigma, base.sigma_inv, t});
    std::vector<BucketSet> rounds = bucketize_rounds(x, *win, params, tracker);
    if (!state.accumulated.entries.empty()) {
        const auto pred = predict_buckets_rounds(state.accumulated, *win, params);
        for (size_t r = 0; r < rounds.size(); ++r) rounds[r] = subtract(rounds[r], pred[r]);
    }
    state.samples_round_sum += static_cast<int64_t>(taus.size()) * win->w;

    const int64_t budget = std::min(state.k_m, state.b_m);
    std::vector<int64_t> order(static_cast<size_t>(state.b_m));
    std::iota(order.begin(), order.end(), 0);
    const auto& y0 = rounds[0].values;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        return std::abs(y0[static_cast<size_t>(a)]) > std::abs(y0[static_cast<size_t>(b)]);
    });
    const double threshold = 0.2 * std::abs(y0[static_cast<size_t>(order[static_cast<size_t>(budget - 1)])]);
    std::vector<int64_t> cand;
    for (int64_t rank = 0; rank < budget; ++rank)
        if (std::abs(y0[static_cast<size_t>(order[rank])]) > threshold) cand.push_back(order[rank]);
    SparseSpectrum found;
    found.n = n;
    if (!cand.empty()) {
        const auto outs = locate_frequencies(cand, rounds, cfg, *win);
        std::vector<cplx> ys;
        std::vector<int64_t> us, fs;
        for (size_t i = 0; i < cand.size(); ++i)
            if (outs[i]) {
                ys.push_back(y0[static_cast<size_t>(cand[i])]);
                us.push_back(outs[i]->u);
            }
        if (!us.empty()) {
            std::vector<cplx> vals(us.size());
            std::vector<int32_t> status(us.size());
            char err[1024] = {0};
            throw_status(msfft_estimate_values(win->n, win->b, win->delta,
                                               reinterpret_cast<const double*>(ys.data()),
                                               us.data(), static_cast<int64_t>(us.size()),
                                               reinterpret_cast<double*>(vals.data()),
                                               status.data(), MSFFT_HOST, err, sizeof(err)),
                         err);
            for (size_t i = 0; i < us.size(); ++i) {  // rank order
                if (status[i] != 0) continue;       // estimate_value threw: skipped
                const uint64_t f = (static_cast<uint64_t>(base.sigma_inv) *
                                    static_cast<uint64_t>(us[i])) & static_cast<uint64_t>(n - 1);
                found.entries[static_cast<int64_t>(f)] += vals[i];
            }
        }
    }
    for (const auto& [f, c] : found.entries) state.accumulated.entries[f] += c;
    state.accumulated.n = n;
    state.k_m = (state.k_m + 1) / 2;
    state.b_m = state.b_m > 32 ? state.b_m / 2 : state.b_m;
    ++state.m;
    return found;
}

}  // namespace msfft_b200

#ifdef MSFFT_B200_AS_MSFFT
namespace msfft = msfft_b200;
#endif
