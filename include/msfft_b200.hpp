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

#include <complex>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "msfft_b200.h"

namespace msfft_b200 {

using cplx = std::complex<double>;

struct ComplexSignal {
    int64_t n = 0;
    std::vector<cplx> samples;
};

struct SparseSpectrum {
    int64_t n = 0;
    std::map<int64_t, cplx> entries;
};

struct MultiscaleConfig {
    int64_t l = 16;
    double q = 1.0;
    double shrink() const { return static_cast<double>(l) / (q + 1.0); }
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

inline SfftResult sfft4(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
                        uint64_t seed, double delta = 1e-8) {
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
    std::vector<double> g_time;
};

struct PermutationParams {  // bucketize.hpp:16-20
    int64_t sigma = 1, sigma_inv = 1, tau = 0;
};

struct BucketSet {  // bucketize.hpp:24-30
    int64_t n = 0, b = 0;
    std::vector<cplx> values;
    PermutationParams params;
    int64_t samples_read = 0;
};

struct LocateOutcome {  // locate.hpp:42-45
    int64_t u = 0;
    int stages = 0;
};

// get_flat_window (window.cpp:179-193): designed on the GPU, bit-identical taps.
inline std::shared_ptr<const FlatWindow> get_flat_window(int64_t n, int64_t b, double delta) {
    auto win = std::make_shared<FlatWindow>();
    char err[1024] = {0};
    int64_t w = 0;
    throw_status(msfft_window(n, b, delta, -1, &w, nullptr, 0, err, sizeof(err)), err);
    win->g_time.resize(static_cast<size_t>(w));
    throw_status(msfft_window(n, b, delta, -1, &w, win->g_time.data(), w, err, sizeof(err)), err);
    win->n = n;
    win->b = b;
    win->l_width = n / b;
    win->w = w;
    win->delta = delta;
    return win;
}

// bucketize of one signal under several permutations in one launch.
inline std::vector<BucketSet> bucketize_rounds(const ComplexSignal& x, const FlatWindow& win,
                                               const std::vector<PermutationParams>& params) {
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
    std::vector<BucketSet> out(params.size());
    for (size_t r = 0; r < params.size(); ++r) {
        out[r].n = x.n;
        out[r].b = win.b;
        out[r].values.assign(vals.begin() + r * win.b, vals.begin() + (r + 1) * win.b);
        out[r].params = params[r];
        out[r].samples_read = w;
    }
    return out;
}

inline BucketSet bucketize(const ComplexSignal& x, const FlatWindow& win,
                           const PermutationParams& params) {
    return bucketize_rounds(x, win, {params})[0];
}

inline BucketSet predict_buckets(const SparseSpectrum& known, const FlatWindow& win,
                                 const PermutationParams& params) {
    if (known.n != win.n) throw std::invalid_argument("predict_buckets: size mismatch");
    std::vector<int64_t> f;
    std::vector<double> c;
    detail::spectrum_arrays(known, f, c);
    BucketSet out;
    out.n = win.n;
    out.b = win.b;
    out.values.resize(static_cast<size_t>(win.b));
    out.params = params;
    char err[1024] = {0};
    throw_status(msfft_predict_buckets(win.n, win.b, win.delta, f.data(), c.data(),
                                       static_cast<int64_t>(f.size()), &params.sigma,
                                       &params.tau, 1, reinterpret_cast<double*>(out.values.data()),
                                       MSFFT_HOST, err, sizeof(err)),
                 err);
    return out;
}

inline BucketSet subtract(const BucketSet& a, const BucketSet& b_set) {  // bucketize.cpp:97-104
    if (a.b != b_set.b || a.n != b_set.n || a.params.sigma != b_set.params.sigma ||
        a.params.tau != b_set.params.tau)
        throw std::invalid_argument("subtract: bucket sets are not from the same round");
    BucketSet out = a;
    for (size_t i = 0; i < out.values.size(); ++i) out.values[i] -= b_set.values[i];
    return out;
}

// locate_frequency for many buckets against one round set (one launch).
inline std::vector<std::optional<LocateOutcome>> locate_frequencies(
    const std::vector<int64_t>& buckets, const std::vector<BucketSet>& rounds,
    const MultiscaleConfig& cfg, const FlatWindow& win) {
    if (rounds.empty()) throw std::invalid_argument("locate_frequency: no rounds");
    std::vector<cplx> vals;
    std::vector<int64_t> tau;
    for (const auto& r : rounds) {
        vals.insert(vals.end(), r.values.begin(), r.values.end());
        tau.push_back(r.params.tau);
    }
    std::vector<int64_t> u(buckets.size());
    std::vector<int32_t> st(buckets.size()), status(buckets.size());
    char err[1024] = {0};
    throw_status(msfft_locate_frequency(win.n, win.b, cfg.l, cfg.q, buckets.data(),
                                        static_cast<int64_t>(buckets.size()),
                                        reinterpret_cast<const double*>(vals.data()), tau.data(),
                                        static_cast<int64_t>(rounds.size()), u.data(), st.data(),
                                        status.data(), MSFFT_HOST, err, sizeof(err)),
                 err);
    std::vector<std::optional<LocateOutcome>> out(buckets.size());
    for (size_t i = 0; i < buckets.size(); ++i)
        if (status[i] == 0) out[i] = LocateOutcome{u[i], st[i]};
    return out;
}

inline std::optional<LocateOutcome> locate_frequency(int64_t bucket,
                                                     const std::vector<BucketSet>& rounds,
                                                     const MultiscaleConfig& cfg,
                                                     const FlatWindow& win) {
    return locate_frequencies({bucket}, rounds, cfg, win)[0];
}

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

}  // namespace msfft_b200

#ifdef MSFFT_B200_AS_MSFFT
namespace msfft = msfft_b200;
#endif
