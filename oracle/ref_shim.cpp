// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle_api.h).
//
// Exposes the reference library's public API (compiled unmodified from
// /root/reference/proj/src by oracle/Makefile) through the C ABI in
// oracle_api.h so Python tests and the bench's CPU arm can drive it.  Every
// number this file returns is produced by the reference's own functions;
// the only logic here is marshalling, plus orc_sfft4_trace, which replays
// msfft::run_iteration (proj/src/sfft4.cpp:38-113) step by step through the
// same public calls so per-stage intermediates can be captured.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "msfft/bucketize.hpp"
#include "msfft/io.hpp"
#include "msfft/phase_mc.hpp"
#include "msfft/locate.hpp"
#include "msfft/rng.hpp"
#include "msfft/sfft4.hpp"
#include "msfft/signal.hpp"
#include "msfft/window.hpp"
#include "oracle_api.h"

using namespace msfft;

namespace {

void put_err(char* err, int64_t errlen, const char* msg) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, msg, static_cast<size_t>(errlen - 1));
    err[errlen - 1] = '\0';
}

template <class F>
int guard(char* err, int64_t errlen, F&& fn) {
    try {
        fn();
        return ORC_OK;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return ORC_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        put_err(err, errlen, e.what());
        return ORC_DOMAIN_ERROR;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return ORC_OTHER;
    }
}

ComplexSignal make_signal(int64_t n, const double* x) {
    ComplexSignal s;
    s.n = n;
    s.samples.resize(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) s.samples[j] = cplx(x[2 * j], x[2 * j + 1]);
    return s;
}

int64_t ceil_log2_i(int64_t k) {
    int64_t r = 0;
    while ((int64_t{1} << r) < k) ++r;
    return r;
}

int64_t next_b(int64_t b) { return b > 32 ? b / 2 : b; }

void write_result(const SfftResult& res, int64_t cap, int64_t* out_f, double* out_c,
                  int64_t* out_count, int64_t* stats_i, double* stats_d) {
    int64_t i = 0;
    for (const auto& [f, c] : res.spectrum.entries) {
        if (i < cap) {
            out_f[i] = f;
            out_c[2 * i] = c.real();
            out_c[2 * i + 1] = c.imag();
        }
        ++i;
    }
    *out_count = i;
    if (stats_i) {
        stats_i[0] = res.stats.samples_used;
        stats_i[1] = res.stats.samples_round_sum;
        stats_i[2] = res.stats.iterations;
        stats_i[3] = res.stats.b_first;
        for (size_t m = 0; m < res.stats.stage_counts.size() && m < ORC_MAX_ITERS; ++m)
            stats_i[4 + m] = res.stats.stage_counts[m];
    }
    if (stats_d) {
        stats_d[0] = res.stats.sample_fraction;
        stats_d[1] = res.stats.runtime_ms;
    }
}

SparseSpectrum make_spectrum(int64_t n, int64_t count, const int64_t* f, const double* c) {
    SparseSpectrum s;
    s.n = n;
    for (int64_t i = 0; i < count; ++i) s.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    return s;
}

void put_cx(const std::vector<cplx>& v, double* out) {
    for (size_t j = 0; j < v.size(); ++j) {
        out[2 * j] = v[j].real();
        out[2 * j + 1] = v[j].imag();
    }
}

}  // namespace

extern "C" {

const char* orc_kind(void) { return "reference"; }

uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }

int orc_mod_inverse(int64_t sigma, int64_t n, int64_t* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] { *out = mod_inverse(sigma, n); });
}

int64_t orc_bucket_of(int64_t u, int64_t l_width, int64_t b) { return bucket_of(u, l_width, b); }

int64_t orc_tau_schedule(double region_length, int64_t n) { return tau_schedule(region_length, n); }

int orc_stage_count(double region_length, int64_t l, double q) {
    MultiscaleConfig cfg{l, q};
    return stage_count(region_length, cfg);
}

int orc_check_parameter_bounds(double max_dphi, int64_t l, double q, int* l_ok, double* q_min,
                               char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const ParameterBounds pb = check_parameter_bounds(max_dphi, l, q);
        *l_ok = pb.l_ok ? 1 : 0;
        *q_min = pb.q_min;
    });
}

int orc_cfg_validate(int64_t l, double q, char* err, int64_t errlen) {
    return guard(err, errlen, [&] { MultiscaleConfig{l, q}.validate(); });
}

int orc_random_params(int64_t n, uint64_t seed, int64_t count, int64_t* sigma, int64_t* sigma_inv,
                      char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        Rng rng(seed);
        for (int64_t i = 0; i < count; ++i) {
            const PermutationParams p = random_params(n, rng, 0);
            sigma[i] = p.sigma;
            sigma_inv[i] = p.sigma_inv;
        }
    });
}

int orc_initial_bucket_count(int64_t n, int64_t k, double delta, int64_t* out, char* err,
                             int64_t errlen) {
    return guard(err, errlen, [&] { *out = initial_bucket_count(n, k, delta); });
}

int orc_plan_build(int64_t n, int64_t k, int64_t l, double q, uint64_t seed, double delta,
                   orc_plan* plan, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        std::memset(plan, 0, sizeof(*plan));
        MultiscaleConfig cfg{l, q};
        cfg.validate();
        if (k < 1 || k > n / 8) throw std::invalid_argument("sfft4: need 1 <= K <= n/8");
        const int iters = static_cast<int>(ceil_log2_i(k)) + 2;
        if (iters > ORC_MAX_ITERS) throw std::invalid_argument("plan: too many iterations");
        int64_t b = initial_bucket_count(n, k, delta);
        plan->b_first = b;
        plan->iterations = iters;
        Rng rng(seed);
        int64_t k_m = k;
        int ntau = 0;
        for (int m = 0; m < iters; ++m) {
            const auto win = get_flat_window(n, b, delta);
            const PermutationParams p = random_params(n, rng, 0);
            const int stages = stage_count(static_cast<double>(win->l_width), cfg);
            plan->b[m] = b;
            plan->w[m] = win->w;
            plan->rounds[m] = stages + 1;
            plan->k_m[m] = k_m;
            plan->budget[m] = std::min(k_m, b);
            plan->sigma[m] = p.sigma;
            plan->sigma_inv[m] = p.sigma_inv;
            if (ntau + stages + 1 > ORC_MAX_ROUNDS)
                throw std::invalid_argument("plan: too many rounds");
            plan->taus[ntau++] = 0;
            double len = static_cast<double>(win->l_width);
            for (int s = 0; s < stages; ++s) {
                plan->taus[ntau++] = tau_schedule(len, n);
                len *= (cfg.q + 1.0) / static_cast<double>(cfg.l);
            }
            k_m = (k_m + 1) / 2;
            b = next_b(b);
        }
    });
}

int orc_window(int64_t n, int64_t b, double delta, int64_t* w, double* taps, int64_t taps_cap,
               char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        *w = win->w;
        if (taps && taps_cap >= win->w)
            std::memcpy(taps, win->g_time.data(), sizeof(double) * static_cast<size_t>(win->w));
    });
}

int orc_response_at(int64_t n, int64_t b, double delta, const int64_t* idx, int64_t count,
                    double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        for (int64_t i = 0; i < count; ++i) out[i] = win->response_at(idx[i]);
    });
}

int orc_bucketize(int64_t n, const double* x, int64_t b, double delta, int64_t sigma, int64_t tau,
                  double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        const ComplexSignal s = make_signal(n, x);
        PermutationParams p;
        p.sigma = sigma;
        p.sigma_inv = mod_inverse(sigma, n);
        p.tau = tau;
        const BucketSet set = bucketize(s, *win, p);
        for (int64_t i = 0; i < b; ++i) {
            out[2 * i] = set.values[i].real();
            out[2 * i + 1] = set.values[i].imag();
        }
    });
}

int orc_predict(int64_t n, int64_t b, double delta, int64_t nk, const int64_t* f, const double* c,
                int64_t sigma, int64_t tau, double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        SparseSpectrum known;
        known.n = n;
        for (int64_t i = 0; i < nk; ++i) known.entries[f[i]] += cplx(c[2 * i], c[2 * i + 1]);
        PermutationParams p;
        p.sigma = sigma;
        p.sigma_inv = mod_inverse(sigma, n);
        p.tau = tau;
        const BucketSet set = predict_buckets(known, *win, p);
        for (int64_t i = 0; i < b; ++i) {
            out[2 * i] = set.values[i].real();
            out[2 * i + 1] = set.values[i].imag();
        }
    });
}

int orc_locate(int64_t n, int64_t b, double delta, int64_t l, double q, int64_t bucket,
               int64_t nrounds, const int64_t* taus, const double* round_vals, int64_t* u,
               int* stages, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        std::vector<BucketSet> rounds(static_cast<size_t>(nrounds));
        for (int64_t r = 0; r < nrounds; ++r) {
            BucketSet& s = rounds[r];
            s.n = n;
            s.b = b;
            s.params.tau = taus[r];
            s.values.resize(static_cast<size_t>(b));
            for (int64_t i = 0; i < b; ++i)
                s.values[i] = cplx(round_vals[2 * (r * b + i)], round_vals[2 * (r * b + i) + 1]);
        }
        const auto out = locate_frequency(bucket, rounds, MultiscaleConfig{l, q}, *win);
        *u = out ? out->u : -1;
        *stages = out ? out->stages : 0;
    });
}

int orc_estimate_value(int64_t n, int64_t b, double delta, double y_re, double y_im, int64_t u,
                       double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto win = get_flat_window(n, b, delta);
        const cplx v = estimate_value(cplx(y_re, y_im), u, *win);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int orc_sfft4(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
              double delta, int64_t cap, int64_t* out_f, double* out_c, int64_t* out_count,
              int64_t* stats_i, double* stats_d, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const ComplexSignal s = make_signal(n, x);
        const SfftResult res = sfft4(s, k, MultiscaleConfig{l, q}, seed, delta);
        write_result(res, cap, out_f, out_c, out_count, stats_i, stats_d);
    });
}

int orc_sfft4_trace(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
                    double delta, double* pre, double* post, int64_t* sel_bucket, int64_t* sel_u,
                    int32_t* sel_status, double* sel_value, int64_t* sel_f, int64_t cap,
                    int64_t* out_f, double* out_c, int64_t* out_count, char* err,
                    int64_t errlen) {
    return guard(err, errlen, [&] {
        const ComplexSignal xs = make_signal(n, x);
        const MultiscaleConfig cfg{l, q};
        xs.validate();
        cfg.validate();
        if (k < 1 || k > n / 8) throw std::invalid_argument("sfft4: need 1 <= K <= n/8");
        const int iters = static_cast<int>(ceil_log2_i(k)) + 2;
        IterationState state;
        state.k_m = k;
        state.b_m = initial_bucket_count(n, k, delta);
        state.delta = delta;
        state.accumulated.n = n;
        Rng rng(seed);
        int64_t voff = 0, soff = 0;
        for (int m = 0; m < iters; ++m) {
            // Mirrors run_iteration (proj/src/sfft4.cpp:38-113) call for call.
            const auto win = get_flat_window(n, state.b_m, delta);
            PermutationParams base = random_params(n, rng, 0);
            const int stages = stage_count(static_cast<double>(win->l_width), cfg);
            std::vector<int64_t> taus{0};
            double len = static_cast<double>(win->l_width);
            for (int s = 0; s < stages; ++s) {
                taus.push_back(tau_schedule(len, n));
                len *= (cfg.q + 1.0) / static_cast<double>(cfg.l);
            }
            std::vector<BucketSet> rounds;
            for (int64_t tau : taus) {
                PermutationParams p = base;
                p.tau = tau;
                BucketSet set = bucketize(xs, *win, p);
                for (int64_t i = 0; i < state.b_m; ++i) {
                    pre[2 * (voff + i)] = set.values[i].real();
                    pre[2 * (voff + i) + 1] = set.values[i].imag();
                }
                if (!state.accumulated.entries.empty())
                    set = subtract(set, predict_buckets(state.accumulated, *win, p));
                for (int64_t i = 0; i < state.b_m; ++i) {
                    post[2 * (voff + i)] = set.values[i].real();
                    post[2 * (voff + i) + 1] = set.values[i].imag();
                }
                voff += state.b_m;
                rounds.push_back(std::move(set));
            }
            const int64_t budget = std::min(state.k_m, state.b_m);
            std::vector<int64_t> order(static_cast<size_t>(state.b_m));
            std::iota(order.begin(), order.end(), 0);
            const auto& y0 = rounds[0].values;
            std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b2) {
                return std::abs(y0[a]) > std::abs(y0[b2]);
            });
            const double threshold = 0.2 * std::abs(y0[order[budget - 1]]);
            SparseSpectrum found;
            found.n = n;
            for (int64_t rank = 0; rank < budget; ++rank) {
                const int64_t slot = soff + rank;
                const int64_t bucket = order[rank];
                sel_bucket[slot] = bucket;
                sel_u[slot] = -1;
                sel_f[slot] = -1;
                sel_value[2 * slot] = sel_value[2 * slot + 1] = 0.0;
                if (!(std::abs(y0[bucket]) > threshold)) {
                    sel_status[slot] = 1;
                    continue;
                }
                const auto outcome = locate_frequency(bucket, rounds, cfg, *win);
                if (!outcome) {
                    sel_status[slot] = 2;
                    continue;
                }
                sel_u[slot] = outcome->u;
                cplx value;
                try {
                    value = estimate_value(y0[bucket], outcome->u, *win);
                } catch (const std::domain_error&) {
                    sel_status[slot] = 3;
                    continue;
                }
                const int64_t f = (base.sigma_inv * outcome->u) % n;
                sel_status[slot] = 0;
                sel_value[2 * slot] = value.real();
                sel_value[2 * slot + 1] = value.imag();
                sel_f[slot] = f;
                found.entries[f] += value;
            }
            soff += budget;
            for (const auto& [f, c] : found.entries) state.accumulated.entries[f] += c;
            state.k_m = (state.k_m + 1) / 2;
            state.b_m = next_b(state.b_m);
        }
        // K-prune, as sfft4 (proj/src/sfft4.cpp:170-178).
        std::vector<std::pair<int64_t, cplx>> entries(state.accumulated.entries.begin(),
                                                      state.accumulated.entries.end());
        std::stable_sort(entries.begin(), entries.end(), [](const auto& a, const auto& b2) {
            return std::abs(a.second) > std::abs(b2.second);
        });
        if (static_cast<int64_t>(entries.size()) > k) entries.resize(static_cast<size_t>(k));
        SfftResult res;
        res.spectrum.n = n;
        for (const auto& [f, c] : entries) res.spectrum.entries[f] = c;
        write_result(res, cap, out_f, out_c, out_count, nullptr, nullptr);
    });
}

int orc_sfft4_batch_c64(int64_t nsig, int64_t n, const float* x, int64_t k, int64_t l, double q,
                        const uint64_t* seeds, double delta, int threads, int64_t cap,
                        int64_t* out_f, double* out_c, int64_t* out_count, double* wall_ms,
                        char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        // Pre-resolve the window schedule, as sfft4 itself does before its
        // timer (proj/src/sfft4.cpp:146-154).
        {
            int64_t b = initial_bucket_count(n, k, delta);
            for (int m = 0; m < static_cast<int>(ceil_log2_i(k)) + 2; ++m) {
                get_flat_window(n, b, delta);
                b = next_b(b);
            }
        }
        const int nthreads = std::max(1, std::min<int>(threads, static_cast<int>(nsig)));
        std::atomic<int64_t> next{0};
        std::vector<std::string> errors(static_cast<size_t>(nthreads));
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (;;) {
                        const int64_t i = next.fetch_add(1);
                        if (i >= nsig) break;
                        ComplexSignal s;
                        s.n = n;
                        s.samples.resize(static_cast<size_t>(n));
                        const float* xi = x + 2 * n * i;
                        for (int64_t j = 0; j < n; ++j)
                            s.samples[j] = cplx(static_cast<double>(xi[2 * j]),
                                                static_cast<double>(xi[2 * j + 1]));
                        const SfftResult res = sfft4(s, k, MultiscaleConfig{l, q}, seeds[i], delta);
                        write_result(res, cap, out_f + cap * i, out_c + 2 * cap * i, out_count + i,
                                     nullptr, nullptr);
                    }
                } catch (const std::exception& e) {
                    errors[t] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        const auto t1 = std::chrono::steady_clock::now();
        *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (const auto& e : errors)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int orc_generate_test_signal(int64_t n, int64_t k, uint64_t seed, double* x, int64_t* f,
                             double* c, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        auto [sig, truth] = generate_test_signal(n, k, seed);
        for (int64_t j = 0; j < n; ++j) {
            x[2 * j] = sig.samples[j].real();
            x[2 * j + 1] = sig.samples[j].imag();
        }
        int64_t i = 0;
        for (const auto& [pos, val] : truth.entries) {
            f[i] = pos;
            c[2 * i] = val.real();
            c[2 * i + 1] = val.imag();
            ++i;
        }
    });
}

int orc_add_awgn(int64_t n, double* x, double snr_db, uint64_t seed, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const ComplexSignal s = make_signal(n, x);
        const ComplexSignal o = add_awgn(s, snr_db, seed);
        for (int64_t j = 0; j < n; ++j) {
            x[2 * j] = o.samples[j].real();
            x[2 * j + 1] = o.samples[j].imag();
        }
    });
}

int orc_dft_dense(int64_t n, const double* x, double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] { put_cx(dft_dense(make_signal(n, x)), out); });
}

int orc_idft_dense(int64_t n, const double* spec, double* out, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        std::vector<cplx> v(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) v[j] = cplx(spec[2 * j], spec[2 * j + 1]);
        put_cx(idft_dense(v).samples, out);
    });
}

int orc_synthesize(int64_t n, int64_t count, const int64_t* f, const double* c, double* x,
                   char* err, int64_t errlen) {
    return guard(err, errlen,
                 [&] { put_cx(synthesize(make_spectrum(n, count, f, c)).samples, x); });
}

int orc_error_metrics(int64_t n, int64_t tcount, const int64_t* tf, const double* tc,
                      int64_t ecount, const int64_t* ef, const double* ec, int64_t k,
                      int64_t* out_l0, double* out_l1, double* out_l2, char* err,
                      int64_t errlen) {
    return guard(err, errlen, [&] {
        const EvalMetrics m = error_metrics(make_spectrum(n, tcount, tf, tc),
                                            make_spectrum(n, ecount, ef, ec), k);
        *out_l0 = m.l0_err;
        *out_l1 = m.l1_err;
        *out_l2 = m.l2_err;
    });
}

// bench.cpp:33-46 keeps top_k_spectrum in an anonymous namespace, so it is
// not linkable; this is the same std::nth_element call with the same
// comparator (the only restated logic in this file besides the trace).
int orc_top_k_spectrum(int64_t n, const double* spec, int64_t k, int64_t* out_f, double* out_c,
                       int64_t* out_count, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        std::vector<cplx> spectrum(static_cast<size_t>(n));
        for (int64_t j = 0; j < n; ++j) spectrum[j] = cplx(spec[2 * j], spec[2 * j + 1]);
        std::vector<int64_t> idx(spectrum.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int64_t>(i);
        const size_t keep = std::min<size_t>(static_cast<size_t>(k), idx.size());
        std::nth_element(idx.begin(), idx.begin() + keep, idx.end(), [&](int64_t a, int64_t b) {
            return std::abs(spectrum[static_cast<size_t>(a)]) >
                   std::abs(spectrum[static_cast<size_t>(b)]);
        });
        SparseSpectrum out;
        out.n = n;
        for (size_t i = 0; i < keep; ++i) out.entries[idx[i]] = spectrum[static_cast<size_t>(idx[i])];
        int64_t i = 0;
        for (const auto& [f, c] : out.entries) {
            out_f[i] = f;
            out_c[2 * i] = c.real();
            out_c[2 * i + 1] = c.imag();
            ++i;
        }
        *out_count = i;
    });
}

int orc_write_signal_file(const char* path, int64_t n, const double* x, char* err,
                          int64_t errlen) {
    return guard(err, errlen, [&] { write_signal_file(path, make_signal(n, x)); });
}

int orc_read_signal_file(const char* path, int64_t cap, double* x, int64_t* n, char* err,
                         int64_t errlen) {
    return guard(err, errlen, [&] {
        const ComplexSignal s = read_signal_file(path);
        *n = s.n;
        if (s.n <= cap) put_cx(s.samples, x);
    });
}

int orc_write_truth_csv(const char* path, int64_t n, int64_t count, const int64_t* f,
                        const double* c, char* err, int64_t errlen) {
    return guard(err, errlen, [&] { write_truth_csv(path, make_spectrum(n, count, f, c)); });
}

int orc_read_truth_csv(const char* path, int64_t n, int64_t cap, int64_t* f, double* c,
                       int64_t* count, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        const SparseSpectrum s = read_truth_csv(path, n);
        int64_t i = 0;
        for (const auto& [pos, val] : s.entries) {
            if (i < cap) {
                f[i] = pos;
                c[2 * i] = val.real();
                c[2 * i + 1] = val.imag();
            }
            ++i;
        }
        *count = i;
    });
}

int orc_phase_experiment(int64_t n, int64_t k, int64_t b, const double* snr, int64_t nsnr,
                         int64_t trials, uint64_t seed, double* out_hist, char* err,
                         int64_t errlen) {
    return guard(err, errlen, [&] {
        const auto hs = run_phase_experiment(n, k, b, std::vector<double>(snr, snr + nsnr), trials,
                                             seed);
        for (size_t i = 0; i < hs.size(); ++i) {
            double* o = out_hist + 73 * i;
            for (int j = 0; j < PhaseErrorHistogram::kBinCount; ++j) o[j] = hs[i].bin_mass[j];
            o[70] = hs[i].p50;
            o[71] = hs[i].p99;
            o[72] = hs[i].max;
        }
    });
}

// run_phase_experiment's accept loop for one SNR (phase_mc.cpp:175-186),
// keeping each accepted trial's details (sample_phase_error discards them).
int orc_phase_trials(int64_t n, int64_t k, int64_t b, double snr, int64_t si, int64_t trials,
                     uint64_t seed, int64_t* out_i, double* out_d, char* err, int64_t errlen) {
    return guard(err, errlen, [&] {
        Rng rng = Rng::stream(seed, 0x5eed0000ull + static_cast<uint64_t>(si));
        int64_t got = 0, attempts = 0;
        const int64_t cap = 200 * trials + 1000;
        while (got < trials) {
            if (++attempts > cap) throw std::runtime_error("run_phase_experiment: rejection rate too high");
            const auto t = sample_phase_trial(n, k, b, snr, rng);
            if (!t) continue;
            out_i[3 * got] = t->u;
            out_i[3 * got + 1] = t->bucket;
            out_i[3 * got + 2] = t->tau;
            double* d = out_d + 7 * got;
            d[0] = t->y0.real();
            d[1] = t->y0.imag();
            d[2] = t->y_tau.real();
            d[3] = t->y_tau.imag();
            d[4] = t->measured_phi;
            d[5] = t->true_phi;
            d[6] = t->dphi;
            ++got;
        }
    });
}

}  // extern "C"
