// msfft_port.cpp -- TEST INFRASTRUCTURE ONLY (see ../oracle_api.h).
//
// An independent CPU restatement of the sFFT4.0 hot path, written from the
// reference's algorithm (file:line citations below) so the tests and the
// bench's CPU leg still have an oracle where the reference sources are not
// available.  It is pinned against the golden fixtures produced by the
// reference itself (tests/test_oracle_golden.py): windows, plans and sfft4
// outputs bit-for-bit.  Arithmetic deliberately keeps the reference's
// operation order (std::complex<double> -> the same libgcc/libm calls, no
// FMA: built with -ffp-contract=off); large n-point transforms split each
// radix-2 stage across threads, which does not change any butterfly.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "oracle_api.h"

namespace port {

using cx = std::complex<double>;
const double kTau = 6.283185307179586476925286766559;  // 2*pi (locate.cpp:10)

// ---------------------------------------------------------------- RNG
// proj/include/msfft/rng.hpp:9-59
uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

struct Gen {
    std::mt19937_64 e;
    bool spare_ok = false;
    double spare = 0.0;
    explicit Gen(uint64_t s) : e(s) {}
    uint64_t draw() { return e(); }
    uint64_t under(uint64_t bound) {  // (u64 * bound) >> 64
        return static_cast<uint64_t>((static_cast<unsigned __int128>(draw()) * bound) >> 64);
    }
    double unit() { return static_cast<double>(draw() >> 11) * 0x1.0p-53; }
    double normal() {  // Box-Muller with a cached second variate
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        double a = unit(), c = unit();
        while (a == 0.0) a = unit();
        const double rad = std::sqrt(-2.0 * std::log(a));
        const double ang = kTau * c;
        spare = rad * std::sin(ang);
        spare_ok = true;
        return rad * std::cos(ang);
    }
};

bool pow2(uint64_t v) { return v && !(v & (v - 1)); }

// ---------------------------------------------------------------- FFT
// Radix-2 DIT, unnormalised; sign < 0 forward (proj/src/fft.cpp:32-66).
std::mutex tw_mu;
std::map<size_t, std::shared_ptr<std::vector<cx>>> tw_cache;

std::shared_ptr<std::vector<cx>> twiddles(size_t n) {
    std::lock_guard<std::mutex> g(tw_mu);
    auto& slot = tw_cache[n];
    if (!slot) {
        slot = std::make_shared<std::vector<cx>>(n / 2);
        const double step = -2.0 * 3.141592653589793 / static_cast<double>(n);
        for (size_t k = 0; k < n / 2; ++k) {
            const double a = step * static_cast<double>(k);
            (*slot)[k] = cx(std::cos(a), std::sin(a));
        }
    }
    return slot;
}

template <class F>
void parallel_for(size_t count, size_t grain, F&& body) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(hw, std::max<size_t>(1, count / grain));
    if (nt <= 1) {
        body(size_t{0}, count);
        return;
    }
    std::vector<std::thread> ts;
    const size_t per = (count + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t)
        ts.emplace_back([&, t] { body(std::min(count, t * per), std::min(count, (t + 1) * per)); });
    for (auto& th : ts) th.join();
}

void fft(std::vector<cx>& a, int sign) {
    const size_t n = a.size();
    if (n <= 1) return;
    if (!pow2(n)) throw std::invalid_argument("fft_radix2: size must be a power of two");
    int bits = 0;
    while ((size_t{1} << bits) < n) ++bits;
    for (size_t i = 0; i < n; ++i) {
        size_t r = 0;
        for (int k = 0; k < bits; ++k) r |= ((i >> k) & 1u) << (bits - 1 - k);
        if (r > i) std::swap(a[i], a[r]);
    }
    const auto tw = twiddles(n);
    for (size_t len = 2; len <= n; len <<= 1) {
        const size_t half = len / 2, stride = n / len;
        parallel_for(n / len, size_t{1} << 14, [&](size_t b0, size_t b1) {
            for (size_t blk = b0; blk < b1; ++blk) {
                const size_t base = blk * len;
                for (size_t j = 0; j < half; ++j) {
                    cx w = (*tw)[j * stride];
                    if (sign > 0) w = std::conj(w);
                    const cx t = a[base + j + half] * w;
                    a[base + j + half] = a[base + j] - t;
                    a[base + j] += t;
                }
            }
        });
    }
}

// ---------------------------------------------------------------- window
// design_flat_window (proj/src/window.cpp:105-177) and helpers (:19-85).
struct Window {
    int64_t n = 0, b = 0, L = 0, w = 0;
    double delta = 0;
    std::vector<double> g;  // g[(w-1)/2 + t], |t| <= (w-1)/2
    double resp(int64_t i) const {  // response_at (window.cpp:89-99)
        const int64_t h = (w - 1) / 2;
        int64_t r = i % n;
        if (r < 0) r += n;
        double s = g[h];
        for (int64_t t = 1; t <= h; ++t)
            s += 2.0 * g[h + t] * std::cos(kTau * static_cast<double>((r * t) % n) /
                                           static_cast<double>(n));
        return s / static_cast<double>(n);
    }
};

std::vector<double> tails(double sg, int64_t maxd) {
    const int64_t reach = std::min<int64_t>(maxd, static_cast<int64_t>(sg * 42.0) + 2);
    std::vector<double> p(reach + 1);
    for (int64_t m = 0; m <= reach; ++m)
        p[m] = std::exp(-0.5 * static_cast<double>(m) * static_cast<double>(m) / (sg * sg));
    double tot = p[0];
    for (int64_t m = 1; m <= reach; ++m) tot += 2.0 * p[m];
    std::vector<double> out(maxd + 2, 0.0);
    double run = 0.0;
    for (int64_t d = std::min(reach, maxd + 1); d >= 0; --d) {
        run += p[d];
        out[d] = run / tot;
    }
    return out;
}

double ripple(double sg, int64_t L, int64_t c) {
    const auto t = tails(sg, L + c + 2);
    return std::max(t[c - L / 2 + 1] + t[c + L / 2 + 1], t[L - c]);
}

bool band_ok(const std::vector<double>& full, int64_t n, int64_t w, int64_t L, double delta) {
    const int64_t h = (w - 1) / 2;
    std::vector<cx> v(n, cx(0.0, 0.0));
    v[0] = full[0];
    for (int64_t t = 1; t <= h; ++t) {
        v[t] = full[t];
        v[n - t] = full[n - t];
    }
    fft(v, -1);
    const double sc = 1.0 / static_cast<double>(n);
    double pass = 0.0, stop = 0.0, trans = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        v[i] *= sc;
        const double m = std::abs(v[i]);
        const int64_t d = std::min(i, n - i);
        if (d <= L / 2) pass = std::max(pass, std::abs(m - 1.0));
        else if (d >= L) stop = std::max(stop, m);
        else trans = std::max(trans, m);
    }
    return pass <= delta && stop <= delta && trans <= 1.0 + delta;
}

Window design(int64_t n, int64_t b, double delta) {
    if (n < 16 || !pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("design_flat_window: n must be a power of two >= 16");
    if (b < 4 || b > n / 4 || !pow2(static_cast<uint64_t>(b)))
        throw std::invalid_argument("design_flat_window: need b a power of two, 4 <= b <= n/4");
    if (!(delta > 0.0 && delta < 0.1))
        throw std::invalid_argument("design_flat_window: delta must be in (0, 0.1)");
    const int64_t L = n / b, c = 3 * L / 4;
    double lo = static_cast<double>(L) / 80.0, hi = static_cast<double>(L);
    if (ripple(lo, L, c) > 0.5 * delta)
        throw std::invalid_argument("design_flat_window: infeasible (n, b, delta)");
    for (int k = 0; k < 64; ++k) {
        const double mid = 0.5 * (lo + hi);
        (ripple(mid, L, c) <= 0.5 * delta ? lo : hi) = mid;
    }
    const auto t = tails(lo, n / 2 + c + 2);
    std::vector<cx> ideal(n);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t d = std::min(i, n - i);
        ideal[i] = d <= c ? 1.0 - t[c - d + 1] - t[c + d + 1] : t[d - c] - t[d + c + 1];
    }
    fft(ideal, +1);
    std::vector<double> full(n);
    for (int64_t j = 0; j < n; ++j) full[j] = ideal[j].real();
    for (int64_t k = 1; k < n - k; ++k) full[k] = full[n - k] = 0.5 * (full[k] + full[n - k]);
    int64_t whi = n - 1;
    if (!band_ok(full, n, whi, L, delta))
        throw std::invalid_argument("design_flat_window: no support w <= n-1 passes the band check");
    int64_t wlo = 1;
    while (wlo < whi) {
        int64_t mid = wlo + (whi - wlo) / 2;
        if (!(mid & 1)) --mid;
        if (band_ok(full, n, mid, L, delta)) whi = mid;
        else wlo = mid + 2;
    }
    Window W;
    W.n = n;
    W.b = b;
    W.L = L;
    W.w = whi;
    W.delta = delta;
    const int64_t h = (whi - 1) / 2;
    W.g.assign(whi, 0.0);
    W.g[h] = full[0];
    for (int64_t k = 1; k <= h; ++k) {
        W.g[h + k] = full[k];
        W.g[h - k] = full[n - k];
    }
    return W;
}

std::mutex win_mu;
std::map<std::tuple<int64_t, int64_t, double>, std::shared_ptr<const Window>> win_cache;

std::shared_ptr<const Window> window(int64_t n, int64_t b, double delta) {
    const auto key = std::make_tuple(n, b, delta);
    {
        std::lock_guard<std::mutex> g(win_mu);
        auto it = win_cache.find(key);
        if (it != win_cache.end()) return it->second;
    }
    auto w = std::make_shared<const Window>(design(n, b, delta));
    std::lock_guard<std::mutex> g(win_mu);
    return win_cache.emplace(key, w).first->second;
}

// ---------------------------------------------------------------- plan
int64_t inverse_odd(int64_t s, int64_t n) {  // extended Euclid (bucketize.cpp:21-37)
    if (n < 2 || !pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("mod_inverse: n must be a power of two");
    if (s % 2 == 0) throw std::invalid_argument("mod_inverse: sigma must be odd");
    int64_t a = n, b = ((s % n) + n) % n, x0 = 0, x1 = 1;
    while (b) {
        const int64_t q = a / b;
        std::tie(a, b) = std::make_pair(b, a - q * b);
        std::tie(x0, x1) = std::make_pair(x1, x0 - q * x1);
    }
    return ((x0 % n) + n) % n;
}

void check_cfg(int64_t l, double q) {  // locate.cpp:25-30
    if (l < 2) throw std::invalid_argument("MultiscaleConfig: l must be >= 2");
    if (q < 0.0) throw std::invalid_argument("MultiscaleConfig: q must be >= 0");
    if (!(static_cast<double>(l) / (q + 1.0) > 1.0))
        throw std::invalid_argument("MultiscaleConfig: l/(q+1) must exceed 1");
}

int64_t tau_for(double len, int64_t n) {  // locate.cpp:39-42
    return std::clamp<int64_t>(std::llround(static_cast<double>(n) / len), 1, n - 1);
}

int stages_for(double len, int64_t l, double q) {  // locate.cpp:44-53
    const double s = static_cast<double>(l) / (q + 1.0);
    int r = 0;
    for (double acc = 1.0; acc * (1.0 + 1e-12) < len; acc *= s) ++r;
    return r;
}

int64_t first_b(int64_t n, int64_t k, double delta) {  // sfft4.cpp:115-129
    int64_t b = 4;
    while (b < 4 * k) b *= 2;
    b = std::max<int64_t>(std::min(b, n / 4), 4);
    for (;;) {
        try {
            window(n, b, delta);
            return b;
        } catch (const std::invalid_argument&) {
            if (b <= 4) throw;
            b /= 2;
        }
    }
}

int iterations_for(int64_t k) {  // ceil_log2(k) + 2 (sfft4.cpp:14-18, 138)
    int r = 0;
    while ((int64_t{1} << r) < k) ++r;
    return r + 2;
}

// ---------------------------------------------------------------- rounds
// One bucketization round (bucketize.hpp:63-86): fold, b-point FFT, 1/n.
std::vector<cx> encode_round(const std::vector<cx>& x, const Window& W, int64_t sigma, int64_t tau,
                             std::vector<uint8_t>* seen, int64_t* distinct) {
    const int64_t n = W.n, b = W.b, h = (W.w - 1) / 2;
    std::vector<cx> fold(b, cx(0.0, 0.0));
    for (int64_t t = -h; t <= h; ++t) {
        const int64_t src = (sigma * (((t - tau) % n + n) % n)) % n;
        if (seen && !(*seen)[src]) {
            (*seen)[src] = 1;
            ++*distinct;
        }
        fold[((t % b) + b) % b] += W.g[h + t] * x[src];
    }
    fft(fold, -1);
    const double sc = 1.0 / static_cast<double>(n);
    for (auto& v : fold) v *= sc;
    return fold;
}

cx root(int64_t n, int64_t e) {  // bucketize.cpp:12-18
    int64_t r = e % n;
    if (r < 0) r += n;
    const double a = -kTau * static_cast<double>(r) / static_cast<double>(n);
    return cx(std::cos(a), std::sin(a));
}

int64_t nearest_bucket(int64_t u, int64_t L) {  // floor(u/L + 0.5)
    return static_cast<int64_t>(std::floor(static_cast<double>(u) / static_cast<double>(L) + 0.5));
}

// predict_buckets (bucketize.cpp:70-95): three buckets per known tone.
std::vector<cx> predict(const std::map<int64_t, cx>& known, const Window& W, int64_t sigma,
                        int64_t tau) {
    const int64_t n = W.n, b = W.b, L = W.L;
    std::vector<cx> out(b, cx(0.0, 0.0));
    for (const auto& kv : known) {
        const int64_t u = (sigma * kv.first) % n;
        const int64_t i = nearest_bucket(u, L);
        const cx rot = root(n, tau * u);
        for (int64_t j = i - 1; j <= i + 1; ++j)
            out[((j % b) + b) % b] += W.resp(j * L - u) * kv.second * rot;
    }
    return out;
}

// ---------------------------------------------------------------- locate
double arg01(cx z) {  // phase_of (locate.cpp:32-37)
    if (z == cx(0.0, 0.0)) throw std::domain_error("phase_of: zero value");
    double a = std::atan2(z.imag(), z.real());
    if (a < 0.0) a += kTau;
    return a + 0.0;
}

double phase_at(double u, int64_t tau, int64_t n) {  // locate.cpp:19-23
    double v = std::fmod(u * static_cast<double>(tau), static_cast<double>(n));
    if (v < 0) v += static_cast<double>(n);
    return v * kTau / static_cast<double>(n);
}

double wrap_dist(double a, double b) {  // locate.cpp:14-17
    const double d = std::fmod(std::fabs(a - b), kTau);
    return std::min(d, kTau - d);
}

// locate_frequency (locate.cpp:83-123).  rounds[r][bucket]; -1 = nullopt.
int64_t locate(int64_t bucket, const std::vector<std::vector<cx>>& rounds,
               const std::vector<int64_t>& taus, int64_t l, double q, const Window& W,
               int* used) {
    check_cfg(l, q);
    if (rounds.empty()) throw std::invalid_argument("locate_frequency: no rounds");
    if (taus[0] != 0) throw std::invalid_argument("locate_frequency: round 0 must have tau = 0");
    if (static_cast<int>(rounds.size()) < stages_for(static_cast<double>(W.L), l, q) + 1)
        throw std::invalid_argument("locate_frequency: not enough rounds for the schedule");
    const int64_t n = W.n;
    const cx y0 = rounds[0][bucket];
    if (y0 == cx(0.0, 0.0)) return -1;
    double lo = (2.0 * static_cast<double>(bucket) - 1.0) * static_cast<double>(W.L) / 2.0;
    double len = static_cast<double>(W.L);
    int st = 0;
    while (len > 1.0 + 1e-9) {
        ++st;
        const cx yt = rounds[st][bucket];
        if (yt == cx(0.0, 0.0)) return -1;
        const double phi = arg01(y0 / yt);
        const double blk = len / static_cast<double>(l);
        int64_t best = 0;
        double bd = INFINITY;
        for (int64_t j = 0; j < l; ++j) {
            const double d =
                wrap_dist(phase_at(lo + (static_cast<double>(j) + 0.5) * blk, taus[st], n), phi);
            if (d < bd) {
                bd = d;
                best = j;
            }
        }
        lo = lo + (static_cast<double>(best) - q / 2.0) * blk;
        len = len * (q + 1.0) / static_cast<double>(l);
    }
    const double hi = lo + len;
    int64_t u = static_cast<int64_t>(std::ceil(lo));
    if (!(static_cast<double>(u) < hi)) u = std::llround(0.5 * (lo + hi));
    u %= n;
    if (u < 0) u += n;
    if (used) *used = st;
    return u;
}

cx estimate(cx y0, int64_t u, const Window& W) {  // sfft4.cpp:27-36
    const double g = W.resp(nearest_bucket(u, W.L) * W.L - u);
    if (std::fabs(g) < 0.5)
        throw std::domain_error("estimate_value: located position outside the pass region");
    return y0 / g;
}

// ---------------------------------------------------------------- sfft4
struct Trace {
    std::vector<cx> pre, post;
    std::vector<int64_t> sel_bucket, sel_u, sel_f;
    std::vector<int32_t> sel_status;
    std::vector<cx> sel_value;
};

struct Out {
    std::map<int64_t, cx> spec;
    int64_t samples_used = 0, round_sum = 0, b_first = 0;
    std::vector<int> stages;
    double ms = 0.0;
};

void check_signal(int64_t n, const std::vector<cx>& x) {  // signal.cpp:18-26
    if (n < 4 || !pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
    if (static_cast<int64_t>(x.size()) != n)
        throw std::invalid_argument("ComplexSignal: sample count != n");
    for (const cx& v : x)
        if (!std::isfinite(v.real()) || !std::isfinite(v.imag()))
            throw std::invalid_argument("ComplexSignal: non-finite sample");
}

// sfft4 (proj/src/sfft4.cpp:131-187) with run_iteration (:38-113) inlined.
Out transform(const std::vector<cx>& x, int64_t k, int64_t l, double q, uint64_t seed,
              double delta, Trace* tr) {
    const int64_t n = static_cast<int64_t>(x.size());
    check_signal(n, x);
    check_cfg(l, q);
    if (k < 1 || k > n / 8) throw std::invalid_argument("sfft4: need 1 <= K <= n/8");
    const int iters = iterations_for(k);
    int64_t b = first_b(n, k, delta);
    Out out;
    out.b_first = b;
    {
        int64_t bb = b;
        for (int m = 0; m < iters; ++m, bb = bb > 32 ? bb / 2 : bb) window(n, bb, delta);
    }
    std::vector<uint8_t> seen(n, 0);
    Gen rng(seed);
    std::map<int64_t, cx> acc;
    int64_t km = k;
    const auto t0 = std::chrono::steady_clock::now();
    for (int m = 0; m < iters; ++m) {
        check_signal(n, x);  // the reference re-validates every iteration (sfft4.cpp:42)
        const auto W = window(n, b, delta);
        const int64_t sg = 2 * static_cast<int64_t>(rng.under(static_cast<uint64_t>(n / 2))) + 1;
        const int64_t sgi = inverse_odd(sg, n);
        const int st = stages_for(static_cast<double>(W->L), l, q);
        std::vector<int64_t> taus{0};
        double len = static_cast<double>(W->L);
        for (int s = 0; s < st; ++s) {
            taus.push_back(tau_for(len, n));
            len *= (q + 1.0) / static_cast<double>(l);
        }
        std::vector<std::vector<cx>> rounds;
        for (int64_t tau : taus) {
            auto r = encode_round(x, *W, sg, tau, &seen, &out.samples_used);
            if (tr) tr->pre.insert(tr->pre.end(), r.begin(), r.end());
            if (!acc.empty()) {
                const auto p = predict(acc, *W, sg, tau);
                for (int64_t i = 0; i < b; ++i) r[i] -= p[i];
            }
            if (tr) tr->post.insert(tr->post.end(), r.begin(), r.end());
            rounds.push_back(std::move(r));
        }
        out.round_sum += static_cast<int64_t>(taus.size()) * W->w;
        out.stages.push_back(st);
        const int64_t budget = std::min(km, b);
        std::vector<int64_t> ord(b);
        for (int64_t i = 0; i < b; ++i) ord[i] = i;
        const auto& y0 = rounds[0];
        std::stable_sort(ord.begin(), ord.end(),
                         [&](int64_t a, int64_t c) { return std::abs(y0[a]) > std::abs(y0[c]); });
        const double thr = 0.2 * std::abs(y0[ord[budget - 1]]);
        std::map<int64_t, cx> found;
        for (int64_t rk = 0; rk < budget; ++rk) {
            const int64_t bk = ord[rk];
            int32_t status = 0;
            int64_t u = -1, f = -1;
            cx v(0.0, 0.0);
            if (!(std::abs(y0[bk]) > thr)) {
                status = 1;
            } else {
                u = locate(bk, rounds, taus, l, q, *W, nullptr);
                if (u < 0) {
                    status = 2;
                } else {
                    try {
                        v = estimate(y0[bk], u, *W);
                        f = (sgi * u) % n;
                        found[f] += v;
                    } catch (const std::domain_error&) {
                        status = 3;
                        v = cx(0.0, 0.0);
                    }
                }
            }
            if (tr) {
                tr->sel_bucket.push_back(bk);
                tr->sel_u.push_back(u);
                tr->sel_status.push_back(status);
                tr->sel_value.push_back(v);
                tr->sel_f.push_back(f);
            }
        }
        for (const auto& kv : found) acc[kv.first] += kv.second;
        km = (km + 1) / 2;
        b = b > 32 ? b / 2 : b;
    }
    out.ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::vector<std::pair<int64_t, cx>> items(acc.begin(), acc.end());
    std::stable_sort(items.begin(), items.end(), [](const std::pair<int64_t, cx>& a,
                                                     const std::pair<int64_t, cx>& c) {
        return std::abs(a.second) > std::abs(c.second);
    });
    if (static_cast<int64_t>(items.size()) > k) items.resize(k);
    for (const auto& kv : items) out.spec[kv.first] = kv.second;
    return out;
}

// ---------------------------------------------------------------- signals
// SparseSpectrum::validate (signal.cpp:28-39).
void check_spectrum(int64_t n, const std::map<int64_t, cx>& spec) {
    if (n < 4 || !pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("SparseSpectrum: n must be a power of two >= 4");
    if (static_cast<int64_t>(spec.size()) > n)
        throw std::invalid_argument("SparseSpectrum: more entries than n");
    for (const auto& kv : spec) {
        if (kv.first < 0 || kv.first >= n)
            throw std::invalid_argument("SparseSpectrum: position out of range");
        if (!std::isfinite(kv.second.real()) || !std::isfinite(kv.second.imag()))
            throw std::invalid_argument("SparseSpectrum: non-finite coefficient");
    }
}

// synthesize (signal.cpp:76-98): per tone in ascending position, a phasor
// recurrence re-seeded from cos/sin every 1024 samples, summed into x.
void synth(int64_t n, const std::map<int64_t, cx>& truth, std::vector<cx>& x) {
    check_spectrum(n, truth);
    x.assign(n, cx(0.0, 0.0));
    for (const auto& kv : truth) {
        const double step = kTau * static_cast<double>(kv.first) / static_cast<double>(n);
        const cx mul(std::cos(step), std::sin(step));
        cx ph(1.0, 0.0);
        for (int64_t j = 0; j < n; ++j) {
            if (j % 1024 == 0) {
                const double a = step * static_cast<double>(j % n);
                ph = cx(std::cos(a), std::sin(a));
            }
            x[j] += kv.second * ph;
            ph *= mul;
        }
    }
}

// dft_dense (signal.cpp:41-48): forward radix-2 with 1/n; idft_dense
// (:50-58): the unnormalised inverse.
std::vector<cx> dense(std::vector<cx> v, int sign) {
    if (sign < 0) {
        check_signal(static_cast<int64_t>(v.size()), v);
    } else if (v.size() < 4 || !pow2(v.size())) {
        throw std::invalid_argument("idft_dense: size must be a power of two >= 4");
    }
    fft(v, sign);
    if (sign < 0) {
        const double scale = 1.0 / static_cast<double>(v.size());
        for (cx& z : v) z *= scale;
    }
    return v;
}

struct Metrics {
    int64_t l0 = 0;
    double l1 = 0.0, l2 = 0.0;
};

// error_metrics (signal.cpp:154-184): over the union of supports in
// ascending position, absent entries read as zero.
Metrics metrics(int64_t n_truth, const std::map<int64_t, cx>& truth, int64_t n_est,
                const std::map<int64_t, cx>& est, int64_t k) {
    if (n_truth != n_est) throw std::invalid_argument("error_metrics: size mismatch");
    std::map<int64_t, bool> support;
    for (const auto& kv : truth) support[kv.first] = true;
    for (const auto& kv : est) support[kv.first] = true;
    if (k <= 0) {
        if (!support.empty())
            throw std::invalid_argument("error_metrics: k = 0 with nonempty support union");
        return {};
    }
    Metrics m;
    double sa = 0.0, sq = 0.0;
    for (const auto& kv : support) {
        const auto t = truth.find(kv.first);
        const auto e = est.find(kv.first);
        const cx tv = t == truth.end() ? cx(0, 0) : t->second;
        const cx ev = e == est.end() ? cx(0, 0) : e->second;
        const double d = std::abs(tv - ev);
        sa += d;
        sq += d * d;
        if (d > 1e-6) ++m.l0;
    }
    m.l1 = sa / static_cast<double>(k);
    m.l2 = std::sqrt(sq / static_cast<double>(k));
    return m;
}

// top_k_spectrum (bench.cpp:33-46): partial selection by |X| descending.
std::map<int64_t, cx> top_k(const std::vector<cx>& spec, int64_t n, int64_t k) {
    std::vector<int64_t> idx(spec.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = static_cast<int64_t>(i);
    const size_t keep = std::min<size_t>(static_cast<size_t>(k), idx.size());
    std::nth_element(idx.begin(), idx.begin() + keep, idx.end(), [&](int64_t a, int64_t b) {
        return std::abs(spec[static_cast<size_t>(a)]) > std::abs(spec[static_cast<size_t>(b)]);
    });
    std::map<int64_t, cx> out;
    (void)n;
    for (size_t i = 0; i < keep; ++i) out[idx[i]] = spec[static_cast<size_t>(idx[i])];
    return out;
}

// MSFT signal file (io.cpp:17-55): "MSFT" + 4 zero bytes, u64 n, n
// little-endian float64 (re, im) pairs; validated on both sides.
void write_file(const std::string& path, const std::vector<cx>& x) {
    check_signal(static_cast<int64_t>(x.size()), x);
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error("write_signal_file: cannot open " + path);
    const char magic[8] = {'M', 'S', 'F', 'T', 0, 0, 0, 0};
    const uint64_t n = x.size();
    bool ok = std::fwrite(magic, 1, 8, f) == 8 && std::fwrite(&n, 8, 1, f) == 1 &&
              std::fwrite(x.data(), 16, x.size(), f) == x.size();
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write_signal_file: write failed for " + path);
}

std::vector<cx> read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("read_signal_file: cannot open " + path);
    char magic[8] = {};
    const size_t got = std::fread(magic, 1, 8, f);
    if (got != 8 || std::memcmp(magic, "MSFT", 4) != 0) {
        std::fclose(f);
        throw std::runtime_error("read_signal_file: bad magic in " + path);
    }
    uint64_t n = 0;
    if (std::fread(&n, 8, 1, f) != 1 || !pow2(n) || n < 4 || n > (uint64_t{1} << 30)) {
        std::fclose(f);
        throw std::runtime_error("read_signal_file: bad length field in " + path);
    }
    std::vector<cx> x(n);
    const size_t rd = std::fread(x.data(), 16, n, f);
    std::fclose(f);
    if (rd != n) throw std::runtime_error("read_signal_file: truncated file " + path);
    check_signal(static_cast<int64_t>(n), x);
    return x;
}

// Truth CSV (io.cpp:57-92): header, then "position,re,im" with %.17g.
void write_csv(const std::string& path, const std::map<int64_t, cx>& truth) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw std::runtime_error("write_truth_csv: cannot open " + path);
    bool ok = std::fputs("position,re,im\n", f) >= 0;
    for (const auto& kv : truth)
        ok = ok && std::fprintf(f, "%lld,%.17g,%.17g\n", static_cast<long long>(kv.first),
                                kv.second.real(), kv.second.imag()) > 0;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error("write_truth_csv: write failed for " + path);
}

std::map<int64_t, cx> read_csv(const std::string& path, int64_t n) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) throw std::runtime_error("read_truth_csv: cannot open " + path);
    std::map<int64_t, cx> truth;
    std::string line;
    int ch;
    bool header = true;
    auto flush_line = [&] {
        if (header) {
            header = false;
        } else if (!line.empty()) {
            const size_t a = line.find(','), b = a == std::string::npos ? a : line.find(',', a + 1);
            const int64_t pos = std::stoll(line.substr(0, a));
            const double re = std::stod(line.substr(a + 1, b - a - 1));
            const double im = std::stod(line.substr(b + 1));
            truth[pos] = cx(re, im);
        }
        line.clear();
    };
    while ((ch = std::fgetc(f)) != EOF) {
        if (ch == '\n') flush_line(); else line.push_back(static_cast<char>(ch));
    }
    if (!line.empty()) flush_line();
    std::fclose(f);
    check_spectrum(n, truth);
    return truth;
}

// generate_test_signal (signal.cpp:100-127): Floyd sampling + synthesize.
void make_signal(int64_t n, int64_t k, uint64_t seed, std::vector<cx>& x,
                 std::map<int64_t, cx>& truth) {
    if (n < 4 || !pow2(static_cast<uint64_t>(n)))
        throw std::invalid_argument("random_sparse_spectrum: bad n");
    if (k < 0 || k > n) throw std::invalid_argument("random_sparse_spectrum: k out of range");
    Gen rng(seed);
    std::vector<int64_t> pos;
    std::map<int64_t, bool> have;
    for (int64_t j = n - k; j < n; ++j) {
        const int64_t t = static_cast<int64_t>(rng.under(static_cast<uint64_t>(j) + 1));
        if (!have.emplace(t, true).second) have.emplace(j, true);
    }
    truth.clear();
    for (const auto& kv : have) {
        const double ph = kTau * rng.unit();
        truth[kv.first] = cx(std::cos(ph), std::sin(ph));
    }
    synth(n, truth, x);
}

// add_awgn (signal.cpp:129-152): realised power ratio.
void awgn(std::vector<cx>& x, double snr_db, uint64_t seed) {
    check_signal(static_cast<int64_t>(x.size()), x);
    if (std::isinf(snr_db) && snr_db > 0) return;
    if (!std::isfinite(snr_db))
        throw std::invalid_argument("add_awgn: snr_db must be finite or +infinity");
    double ps = 0.0;
    for (const cx& v : x) ps += std::norm(v);
    Gen rng(seed);
    std::vector<cx> z(x.size());
    double pn = 0.0;
    for (cx& g : z) {
        // signal.cpp:140 builds cplx(rng.gaussian(), rng.gaussian()); the
        // argument order is unspecified and GCC evaluates it right to left,
        // so the imaginary part takes the first draw.
        const double im = rng.normal();
        const double re = rng.normal();
        g = cx(re, im);
        pn += std::norm(g);
    }
    const double target = ps * std::pow(10.0, -snr_db / 10.0);
    const double sc = pn > 0.0 ? std::sqrt(target / pn) : 0.0;
    for (size_t j = 0; j < x.size(); ++j) x[j] += sc * z[j];
}

}  // namespace port

// ================================================================ C ABI
namespace {

void copy_err(char* err, int64_t len, const char* msg) {
    if (!err || len <= 0) return;
    std::strncpy(err, msg, static_cast<size_t>(len - 1));
    err[len - 1] = '\0';
}

template <class F>
int wrap(char* err, int64_t len, F&& fn) {
    try {
        fn();
        return ORC_OK;
    } catch (const std::invalid_argument& e) {
        copy_err(err, len, e.what());
        return ORC_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        copy_err(err, len, e.what());
        return ORC_DOMAIN_ERROR;
    } catch (const std::exception& e) {
        copy_err(err, len, e.what());
        return ORC_OTHER;
    }
}

std::vector<port::cx> as_cx(int64_t n, const double* x) {
    std::vector<port::cx> v(n);
    for (int64_t j = 0; j < n; ++j) v[j] = port::cx(x[2 * j], x[2 * j + 1]);
    return v;
}

void emit(const std::map<int64_t, port::cx>& spec, int64_t cap, int64_t* f, double* c,
          int64_t* count) {
    int64_t i = 0;
    for (const auto& kv : spec) {
        if (i < cap) {
            f[i] = kv.first;
            c[2 * i] = kv.second.real();
            c[2 * i + 1] = kv.second.imag();
        }
        ++i;
    }
    *count = i;
}

}  // namespace

extern "C" {

const char* orc_kind(void) { return "port"; }
uint64_t orc_splitmix64(uint64_t x) { return port::mix64(x); }

int orc_mod_inverse(int64_t sigma, int64_t n, int64_t* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] { *out = port::inverse_odd(sigma, n); });
}

int64_t orc_bucket_of(int64_t u, int64_t l_width, int64_t b) {
    const int64_t i = port::nearest_bucket(u, l_width);
    return ((i % b) + b) % b;
}

int64_t orc_tau_schedule(double len, int64_t n) { return port::tau_for(len, n); }
int orc_stage_count(double len, int64_t l, double q) { return port::stages_for(len, l, q); }

int orc_check_parameter_bounds(double max_dphi, int64_t l, double, int* l_ok, double* q_min,
                               char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {  // locate.cpp:125-133
        if (!(max_dphi > 0.0))
            throw std::invalid_argument("check_parameter_bounds: max_dphi must be positive");
        *l_ok = static_cast<double>(l) <= 3.141592653589793 / max_dphi;
        *q_min = max_dphi * static_cast<double>(l) / 3.141592653589793;
    });
}

int orc_cfg_validate(int64_t l, double q, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] { port::check_cfg(l, q); });
}

int orc_random_params(int64_t n, uint64_t seed, int64_t count, int64_t* sigma, int64_t* sigma_inv,
                      char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        if (n < 4 || !port::pow2(static_cast<uint64_t>(n)))
            throw std::invalid_argument("random_params: bad n");
        port::Gen g(seed);
        for (int64_t i = 0; i < count; ++i) {
            sigma[i] = 2 * static_cast<int64_t>(g.under(static_cast<uint64_t>(n / 2))) + 1;
            sigma_inv[i] = port::inverse_odd(sigma[i], n);
        }
    });
}

int orc_initial_bucket_count(int64_t n, int64_t k, double delta, int64_t* out, char* err,
                             int64_t errlen) {
    return wrap(err, errlen, [&] { *out = port::first_b(n, k, delta); });
}

int orc_plan_build(int64_t n, int64_t k, int64_t l, double q, uint64_t seed, double delta,
                   orc_plan* plan, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        std::memset(plan, 0, sizeof(*plan));
        port::check_cfg(l, q);
        if (k < 1 || k > n / 8) throw std::invalid_argument("sfft4: need 1 <= K <= n/8");
        const int iters = port::iterations_for(k);
        int64_t b = port::first_b(n, k, delta);
        plan->b_first = b;
        plan->iterations = iters;
        port::Gen g(seed);
        int64_t km = k;
        int nt = 0;
        for (int m = 0; m < iters; ++m) {
            const auto W = port::window(n, b, delta);
            const int st = port::stages_for(static_cast<double>(W->L), l, q);
            plan->b[m] = b;
            plan->w[m] = W->w;
            plan->rounds[m] = st + 1;
            plan->k_m[m] = km;
            plan->budget[m] = std::min(km, b);
            plan->sigma[m] = 2 * static_cast<int64_t>(g.under(static_cast<uint64_t>(n / 2))) + 1;
            plan->sigma_inv[m] = port::inverse_odd(plan->sigma[m], n);
            if (nt + st + 1 > ORC_MAX_ROUNDS) throw std::invalid_argument("plan: too many rounds");
            plan->taus[nt++] = 0;
            double len = static_cast<double>(W->L);
            for (int s = 0; s < st; ++s) {
                plan->taus[nt++] = port::tau_for(len, n);
                len *= (q + 1.0) / static_cast<double>(l);
            }
            km = (km + 1) / 2;
            b = b > 32 ? b / 2 : b;
        }
    });
}

int orc_window(int64_t n, int64_t b, double delta, int64_t* w, double* taps, int64_t cap,
               char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        *w = W->w;
        if (taps && cap >= W->w) std::memcpy(taps, W->g.data(), sizeof(double) * W->w);
    });
}

int orc_response_at(int64_t n, int64_t b, double delta, const int64_t* idx, int64_t count,
                    double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        for (int64_t i = 0; i < count; ++i) out[i] = W->resp(idx[i]);
    });
}

int orc_bucketize(int64_t n, const double* x, int64_t b, double delta, int64_t sigma, int64_t tau,
                  double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        port::inverse_odd(sigma, n);
        const auto r = port::encode_round(as_cx(n, x), *W, sigma, tau, nullptr, nullptr);
        std::memcpy(out, r.data(), sizeof(double) * 2 * b);
    });
}

int orc_predict(int64_t n, int64_t b, double delta, int64_t nk, const int64_t* f, const double* c,
                int64_t sigma, int64_t tau, double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        std::map<int64_t, port::cx> known;
        for (int64_t i = 0; i < nk; ++i) known[f[i]] += port::cx(c[2 * i], c[2 * i + 1]);
        const auto p = port::predict(known, *W, sigma, tau);
        std::memcpy(out, p.data(), sizeof(double) * 2 * b);
    });
}

int orc_locate(int64_t n, int64_t b, double delta, int64_t l, double q, int64_t bucket,
               int64_t nrounds, const int64_t* taus, const double* vals, int64_t* u, int* stages,
               char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        std::vector<std::vector<port::cx>> rounds(nrounds);
        for (int64_t r = 0; r < nrounds; ++r) rounds[r] = as_cx(b, vals + 2 * r * b);
        int used = 0;
        *u = port::locate(bucket, rounds, std::vector<int64_t>(taus, taus + nrounds), l, q, *W,
                          &used);
        *stages = *u < 0 ? 0 : used;
    });
}

int orc_estimate_value(int64_t n, int64_t b, double delta, double yr, double yi, int64_t u,
                       double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto W = port::window(n, b, delta);
        const port::cx v = port::estimate(port::cx(yr, yi), u, *W);
        out[0] = v.real();
        out[1] = v.imag();
    });
}

int orc_sfft4(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
              double delta, int64_t cap, int64_t* out_f, double* out_c, int64_t* out_count,
              int64_t* si, double* sd, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto o = port::transform(as_cx(n, x), k, l, q, seed, delta, nullptr);
        emit(o.spec, cap, out_f, out_c, out_count);
        if (si) {
            si[0] = o.samples_used;
            si[1] = o.round_sum;
            si[2] = static_cast<int64_t>(o.stages.size());
            si[3] = o.b_first;
            for (size_t m = 0; m < o.stages.size() && m < ORC_MAX_ITERS; ++m) si[4 + m] = o.stages[m];
        }
        if (sd) {
            sd[0] = static_cast<double>(o.samples_used) / static_cast<double>(n);
            sd[1] = o.ms;
        }
    });
}

int orc_sfft4_trace(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
                    double delta, double* pre, double* post, int64_t* sel_bucket, int64_t* sel_u,
                    int32_t* sel_status, double* sel_value, int64_t* sel_f, int64_t cap,
                    int64_t* out_f, double* out_c, int64_t* out_count, char* err,
                    int64_t errlen) {
    return wrap(err, errlen, [&] {
        port::Trace tr;
        const auto o = port::transform(as_cx(n, x), k, l, q, seed, delta, &tr);
        std::memcpy(pre, tr.pre.data(), sizeof(double) * 2 * tr.pre.size());
        std::memcpy(post, tr.post.data(), sizeof(double) * 2 * tr.post.size());
        for (size_t i = 0; i < tr.sel_bucket.size(); ++i) {
            sel_bucket[i] = tr.sel_bucket[i];
            sel_u[i] = tr.sel_u[i];
            sel_status[i] = tr.sel_status[i];
            sel_value[2 * i] = tr.sel_value[i].real();
            sel_value[2 * i + 1] = tr.sel_value[i].imag();
            sel_f[i] = tr.sel_f[i];
        }
        emit(o.spec, cap, out_f, out_c, out_count);
    });
}

int orc_sfft4_batch_c64(int64_t nsig, int64_t n, const float* x, int64_t k, int64_t l, double q,
                        const uint64_t* seeds, double delta, int threads, int64_t cap,
                        int64_t* out_f, double* out_c, int64_t* out_count, double* wall_ms,
                        char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        {
            int64_t b = port::first_b(n, k, delta);
            for (int m = 0; m < port::iterations_for(k); ++m, b = b > 32 ? b / 2 : b)
                port::window(n, b, delta);
        }
        std::atomic<int64_t> next{0};
        std::vector<std::string> errs(std::max(1, threads));
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, threads); ++t)
            pool.emplace_back([&, t] {
                try {
                    for (int64_t i; (i = next.fetch_add(1)) < nsig;) {
                        std::vector<port::cx> s(n);
                        for (int64_t j = 0; j < n; ++j)
                            s[j] = port::cx(x[2 * (n * i + j)], x[2 * (n * i + j) + 1]);
                        const auto o = port::transform(s, k, l, q, seeds[i], delta, nullptr);
                        emit(o.spec, cap, out_f + cap * i, out_c + 2 * cap * i, out_count + i);
                    }
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        for (auto& th : pool) th.join();
        *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                       .count();
        for (const auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int orc_generate_test_signal(int64_t n, int64_t k, uint64_t seed, double* x, int64_t* f,
                             double* c, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        std::vector<port::cx> s;
        std::map<int64_t, port::cx> truth;
        port::make_signal(n, k, seed, s, truth);
        std::memcpy(x, s.data(), sizeof(double) * 2 * n);
        int64_t i = 0;
        for (const auto& kv : truth) {
            f[i] = kv.first;
            c[2 * i] = kv.second.real();
            c[2 * i + 1] = kv.second.imag();
            ++i;
        }
    });
}

int orc_add_awgn(int64_t n, double* x, double snr_db, uint64_t seed, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        auto s = as_cx(n, x);
        port::awgn(s, snr_db, seed);
        std::memcpy(x, s.data(), sizeof(double) * 2 * n);
    });
}

int orc_dft_dense(int64_t n, const double* x, double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto v = port::dense(as_cx(n, x), -1);
        std::memcpy(out, v.data(), sizeof(double) * 2 * n);
    });
}

int orc_idft_dense(int64_t n, const double* spec, double* out, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto v = port::dense(as_cx(n, spec), +1);
        std::memcpy(out, v.data(), sizeof(double) * 2 * n);
    });
}

static std::map<int64_t, port::cx> as_spec(int64_t count, const int64_t* f, const double* c) {
    std::map<int64_t, port::cx> m;
    for (int64_t i = 0; i < count; ++i) m[f[i]] = port::cx(c[2 * i], c[2 * i + 1]);
    return m;
}

int orc_synthesize(int64_t n, int64_t count, const int64_t* f, const double* c, double* x,
                   char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        std::vector<port::cx> v;
        port::synth(n, as_spec(count, f, c), v);
        std::memcpy(x, v.data(), sizeof(double) * 2 * n);
    });
}

int orc_error_metrics(int64_t n, int64_t tcount, const int64_t* tf, const double* tc,
                      int64_t ecount, const int64_t* ef, const double* ec, int64_t k,
                      int64_t* out_l0, double* out_l1, double* out_l2, char* err,
                      int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto m = port::metrics(n, as_spec(tcount, tf, tc), n, as_spec(ecount, ef, ec), k);
        *out_l0 = m.l0;
        *out_l1 = m.l1;
        *out_l2 = m.l2;
    });
}

int orc_top_k_spectrum(int64_t n, const double* spec, int64_t k, int64_t* out_f, double* out_c,
                       int64_t* out_count, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] {
        emit(port::top_k(as_cx(n, spec), n, k), k, out_f, out_c, out_count);
    });
}

int orc_write_signal_file(const char* path, int64_t n, const double* x, char* err,
                          int64_t errlen) {
    return wrap(err, errlen, [&] { port::write_file(path, as_cx(n, x)); });
}

int orc_read_signal_file(const char* path, int64_t cap, double* x, int64_t* n, char* err,
                         int64_t errlen) {
    return wrap(err, errlen, [&] {
        const auto v = port::read_file(path);
        *n = static_cast<int64_t>(v.size());
        if (*n <= cap) std::memcpy(x, v.data(), sizeof(double) * 2 * v.size());
    });
}

int orc_write_truth_csv(const char* path, int64_t n, int64_t count, const int64_t* f,
                        const double* c, char* err, int64_t errlen) {
    (void)n;
    return wrap(err, errlen, [&] { port::write_csv(path, as_spec(count, f, c)); });
}

int orc_read_truth_csv(const char* path, int64_t n, int64_t cap, int64_t* f, double* c,
                       int64_t* count, char* err, int64_t errlen) {
    return wrap(err, errlen, [&] { emit(port::read_csv(path, n), cap, f, c, count); });
}

}  // extern "C"
