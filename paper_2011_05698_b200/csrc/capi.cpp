// capi.cpp -- extern "C" boundary (include/msfft_b200.h).  Maps the C++
// exception taxonomy of the reference onto status codes + messages.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "../../include/msfft_b200.h"
#include "engine.hpp"
#include "host_plan.hpp"
#include "window.hpp"

using namespace msfft_b200;

namespace {

void put_err(char* err, size_t errlen, const char* msg) {
    if (!err || errlen == 0) return;
    std::strncpy(err, msg, errlen - 1);
    err[errlen - 1] = '\0';
}

template <class F>
int guarded(char* err, size_t errlen, F&& fn) {
    try {
        fn();
        return MSFFT_OK;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return MSFFT_ERR_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        put_err(err, errlen, e.what());
        return MSFFT_ERR_DOMAIN;
    } catch (const CudaError& e) {
        put_err(err, errlen, e.what());
        return MSFFT_ERR_CUDA;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return MSFFT_ERR_RUNTIME;
    }
}

int current_or(int device) {
    if (device >= 0) return device;
    int d = 0;
    MSFFT_CUDA(cudaGetDevice(&d));
    return d;
}

void require_device() {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw CudaError("msfft_b200: no CUDA device available (there is no CPU fallback)");
}

// True if any of the n samples is non-finite (host copy of the input).
bool has_non_finite(const void* x, int64_t n, bool c128, bool on_device) {
    const size_t bytes = static_cast<size_t>(n) * (c128 ? 16 : 8);
    std::vector<unsigned char> buf;
    const unsigned char* p = static_cast<const unsigned char*>(x);
    if (on_device) {
        buf.resize(bytes);
        MSFFT_CUDA(cudaMemcpy(buf.data(), x, bytes, cudaMemcpyDeviceToHost));
        p = buf.data();
    }
    for (int64_t j = 0; j < 2 * n; ++j) {
        double v;
        if (c128) {
            std::memcpy(&v, p + 8 * j, 8);
        } else {
            float f;
            std::memcpy(&f, p + 4 * j, 4);
            v = f;
        }
        if (!std::isfinite(v)) return true;
    }
    return false;
}

void fill_stats(const SchedulePlan& sp, msfft_stats* st) {
    std::memset(st, 0, sizeof(*st));
    st->samples_round_sum = sp.samples_round_sum;
    st->iterations = sp.iterations;
    st->b_first = sp.b_first;
    for (int m = 0; m < sp.iterations && m < MSFFT_MAX_ITERATIONS; ++m)
        st->stage_counts[m] = sp.iters[m].stages;
}

}  // namespace

struct msfft_plan_s {
    std::shared_ptr<Plan> plan;
};

extern "C" {

const char* msfft_version(void) { return "msfft_b200 1.0 (sm_100a)"; }

int msfft_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

int msfft_sfft4(const void* x, int64_t n, int32_t dtype, int32_t x_location, int64_t k,
                int64_t l, double q, uint64_t seed, double delta, int64_t cap, int64_t* out_f,
                double* out_c, int64_t* out_count, msfft_stats* stats, char* err,
                size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const bool c128 = dtype == MSFFT_C128;
        if (dtype != MSFFT_C128 && dtype != MSFFT_C64)
            throw std::invalid_argument("msfft_sfft4: unknown dtype");
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
        const bool on_dev = x_location == MSFFT_DEVICE;
        std::shared_ptr<Plan> plan;
        try {
            plan = cached_plan(n, k, l, q, delta, c128, current_or(-1));
        } catch (const std::invalid_argument&) {
            // sfft4 validates x before its other arguments (sfft4.cpp:133-135)
            if (has_non_finite(x, n, c128, on_dev))
                throw std::invalid_argument("ComplexSignal: non-finite sample");
            throw;
        }
        std::lock_guard<std::mutex> lock(plan->mutex());
        std::vector<int64_t> f(static_cast<size_t>(k));
        std::vector<double> c(static_cast<size_t>(2 * k));
        int64_t count = 0;
        ExecOptions opt;
        opt.x_on_device = on_dev;
        double ms = 0.0;
        plan->execute(1, x, n, &seed, f.data(), c.data(), &count, opt, &ms);
        *out_count = count;
        for (int64_t i = 0; i < count && i < cap; ++i) {
            out_f[i] = f[i];
            out_c[2 * i] = c[2 * i];
            out_c[2 * i + 1] = c[2 * i + 1];
        }
        if (stats) {
            const SchedulePlan& sp = plan->schedule();
            fill_stats(sp, stats);
            std::vector<int64_t> sg(sp.iterations), sgi(sp.iterations);
            draw_sigmas(seed, n, sp.iterations, sg.data(), sgi.data());
            stats->samples_used = count_samples_used(sp, sg.data());
            stats->sample_fraction =
                static_cast<double>(stats->samples_used) / static_cast<double>(n);
            stats->runtime_ms = ms;
        }
    });
}

int msfft_plan_create(int64_t n, int64_t k, int64_t l, double q, double delta, int32_t dtype,
                      int32_t device, msfft_plan* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (dtype != MSFFT_C128 && dtype != MSFFT_C64)
            throw std::invalid_argument("msfft_plan_create: unknown dtype");
        auto p = std::make_shared<Plan>(n, k, l, q, delta, dtype == MSFFT_C128,
                                        current_or(device));
        *out = new msfft_plan_s{std::move(p)};
    });
}

void msfft_plan_destroy(msfft_plan plan) { delete plan; }

int msfft_plan_stats(msfft_plan plan, msfft_stats* stats) {
    if (!plan || !stats) return MSFFT_ERR_INVALID_ARGUMENT;
    fill_stats(plan->plan->schedule(), stats);
    return MSFFT_OK;
}

int64_t msfft_plan_launches(msfft_plan plan, int64_t batch, uint32_t flags) {
    if (!plan) return -1;
    return plan->plan->launches(batch, !(flags & MSFFT_FLAG_ASSUME_VALID),
                                (flags & MSFFT_FLAG_SERIAL) != 0);
}

int msfft_execute(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                  int32_t x_location, const uint64_t* seeds, int64_t* out_f, double* out_c,
                  int64_t* out_count, int32_t out_location, uint32_t flags, void* stream,
                  double* device_ms, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_execute: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        ExecOptions opt;
        opt.x_on_device = x_location == MSFFT_DEVICE;
        opt.out_on_device = out_location == MSFFT_DEVICE;
        opt.assume_valid = (flags & MSFFT_FLAG_ASSUME_VALID) != 0;
        opt.stage_times = (flags & MSFFT_FLAG_STAGE_TIMES) != 0;
        opt.force_serial = (flags & MSFFT_FLAG_SERIAL) != 0;
        opt.stream = static_cast<cudaStream_t>(stream);
        plan->plan->execute(batch, x, x_stride, seeds, out_f, out_c, out_count, opt, device_ms);
    });
}

int64_t msfft_plan_ingest_samples(msfft_plan plan) {
    if (!plan) return -1;
    return plan->plan->ingest_samples_per_signal();
}

int64_t msfft_plan_values_per_signal(msfft_plan plan) {
    if (!plan) return -1;
    return plan->plan->values_per_signal();
}

int msfft_encode_values(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                        int64_t x_lo, int64_t x_hi, const uint64_t* seeds, double* y,
                        uint32_t flags, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_encode_values: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        plan->plan->encode_values(batch, x, x_stride, x_lo, x_hi, seeds,
                                  reinterpret_cast<double2*>(y),
                                  !(flags & MSFFT_FLAG_ASSUME_VALID),
                                  static_cast<cudaStream_t>(stream));
    });
}

int msfft_decode_values(msfft_plan plan, int64_t batch, double* y, const uint64_t* seeds,
                        int64_t* out_f, double* out_c, int64_t* out_count, void* stream,
                        char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_decode_values: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        plan->plan->decode_values(batch, reinterpret_cast<double2*>(y), seeds, out_f,
                                  reinterpret_cast<double2*>(out_c), out_count,
                                  static_cast<cudaStream_t>(stream));
    });
}

int msfft_sigma_plan(uint64_t seed, int64_t n, int32_t iterations, int64_t* sigma,
                     int64_t* sigma_inv, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { draw_sigmas(seed, n, iterations, sigma, sigma_inv); });
}

int msfft_tau_plan(double l_width, int64_t n, int64_t l, double q, int64_t* taus,
                   int32_t cap, int32_t* rounds, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        validate_cfg(l, q);
        const int stages = stage_count(l_width, l, q);
        *rounds = stages + 1;
        if (stages + 1 > cap) throw std::invalid_argument("msfft_tau_plan: cap too small");
        taus[0] = 0;
        double len = l_width;
        for (int s = 0; s < stages; ++s) {
            taus[s + 1] = tau_schedule(len, n);
            len *= (q + 1.0) / static_cast<double>(l);
        }
    });
}

int msfft_plan_gather_traffic(msfft_plan plan, int64_t batch, const uint64_t* seeds,
                              int64_t* loads, int64_t* sectors) {
    if (!plan || !seeds || !loads || !sectors) return MSFFT_ERR_INVALID_ARGUMENT;
    const SchedulePlan& sp = plan->plan->schedule();
    const int elem = plan->plan->c128() ? 16 : 8;
    const int nt = static_cast<int>(std::max<unsigned>(1u, std::thread::hardware_concurrency()));
    std::vector<int64_t> L(nt, 0), S(nt, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            std::vector<int64_t> sg(sp.iterations), sgi(sp.iterations);
            for (int64_t s = t; s < batch; s += nt) {
                draw_sigmas(seeds[s], sp.n, sp.iterations, sg.data(), sgi.data());
                gather_traffic(sp, sg.data(), elem, &L[t], &S[t]);
            }
        });
    for (auto& th : pool) th.join();
    *loads = 0;
    *sectors = 0;
    for (int t = 0; t < nt; ++t) {
        *loads += L[t];
        *sectors += S[t];
    }
    return MSFFT_OK;
}

int msfft_plan_stage_times(msfft_plan plan, double* ms3) {
    if (!plan || !ms3) return MSFFT_ERR_INVALID_ARGUMENT;
    for (int i = 0; i < 3; ++i) ms3[i] = plan->plan->stage_ms()[i];
    return MSFFT_OK;
}

int msfft_window(int64_t n, int64_t b, double delta, int32_t device, int64_t* w, double* taps,
                 int64_t taps_cap, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (device >= 0) MSFFT_CUDA(cudaSetDevice(device));
        auto win = get_device_window(n, b, delta);
        *w = win->w;
        if (taps && taps_cap >= win->w)
            std::memcpy(taps, win->taps.data(), sizeof(double) * static_cast<size_t>(win->w));
    });
}

int msfft_window_response(int64_t n, int64_t b, double delta, int32_t device,
                          const int64_t* idx, int64_t count, double* out, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (device >= 0) MSFFT_CUDA(cudaSetDevice(device));
        auto win = get_device_window(n, b, delta);
        std::vector<double> table(static_cast<size_t>(2 * win->gmax + 1));
        MSFFT_CUDA(cudaMemcpy(table.data(), win->d_ghat, sizeof(double) * table.size(),
                              cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < count; ++i) {
            if (idx[i] < -win->gmax || idx[i] > win->gmax)
                throw std::invalid_argument("msfft_window_response: offset outside the table");
            out[i] = table[static_cast<size_t>(idx[i] + win->gmax)];
        }
    });
}

int msfft_trace(const void* x, int64_t n, int32_t dtype, int64_t k, int64_t l, double q,
                uint64_t seed, double delta, double* pre, double* post, int64_t* sel_bucket,
                int64_t* sel_f, double* sel_value, int64_t cap, int64_t* out_f, double* out_c,
                int64_t* out_count, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const bool c128 = dtype == MSFFT_C128;
        auto plan = cached_plan(n, k, l, q, delta, c128, current_or(-1));
        std::lock_guard<std::mutex> lock(plan->mutex());
        std::vector<int64_t> f(static_cast<size_t>(k));
        std::vector<double> c(static_cast<size_t>(2 * k));
        int64_t count = 0;
        ExecOptions opt;
        opt.pre = pre;
        opt.post = post;
        opt.sel_bucket = sel_bucket;
        opt.sel_f = sel_f;
        opt.sel_value = sel_value;
        plan->execute(1, x, n, &seed, f.data(), c.data(), &count, opt, nullptr);
        *out_count = count;
        for (int64_t i = 0; i < count && i < cap; ++i) {
            out_f[i] = f[i];
            out_c[2 * i] = c[2 * i];
            out_c[2 * i + 1] = c[2 * i + 1];
        }
    });
}

}  // extern "C"
