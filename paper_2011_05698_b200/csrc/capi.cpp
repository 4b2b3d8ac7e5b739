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
#include "components.hpp"
#include "engine.hpp"
#include "host_plan.hpp"
#include "phase_mc.hpp"
#include "signal_io.hpp"
#include "signal_ops.hpp"
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
        PlanLease lease;
        try {
            lease = lease_plan(n, k, l, q, delta, c128, current_or(-1));
        } catch (const std::invalid_argument&) {
            // sfft4 validates x before its other arguments (sfft4.cpp:133-135)
            if (has_non_finite(x, n, c128, on_dev))
                throw std::invalid_argument("ComplexSignal: non-finite sample");
            throw;
        }
        Plan* plan = lease.plan.get();
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
        opt.async_call = (flags & MSFFT_FLAG_ASYNC) != 0;
        opt.stream = static_cast<cudaStream_t>(stream);
        plan->plan->execute(batch, x, x_stride, seeds, out_f, out_c, out_count, opt, device_ms);
    });
}

int msfft_plan_sync(msfft_plan plan, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_plan_sync: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        plan->plan->sync(static_cast<cudaStream_t>(stream));
    });
}

int64_t msfft_plan_ingest_samples(msfft_plan plan) {
    if (!plan) return -1;
    return plan->plan->ingest_samples_per_signal();
}

int msfft_validate_signal(const void* x, int64_t n, int64_t sample_count, int64_t batch,
                          int64_t x_stride, int32_t dtype, int32_t x_location, void* stream,
                          double* device_ms, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        // ComplexSignal::validate (proj/src/signal.cpp:18-26), same check order
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
        if (sample_count != n) throw std::invalid_argument("ComplexSignal: sample count != n");
        if (dtype != MSFFT_C128 && dtype != MSFFT_C64)
            throw std::invalid_argument("msfft_validate_signal: unknown dtype");
        if (batch < 0 || x_stride < n)
            throw std::invalid_argument("msfft_validate_signal: need batch >= 0 and x_stride >= n");
        const bool c128 = dtype == MSFFT_C128;
        if (device_ms) *device_ms = 0.0;
        if (batch == 0) return;
        if (x_location != MSFFT_DEVICE) {
            const size_t row = static_cast<size_t>(x_stride) * (c128 ? 16 : 8);
            for (int64_t s = 0; s < batch; ++s)
                if (has_non_finite(static_cast<const unsigned char*>(x) + s * row, n, c128, false))
                    throw std::invalid_argument("ComplexSignal: non-finite sample");
            return;
        }
        require_device();
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        int32_t* d_bad = nullptr;
        MSFFT_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(int32_t), st));
        MSFFT_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), st));
        cudaEvent_t ev[2];
        MSFFT_CUDA(cudaEventCreate(&ev[0]));
        MSFFT_CUDA(cudaEventCreate(&ev[1]));
        MSFFT_CUDA(cudaEventRecord(ev[0], st));
        launch_validate(x, c128, n, x_stride, batch, d_bad, st);
        MSFFT_CUDA(cudaEventRecord(ev[1], st));
        int32_t bad = 0;
        MSFFT_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaFreeAsync(d_bad, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        MSFFT_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        if (device_ms) *device_ms = ms;
        if (bad) throw std::invalid_argument("ComplexSignal: non-finite sample");
    });
}

int msfft_plan_copy_bytes(msfft_plan plan, int64_t* h2d, int64_t* d2h) {
    if (!plan) return MSFFT_ERR_INVALID_ARGUMENT;
    if (h2d) *h2d = plan->plan->last_h2d_bytes();
    if (d2h) *d2h = plan->plan->last_d2h_bytes();
    return MSFFT_OK;
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

int msfft_encode_values_part(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                             int64_t part, int64_t parts, const uint64_t* seeds, double* y,
                             uint32_t flags, void* stream, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_encode_values_part: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        plan->plan->encode_values_part(batch, x, x_stride, part, parts, seeds,
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

int msfft_decode_folds(msfft_plan plan, int64_t batch, double* y, const uint64_t* seeds,
                       int64_t* out_f, double* out_c, int64_t* out_count, void* stream,
                       char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!plan) throw std::invalid_argument("msfft_decode_folds: null plan");
        std::lock_guard<std::mutex> lock(plan->plan->mutex());
        plan->plan->decode_values(batch, reinterpret_cast<double2*>(y), seeds, out_f,
                                  reinterpret_cast<double2*>(out_c), out_count,
                                  static_cast<cudaStream_t>(stream), true);
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

int msfft_mod_inverse(int64_t sigma, int64_t n, int64_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *out = mod_inverse(sigma, n); });
}

int64_t msfft_bucket_of(int64_t u, int64_t l_width, int64_t b) {
    if (l_width <= 0 || b <= 0) return -1;
    return bucket_of(u, l_width, b);
}

int msfft_stage_count(double region_length, int64_t l, double q, int32_t* out, char* err,
                      size_t errlen) {
    return guarded(err, errlen, [&] {
        // the reference loops forever when l/(q+1) <= 1; report the config error
        if (!(static_cast<double>(l) / (q + 1.0) > 1.0)) validate_cfg(l, q);
        *out = stage_count(region_length, l, q);
    });
}

int msfft_tau_schedule(double region_length, int64_t n, int64_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (n < 2) throw std::invalid_argument("tau_schedule: need n >= 2");
        *out = tau_schedule(region_length, n);
    });
}

int msfft_config_validate(int64_t l, double q, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { validate_cfg(l, q); });
}

int msfft_check_parameter_bounds(double max_dphi, int64_t l, double q, int32_t* l_ok,
                                 double* q_min, char* err, size_t errlen) {
    (void)q;  // unused by the reference as well (locate.cpp:125)
    return guarded(err, errlen, [&] {
        bool ok = false;
        check_parameter_bounds(max_dphi, l, &ok, q_min);
        *l_ok = ok ? 1 : 0;
    });
}

int msfft_initial_bucket_count(int64_t n, int64_t k, double delta, int64_t* out, char* err,
                               size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        int64_t b = 4;
        while (b < 4 * k) b *= 2;
        b = std::min(b, n / 4);
        b = std::max<int64_t>(b, 4);
        for (;;) {
            try {
                window_support(n, b, delta);  // get_flat_window on the GPU designer
                *out = b;
                return;
            } catch (const std::invalid_argument&) {
                if (b <= 4) throw;
                b /= 2;
            }
        }
    });
}

int msfft_phase_of(const double* z, int64_t count, double* phase, int32_t* status, char* err,
                   size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        phase_of_host(z, count, phase, status, nullptr);
    });
}

int msfft_position_phase(const double* u, const int64_t* tau, int64_t count, int64_t n,
                         double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (n < 2 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("position_phase: n must be a power of two");
        position_phase_host(u, tau, count, n, out, nullptr);
    });
}

int msfft_circular_phase_distance(const double* a, const double* b, int64_t count, double* out,
                                  char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        circular_phase_distance_host(a, b, count, out, nullptr);
    });
}

int msfft_locate_step(const double* phi, const int64_t* tau, const msfft_locate_region* region,
                      int64_t count, int64_t l, double q, int64_t n, msfft_locate_region* out,
                      char* err, size_t errlen) {
    static_assert(sizeof(msfft_locate_region) == sizeof(LocateRegionDev), "region layout");
    return guarded(err, errlen, [&] {
        require_device();
        if (n < 2 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("locate_step: n must be a power of two");
        if (l < 1) throw std::invalid_argument("MultiscaleConfig: l must be >= 2");
        locate_step_host(phi, tau, reinterpret_cast<const LocateRegionDev*>(region), count, l, q,
                         n, reinterpret_cast<LocateRegionDev*>(out), nullptr);
    });
}

int msfft_bucketize_taps(int64_t n, int64_t b, double delta, const double* values, int64_t rounds,
                         double* out, int64_t* samples_read, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const int64_t w = bucketize_taps_host(n, b, delta, values, rounds, out, nullptr);
        if (samples_read) *samples_read = w;
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
        window_response_list(n, b, delta, idx, count, out);
    });
}

int msfft_trace(const void* x, int64_t n, int32_t dtype, int64_t k, int64_t l, double q,
                uint64_t seed, double delta, double* pre, double* post, int64_t* sel_bucket,
                int64_t* sel_f, double* sel_value, int64_t cap, int64_t* out_f, double* out_c,
                int64_t* out_count, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const bool c128 = dtype == MSFFT_C128;
        PlanLease lease = lease_plan(n, k, l, q, delta, c128, current_or(-1));
        Plan* plan = lease.plan.get();
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

// ---- signal helpers -----------------------------------------

namespace {

size_t elem_of(int32_t dtype) {
    if (dtype != MSFFT_C128 && dtype != MSFFT_C64) throw std::invalid_argument("msfft: unknown dtype");
    return dtype == MSFFT_C128 ? 16 : 8;
}

// Device view of a caller buffer: the buffer itself, or a device copy that
// is written back (when `out`) for host buffers.
struct DeviceView {
    void* host = nullptr;
    void* dev = nullptr;
    size_t bytes = 0;
    DeviceBuffer<unsigned char> own;
    DeviceView(void* p, size_t b, bool on_device, bool copy_in) : bytes(b) {
        if (on_device) {
            dev = p;
            return;
        }
        host = p;
        own.reset(b);
        dev = own.get();
        if (copy_in && b) MSFFT_CUDA(cudaMemcpy(dev, p, b, cudaMemcpyHostToDevice));
    }
    void write_back() {
        if (host && bytes) MSFFT_CUDA(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost));
    }
};

}  // namespace

int msfft_generate_test_signal(int64_t n, int64_t k, uint64_t seed, int32_t dtype,
                               int32_t location, void* x, int64_t* truth_f, double* truth_c,
                               int32_t* bit_exact, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const size_t esz = elem_of(dtype);
        std::vector<int64_t> f;
        std::vector<double> c;
        random_sparse_spectrum(n, k, seed, f, c);
        DeviceView v(x, static_cast<size_t>(n) * esz, location == MSFFT_DEVICE, false);
        const bool exact = synthesize_device(n, f.data(), c.data(), static_cast<int64_t>(f.size()),
                                             dtype == MSFFT_C128, v.dev, nullptr);
        v.write_back();
        for (size_t i = 0; i < f.size(); ++i) {
            truth_f[i] = f[i];
            truth_c[2 * i] = c[2 * i];
            truth_c[2 * i + 1] = c[2 * i + 1];
        }
        if (bit_exact) *bit_exact = exact ? 1 : 0;
    });
}

int msfft_synthesize(int64_t n, const int64_t* f, const double* c, int64_t count, int32_t dtype,
                     int32_t location, void* x, int32_t* bit_exact, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const size_t esz = elem_of(dtype);
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("SparseSpectrum: n must be a power of two >= 4");
        DeviceView v(x, static_cast<size_t>(n) * esz, location == MSFFT_DEVICE, false);
        const bool exact = synthesize_device(n, f, c, count, dtype == MSFFT_C128, v.dev, nullptr);
        v.write_back();
        if (bit_exact) *bit_exact = exact ? 1 : 0;
    });
}

int msfft_add_awgn(void* x, int64_t n, int32_t dtype, int32_t location, double snr_db,
                   uint64_t seed, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const size_t esz = elem_of(dtype);
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
        DeviceView v(x, static_cast<size_t>(n) * esz, location == MSFFT_DEVICE, true);
        awgn_device(v.dev, dtype == MSFFT_C128, n, snr_db, seed, nullptr);
        v.write_back();
    });
}

int msfft_dft_dense(const void* x, int64_t n, int64_t batch, int32_t dtype, int32_t location,
                    double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const size_t esz = elem_of(dtype);
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
        const bool dev = location == MSFFT_DEVICE;
        DeviceView in(const_cast<void*>(x), static_cast<size_t>(n * batch) * esz, dev, true);
        DeviceView o(out, static_cast<size_t>(n * batch) * 16, dev, false);
        dense_dft_device(in.dev, dtype == MSFFT_C128, n, batch, static_cast<double2*>(o.dev), -1,
                         nullptr);
        o.write_back();
    });
}

int msfft_idft_dense(const double* spec, int64_t n, int64_t batch, int32_t location, double* out,
                     char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("idft_dense: size must be a power of two >= 4");
        const bool dev = location == MSFFT_DEVICE;
        DeviceView in(const_cast<double*>(spec), static_cast<size_t>(n * batch) * 16, dev, true);
        DeviceView o(out, static_cast<size_t>(n * batch) * 16, dev, false);
        dense_dft_device(in.dev, true, n, batch, static_cast<double2*>(o.dev), +1, nullptr);
        o.write_back();
    });
}

int msfft_top_k_spectrum(const double* spec, int64_t n, int64_t k, int32_t location,
                         int64_t* out_f, double* out_c, int64_t* out_count, char* err,
                         size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        DeviceView in(const_cast<double*>(spec), static_cast<size_t>(n) * 16,
                      location == MSFFT_DEVICE, true);
        *out_count = top_k_device(static_cast<const double2*>(in.dev), n, k, out_f, out_c, nullptr);
    });
}

int msfft_error_metrics(int64_t truth_n, const int64_t* truth_f, const double* truth_c,
                        int64_t truth_count, int64_t est_n, const int64_t* est_f,
                        const double* est_c, int64_t est_count, int64_t k,
                        msfft_eval_metrics* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const EvalMetrics m = error_metrics(truth_n, truth_f, truth_c, truth_count, est_n, est_f,
                                            est_c, est_count, k);
        out->l0_err = m.l0;
        out->l1_err = m.l1;
        out->l2_err = m.l2;
    });
}

int msfft_signal_file_length(const char* path, int64_t* n, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *n = signal_file_length(path); });
}

int msfft_read_signal_file(const char* path, int32_t dtype, int32_t location, void* x,
                           int64_t cap, int64_t* n, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const size_t esz = elem_of(dtype);
        (void)esz;
        *n = read_signal_file(path, dtype == MSFFT_C128, location == MSFFT_DEVICE, x, cap);
    });
}

int msfft_write_signal_file(const char* path, const void* x, int64_t n, int32_t dtype,
                            int32_t location, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        elem_of(dtype);
        write_signal_file(path, x, n, dtype == MSFFT_C128, location == MSFFT_DEVICE);
    });
}

int msfft_write_truth_csv(const char* path, const int64_t* f, const double* c, int64_t count,
                          char* err, size_t errlen) {
    return guarded(err, errlen, [&] { write_truth_csv(path, f, c, count); });
}

int msfft_read_truth_csv(const char* path, int64_t n, int64_t* f, double* c, int64_t cap,
                         int64_t* count, char* err, size_t errlen) {
    return guarded(err, errlen, [&] { *count = read_truth_csv(path, n, f, c, cap); });
}

int msfft_phase_experiment(int64_t n, int64_t k, int64_t b, const double* snr_list, int64_t nsnr,
                           int64_t trials, uint64_t seed, msfft_phase_histogram* out,
                           msfft_phase_trial* trials_out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        std::vector<std::vector<PhaseTrialOut>> tr;
        const auto hs = phase_experiment(n, k, b, std::vector<double>(snr_list, snr_list + nsnr),
                                         trials, seed, trials_out ? &tr : nullptr);
        for (size_t i = 0; i < hs.size(); ++i) {
            msfft_phase_histogram& o = out[i];
            o.snr_db = hs[i].snr_db;
            o.n = hs[i].n;
            o.k = hs[i].k;
            o.l_width = hs[i].l_width;
            o.trials = hs[i].trials;
            for (int j = 0; j < MSFFT_PHASE_BINS; ++j) o.bin_mass[j] = hs[i].bin_mass[j];
            o.p50 = hs[i].p50;
            o.p99 = hs[i].p99;
            o.max = hs[i].max;
            if (trials_out)
                for (size_t t = 0; t < tr[i].size(); ++t) {
                    const PhaseTrialOut& a = tr[i][t];
                    msfft_phase_trial& d = trials_out[i * static_cast<size_t>(trials) + t];
                    d.dphi = a.dphi;
                    d.u = a.u;
                    d.bucket = a.bucket;
                    d.tau = a.tau;
                    d.y0[0] = a.y0[0];
                    d.y0[1] = a.y0[1];
                    d.y_tau[0] = a.y_tau[0];
                    d.y_tau[1] = a.y_tau[1];
                    d.measured_phi = a.measured_phi;
                    d.true_phi = a.true_phi;
                }
        }
    });
}


int msfft_bucketize(const void* x, int64_t n, int32_t dtype, int32_t x_location, int64_t b,
                    double delta, const int64_t* sigma, const int64_t* tau, int64_t rounds,
                    double* values, int32_t values_location, int64_t* samples_read, char* err,
                    size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const size_t esz = elem_of(dtype);
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
            throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
        if (rounds < 1) throw std::invalid_argument("bucketize: rounds must be >= 1");
        DeviceView in(const_cast<void*>(x), static_cast<size_t>(n) * esz,
                      x_location == MSFFT_DEVICE, true);
        DeviceView out(values, static_cast<size_t>(rounds * b) * 16,
                       values_location == MSFFT_DEVICE, false);
        const int64_t w = bucketize_device(in.dev, dtype == MSFFT_C128, n, b, delta, sigma, tau,
                                           rounds, static_cast<double2*>(out.dev), nullptr);
        out.write_back();
        if (samples_read) *samples_read = w;
    });
}

int msfft_predict_buckets(int64_t n, int64_t b, double delta, const int64_t* f, const double* c,
                          int64_t count, const int64_t* sigma, const int64_t* tau,
                          int64_t rounds, double* values, int32_t location, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        if (rounds < 1) throw std::invalid_argument("predict_buckets: rounds must be >= 1");
        if (count < 0) throw std::invalid_argument("predict_buckets: negative tone count");
        const bool dev = location == MSFFT_DEVICE;
        if (!dev) {  // SparseSpectrum is a std::map: ascending, unique positions
            for (int64_t i = 0; i < count; ++i)
                if (f[i] < 0 || f[i] >= n || (i > 0 && f[i] <= f[i - 1]))
                    throw std::invalid_argument(
                        "predict_buckets: positions must be strictly ascending in [0, n)");
        }
        DeviceView df(const_cast<int64_t*>(f), static_cast<size_t>(count) * 8, dev, true);
        DeviceView dc(const_cast<double*>(c), static_cast<size_t>(count) * 16, dev, true);
        DeviceView out(values, static_cast<size_t>(rounds * b) * 16, dev, false);
        predict_buckets_device(n, b, delta, static_cast<const int64_t*>(df.dev),
                               static_cast<const double2*>(dc.dev), count, sigma, tau, rounds,
                               static_cast<double2*>(out.dev), nullptr);
        out.write_back();
    });
}

int msfft_locate_frequency(int64_t n, int64_t b, int64_t l, double q, const int64_t* buckets,
                           int64_t count, const double* rounds, const int64_t* tau,
                           int64_t nrounds, int64_t* u, int32_t* stages, int32_t* status,
                           int32_t location, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        validate_cfg(l, q);
        if (nrounds < 1) throw std::invalid_argument("locate_frequency: no rounds");
        if (tau[0] != 0) throw std::invalid_argument("locate_frequency: round 0 must have tau = 0");
        if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)) || b < 1 ||
            !is_pow2_u(static_cast<uint64_t>(b)) || b > n)
            throw std::invalid_argument("locate_frequency: n and b must be powers of two, b <= n");
        const int needed = stage_count(static_cast<double>(n / b), l, q);
        if (nrounds < needed + 1)
            throw std::invalid_argument("locate_frequency: not enough rounds for the schedule");
        const bool dev = location == MSFFT_DEVICE;
        DeviceView db(const_cast<int64_t*>(buckets), static_cast<size_t>(count) * 8, dev, true);
        if (!dev)
            for (int64_t i = 0; i < count; ++i)
                if (buckets[i] < 0 || buckets[i] >= b)
                    throw std::invalid_argument("locate_frequency: bucket out of range");
        DeviceView dr(const_cast<double*>(rounds), static_cast<size_t>(nrounds * b) * 16, dev,
                      true);
        DeviceView du(u, static_cast<size_t>(count) * 8, dev, false);
        DeviceView ds(stages, static_cast<size_t>(count) * 4, dev, false);
        DeviceView dst(status, static_cast<size_t>(count) * 4, dev, false);
        locate_frequency_device(n, b, l, q, static_cast<const int64_t*>(db.dev), count,
                                static_cast<const double2*>(dr.dev), tau, nrounds,
                                static_cast<int64_t*>(du.dev), static_cast<int32_t*>(ds.dev),
                                static_cast<int32_t*>(dst.dev), nullptr);
        du.write_back();
        ds.write_back();
        dst.write_back();
        std::vector<int32_t> st(static_cast<size_t>(count));
        if (count)
            MSFFT_CUDA(cudaMemcpy(st.data(), dst.dev, st.size() * 4, cudaMemcpyDeviceToHost));
        for (const int32_t code : st) {  // first failing bucket in input order
            if (code == 2) throw std::domain_error("phase_of: zero value");
            if (code == 3)
                throw std::invalid_argument("locate_frequency: not enough rounds for the schedule");
            if (code == 4) throw std::invalid_argument("locate_frequency: bucket out of range");
        }
    });
}

int msfft_estimate_values(int64_t n, int64_t b, double delta, const double* y0, const int64_t* u,
                          int64_t count, double* out, int32_t* status, int32_t location,
                          char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        require_device();
        const bool dev = location == MSFFT_DEVICE;
        DeviceView dy(const_cast<double*>(y0), static_cast<size_t>(count) * 16, dev, true);
        DeviceView du(const_cast<int64_t*>(u), static_cast<size_t>(count) * 8, dev, true);
        DeviceView dout(out, static_cast<size_t>(count) * 16, dev, false);
        DeviceView dst(status, static_cast<size_t>(count) * 4, dev, false);
        estimate_values_device(n, b, delta, static_cast<const double2*>(dy.dev),
                               static_cast<const int64_t*>(du.dev), count,
                               static_cast<double2*>(dout.dev), static_cast<int32_t*>(dst.dev),
                               nullptr);
        dout.write_back();
        dst.write_back();
    });
}

}  // extern "C"
