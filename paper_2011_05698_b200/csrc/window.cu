// window.cu -- GPU flat-window designer, response table and device cache.
// Compiled with --fmad=false (see common.cuh).
//
// The design follows proj/src/window.cpp:105-177 step for step:
//   1. parameter checks (:106-111) with the reference's messages;
//   2. boxcar half-width c = 3L/4 (:114);
//   3. sigma = 64-step bisection on [L/80, L] of the analytic ripple
//      (:118-128; gaussian_tails :19-35, ideal_ripple :39-45) -- host, same
//      libm exp, same summation order;
//   4. ideal response from the discrete Gaussian CDF (:131-138) -- device;
//   5. inverse n-point FFT (:139) -- device, bit-identical radix-2;
//   6. real part + symmetrisation (:140-144) -- device;
//   7. binary search over odd w of the truncation check (:147-158; :71-85,
//      band scan :53-67) -- one device FFT + max-reduction per probe;
//   8. tap extraction (:169-175).
// Then the response table G_d (window.cpp:89-99) is evaluated on the device
// for every offset predict/estimate can ask for.
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"
#include "host_plan.hpp"
#include "window.hpp"

namespace msfft_b200 {

namespace {

// Suffix masses of the normalised discrete Gaussian (window.cpp:19-35).
// Only the first `top + 1` entries can be non-zero; the vector stops there
// and callers read indices beyond its end as 0.
std::vector<double> gaussian_suffix(double sigma, int64_t max_d) {
    const int64_t reach = std::min<int64_t>(max_d, static_cast<int64_t>(sigma * 42.0) + 2);
    std::vector<double> dens(static_cast<size_t>(reach + 1));
    auto fill = [&](int64_t lo, int64_t hi) {
        for (int64_t m = lo; m < hi; ++m)
            dens[m] = std::exp(-0.5 * static_cast<double>(m) * static_cast<double>(m) /
                               (sigma * sigma));
    };
    if (reach < (1 << 18)) {
        fill(0, reach + 1);
    } else {
        const int nt = static_cast<int>(
            std::max<unsigned>(1u, std::min<unsigned>(16u, std::thread::hardware_concurrency())));
        std::vector<std::thread> pool;
        const int64_t per = (reach + 1 + nt - 1) / nt;
        for (int i = 0; i < nt; ++i)
            pool.emplace_back(fill, std::min(reach + 1, i * per), std::min(reach + 1, (i + 1) * per));
        for (auto& th : pool) th.join();
    }
    double total = dens[0];
    for (int64_t m = 1; m <= reach; ++m) total += 2.0 * dens[m];
    const int64_t top = std::min(reach, max_d + 1);
    std::vector<double> tail(static_cast<size_t>(top + 1));
    double acc = 0.0;
    for (int64_t d = top; d >= 0; --d) {
        acc += dens[d];
        tail[d] = acc / total;
    }
    return tail;
}

inline double tail_at(const std::vector<double>& t, int64_t i) {
    return i < static_cast<int64_t>(t.size()) ? t[i] : 0.0;
}

// Worst-case band deviation of the untruncated response (window.cpp:39-45).
double analytic_ripple(double sigma, int64_t L, int64_t c) {
    const int64_t half = L / 2;
    const auto tail = gaussian_suffix(sigma, L + c + 2);
    const double pass = tail_at(tail, c - half + 1) + tail_at(tail, c + half + 1);
    const double stop = tail_at(tail, L - c);
    return std::max(pass, stop);
}

__global__ void ideal_kernel(double2* __restrict__ out, int64_t n, int64_t c,
                             const double* __restrict__ tail, int64_t ntail) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto T = [&](int64_t j) { return j < ntail ? tail[j] : 0.0; };
    const int64_t d = i < n - i ? i : n - i;
    const double v = d <= c ? 1.0 - T(c - d + 1) - T(c + d + 1) : T(d - c) - T(d + c + 1);
    out[i] = make_double2(v, 0.0);
}

// g[t] = Re ideal[t], then g[t] = g[n-t] = (g[t] + g[n-t]) / 2 for 0 < t < n-t.
__global__ void symmetrize_kernel(double* __restrict__ g, const double2* __restrict__ ideal,
                                  int64_t n) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t u = t < n - t ? t : n - t;
    if (u == 0 || u == n - u) {
        g[t] = ideal[t].x;
    } else {
        g[t] = 0.5 * (ideal[u].x + ideal[n - u].x);
    }
}

__global__ void truncate_kernel(double2* __restrict__ out, const double* __restrict__ g,
                                int64_t n, int64_t h) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool keep = (i <= h) || (i >= n - h);
    out[i] = make_double2(keep ? g[i] : 0.0, 0.0);
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Band scan of the scaled response (window.cpp:53-67, 80-84).  maxes:
// [pass_dev, stop_max, trans_max] as non-negative double bit patterns.
__global__ void band_scan_kernel(const double2* __restrict__ v, int64_t n, int64_t L,
                                 double scale, unsigned long long* __restrict__ maxes) {
    double pass = 0.0, stop = 0.0, trans = 0.0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 z = v[i];
        const double mag = cabs_ref(z.x * scale, z.y * scale);
        const int64_t d = i < n - i ? i : n - i;
        if (d <= L / 2)
            pass = fmax(pass, fabs(mag - 1.0));
        else if (d >= L)
            stop = fmax(stop, mag);
        else
            trans = fmax(trans, mag);
    }
    pass = warp_max(pass);
    stop = warp_max(stop);
    trans = warp_max(trans);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&maxes[0], static_cast<unsigned long long>(__double_as_longlong(pass)));
        atomicMax(&maxes[1], static_cast<unsigned long long>(__double_as_longlong(stop)));
        atomicMax(&maxes[2], static_cast<unsigned long long>(__double_as_longlong(trans)));
    }
}

__global__ void extract_taps_kernel(double* __restrict__ taps, const double* __restrict__ g,
                                    int64_t n, int64_t h) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t > h) return;
    taps[h + t] = g[t];
    taps[h - t] = g[t == 0 ? 0 : n - t];
    if (t == 0) taps[2 * h + 1] = 0.0;  // pad to an even length
}

// G_d = response_at(d) (window.cpp:89-99) for d in [-gmax, gmax]: the same
// sequential series over t with the same argument reduction
// (i0 * t mod n) * 2pi / n; only libm's cos is replaced by CUDA's.
__global__ void response_table_kernel(double* __restrict__ ghat, const double* __restrict__ taps,
                                      int64_t n, int64_t h, int64_t gmax) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx > 2 * gmax) return;
    const int64_t d = idx - gmax;
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const uint64_t i0 = static_cast<uint64_t>(d) & mask;  // d mod n, n a power of two
    const double nd = static_cast<double>(n);
    double acc = taps[h];
    for (int64_t t = 1; t <= h; ++t) {
        const uint64_t m = (i0 * static_cast<uint64_t>(t)) & mask;
        const double a = kTwoPi * static_cast<double>(m) / nd;
        acc += 2.0 * taps[h + t] * cos(a);
    }
    ghat[idx] = acc / nd;
}

// Wide windows (few entries, h up to ~10^6): a warp per entry, lanes take
// every 32nd tap, then a shuffle reduction.  The summation order differs from
// the sequential series only by rounding (the table is cos-limited anyway).
__global__ void response_table_warp_kernel(double* __restrict__ ghat,
                                           const double* __restrict__ taps, int64_t n,
                                           int64_t h, int64_t gmax) {
    const int64_t idx = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (idx > 2 * gmax) return;
    const int64_t d = idx - gmax;
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const uint64_t i0 = static_cast<uint64_t>(d) & mask;
    const double nd = static_cast<double>(n);
    double acc = 0.0;
    for (int64_t t = 1 + lane; t <= h; t += 32) {
        const uint64_t m = (i0 * static_cast<uint64_t>(t)) & mask;
        acc += 2.0 * taps[h + t] * cos(kTwoPi * static_cast<double>(m) / nd);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) ghat[idx] = (taps[h] + acc) / nd;
}

// response_at(idx[k]) for arbitrary offsets (any residue mod n): the same
// two series as the table kernels above, chosen by the same h threshold, so
// an offset inside the table gets exactly the table's value.
__global__ void response_list_kernel(double* __restrict__ out, const int64_t* __restrict__ idx,
                                     int64_t count, const double* __restrict__ taps, int64_t n,
                                     int64_t h, int warp_per_entry) {
    const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t k = warp_per_entry ? (gt >> 5) : gt;
    const int lane = warp_per_entry ? static_cast<int>(threadIdx.x & 31) : 0;
    if (k >= count) return;
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    const uint64_t i0 = static_cast<uint64_t>(idx[k]) & mask;
    const double nd = static_cast<double>(n);
    if (!warp_per_entry) {
        double acc = taps[h];
        for (int64_t t = 1; t <= h; ++t) {
            const uint64_t m = (i0 * static_cast<uint64_t>(t)) & mask;
            const double a = kTwoPi * static_cast<double>(m) / nd;
            acc += 2.0 * taps[h + t] * cos(a);
        }
        out[k] = acc / nd;
        return;
    }
    double acc = 0.0;
    for (int64_t t = 1 + lane; t <= h; t += 32) {
        const uint64_t m = (i0 * static_cast<uint64_t>(t)) & mask;
        acc += 2.0 * taps[h + t] * cos(kTwoPi * static_cast<double>(m) / nd);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[k] = (taps[h] + acc) / nd;
}

struct Key {
    int device;
    int64_t n, b;
    double delta;
    bool operator<(const Key& o) const {
        return std::tie(device, n, b, delta) < std::tie(o.device, o.n, o.b, o.delta);
    }
};

std::mutex g_mu;
std::map<Key, std::shared_ptr<const DeviceWindow>> g_cache;
std::map<Key, std::string> g_infeasible;

unsigned blocks_for(int64_t n, int threads) {
    return static_cast<unsigned>((n + threads - 1) / threads);
}

std::shared_ptr<DeviceWindow> design_on_device(int device, int64_t n, int64_t b, double delta) {
    if (n < 16 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("design_flat_window: n must be a power of two >= 16");
    if (b < 4 || b > n / 4 || !is_pow2_u(static_cast<uint64_t>(b)))
        throw std::invalid_argument("design_flat_window: need b a power of two, 4 <= b <= n/4");
    if (!(delta > 0.0 && delta < 0.1))
        throw std::invalid_argument("design_flat_window: delta must be in (0, 0.1)");
    if (n > (int64_t{1} << 30))
        throw std::invalid_argument("design_flat_window: n above 2^30 is not supported");

    const int64_t L = n / b;
    const int64_t c = 3 * L / 4;
    double lo = static_cast<double>(L) / 80.0, hi = static_cast<double>(L);
    if (analytic_ripple(lo, L, c) > 0.5 * delta)
        throw std::invalid_argument("design_flat_window: infeasible (n, b, delta)");
    for (int iter = 0; iter < 64; ++iter) {
        const double mid = 0.5 * (lo + hi);
        if (analytic_ripple(mid, L, c) <= 0.5 * delta)
            lo = mid;
        else
            hi = mid;
    }
    const double sigma = lo;
    const auto tail = gaussian_suffix(sigma, n / 2 + c + 2);

    cudaStream_t st;
    MSFFT_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{st};

    DeviceBuffer<double> d_tail(tail.size());
    MSFFT_CUDA(cudaMemcpyAsync(d_tail.get(), tail.data(), tail.size() * sizeof(double),
                               cudaMemcpyHostToDevice, st));
    DeviceBuffer<double2> work(static_cast<size_t>(n));
    DeviceBuffer<double> g(static_cast<size_t>(n));
    DeviceBuffer<unsigned long long> maxes(3);
    const int T = 256;
    ideal_kernel<<<blocks_for(n, T), T, 0, st>>>(work.get(), n, c, d_tail.get(),
                                                  static_cast<int64_t>(tail.size()));
    MSFFT_LAUNCH_CHECK("ideal_kernel");
    fft_radix2_batched(work.get(), n, 1, 1, n, +1, 1.0, st);
    symmetrize_kernel<<<blocks_for(n, T), T, 0, st>>>(g.get(), work.get(), n);
    MSFFT_LAUNCH_CHECK("symmetrize_kernel");

    const double scale = 1.0 / static_cast<double>(n);
    auto passes = [&](int64_t w) {
        const int64_t h = (w - 1) / 2;
        truncate_kernel<<<blocks_for(n, T), T, 0, st>>>(work.get(), g.get(), n, h);
        MSFFT_LAUNCH_CHECK("truncate_kernel");
        fft_radix2_batched(work.get(), n, 1, 1, n, -1, 1.0, st);
        MSFFT_CUDA(cudaMemsetAsync(maxes.get(), 0, 3 * sizeof(unsigned long long), st));
        const unsigned nb = std::min<unsigned>(blocks_for(n, T), 148u * 8u);
        band_scan_kernel<<<nb, T, 0, st>>>(work.get(), n, L, scale, maxes.get());
        MSFFT_LAUNCH_CHECK("band_scan_kernel");
        unsigned long long hm[3];
        MSFFT_CUDA(cudaMemcpyAsync(hm, maxes.get(), sizeof(hm), cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        double m[3];
        for (int i = 0; i < 3; ++i) std::memcpy(&m[i], &hm[i], sizeof(double));
        return m[0] <= delta && m[1] <= delta && m[2] <= 1.0 + delta;
    };
    int64_t w_hi = n - 1;
    if (!passes(w_hi))
        throw std::invalid_argument(
            "design_flat_window: no support w <= n-1 passes the band check");
    int64_t w_lo = 1;
    while (w_lo < w_hi) {
        int64_t mid = w_lo + (w_hi - w_lo) / 2;
        if (mid % 2 == 0) --mid;
        if (passes(mid))
            w_hi = mid;
        else
            w_lo = mid + 2;
    }
    const int64_t w = w_hi;
    const int64_t h = (w - 1) / 2;

    auto win = std::make_shared<DeviceWindow>();
    win->device = device;
    win->n = n;
    win->b = b;
    win->l_width = L;
    win->w = w;
    win->h = h;
    win->delta = delta;
    win->gmax = 3 * L / 2 + 1;
    MSFFT_CUDA(cudaMalloc(&win->d_taps, sizeof(double) * static_cast<size_t>(w + 1)));
    MSFFT_CUDA(cudaMalloc(&win->d_ghat, sizeof(double) * static_cast<size_t>(2 * win->gmax + 1)));
    extract_taps_kernel<<<blocks_for(h + 1, T), T, 0, st>>>(win->d_taps, g.get(), n, h);
    MSFFT_LAUNCH_CHECK("extract_taps_kernel");
    if (h <= 8192) {
        response_table_kernel<<<blocks_for(2 * win->gmax + 1, 128), 128, 0, st>>>(
            win->d_ghat, win->d_taps, n, h, win->gmax);
    } else {
        response_table_warp_kernel<<<blocks_for((2 * win->gmax + 1) * 32, 256), 256, 0, st>>>(
            win->d_ghat, win->d_taps, n, h, win->gmax);
    }
    MSFFT_LAUNCH_CHECK("response_table_kernel");
    win->taps.resize(static_cast<size_t>(w));
    MSFFT_CUDA(cudaMemcpyAsync(win->taps.data(), win->d_taps, sizeof(double) * w,
                               cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaStreamSynchronize(st));
    return win;
}

}  // namespace

DeviceWindow::~DeviceWindow() {
    // Windows live in a process-lifetime cache; freeing at static destruction
    // can race CUDA teardown, so only free when the context is still alive.
    if (d_taps || d_ghat) {
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess) {
            cudaFree(d_taps);
            cudaFree(d_ghat);
        }
    }
}

std::shared_ptr<const DeviceWindow> get_device_window(int64_t n, int64_t b, double delta) {
    int device = 0;
    MSFFT_CUDA(cudaGetDevice(&device));
    const Key key{device, n, b, delta};
    {
        std::lock_guard<std::mutex> lock(g_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) return it->second;
        auto bad = g_infeasible.find(key);
        if (bad != g_infeasible.end()) throw std::invalid_argument(bad->second);
    }
    std::shared_ptr<const DeviceWindow> win;
    try {
        win = design_on_device(device, n, b, delta);
    } catch (const std::invalid_argument& e) {
        std::lock_guard<std::mutex> lock(g_mu);
        g_infeasible.emplace(key, e.what());
        throw;
    }
    std::lock_guard<std::mutex> lock(g_mu);
    auto [it, inserted] = g_cache.emplace(key, win);
    return it->second;
}

int64_t window_support(int64_t n, int64_t b, double delta) {
    return get_device_window(n, b, delta)->w;
}

void window_response_list(int64_t n, int64_t b, double delta, const int64_t* idx, int64_t count,
                          double* out) {
    auto win = get_device_window(n, b, delta);
    if (count <= 0) return;
    int64_t* d_idx = nullptr;
    double* d_out = nullptr;
    MSFFT_CUDA(cudaMalloc(&d_idx, sizeof(int64_t) * count));
    MSFFT_CUDA(cudaMalloc(&d_out, sizeof(double) * count));
    MSFFT_CUDA(cudaMemcpy(d_idx, idx, sizeof(int64_t) * count, cudaMemcpyHostToDevice));
    const int wpe = win->h > 8192 ? 1 : 0;
    const int64_t threads = wpe ? count * 32 : count;
    response_list_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256>>>(
        d_out, d_idx, count, win->d_taps, n, win->h, wpe);
    const cudaError_t le = cudaGetLastError();
    cudaError_t ce = cudaSuccess;
    if (le == cudaSuccess) ce = cudaMemcpy(out, d_out, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(d_idx);
    cudaFree(d_out);
    MSFFT_CUDA(le);
    MSFFT_CUDA(ce);
}

}  // namespace msfft_b200
