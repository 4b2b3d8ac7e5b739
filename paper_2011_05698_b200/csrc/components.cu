// components.cu -- bucketize / predict_buckets / locate_frequency /
// estimate_value as batched device functions (see components.hpp).
#include "components.hpp"

#include <algorithm>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"
#include "window.hpp"

namespace msfft_b200 {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ double2 load_sample(const float2* x, int64_t i) {
    const float2 v = __ldg(x + i);
    return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}
__device__ __forceinline__ double2 load_sample(const double2* x, int64_t i) { return __ldg(x + i); }

// One thread per (round, bin): the taps t = bin (mod b) in ascending t, as
// fold[bin] += g[h+t] * x[sigma*((t - tau) mod n) mod n] (bucketize.hpp:69-74).
template <class T>
__global__ void __launch_bounds__(kT)
bucketize_kernel(const T* __restrict__ x, int64_t n, int64_t b, int64_t h,
                 const double* __restrict__ taps, const int64_t* __restrict__ sigma,
                 const int64_t* __restrict__ tau, double2* __restrict__ out) {
    const int64_t bin = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int r = blockIdx.y;
    if (bin >= b) return;
    const int64_t nmask = n - 1, sg = sigma[r], tu = tau[r];
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t t = -h + ((bin + h) & (b - 1)); t <= h; t += b) {
        const int64_t src = (sg * ((t - tu) & nmask)) & nmask;
        const double g = taps[h + t];
        const double2 v = load_sample(x, src);
        acc.x += g * v.x;
        acc.y += g * v.y;
    }
    out[static_cast<int64_t>(r) * b + bin] = acc;
}

// predict step 1, one thread per (round, tone): owning bucket, G*c for the
// three buckets j = i-1, i, i+1 and the rotation (bucketize.cpp:84-91).
__global__ void predict_tones(int64_t n, int64_t L, const int64_t* __restrict__ f,
                             const double2* __restrict__ c, int64_t count,
                             const int64_t* __restrict__ sigma, const int64_t* __restrict__ tau,
                             const double* __restrict__ ghat, int64_t gmax,
                             int64_t* __restrict__ home, double2* __restrict__ gc,
                             double2* __restrict__ rot) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int r = blockIdx.y;
    if (t >= count) return;
    const int64_t nmask = n - 1;
    const double inv_n = 1.0 / static_cast<double>(n), invL = 1.0 / static_cast<double>(L);
    const int64_t u = (sigma[r] * f[t]) & nmask;
    const int64_t i = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
    const int64_t e = (tau[r] * u) & nmask;
    const double a = -kTwoPi * static_cast<double>(e) * inv_n;
    double s, co;
    sincos(a, &s, &co);
    const int64_t k = static_cast<int64_t>(r) * count + t;
    home[k] = i;
    rot[k] = make_double2(co, s);
    const double2 cv = c[t];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double g = ghat[(i - 1 + d) * L - u + gmax];
        gc[k * 3 + d] = make_double2(g * cv.x, g * cv.y);
    }
}

// predict step 2, one thread per (round, bucket): contributions in ascending f.
__global__ void __launch_bounds__(kT)
predict_sum(int64_t b, int64_t count, const int64_t* __restrict__ home,
            const double2* __restrict__ gc, const double2* __restrict__ rot,
            double2* __restrict__ out) {
    const int64_t beta = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int r = blockIdx.y;
    if (beta >= b) return;
    const int64_t base = static_cast<int64_t>(r) * count;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t t = 0; t < count; ++t) {
        const int64_t i = home[base + t];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (((i - 1 + d) & (b - 1)) == beta) {
                const double2 v = cmul(gc[(base + t) * 3 + d], rot[base + t]);
                acc.x += v.x;
                acc.y += v.y;
            }
        }
    }
    out[static_cast<int64_t>(r) * b + beta] = acc;
}

// locate_frequency (locate.cpp:83-123), one thread per bucket.
__global__ void locate_kernel(int64_t n, int64_t b, int64_t l, double q,
                              const int64_t* __restrict__ bucket, int64_t count,
                              const double2* __restrict__ rounds, const int64_t* __restrict__ tau,
                              int64_t nrounds, int64_t* __restrict__ u_out,
                              int32_t* __restrict__ stages_out, int32_t* __restrict__ status) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    const int64_t beta = bucket[k];
    const int64_t L = n / b;
    const double inv_n = 1.0 / static_cast<double>(n);
    u_out[k] = -1;
    stages_out[k] = 0;
    if (beta < 0 || beta >= b) {
        status[k] = 4;
        return;
    }
    const double2 y0 = rounds[beta];
    if (y0.x == 0.0 && y0.y == 0.0) {
        status[k] = 1;
        return;
    }
    double u_min = (2.0 * static_cast<double>(beta) - 1.0) * static_cast<double>(L) / 2.0;
    double len = static_cast<double>(L);
    int stages = 0;
    while (len > 1.0 + 1e-9) {
        ++stages;
        if (stages >= nrounds) {
            status[k] = 3;
            return;
        }
        const double2 yt = rounds[static_cast<int64_t>(stages) * b + beta];
        if (yt.x == 0.0 && yt.y == 0.0) {
            status[k] = 1;
            return;
        }
        const double2 z = cdiv_ref(y0.x, y0.y, yt.x, yt.y);
        if (z.x == 0.0 && z.y == 0.0) {
            status[k] = 2;
            return;
        }
        double phi = atan2(z.y, z.x);
        if (phi < 0.0) phi += kTwoPi;
        phi = phi + 0.0;
        const int64_t tu = tau[stages];
        const double rblk = len / static_cast<double>(l);
        int64_t best = 0;
        double best_d = INFINITY;
        for (int64_t j = 0; j < l; ++j) {
            const double center = u_min + (static_cast<double>(j) + 0.5) * rblk;
            const double d = circular_phase_distance(position_phase(center, tu, n, inv_n), phi);
            if (d < best_d) {
                best_d = d;
                best = j;
            }
        }
        u_min = u_min + (static_cast<double>(best) - q / 2.0) * rblk;
        len = len * (q + 1.0) / static_cast<double>(l);
    }
    const double lo = u_min, hi = u_min + len;
    int64_t u = static_cast<int64_t>(ceil(lo));
    if (!(static_cast<double>(u) < hi)) u = llround(0.5 * (lo + hi));
    u %= n;
    if (u < 0) u += n;
    u_out[k] = u;
    stages_out[k] = stages;
    status[k] = 0;
}

// estimate_value (sfft4.cpp:27-36), one thread per pair.
__global__ void estimate_kernel(int64_t n, int64_t L, const double* __restrict__ ghat,
                                int64_t gmax, const double2* __restrict__ y0,
                                const int64_t* __restrict__ u, int64_t count,
                                double2* __restrict__ out, int32_t* __restrict__ status) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    const int64_t uk = u[k];
    const int64_t i =
        static_cast<int64_t>(floor(static_cast<double>(uk) / static_cast<double>(L) + 0.5));
    const int64_t d = i * L - uk;
    MSFFT_DCHECK(d >= -gmax && d <= gmax);
    const double g = ghat[d + gmax];
    if (fabs(g) < 0.5) {
        status[k] = 1;
        out[k] = make_double2(0.0, 0.0);
        return;
    }
    status[k] = 0;
    out[k] = make_double2(y0[k].x / g, y0[k].y / g);
}

unsigned blocks_for(int64_t count) { return static_cast<unsigned>((count + kT - 1) / kT); }

void check_rounds(int64_t rounds) {
    if (rounds < 1 || rounds > 65535)
        throw std::invalid_argument("msfft: rounds must be in [1, 65535]");
}

}  // namespace

int64_t bucketize_device(const void* d_x, bool c128, int64_t n, int64_t b, double delta,
                         const int64_t* sigma, const int64_t* tau, int64_t rounds, double2* d_out,
                         cudaStream_t st) {
    check_rounds(rounds);
    auto win = get_device_window(n, b, delta);
    DeviceBuffer<int64_t> d_sig(rounds), d_tau(rounds);
    MSFFT_CUDA(cudaMemcpyAsync(d_sig.get(), sigma, sizeof(int64_t) * rounds,
                               cudaMemcpyHostToDevice, st));
    MSFFT_CUDA(cudaMemcpyAsync(d_tau.get(), tau, sizeof(int64_t) * rounds,
                               cudaMemcpyHostToDevice, st));
    const dim3 grid(blocks_for(b), static_cast<unsigned>(rounds));
    if (c128)
        bucketize_kernel<double2><<<grid, kT, 0, st>>>(static_cast<const double2*>(d_x), n, b,
                                                       win->h, win->d_taps, d_sig.get(),
                                                       d_tau.get(), d_out);
    else
        bucketize_kernel<float2><<<grid, kT, 0, st>>>(static_cast<const float2*>(d_x), n, b,
                                                      win->h, win->d_taps, d_sig.get(),
                                                      d_tau.get(), d_out);
    MSFFT_LAUNCH_CHECK("bucketize_kernel");
    fft_radix2_batched(d_out, b, rounds, rounds, 0, -1, 1.0 / static_cast<double>(n), st);
    MSFFT_CUDA(cudaStreamSynchronize(st));  // the plan copies die with this scope
    return win->w;
}

void predict_buckets_device(int64_t n, int64_t b, double delta, const int64_t* d_f,
                            const double2* d_c, int64_t count, const int64_t* sigma,
                            const int64_t* tau, int64_t rounds, double2* d_out, cudaStream_t st) {
    check_rounds(rounds);
    auto win = get_device_window(n, b, delta);
    if (count == 0) {
        MSFFT_CUDA(cudaMemsetAsync(d_out, 0, sizeof(double2) * b * rounds, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        return;
    }
    DeviceBuffer<int64_t> d_sig(rounds), d_tau(rounds), home(count * rounds);
    DeviceBuffer<double2> gc(3 * count * rounds), rot(count * rounds);
    MSFFT_CUDA(cudaMemcpyAsync(d_sig.get(), sigma, sizeof(int64_t) * rounds,
                               cudaMemcpyHostToDevice, st));
    MSFFT_CUDA(cudaMemcpyAsync(d_tau.get(), tau, sizeof(int64_t) * rounds,
                               cudaMemcpyHostToDevice, st));
    predict_tones<<<dim3(blocks_for(count), static_cast<unsigned>(rounds)), kT, 0, st>>>(
        n, win->l_width, d_f, d_c, count, d_sig.get(), d_tau.get(), win->d_ghat, win->gmax,
        home.get(), gc.get(), rot.get());
    MSFFT_LAUNCH_CHECK("predict_tones");
    predict_sum<<<dim3(blocks_for(b), static_cast<unsigned>(rounds)), kT, 0, st>>>(
        b, count, home.get(), gc.get(), rot.get(), d_out);
    MSFFT_LAUNCH_CHECK("predict_sum");
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void locate_frequency_device(int64_t n, int64_t b, int64_t l, double q, const int64_t* d_bucket,
                             int64_t count, const double2* d_rounds, const int64_t* tau,
                             int64_t nrounds, int64_t* d_u, int32_t* d_stages, int32_t* d_status,
                             cudaStream_t st) {
    if (count == 0) return;
    DeviceBuffer<int64_t> d_tau(nrounds);
    MSFFT_CUDA(cudaMemcpyAsync(d_tau.get(), tau, sizeof(int64_t) * nrounds,
                               cudaMemcpyHostToDevice, st));
    locate_kernel<<<blocks_for(count), kT, 0, st>>>(n, b, l, q, d_bucket, count, d_rounds,
                                                    d_tau.get(), nrounds, d_u, d_stages,
                                                    d_status);
    MSFFT_LAUNCH_CHECK("locate_kernel");
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void estimate_values_device(int64_t n, int64_t b, double delta, const double2* d_y0,
                            const int64_t* d_u, int64_t count, double2* d_out, int32_t* d_status,
                            cudaStream_t st) {
    auto win = get_device_window(n, b, delta);
    if (count == 0) return;
    estimate_kernel<<<blocks_for(count), kT, 0, st>>>(n, win->l_width, win->d_ghat, win->gmax,
                                                      d_y0, d_u, count, d_out, d_status);
    MSFFT_LAUNCH_CHECK("estimate_kernel");
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

}  // namespace msfft_b200
