// phase_mc.cu -- see phase_mc.hpp.  Compiled with --fmad=false.
#include <algorithm>
#include <cmath>
#include <complex>
#include <memory>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"
#include "host_plan.hpp"
#include "phase_mc.hpp"
#include "signal_ops.hpp"
#include "window.hpp"

namespace msfft_b200 {

namespace {

constexpr double kTwoPiRef = 6.283185307179586476925286766559;  // 2 * std::numbers::pi
constexpr int kPhaseThreads = 256;
constexpr int64_t kMaxBatch = 4096;  // candidate trials per launch

uint64_t splitmix64_h(uint64_t x) {  // rng.hpp:9-14
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// indexed_noise (phase_mc.cpp:20-30): counter-based complex Gaussian keyed by
// the time index.
__device__ __forceinline__ double2 indexed_noise(uint64_t seed, int64_t idx, double scale) {
    if (scale == 0.0) return make_double2(0.0, 0.0);
    const uint64_t a = splitmix64_d(seed ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(idx + 1)));
    const uint64_t b = splitmix64_d(a);
    const double u1 = static_cast<double>((a >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    const double r = sqrt(-log(u1));
    double s, c;
    sincos(kTwoPi * u2, &s, &c);
    return make_double2(scale * (r * c), scale * (r * s));
}

// One CTA per (candidate trial, round): the fold of bucketize_fn
// (bucketize.hpp:63-86) over the lazy tone source (phase_mc.cpp:34-90) --
// per bin the taps t = bin (mod b) in increasing t, g[h+t] * v(t) with
// v(t) = noise(src) + sum over tones (ascending f) of c e^{2 pi i u (t - tau)/n}
// -- then the reference's radix-2 DIT in shared memory and value `chosen`/n.
__global__ void __launch_bounds__(kPhaseThreads)
phase_bucket_kernel(int64_t n, int64_t b, int log2b, int64_t h, const double* __restrict__ taps,
                    const double2* __restrict__ tw, int64_t tau1, double noise_scale, int64_t k,
                    const int64_t* __restrict__ sigma, const uint64_t* __restrict__ nseed,
                    const int32_t* __restrict__ chosen, const int64_t* __restrict__ tone_u,
                    const double2* __restrict__ tone_c, double2* __restrict__ y) {
    extern __shared__ double2 fold[];
    const int64_t cand = blockIdx.x;
    const int r = blockIdx.y;
    const int64_t tau = r ? tau1 : 0;
    const int64_t mask = n - 1;
    const int64_t sg = sigma[cand];
    const uint64_t seed = nseed[cand];
    const int64_t* U = tone_u + cand * k;
    const double2* Cf = tone_c + cand * k;
    const double dn = static_cast<double>(n);
    for (int64_t c = threadIdx.x; c < b; c += kPhaseThreads) {
        double2 acc = make_double2(0.0, 0.0);
        for (int64_t t = -h + ((c + h) & (b - 1)); t <= h; t += b) {
            const int64_t s = (t - tau) & mask;     // ((t - tau) % n + n) % n
            const int64_t src = (sg * s) & mask;    // sigma * src % n
            double2 v = indexed_noise(seed, src, noise_scale);
            for (int64_t j = 0; j < k; ++j) {
                const int64_t e = (U[j] * s) & mask;
                const double a = kTwoPi * static_cast<double>(e) / dn;
                double sn, cs;
                sincos(a, &sn, &cs);
                const double2 ph = cmul(Cf[j], make_double2(cs, sn));
                v.x += ph.x;
                v.y += ph.y;
            }
            const double g = taps[h + t];
            acc.x += g * v.x;
            acc.y += g * v.y;
        }
        fold[bitrev_bits(static_cast<unsigned>(c), log2b)] = acc;
    }
    __syncthreads();
    for (int st = 1; st <= log2b; ++st) {
        const int64_t half = int64_t{1} << (st - 1);
        for (int64_t bf = threadIdx.x; bf < b / 2; bf += kPhaseThreads) {
            const int64_t blk = bf >> (st - 1), off = bf & (half - 1);
            const int64_t j = (blk << st) + off;
            const double2 w = tw[off << (log2b - st)];
            const double2 x0 = fold[j];
            const double2 tv = cmul(fold[j + half], w);
            fold[j + half] = make_double2(x0.x - tv.x, x0.y - tv.y);
            fold[j] = make_double2(x0.x + tv.x, x0.y + tv.y);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double scale = 1.0 / dn;
        const double2 v = fold[chosen[cand]];
        y[cand * 2 + r] = make_double2(v.x * scale, v.y * scale);
    }
}

struct Candidate {
    int64_t sigma = 0, u = 0;
    uint64_t nseed = 0;
    int32_t chosen = -1;
    std::vector<int64_t> tone_u;
    std::vector<double> tone_c;
};

// locate.cpp:14-23, 32-37 on the host (libm), as the reference evaluates them.
double phase_of_h(double re, double im) {
    if (re == 0.0 && im == 0.0) throw std::domain_error("phase_of: zero value");
    double a = std::atan2(im, re);
    if (a < 0.0) a += kTwoPiRef;
    return a + 0.0;
}

double position_phase_h(double u, int64_t tau, int64_t n) {
    double x = std::fmod(u * static_cast<double>(tau), static_cast<double>(n));
    if (x < 0) x += static_cast<double>(n);
    return x * kTwoPiRef / static_cast<double>(n);
}

double circular_distance_h(double a, double b) {
    const double d = std::fmod(std::fabs(a - b), kTwoPiRef);
    return std::min(d, kTwoPiRef - d);
}

}  // namespace

std::vector<PhaseHistogramOut> phase_experiment(int64_t n, int64_t k, int64_t b,
                                                const std::vector<double>& snr_list,
                                                int64_t trials, uint64_t seed,
                                                std::vector<std::vector<PhaseTrialOut>>* trials_out) {
    if (trials < 1) throw std::invalid_argument("run_phase_experiment: trials must be >= 1");
    std::vector<PhaseHistogramOut> out;
    if (trials_out) trials_out->assign(snr_list.size(), {});
    for (size_t si = 0; si < snr_list.size(); ++si) {
        const double snr_db = snr_list[si];
        HostRng rng(splitmix64_h(seed ^ splitmix64_h(0x5eed0000ull + si)));  // Rng::stream
        std::vector<double> samples;
        std::vector<PhaseTrialOut> accepted;
        int64_t attempts = 0;
        const int64_t attempt_cap = 200 * trials + 1000;
        while (static_cast<int64_t>(samples.size()) < trials) {
            // ---- replay attempts on the host until the batch is full
            const int64_t need = std::min<int64_t>(trials - static_cast<int64_t>(samples.size()),
                                                   kMaxBatch);
            std::vector<Candidate> batch;
            std::shared_ptr<const DeviceWindow> win;
            int64_t tau1 = 0;
            double noise_scale = 0.0;
            while (static_cast<int64_t>(batch.size()) < need) {
                if (++attempts > attempt_cap)
                    throw std::runtime_error("run_phase_experiment: rejection rate too high");
                // sample_phase_trial (phase_mc.cpp:94-151)
                if (k < 1) throw std::invalid_argument("sample_phase_trial: need k >= 1");
                const bool noisy = std::isfinite(snr_db);
                if (!noisy && !(std::isinf(snr_db) && snr_db > 0))
                    throw std::invalid_argument("sample_phase_trial: bad snr_db");
                win = get_device_window(n, b, noisy ? 1e-6 : 1e-8);
                const int64_t L = win->l_width;
                Candidate cd;
                std::vector<int64_t> f;
                std::vector<double> c;
                random_sparse_spectrum(n, k, rng, f, c);
                cd.sigma = 2 * static_cast<int64_t>(rng.below(static_cast<uint64_t>(n / 2))) + 1;
                cd.nseed = rng.u64();
                noise_scale = noisy ? std::sqrt(static_cast<double>(k) * std::pow(10.0, -snr_db / 10.0))
                                    : 0.0;
                std::vector<int> occ(static_cast<size_t>(b), 0);
                std::vector<int64_t> tone_at(static_cast<size_t>(b), -1);
                cd.tone_u.resize(f.size());
                for (size_t i = 0; i < f.size(); ++i) {
                    const int64_t u = (cd.sigma * f[i]) % n;
                    cd.tone_u[i] = u;
                    const int64_t i_b = static_cast<int64_t>(
                        std::floor(static_cast<double>(u) / static_cast<double>(L) + 0.5));
                    const int64_t bucket = ((i_b % b) + b) % b;  // bucket_of
                    ++occ[static_cast<size_t>(bucket)];
                    tone_at[static_cast<size_t>(bucket)] = u;
                }
                cd.tone_c = std::move(c);
                for (int64_t attempt = 0; attempt < b; ++attempt) {
                    const int64_t cand = static_cast<int64_t>(rng.below(static_cast<uint64_t>(b)));
                    if (occ[static_cast<size_t>(cand)] == 1) {
                        cd.chosen = static_cast<int32_t>(cand);
                        break;
                    }
                }
                if (cd.chosen < 0) continue;  // nullopt: no isolated tone found
                cd.u = tone_at[static_cast<size_t>(cd.chosen)];
                tau1 = tau_schedule(static_cast<double>(L), n);
                batch.push_back(std::move(cd));
            }
            // ---- both bucketizations of every candidate on the device
            const int64_t nc = static_cast<int64_t>(batch.size());
            std::vector<int64_t> hsig(nc), hu(nc * k);
            std::vector<uint64_t> hseed(nc);
            std::vector<int32_t> hch(nc);
            std::vector<double> hc(2 * nc * k);
            for (int64_t i = 0; i < nc; ++i) {
                hsig[i] = batch[i].sigma;
                hseed[i] = batch[i].nseed;
                hch[i] = batch[i].chosen;
                std::copy(batch[i].tone_u.begin(), batch[i].tone_u.end(), hu.begin() + i * k);
                std::copy(batch[i].tone_c.begin(), batch[i].tone_c.end(), hc.begin() + 2 * i * k);
            }
            DeviceBuffer<int64_t> dsig(nc), du(nc * k);
            DeviceBuffer<uint64_t> dseed(nc);
            DeviceBuffer<int32_t> dch(nc);
            DeviceBuffer<double2> dc(nc * k), dy(2 * nc);
            MSFFT_CUDA(cudaMemcpy(dsig.get(), hsig.data(), nc * 8, cudaMemcpyHostToDevice));
            MSFFT_CUDA(cudaMemcpy(du.get(), hu.data(), nc * k * 8, cudaMemcpyHostToDevice));
            MSFFT_CUDA(cudaMemcpy(dseed.get(), hseed.data(), nc * 8, cudaMemcpyHostToDevice));
            MSFFT_CUDA(cudaMemcpy(dch.get(), hch.data(), nc * 4, cudaMemcpyHostToDevice));
            MSFFT_CUDA(cudaMemcpy(dc.get(), hc.data(), nc * k * 16, cudaMemcpyHostToDevice));
            int log2b = 0;
            while ((int64_t{1} << log2b) < b) ++log2b;
            const size_t smem = static_cast<size_t>(b) * sizeof(double2);
            if (smem > 200 * 1024) throw std::invalid_argument("phase_experiment: b too large");
            MSFFT_CUDA(cudaFuncSetAttribute(phase_bucket_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            static_cast<int>(smem)));
            phase_bucket_kernel<<<dim3(static_cast<unsigned>(nc), 2), kPhaseThreads, smem>>>(
                n, b, log2b, win->h, win->d_taps, device_twiddles(b), tau1, noise_scale, k,
                dsig.get(), dseed.get(), dch.get(), du.get(), dc.get(), dy.get());
            MSFFT_LAUNCH_CHECK("phase_bucket_kernel");
            std::vector<double2> hy(2 * nc);
            MSFFT_CUDA(cudaMemcpy(hy.data(), dy.get(), 2 * nc * 16, cudaMemcpyDeviceToHost));
            // ---- accept in attempt order (phase_mc.cpp:137-150)
            for (int64_t i = 0; i < nc && static_cast<int64_t>(samples.size()) < trials; ++i) {
                const double2 y0 = hy[2 * i], y1 = hy[2 * i + 1];
                if ((y0.x == 0.0 && y0.y == 0.0) || (y1.x == 0.0 && y1.y == 0.0)) continue;
                PhaseTrialOut t;
                t.u = batch[i].u;
                t.bucket = batch[i].chosen;
                t.tau = tau1;
                t.y0[0] = y0.x;
                t.y0[1] = y0.y;
                t.y_tau[0] = y1.x;
                t.y_tau[1] = y1.y;
                const std::complex<double> q =
                    std::complex<double>(y0.x, y0.y) / std::complex<double>(y1.x, y1.y);
                t.measured_phi = phase_of_h(q.real(), q.imag());
                t.true_phi = position_phase_h(static_cast<double>(t.u), tau1, n);
                t.dphi = circular_distance_h(t.measured_phi, t.true_phi);
                samples.push_back(t.dphi);
                accepted.push_back(t);
            }
            // candidates beyond `trials` were drawn from a stream nothing reads again
        }
        PhaseHistogramOut hgm;  // phase_mc.cpp:188-209
        hgm.snr_db = snr_db;
        hgm.n = n;
        hgm.k = k;
        hgm.l_width = n / b;
        hgm.trials = trials;
        const double mass = 1.0 / static_cast<double>(trials);
        for (double d : samples) {
            const double lg = d > 0.0 ? std::log10(d) : -6.0;
            int bin = static_cast<int>(std::floor((lg - -6.0) / 0.1));
            bin = std::min(std::max(bin, 0), kPhaseBins - 1);
            hgm.bin_mass[bin] += mass;
        }
        std::sort(samples.begin(), samples.end());
        const auto rank = [&](double p) {
            const int64_t idx = std::min(
                std::max<int64_t>(static_cast<int64_t>(std::ceil(p * static_cast<double>(trials))) - 1, 0),
                trials - 1);
            return samples[static_cast<size_t>(idx)];
        };
        hgm.p50 = rank(0.50);
        hgm.p99 = rank(0.99);
        hgm.max = samples.back();
        out.push_back(hgm);
        if (trials_out) (*trials_out)[si] = std::move(accepted);
    }
    return out;
}

}  // namespace msfft_b200
