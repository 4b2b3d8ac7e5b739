// signal_ops.cu -- see signal_ops.hpp.  Compiled with --fmad=false.
#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <stdexcept>
#include <thread>
#include <vector>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"
#include "host_plan.hpp"
#include "signal_ops.hpp"

namespace msfft_b200 {

namespace {

constexpr double kTwoPiRef = 6.283185307179586476925286766559;  // 2 * std::numbers::pi, signal.cpp:13
constexpr int64_t kResync = 1024;                     // signal.cpp:81
constexpr int64_t kMaxSeedTable = int64_t{1} << 23;   // tone x 1024-block seeds

// ---------------------------------------------------------------- synthesize
constexpr int kSynTile = 128;  // tones per pass (one per thread)
constexpr int kSynSub = 32;    // samples per contribution slab

// One CTA per 1024-sample block.  Per tile of tones: every thread advances
// its tone's phasor over a 32-sample slab and parks c*ph in shared memory;
// then one thread per sample adds the slab's contributions in ascending tone
// order to the sample's running sum -- x[j] receives exactly the reference's
// additions in the reference's order.
template <class OutT>
__global__ void __launch_bounds__(kSynTile)
synth_kernel(int64_t n, int64_t nblk, int64_t count, const double2* __restrict__ mul,
             const double2* __restrict__ coef, const double2* __restrict__ seed_tab,
             const double* __restrict__ steps, OutT* __restrict__ x) {
    extern __shared__ double2 syn_smem[];
    double2* contrib = syn_smem;                            // [kSynTile][kSynSub + 1]
    double2* acc = syn_smem + kSynTile * (kSynSub + 1);     // [block length]
    const int64_t blk = blockIdx.x;
    const int64_t j0 = blk * kResync;
    const int len = static_cast<int>(n < kResync ? n : kResync);
    const int sub = len < kSynSub ? len : kSynSub;
    const int t = threadIdx.x;
    for (int i = t; i < len; i += kSynTile) acc[i] = make_double2(0.0, 0.0);
    for (int64_t tile0 = 0; tile0 < count; tile0 += kSynTile) {
        const int tc = static_cast<int>(count - tile0 < kSynTile ? count - tile0 : kSynTile);
        const bool have = t < tc;
        double2 ph = make_double2(1.0, 0.0), mv = ph, c = make_double2(0.0, 0.0);
        if (have) {
            const int64_t tone = tile0 + t;
            mv = mul[tone];
            c = coef[tone];
            if (seed_tab) {
                ph = seed_tab[tone * nblk + blk];
            } else {
                double s, co;
                sincos(steps[tone] * static_cast<double>(j0), &s, &co);
                ph = make_double2(co, s);
            }
        }
        __syncthreads();  // acc initialised / previous tile's slabs consumed
        for (int s0 = 0; s0 < len; s0 += sub) {
            if (have) {
                for (int i = 0; i < sub; ++i) {
                    contrib[t * (kSynSub + 1) + i] = cmul(c, ph);
                    ph = cmul(ph, mv);
                }
            }
            __syncthreads();
            if (t < sub) {
                double2 a = acc[s0 + t];
                for (int u = 0; u < tc; ++u) {
                    const double2 v = contrib[u * (kSynSub + 1) + t];
                    a.x += v.x;
                    a.y += v.y;
                }
                acc[s0 + t] = a;
            }
            __syncthreads();
        }
    }
    for (int i = t; i < len; i += kSynTile) {
        const double2 a = acc[i];
        if constexpr (sizeof(OutT) == 16) {
            x[j0 + i] = a;
        } else {
            x[j0 + i] = make_float2(static_cast<float>(a.x), static_cast<float>(a.y));
        }
    }
}

// ---------------------------------------------------------------- AWGN
__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
    constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
    constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(kM0, ctr.x), lo0 = kM0 * ctr.x;
        const uint32_t hi1 = __umulhi(kM1, ctr.z), lo1 = kM1 * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
        key.x += kW0;
        key.y += kW1;
    }
    return ctr;
}

// Complex standard-normal pair for sample j (Box-Muller on two 53-bit
// uniforms, rng.hpp:38-49's construction over a counter-based source).
__device__ __forceinline__ double2 noise_at(int64_t j, uint64_t seed) {
    const uint4 r = philox4x32_10(
        make_uint4(static_cast<uint32_t>(j), static_cast<uint32_t>(static_cast<uint64_t>(j) >> 32),
                   0x51u, 0x52u),
        make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
    const uint64_t a = (static_cast<uint64_t>(r.x) << 32) | r.y;
    const uint64_t b = (static_cast<uint64_t>(r.z) << 32) | r.w;
    double u1 = static_cast<double>(a >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    if (u1 == 0.0) u1 = 0x1.0p-54;
    const double rad = sqrt(-2.0 * log(u1));
    double s, c;
    sincos(kTwoPi * u2, &s, &c);
    return make_double2(rad * c, rad * s);
}

template <class T>
__device__ __forceinline__ double2 load_c(const T* p) {
    const T v = *p;
    return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}

constexpr int kRedThreads = 256;

// Per-block partial sums of |x|^2 and |g|^2 (fixed order: deterministic), and
// the finiteness flag of x.
template <class T>
__global__ void __launch_bounds__(kRedThreads)
awgn_power_kernel(const T* __restrict__ x, int64_t n, uint64_t seed, double2* __restrict__ part,
                  int32_t* __restrict__ bad) {
    __shared__ double ss[kRedThreads], sn[kRedThreads];
    double ps = 0.0, pn = 0.0;
    bool ok = true;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * kRedThreads) {
        const double2 v = load_c(x + j);
        ok &= isfinite(v.x) && isfinite(v.y);
        ps += v.x * v.x + v.y * v.y;
        const double2 g = noise_at(j, seed);
        pn += g.x * g.x + g.y * g.y;
    }
    if (!ok) atomicExch(bad, 1);
    ss[threadIdx.x] = ps;
    sn[threadIdx.x] = pn;
    __syncthreads();
    for (int o = kRedThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            ss[threadIdx.x] += ss[threadIdx.x + o];
            sn[threadIdx.x] += sn[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = make_double2(ss[0], sn[0]);
}

template <class T>
__global__ void awgn_add_kernel(T* __restrict__ x, int64_t n, uint64_t seed, double scale) {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 v = load_c(x + j);
        const double2 g = noise_at(j, seed);
        const double re = v.x + scale * g.x, im = v.y + scale * g.y;
        if constexpr (sizeof(T) == 16) {
            x[j] = make_double2(re, im);
        } else {
            x[j] = make_float2(static_cast<float>(re), static_cast<float>(im));
        }
    }
}

// ---------------------------------------------------------------- dense DFT
template <class T>
__global__ void upcast_check_kernel(const T* __restrict__ in, int64_t total,
                                    double2* __restrict__ out, int32_t* __restrict__ bad) {
    bool ok = true;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 v = load_c(in + j);
        ok &= isfinite(v.x) && isfinite(v.y);
        out[j] = v;
    }
    if (!ok) atomicExch(bad, 1);
}

// ---------------------------------------------------------------- top-k
constexpr int kSelBits = 16;
constexpr int kSelBins = 1 << kSelBits;

__global__ void mag_key_kernel(const double2* __restrict__ s, int64_t n,
                               uint64_t* __restrict__ key) {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 v = s[j];
        const double m = cabs_ref(v.x, v.y);
        // |X| >= 0: IEEE bits order like the values; NaN ranks last
        key[j] = m == m ? static_cast<uint64_t>(__double_as_longlong(m)) : 0ull;
    }
}

// Histogram of the next 16-bit digit among keys whose higher digits equal
// `prefix` (under `mask`).
__global__ void digit_hist_kernel(const uint64_t* __restrict__ key, int64_t n, uint64_t prefix,
                                  uint64_t mask, int shift, uint32_t* __restrict__ hist) {
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = key[j];
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & (kSelBins - 1)], 1u);
    }
}

constexpr int kCmpThreads = 256;
constexpr int kCmpPerThread = 16;
constexpr int64_t kCmpChunk = int64_t{kCmpThreads} * kCmpPerThread;

// Pass A: per chunk, the number of keys > thr and == thr.
__global__ void __launch_bounds__(kCmpThreads)
sel_count_kernel(const uint64_t* __restrict__ key, int64_t n, uint64_t thr,
                 int64_t* __restrict__ cnt_gt, int64_t* __restrict__ cnt_eq) {
    __shared__ int gt_s, eq_s;
    if (threadIdx.x == 0) gt_s = eq_s = 0;
    __syncthreads();
    int gt = 0, eq = 0;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kCmpChunk;
    for (int i = threadIdx.x; i < kCmpChunk; i += kCmpThreads) {
        const int64_t j = base + i;
        if (j >= n) break;
        const uint64_t k = key[j];
        gt += k > thr;
        eq += k == thr;
    }
    atomicAdd(&gt_s, gt);
    atomicAdd(&eq_s, eq);
    __syncthreads();
    if (threadIdx.x == 0) {
        cnt_gt[blockIdx.x] = gt_s;
        cnt_eq[blockIdx.x] = eq_s;
    }
}

// Pass B: ordered compaction of the selected indices (key > thr, or key ==
// thr among the first `need_eq` such in index order).  off_sel / off_eq are
// the exclusive prefixes of the chunk counts.
__global__ void __launch_bounds__(kCmpThreads)
sel_write_kernel(const uint64_t* __restrict__ key, const double2* __restrict__ spec, int64_t n,
                 uint64_t thr, int64_t need_eq, const int64_t* __restrict__ off_sel,
                 const int64_t* __restrict__ off_eq, int64_t* __restrict__ out_f,
                 double2* __restrict__ out_c) {
    __shared__ int warp_sel[kCmpThreads / 32], warp_eq[kCmpThreads / 32];
    __shared__ int64_t run_sel, run_eq;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        run_sel = off_sel[blockIdx.x];
        run_eq = off_eq[blockIdx.x];
    }
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kCmpChunk;
    for (int r = 0; r < kCmpPerThread; ++r) {
        const int64_t j = base + static_cast<int64_t>(r) * kCmpThreads + threadIdx.x;
        const uint64_t k = j < n ? key[j] : 0ull;
        const bool is_eq = j < n && k == thr;
        const bool is_gt = j < n && k > thr;
        // equal keys in index order: rank among this round's equals
        const unsigned eq_mask = __ballot_sync(0xffffffffu, is_eq);
        if (lane == 0) warp_eq[wid] = __popc(eq_mask);
        __syncthreads();
        int eq_before = __popc(eq_mask & ((1u << lane) - 1u));
        int eq_total = 0;
        for (int w = 0; w < kCmpThreads / 32; ++w) {
            if (w < wid) eq_before += warp_eq[w];
            eq_total += warp_eq[w];
        }
        const bool take = is_gt || (is_eq && run_eq + eq_before < need_eq);
        const unsigned sel_mask = __ballot_sync(0xffffffffu, take);
        if (lane == 0) warp_sel[wid] = __popc(sel_mask);
        __syncthreads();
        int sel_before = __popc(sel_mask & ((1u << lane) - 1u));
        int sel_total = 0;
        for (int w = 0; w < kCmpThreads / 32; ++w) {
            if (w < wid) sel_before += warp_sel[w];
            sel_total += warp_sel[w];
        }
        if (take) {
            const int64_t pos = run_sel + sel_before;
            out_f[pos] = j;
            out_c[pos] = spec[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            run_sel += sel_total;
            run_eq += eq_total;
        }
        __syncthreads();
    }
}

unsigned grid_for(int64_t work, int threads) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads,
                                                                         148 * 16)));
}

void check_n(int64_t n, const char* who) {
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument(std::string(who) + ": n must be a power of two >= 4");
}

template <class F>
void parallel_for(int64_t items, F&& fn) {
    const int64_t threads =
        std::max<int64_t>(1, std::min<int64_t>(items / 4096 + 1,
                                               std::max(1u, std::thread::hardware_concurrency())));
    if (threads == 1) {
        for (int64_t i = 0; i < items; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < threads; ++w)
        pool.emplace_back([&, w] {
            for (int64_t i = w; i < items; i += threads) fn(i);
        });
    for (auto& th : pool) th.join();
}

}  // namespace

void random_sparse_spectrum(int64_t n, int64_t k, uint64_t seed, std::vector<int64_t>& f,
                            std::vector<double>& c) {
    HostRng rng(seed);
    random_sparse_spectrum(n, k, rng, f, c);
}

void random_sparse_spectrum(int64_t n, int64_t k, HostRng& rng, std::vector<int64_t>& f,
                            std::vector<double>& c) {
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("random_sparse_spectrum: bad n");
    if (k < 0 || k > n) throw std::invalid_argument("random_sparse_spectrum: k out of range");
    std::set<int64_t> positions;  // Floyd's sampling (signal.cpp:107-112)
    for (int64_t j = n - k; j < n; ++j) {
        const int64_t t = static_cast<int64_t>(rng.below(static_cast<uint64_t>(j) + 1));
        if (!positions.insert(t).second) positions.insert(j);
    }
    f.assign(positions.begin(), positions.end());
    c.resize(2 * f.size());
    for (size_t i = 0; i < f.size(); ++i) {
        const double phase = kTwoPiRef * (static_cast<double>(rng.u64() >> 11) * 0x1.0p-53);
        c[2 * i] = std::cos(phase);
        c[2 * i + 1] = std::sin(phase);
    }
}

bool synthesize_device(int64_t n, const int64_t* f, const double* c, int64_t count, bool c128,
                       void* d_x, cudaStream_t st) {
    check_n(n, "SparseSpectrum");  // SparseSpectrum::validate (signal.cpp:28-39)
    if (count > n) throw std::invalid_argument("SparseSpectrum: more entries than n");
    for (int64_t i = 0; i < count; ++i) {
        if (f[i] < 0 || f[i] >= n) throw std::invalid_argument("SparseSpectrum: position out of range");
        if (!std::isfinite(c[2 * i]) || !std::isfinite(c[2 * i + 1]))
            throw std::invalid_argument("SparseSpectrum: non-finite coefficient");
        if (i > 0 && f[i] <= f[i - 1])
            throw std::invalid_argument("synthesize: positions must be strictly ascending");
    }
    const int64_t nblk = (n + kResync - 1) / kResync;
    const bool exact = count * nblk <= kMaxSeedTable;
    std::vector<double2> mul(static_cast<size_t>(std::max<int64_t>(count, 1)));
    std::vector<double> steps(static_cast<size_t>(std::max<int64_t>(count, 1)));
    std::vector<double2> seeds;
    if (exact) seeds.resize(static_cast<size_t>(std::max<int64_t>(count * nblk, 1)));
    parallel_for(count, [&](int64_t t) {
        const double step = kTwoPiRef * static_cast<double>(f[t]) / static_cast<double>(n);
        steps[t] = step;
        mul[t] = make_double2(std::cos(step), std::sin(step));
        if (exact)
            for (int64_t b = 0; b < nblk; ++b) {
                const double a = step * static_cast<double>((b * kResync) % n);
                seeds[t * nblk + b] = make_double2(std::cos(a), std::sin(a));
            }
    });
    DeviceBuffer<double2> d_mul(mul.size()), d_coef(mul.size()), d_seed(seeds.size());
    DeviceBuffer<double> d_steps(steps.size());
    MSFFT_CUDA(cudaMemcpyAsync(d_mul.get(), mul.data(), mul.size() * 16, cudaMemcpyHostToDevice, st));
    if (count)
        MSFFT_CUDA(cudaMemcpyAsync(d_coef.get(), c, count * 16, cudaMemcpyHostToDevice, st));
    MSFFT_CUDA(cudaMemcpyAsync(d_steps.get(), steps.data(), steps.size() * 8,
                               cudaMemcpyHostToDevice, st));
    if (exact)
        MSFFT_CUDA(cudaMemcpyAsync(d_seed.get(), seeds.data(), seeds.size() * 16,
                                   cudaMemcpyHostToDevice, st));
    const size_t smem = sizeof(double2) * (kSynTile * (kSynSub + 1) + kResync);
    if (c128) {
        MSFFT_CUDA(cudaFuncSetAttribute(synth_kernel<double2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        synth_kernel<double2><<<static_cast<unsigned>(nblk), kSynTile, smem, st>>>(
            n, nblk, count, d_mul.get(), d_coef.get(), exact ? d_seed.get() : nullptr,
            d_steps.get(), static_cast<double2*>(d_x));
    } else {
        MSFFT_CUDA(cudaFuncSetAttribute(synth_kernel<float2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
        synth_kernel<float2><<<static_cast<unsigned>(nblk), kSynTile, smem, st>>>(
            n, nblk, count, d_mul.get(), d_coef.get(), exact ? d_seed.get() : nullptr,
            d_steps.get(), static_cast<float2*>(d_x));
    }
    MSFFT_LAUNCH_CHECK("synth_kernel");
    MSFFT_CUDA(cudaStreamSynchronize(st));  // host tables go out of scope
    return exact;
}

void awgn_device(void* d_x, bool c128, int64_t n, double snr_db, uint64_t seed,
                 cudaStream_t st) {
    check_n(n, "ComplexSignal");
    DeviceBuffer<int32_t> bad(1);
    MSFFT_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), st));
    const unsigned blocks = grid_for(n, kRedThreads);
    DeviceBuffer<double2> part(blocks);
    // validation first (add_awgn calls x.validate(), signal.cpp:124), then the
    // sentinel and the snr check
    if (c128)
        awgn_power_kernel<double2><<<blocks, kRedThreads, 0, st>>>(
            static_cast<const double2*>(d_x), n, seed, part.get(), bad.get());
    else
        awgn_power_kernel<float2><<<blocks, kRedThreads, 0, st>>>(
            static_cast<const float2*>(d_x), n, seed, part.get(), bad.get());
    MSFFT_LAUNCH_CHECK("awgn_power_kernel");
    std::vector<double2> hp(blocks);
    int32_t hbad = 0;
    MSFFT_CUDA(cudaMemcpyAsync(hp.data(), part.get(), blocks * 16, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaStreamSynchronize(st));
    if (hbad) throw std::invalid_argument("ComplexSignal: non-finite sample");
    if (std::isinf(snr_db) && snr_db > 0) return;
    if (!std::isfinite(snr_db))
        throw std::invalid_argument("add_awgn: snr_db must be finite or +infinity");
    double sig_power = 0.0, noise_power = 0.0;
    for (const double2& p : hp) {
        sig_power += p.x;
        noise_power += p.y;
    }
    const double target = sig_power * std::pow(10.0, -snr_db / 10.0);
    const double scale = noise_power > 0.0 ? std::sqrt(target / noise_power) : 0.0;
    if (c128)
        awgn_add_kernel<double2><<<grid_for(n, 256), 256, 0, st>>>(static_cast<double2*>(d_x), n,
                                                                   seed, scale);
    else
        awgn_add_kernel<float2><<<grid_for(n, 256), 256, 0, st>>>(static_cast<float2*>(d_x), n,
                                                                  seed, scale);
    MSFFT_LAUNCH_CHECK("awgn_add_kernel");
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void dense_dft_device(const void* d_in, bool in_c128, int64_t n, int64_t batch, double2* d_out,
                      int sign, cudaStream_t st) {
    if (sign < 0)
        check_n(n, "ComplexSignal");
    else if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("idft_dense: size must be a power of two >= 4");
    if (batch <= 0) return;
    const int64_t total = n * batch;
    DeviceBuffer<int32_t> bad(1);
    MSFFT_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int32_t), st));
    if (in_c128)
        upcast_check_kernel<double2><<<grid_for(total, 256), 256, 0, st>>>(
            static_cast<const double2*>(d_in), total, d_out, bad.get());
    else
        upcast_check_kernel<float2><<<grid_for(total, 256), 256, 0, st>>>(
            static_cast<const float2*>(d_in), total, d_out, bad.get());
    MSFFT_LAUNCH_CHECK("upcast_check_kernel");
    if (sign < 0) {
        int32_t hbad = 0;
        MSFFT_CUDA(cudaMemcpyAsync(&hbad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        if (hbad) throw std::invalid_argument("ComplexSignal: non-finite sample");
    }
    fft_radix2_batched(d_out, n, batch, 1, n, sign < 0 ? -1 : 1,
                       sign < 0 ? 1.0 / static_cast<double>(n) : 1.0, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

int64_t top_k_device(const double2* d_spec, int64_t n, int64_t k, int64_t* f, double* c,
                     cudaStream_t st) {
    if (n <= 0) return 0;
    const int64_t keep = std::max<int64_t>(0, std::min(k, n));
    if (keep == 0) return 0;
    DeviceBuffer<uint64_t> key(static_cast<size_t>(n));
    DeviceBuffer<uint32_t> hist(kSelBins);
    mag_key_kernel<<<grid_for(n, 256), 256, 0, st>>>(d_spec, n, key.get());
    MSFFT_LAUNCH_CHECK("mag_key_kernel");
    // radix select of the keep-th largest key, 16 bits per pass
    uint64_t prefix = 0, mask = 0;
    int64_t remaining = keep;  // rank (1-based) of the target within the prefix class
    std::vector<uint32_t> h(kSelBins);
    for (int shift = 64 - kSelBits; shift >= 0; shift -= kSelBits) {
        MSFFT_CUDA(cudaMemsetAsync(hist.get(), 0, kSelBins * sizeof(uint32_t), st));
        digit_hist_kernel<<<grid_for(n, 256), 256, 0, st>>>(key.get(), n, prefix, mask, shift,
                                                            hist.get());
        MSFFT_LAUNCH_CHECK("digit_hist_kernel");
        MSFFT_CUDA(cudaMemcpyAsync(h.data(), hist.get(), kSelBins * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        int d = kSelBins - 1;
        for (; d > 0; --d) {
            if (static_cast<int64_t>(h[d]) >= remaining) break;
            remaining -= h[d];
        }
        prefix |= static_cast<uint64_t>(d) << shift;
        mask |= static_cast<uint64_t>(kSelBins - 1) << shift;
    }
    const uint64_t thr = prefix;
    const int64_t nchunks = (n + kCmpChunk - 1) / kCmpChunk;
    DeviceBuffer<int64_t> cgt(nchunks), ceq(nchunks), osel(nchunks), oeq(nchunks);
    sel_count_kernel<<<static_cast<unsigned>(nchunks), kCmpThreads, 0, st>>>(key.get(), n, thr,
                                                                            cgt.get(), ceq.get());
    MSFFT_LAUNCH_CHECK("sel_count_kernel");
    std::vector<int64_t> hg(nchunks), he(nchunks), hs(nchunks), hq(nchunks);
    MSFFT_CUDA(cudaMemcpyAsync(hg.data(), cgt.get(), nchunks * 8, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaMemcpyAsync(he.data(), ceq.get(), nchunks * 8, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaStreamSynchronize(st));
    int64_t total_gt = 0;
    for (int64_t i = 0; i < nchunks; ++i) total_gt += hg[i];
    const int64_t need_eq = keep - total_gt;
    int64_t run_sel = 0, run_eq = 0;
    for (int64_t i = 0; i < nchunks; ++i) {
        hs[i] = run_sel;
        hq[i] = run_eq;
        const int64_t eq_take = std::max<int64_t>(0, std::min(he[i], need_eq - run_eq));
        run_sel += hg[i] + eq_take;
        run_eq += he[i];
    }
    MSFFT_CUDA(cudaMemcpyAsync(osel.get(), hs.data(), nchunks * 8, cudaMemcpyHostToDevice, st));
    MSFFT_CUDA(cudaMemcpyAsync(oeq.get(), hq.data(), nchunks * 8, cudaMemcpyHostToDevice, st));
    DeviceBuffer<int64_t> of(static_cast<size_t>(keep));
    DeviceBuffer<double2> oc(static_cast<size_t>(keep));
    sel_write_kernel<<<static_cast<unsigned>(nchunks), kCmpThreads, 0, st>>>(
        key.get(), d_spec, n, thr, need_eq, osel.get(), oeq.get(), of.get(), oc.get());
    MSFFT_LAUNCH_CHECK("sel_write_kernel");
    MSFFT_CUDA(cudaMemcpyAsync(f, of.get(), keep * 8, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaMemcpyAsync(c, oc.get(), keep * 16, cudaMemcpyDeviceToHost, st));
    MSFFT_CUDA(cudaStreamSynchronize(st));
    return keep;
}

}  // namespace msfft_b200
