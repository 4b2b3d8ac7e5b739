// fft.cu -- see fft.hpp.  Compiled with --fmad=false.
#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"

namespace msfft_b200 {

namespace {

std::mutex g_tw_mu;
std::map<int64_t, std::unique_ptr<std::vector<double>>> g_host_tw;
std::map<std::pair<int, int64_t>, double2*> g_dev_tw;

// twiddle_table (proj/src/fft.cpp:14-28): step = -2 pi / n, a = step * k.
std::vector<double> make_twiddles(int64_t n) {
    const int64_t half = n / 2;
    std::vector<double> t(static_cast<size_t>(2 * std::max<int64_t>(half, 1)));
    const double step = -2.0 * 3.141592653589793 / static_cast<double>(n);
    auto work = [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) {
            const double a = step * static_cast<double>(k);
            t[2 * k] = std::cos(a);
            t[2 * k + 1] = std::sin(a);
        }
    };
    const int64_t chunk = 1 << 18;
    if (half <= chunk) {
        work(0, half);
    } else {
        const int nt = static_cast<int>(
            std::max<unsigned>(1u, std::min<unsigned>(16u, std::thread::hardware_concurrency())));
        std::vector<std::thread> pool;
        const int64_t per = (half + nt - 1) / nt;
        for (int i = 0; i < nt; ++i)
            pool.emplace_back(work, std::min(half, i * per), std::min(half, (i + 1) * per));
        for (auto& th : pool) th.join();
    }
    return t;
}

__global__ void bitrev_inplace_kernel(double2* __restrict__ data, int64_t size, int log2size,
                                      int64_t inner, int64_t outer_stride, int64_t total) {
    const int64_t gid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (gid >= total) return;
    const int64_t bi = gid / size;
    const unsigned i = static_cast<unsigned>(gid - bi * size);
    const unsigned j = bitrev_bits(i, log2size);
    if (j <= i) return;
    double2* a = data + (bi / inner) * outer_stride + (bi % inner) * size;
    const double2 t = a[i];
    a[i] = a[j];
    a[j] = t;
}

// Stages s0+1 .. s1 (1-based; stage s has butterfly span 2^(s-1)).  A CTA
// owns `lo_tile` consecutive low indices of one high block, i.e. the
// elements j = hi*2^s1 + kk*2^s0 + lo for all kk < 2^(s1-s0).  Every
// butterfly is the reference's:  t = a[j+half]*w; a[j+half] = a[j]-t; a[j] += t.
__global__ void __launch_bounds__(512) stages_kernel(double2* __restrict__ data, int64_t size,
                                                     int64_t inner, int64_t outer_stride,
                                                     int s0, int s1, int lo_tile, int sign,
                                                     const double2* __restrict__ tw,
                                                     double scale) {
    extern __shared__ double2 tile[];
    const int G = s1 - s0;
    const int64_t span = int64_t{1} << s0;       // distance between kk neighbours
    const int64_t tiles_per_hi = span / lo_tile;
    const int64_t groups = (size >> s1) * tiles_per_hi;
    const int64_t bi = blockIdx.x / groups;
    const int64_t g = blockIdx.x - bi * groups;
    const int64_t hi = g / tiles_per_hi;
    const int64_t lo0 = (g - hi * tiles_per_hi) * lo_tile;
    double2* a = data + (bi / inner) * outer_stride + (bi % inner) * size;
    const int nk = 1 << G;
    const int count = nk * lo_tile;
    const int64_t base = (hi << s1) + lo0;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const int kk = e / lo_tile, li = e - kk * lo_tile;
        tile[e] = a[base + static_cast<int64_t>(kk) * span + li];
    }
    __syncthreads();
    for (int s = s0 + 1; s <= s1; ++s) {
        const int hkk = 1 << (s - 1 - s0);   // half span in kk units
        const int64_t step = size >> s;      // twiddle stride n/size
        for (int bf = threadIdx.x; bf < count / 2; bf += blockDim.x) {
            const int li = bf % lo_tile;
            const int p = bf / lo_tile;
            const int blk = p / hkk, off = p - blk * hkk;
            const int kk = blk * 2 * hkk + off;
            const int64_t k = ((static_cast<int64_t>(off) << s0) + lo0 + li) * step;
            double2 w = tw[k];
            if (sign > 0) w.y = -w.y;
            const int e0 = kk * lo_tile + li, e1 = (kk + hkk) * lo_tile + li;
            const double2 x0 = tile[e0];
            const double2 t = cmul(tile[e1], w);
            tile[e1] = make_double2(x0.x - t.x, x0.y - t.y);
            tile[e0] = make_double2(x0.x + t.x, x0.y + t.y);
        }
        __syncthreads();
    }
    const bool do_scale = scale != 1.0;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const int kk = e / lo_tile, li = e - kk * lo_tile;
        double2 v = tile[e];
        if (do_scale) v = make_double2(v.x * scale, v.y * scale);
        a[base + static_cast<int64_t>(kk) * span + li] = v;
    }
}

// Whole transform of one array (size <= kSmemFftMax) in shared memory: the
// bit-reversal permutation folded into the load, then every radix-2 stage
// with the same butterflies and twiddles as stages_kernel (bit-identical).
__global__ void __launch_bounds__(512) fft_smem_kernel(double2* __restrict__ data, int64_t size,
                                                       int log2size, int64_t inner,
                                                       int64_t outer_stride, int sign,
                                                       const double2* __restrict__ tw,
                                                       double scale) {
    extern __shared__ double2 buf[];
    const int64_t bi = blockIdx.x;
    double2* a = data + (bi / inner) * outer_stride + (bi % inner) * size;
    const int n = static_cast<int>(size);
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        buf[bitrev_bits(static_cast<unsigned>(e), log2size)] = a[e];
    __syncthreads();
    for (int s = 1; s <= log2size; ++s) {
        const int half = 1 << (s - 1);
        const int64_t step = size >> s;
        for (int bf = threadIdx.x; bf < n / 2; bf += blockDim.x) {
            const int blk = bf / half, off = bf - blk * half;
            const int e0 = blk * 2 * half + off, e1 = e0 + half;
            double2 w = tw[static_cast<int64_t>(off) * step];
            if (sign > 0) w.y = -w.y;
            const double2 x0 = buf[e0];
            const double2 t = cmul(buf[e1], w);
            buf[e1] = make_double2(x0.x - t.x, x0.y - t.y);
            buf[e0] = make_double2(x0.x + t.x, x0.y + t.y);
        }
        __syncthreads();
    }
    const bool do_scale = scale != 1.0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        double2 v = buf[e];
        if (do_scale) v = make_double2(v.x * scale, v.y * scale);
        a[e] = v;
    }
}

// fft_smem_kernel over several array sets of different sizes in one launch
// (the bucket vectors of every iteration with 256 < b <= kSmemFftMax): the
// CTA's set is found from the cumulative block counts, then the transform is
// fft_smem_kernel's, operation for operation.
struct SmemFftSets {
    int nsets;
    int64_t first[kMaxFftSets + 1];  // first block of each set
    int64_t off[kMaxFftSets], size[kMaxFftSets], inner[kMaxFftSets];
    int log2size[kMaxFftSets];
    int m[kMaxFftSets];
    const double2* tw[kMaxFftSets];
};

__global__ void __launch_bounds__(512) fft_smem_sets_kernel(double2* __restrict__ data,
                                                            const __grid_constant__ SmemFftSets S,
                                                            int64_t outer_stride, int sign,
                                                            double scale, FftGate gate) {
    extern __shared__ double2 buf[];
    int si = 0;
    while (si + 1 < S.nsets && static_cast<int64_t>(blockIdx.x) >= S.first[si + 1]) ++si;
    if (gate.post_done) {
        // gated: let the decode behind this grid be scheduled, then wait for
        // this set's iteration to be encoded (acquire, then drop stale L1)
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (threadIdx.x == 0) {
            const int m = S.m[si];
            for (;;) {
                int32_t v;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v)
                             : "l"(gate.wait_done + m) : "memory");
                if (v >= gate.wait_need[m]) break;
                __nanosleep(64);
            }
            __threadfence();
        }
        __syncthreads();
    }
    const int64_t bi = static_cast<int64_t>(blockIdx.x) - S.first[si];
    const int64_t size = S.size[si];
    const int log2size = S.log2size[si];
    const double2* __restrict__ tw = S.tw[si];
    double2* a = data + S.off[si] + (bi / S.inner[si]) * outer_stride + (bi % S.inner[si]) * size;
    const int n = static_cast<int>(size);
    for (int e = threadIdx.x; e < n; e += blockDim.x)
        buf[bitrev_bits(static_cast<unsigned>(e), log2size)] = a[e];
    __syncthreads();
    for (int s = 1; s <= log2size; ++s) {
        const int half = 1 << (s - 1);
        const int64_t step = size >> s;
        for (int bf = threadIdx.x; bf < n / 2; bf += blockDim.x) {
            const int blk = bf / half, off = bf - blk * half;
            const int e0 = blk * 2 * half + off, e1 = e0 + half;
            double2 w = tw[static_cast<int64_t>(off) * step];
            if (sign > 0) w.y = -w.y;
            const double2 x0 = buf[e0];
            const double2 t = cmul(buf[e1], w);
            buf[e1] = make_double2(x0.x - t.x, x0.y - t.y);
            buf[e0] = make_double2(x0.x + t.x, x0.y + t.y);
        }
        __syncthreads();
    }
    const bool do_scale = scale != 1.0;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        double2 v = buf[e];
        if (do_scale) v = make_double2(v.x * scale, v.y * scale);
        a[e] = v;
    }
    if (gate.post_done) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(gate.post_done + S.m[si], 1);
        }
    }
}

// Arrays larger than one CTA's shared memory (4096 < size <= 2^18), every
// set in two launches instead of a bit-reversal pass plus two stage passes
// per size: pass 1 gathers each 2048-element tile straight from its
// bit-reversed positions and runs stages 1..11 (span 1, as stages_kernel
// with s0 = 0), writing to a scratch copy (in place would overwrite samples
// other tiles still gather); pass 2 runs the remaining stages 12..log2size
// (lo_tile 16, as stages_kernel with s0 = 11) from the scratch back into the
// data, scaling after the last butterfly.  Same butterflies, twiddles and
// order as stages_kernel: bit-identical.
constexpr int kBigPass1 = 11;
struct BigFftSets {
    int nsets;
    int64_t first[kMaxFftSets + 1];  // first block of each set
    int64_t off[kMaxFftSets], size[kMaxFftSets], inner[kMaxFftSets];
    int64_t groups[kMaxFftSets];      // blocks per array
    int log2size[kMaxFftSets], s0[kMaxFftSets], s1[kMaxFftSets], lo_tile[kMaxFftSets];
    const double2* tw[kMaxFftSets];
};

template <bool kGather>
__global__ void __launch_bounds__(512) stages_sets_kernel(const double2* __restrict__ src,
                                                          double2* __restrict__ dst,
                                                          const __grid_constant__ BigFftSets S,
                                                          int64_t outer_stride, int sign,
                                                          double scale) {
    extern __shared__ double2 tile[];
    int si = 0;
    while (si + 1 < S.nsets && static_cast<int64_t>(blockIdx.x) >= S.first[si + 1]) ++si;
    const int64_t blk = static_cast<int64_t>(blockIdx.x) - S.first[si];
    const int64_t bi = blk / S.groups[si];
    const int64_t g = blk - bi * S.groups[si];
    const int64_t size = S.size[si];
    const int s0 = S.s0[si], s1 = S.s1[si], lo_tile = S.lo_tile[si], log2size = S.log2size[si];
    const double2* __restrict__ tw = S.tw[si];
    const int64_t arr = S.off[si] + (bi / S.inner[si]) * outer_stride + (bi % S.inner[si]) * size;
    const double2* a = src + arr;
    double2* d = dst + arr;
    const int G = s1 - s0;
    const int64_t span = int64_t{1} << s0;
    const int64_t tiles_per_hi = span / lo_tile;
    const int64_t hi = g / tiles_per_hi;
    const int64_t lo0 = (g - hi * tiles_per_hi) * lo_tile;
    const int count = (1 << G) * lo_tile;
    const int64_t base = (hi << s1) + lo0;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const int kk = e / lo_tile, li = e - kk * lo_tile;
        const int64_t pos = base + static_cast<int64_t>(kk) * span + li;
        tile[e] = kGather ? a[bitrev_bits(static_cast<unsigned>(pos), log2size)] : a[pos];
    }
    __syncthreads();
    for (int st = s0 + 1; st <= s1; ++st) {
        const int hkk = 1 << (st - 1 - s0);
        const int64_t step = size >> st;
        for (int bf = threadIdx.x; bf < count / 2; bf += blockDim.x) {
            const int li = bf % lo_tile;
            const int p = bf / lo_tile;
            const int blk2 = p / hkk, off = p - blk2 * hkk;
            const int kk = blk2 * 2 * hkk + off;
            const int64_t k = ((static_cast<int64_t>(off) << s0) + lo0 + li) * step;
            double2 w = tw[k];
            if (sign > 0) w.y = -w.y;
            const int e0 = kk * lo_tile + li, e1 = (kk + hkk) * lo_tile + li;
            const double2 x0 = tile[e0];
            const double2 t = cmul(tile[e1], w);
            tile[e1] = make_double2(x0.x - t.x, x0.y - t.y);
            tile[e0] = make_double2(x0.x + t.x, x0.y + t.y);
        }
        __syncthreads();
    }
    const bool do_scale = s1 == log2size && scale != 1.0;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        const int kk = e / lo_tile, li = e - kk * lo_tile;
        double2 v = tile[e];
        if (do_scale) v = make_double2(v.x * scale, v.y * scale);
        d[base + static_cast<int64_t>(kk) * span + li] = v;
    }
}

void smem_fft_attribute(const void* fn) {
    // the attribute is per device
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> ready;
    int dev = 0;
    MSFFT_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (!ready.count({dev, fn})) {
        MSFFT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(double2) * kSmemFftMax)));
        ready.insert({dev, fn});
    }
}

}  // namespace

void fft_radix2_sets(double2* data, const FftSet* sets, int nsets, int64_t batch,
                     int64_t outer_stride, int sign, double scale, cudaStream_t stream,
                     const FftGate* gate, double2* scratch) {
    SmemFftSets S{};
    BigFftSets B{};
    int64_t blocks = 0, max_size = 0;
    for (int i = 0; i < nsets; ++i) {
        const FftSet& f = sets[i];
        if (f.size <= 1 || batch <= 0) continue;
        if (f.size > kSmemFftMax || S.nsets == kMaxFftSets) {
            if (gate) throw CudaError("fft_radix2_sets: gated sets must fit one launch");
            if (scratch && f.size <= (int64_t{1} << (kBigPass1 + 7)) && B.nsets < kMaxFftSets) {
                int lg = 0;
                while ((int64_t{1} << lg) < f.size) ++lg;
                B.off[B.nsets] = f.off;
                B.size[B.nsets] = f.size;
                B.inner[B.nsets] = f.inner;
                B.log2size[B.nsets] = lg;
                B.tw[B.nsets] = device_twiddles(f.size);
                ++B.nsets;
                continue;
            }
            fft_radix2_batched(data + f.off, f.size, batch * f.inner, f.inner, outer_stride, sign,
                               scale, stream);
            continue;
        }
        int lg = 0;
        while ((int64_t{1} << lg) < f.size) ++lg;
        S.first[S.nsets] = blocks;
        S.off[S.nsets] = f.off;
        S.size[S.nsets] = f.size;
        S.inner[S.nsets] = f.inner;
        S.log2size[S.nsets] = lg;
        S.m[S.nsets] = f.m;
        S.tw[S.nsets] = device_twiddles(f.size);
        ++S.nsets;
        blocks += batch * f.inner;
        max_size = std::max(max_size, f.size);
    }
    if (B.nsets > 0) {
        // the two passes over every large set (see stages_sets_kernel)
        BigFftSets P1 = B, P2 = B;
        int64_t b1 = 0, b2 = 0;
        for (int i = 0; i < B.nsets; ++i) {
            P1.s0[i] = 0;
            P1.s1[i] = kBigPass1;
            P1.lo_tile[i] = 1;
            P1.groups[i] = B.size[i] >> kBigPass1;
            P1.first[i] = b1;
            b1 += batch * B.inner[i] * P1.groups[i];
            P2.s0[i] = kBigPass1;
            P2.s1[i] = B.log2size[i];
            P2.lo_tile[i] = 16;
            P2.groups[i] = (B.size[i] >> B.log2size[i]) * ((int64_t{1} << kBigPass1) / 16);
            P2.first[i] = b2;
            b2 += batch * B.inner[i] * P2.groups[i];
        }
        P1.first[B.nsets] = b1;
        P2.first[B.nsets] = b2;
        int g2max = 0;
        for (int i = 0; i < B.nsets; ++i) g2max = std::max(g2max, B.log2size[i] - kBigPass1);
        const size_t smem1 = sizeof(double2) << kBigPass1;
        const size_t smem2 = sizeof(double2) * 16 << g2max;
        smem_attr(stages_sets_kernel<true>, smem1);
        smem_attr(stages_sets_kernel<false>, smem2);
        if (b1 > 0x7fffffff || b2 > 0x7fffffff) throw CudaError("fft_radix2_sets: too many tiles");
        stages_sets_kernel<true><<<static_cast<unsigned>(b1), 512, smem1, stream>>>(
            data, scratch, P1, outer_stride, sign, scale);
        MSFFT_LAUNCH_CHECK("stages_sets_kernel (pass 1)");
        const int t2 = static_cast<int>(std::min<size_t>(512, std::max<size_t>(32, smem2 / 32)));
        stages_sets_kernel<false><<<static_cast<unsigned>(b2), t2, smem2, stream>>>(
            scratch, data, P2, outer_stride, sign, scale);
        MSFFT_LAUNCH_CHECK("stages_sets_kernel (pass 2)");
    }
    if (S.nsets == 0) return;
    S.first[S.nsets] = blocks;
    if (blocks > 0x7fffffff) throw CudaError("fft_radix2_sets: too many arrays");
    smem_fft_attribute(reinterpret_cast<const void*>(fft_smem_sets_kernel));
    const int threads = static_cast<int>(std::min<int64_t>(512, std::max<int64_t>(32, max_size / 2)));
    const FftGate g = gate ? *gate : FftGate{nullptr, nullptr, nullptr};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = sizeof(double2) * static_cast<size_t>(max_size);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = gate ? 1 : 0;
    MSFFT_CUDA(cudaLaunchKernelEx(&cfg, fft_smem_sets_kernel, data, S, outer_stride, sign, scale, g));
    MSFFT_LAUNCH_CHECK("fft_smem_sets_kernel");
}

const double* host_twiddles(int64_t n) {
    std::lock_guard<std::mutex> lock(g_tw_mu);
    auto it = g_host_tw.find(n);
    if (it == g_host_tw.end())
        it = g_host_tw.emplace(n, std::make_unique<std::vector<double>>(make_twiddles(n))).first;
    return it->second->data();
}

const double2* device_twiddles(int64_t n) {
    int dev = 0;
    MSFFT_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lock(g_tw_mu);
        auto it = g_dev_tw.find({dev, n});
        if (it != g_dev_tw.end()) return it->second;
    }
    const double* h = host_twiddles(n);
    const size_t count = static_cast<size_t>(std::max<int64_t>(n / 2, 1));
    double2* d = nullptr;
    MSFFT_CUDA(cudaMalloc(&d, count * sizeof(double2)));
    MSFFT_CUDA(cudaMemcpy(d, h, count * sizeof(double2), cudaMemcpyHostToDevice));
    std::lock_guard<std::mutex> lock(g_tw_mu);
    auto [it, inserted] = g_dev_tw.emplace(std::make_pair(dev, n), d);
    if (!inserted) cudaFree(d);
    return it->second;
}

void fft_radix2_batched(double2* data, int64_t size, int64_t batch, int64_t inner,
                        int64_t outer_stride, int sign, double scale, cudaStream_t stream) {
    if (size <= 1 || batch <= 0) return;
    int log2size = 0;
    while ((int64_t{1} << log2size) < size) ++log2size;
    const double2* tw = device_twiddles(size);
    if (size <= kSmemFftMax && batch <= 0x7fffffff) {
        // one launch, one read and one write of the data
        const size_t smem = sizeof(double2) * static_cast<size_t>(size);
        smem_fft_attribute(reinterpret_cast<const void*>(fft_smem_kernel));
        const int threads = static_cast<int>(std::min<int64_t>(512, std::max<int64_t>(32, size / 2)));
        fft_smem_kernel<<<static_cast<unsigned>(batch), threads, smem, stream>>>(
            data, size, log2size, inner, outer_stride, sign, tw, scale);
        MSFFT_LAUNCH_CHECK("fft_smem_kernel");
        return;
    }
    const int64_t total = size * batch;
    bitrev_inplace_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(
        data, size, log2size, inner, outer_stride, total);
    MSFFT_LAUNCH_CHECK("bitrev_inplace_kernel");
    int s0 = 0;
    while (s0 < log2size) {
        int lo_tile, G;
        if (s0 == 0) {
            lo_tile = 1;
            G = std::min(log2size, 11);
        } else {
            lo_tile = static_cast<int>(std::min<int64_t>(int64_t{1} << s0, 16));
            G = std::min(log2size - s0, lo_tile == 16 ? 7 : 11 - s0);
            if (G < 1) G = 1;
        }
        const int s1 = s0 + G;
        const int64_t groups = (size >> s1) * ((int64_t{1} << s0) / lo_tile);
        const int64_t blocks = groups * batch;
        const size_t smem = sizeof(double2) * (static_cast<size_t>(1) << G) * lo_tile;
        const int threads = static_cast<int>(std::min<size_t>(512, std::max<size_t>(32, smem / 32)));
        const double sc = (s1 == log2size) ? scale : 1.0;
        stages_kernel<<<static_cast<unsigned>(blocks), threads, smem, stream>>>(
            data, size, inner, outer_stride, s0, s1, lo_tile, sign, tw, sc);
        MSFFT_LAUNCH_CHECK("stages_kernel");
        s0 = s1;
    }
}

}  // namespace msfft_b200
