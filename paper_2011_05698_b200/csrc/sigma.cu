// sigma.cu -- per-signal sigma plan on the device.
//
// random_params(n, rng, 0) once per iteration (proj/src/sfft4.cpp:48,
// proj/src/bucketize.cpp:39-48) from Rng(seed) = std::mt19937_64(seed)
// (proj/include/msfft/rng.hpp:21): sigma = 2*below(n/2) + 1 with
// below(B) = (u64 * B) >> 64, sigma_inv = sigma^-1 mod n.  One thread per
// signal reproduces the engine's first outputs exactly: a draw d < 156 only
// needs state words 0..d+1 and 156..156+d of the seeded state after one
// twist, so the thread seeds 156+iters+1 words instead of all 312.
#include <cuda_runtime.h>

#include "cuda_check.hpp"
#include "sigma.hpp"

namespace msfft_b200 {

namespace {

constexpr int kNN = 312, kMM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

#ifdef MSFFT_TIMELINE
__device__ unsigned long long g_sig_tl[2];
#endif

template <int MAXD>
__global__ void sigma_kernel(const uint64_t* __restrict__ seeds, int64_t batch, int iters,
                             int64_t n, int64_t* __restrict__ sigma,
                             int64_t* __restrict__ sigma_inv) {
    // programmatic dependent launch: the next kernel may be scheduled now
    // (it waits for this grid's results with griddepcontrol.wait)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef MSFFT_TIMELINE
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (blockIdx.x == 0 && threadIdx.x == 0) g_sig_tl[0] = t0;
#endif
    const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= batch) return;
    // seeded state words 0..MAXD and kMM..kMM+MAXD
    uint64_t lo[MAXD + 1], hi[MAXD];
    uint64_t v = seeds[s];
    lo[0] = v;
    for (int i = 1; i <= MAXD; ++i) {
        v = 6364136223846793005ull * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
        lo[i] = v;
    }
    for (int i = MAXD + 1; i < kMM; ++i)
        v = 6364136223846793005ull * (v ^ (v >> 62)) + static_cast<uint64_t>(i);
    for (int i = 0; i < MAXD; ++i) {
        v = 6364136223846793005ull * (v ^ (v >> 62)) + static_cast<uint64_t>(kMM + i);
        hi[i] = v;
    }
    const uint64_t half = static_cast<uint64_t>(n / 2);
    const uint64_t mask = static_cast<uint64_t>(n - 1);
    for (int d = 0; d < iters; ++d) {
        // word d after the first twist: mt[d+156] ^ twist(mt[d], mt[d+1])
        const uint64_t x = (lo[d] & kUpper) | (lo[d + 1] & kLower);
        uint64_t xa = x >> 1;
        if (x & 1ull) xa ^= kMatrixA;
        const uint64_t out = temper(hi[d] ^ xa);
        const uint64_t sg = 2ull * __umul64hi(out, half) + 1ull;
        uint64_t inv = sg;  // Newton: correct to 3 bits, doubles each step
        for (int it = 0; it < 6; ++it) inv *= 2ull - sg * inv;
        sigma[s * iters + d] = static_cast<int64_t>(sg);
        sigma_inv[s * iters + d] = static_cast<int64_t>(inv & mask);
    }
#ifdef MSFFT_TIMELINE
    if (s == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g_sig_tl[1]));
#endif
}

}  // namespace

#ifdef MSFFT_TIMELINE
extern "C" int msfft_debug_sigma_timeline(void* dst) {
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_sig_tl, 16));
}
#endif

void launch_sigma(const uint64_t* d_seeds, int64_t batch, int iters, int64_t n, int64_t* d_sigma,
                  int64_t* d_sigma_inv, cudaStream_t stream, bool programmatic) {
    if (batch <= 0) return;
    if (iters > kMaxSigmaIters) throw std::invalid_argument("sigma plan: too many iterations");
    const unsigned blocks = static_cast<unsigned>((batch + 127) / 128);
    if (programmatic) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(128);
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MSFFT_CUDA(cudaLaunchKernelEx(&cfg, sigma_kernel<kMaxSigmaIters>, d_seeds, batch, iters, n,
                                      d_sigma, d_sigma_inv));
    } else {
        sigma_kernel<kMaxSigmaIters><<<blocks, 128, 0, stream>>>(d_seeds, batch, iters, n,
                                                                 d_sigma, d_sigma_inv);
    }
    MSFFT_LAUNCH_CHECK("sigma_kernel");
}

}  // namespace msfft_b200
