// gather_probe.cu -- random 8-/16-byte gather microbenchmark on B200.
// Measures how fast independent random sample loads (the sFFT encode's
// access pattern) stream from HBM for several load flavours, with and
// without the L2 fetch-granularity limit.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
//   ./gather_probe [limit_bytes]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

template <int MODE>
__device__ __forceinline__ float2 ld8(const float2* p) {
    float2 v;
    if (MODE == 0) v = *p;
    else if (MODE == 1) v = __ldcs(p);
    else if (MODE == 2) v = __ldg(p);
    else if (MODE == 3) v = __ldcg(p);
    else if (MODE == 4) asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    else if (MODE == 5) asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(0ull));
    else if (MODE == 6) asm volatile("ld.global.cg.L2::64B.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    else asm volatile("ld.volatile.global.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

template <int MODE, int U>
__global__ void __launch_bounds__(256) gather8(const float2* __restrict__ x, uint64_t mask, int iters,
                                               float* __restrict__ sink, uint64_t salt) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld8<MODE>(x + (mix(tid * 1315423911ull + (uint64_t)(it * U + u) + salt) & mask));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1234.5f) sink[tid] = acc;
}

template <int MODE>
float run(const float2* x, uint64_t n, int blocks, int iters, float* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    gather8<MODE, 8><<<blocks, 256>>>(x, n - 1, iters, sink, 7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    gather8<MODE, 8><<<blocks, 256>>>(x, n - 1, iters, sink, 99);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char** argv) {
    if (argc > 1) {
        size_t lim = atoi(argv[1]);
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, lim);
        printf("set MaxL2FetchGranularity=%zu -> %s\n", lim, cudaGetErrorString(e));
    }
    size_t cur = 0;
    CK(cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity));
    printf("MaxL2FetchGranularity now %zu\n", cur);
    const uint64_t n = 1ull << 31;  // 16 GiB of float2
    float2* x; CK(cudaMalloc(&x, n * sizeof(float2)));
    CK(cudaMemset(x, 0, n * sizeof(float2)));
    float* sink; CK(cudaMalloc(&sink, 148ull * 8 * 256 * 64 * sizeof(float)));
    const int blocks = 148 * 8 * 4, iters = 64;
    const double loads = (double)blocks * 256 * iters * 8;
    const char* names[] = {"default", "ldcs(EF)", "ldg(nc)", "ldcg", "nc.L1::no_allocate", "L1::no_alloc+hint", "cg.L2::64B", "volatile"};
    float ms[8];
    ms[0] = run<0>(x, n, blocks, iters, sink);
    ms[1] = run<1>(x, n, blocks, iters, sink);
    ms[2] = run<2>(x, n, blocks, iters, sink);
    ms[3] = run<3>(x, n, blocks, iters, sink);
    ms[4] = run<4>(x, n, blocks, iters, sink);
    ms[5] = run<5>(x, n, blocks, iters, sink);
    ms[6] = run<6>(x, n, blocks, iters, sink);
    ms[7] = run<7>(x, n, blocks, iters, sink);
    for (int i = 0; i < 8; ++i)
        printf("%-22s %8.3f ms  %7.1f Gloads/s  %7.1f GB/s at 32B/sector\n", names[i], ms[i],
               loads / ms[i] / 1e6, loads * 32 / ms[i] / 1e6);
    return 0;
}
