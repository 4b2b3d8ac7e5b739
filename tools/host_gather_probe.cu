// host_gather_probe.cu -- random 8-byte loads from pinned, mapped HOST memory
// (zero-copy over PCIe) vs a full H2D copy of the same buffer.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x; }
template <int U>
__global__ void gather(const float2* __restrict__ x, uint64_t mask, int iters, float* sink, uint64_t salt) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        float2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcg(x + (mix(tid * 1315423911ull + (uint64_t)(it * U + u) + salt) & mask));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 1234.5f) sink[tid] = acc;
}
int main() {
    const uint64_t n = 1ull << 31;  // 16 GiB of float2
    float2* h; CK(cudaHostAlloc(&h, n * sizeof(float2), cudaHostAllocMapped));
    for (uint64_t i = 0; i < n; i += 4096) h[i] = make_float2(1.f, 2.f);
    float2* dptr; CK(cudaHostGetDevicePointer(&dptr, h, 0));
    float* sink; CK(cudaMalloc(&sink, 1 << 26));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int blocks : {148 * 4, 148 * 16, 148 * 64}) {
        for (int iters : {4, 16}) {
            gather<8><<<blocks, 256>>>(dptr, n - 1, 1, sink, 1);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            gather<8><<<blocks, 256>>>(dptr, n - 1, iters, sink, 99);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            const double loads = (double)blocks * 256 * iters * 8;
            printf("zero-copy blocks %6d iters %3d: %8.3f ms  %7.2f Gloads/s\n", blocks, iters, ms, loads / ms / 1e6);
        }
    }
    float2* d; CK(cudaMalloc(&d, (size_t)1 << 32));
    cudaEventRecord(a);
    CK(cudaMemcpyAsync(d, h, (size_t)1 << 32, cudaMemcpyHostToDevice));
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("H2D 4 GiB pinned: %.3f ms = %.1f GB/s\n", ms, 4.294967296 / ms * 1e3);
    return 0;
}
