// tma_probe.cu -- does the path of a random 16-byte read change how much HBM
// traffic it costs?  LDG (8 B and 16 B), cp.async (LDGSTS, 16 B) and TMA
// bulk copies (cp.async.bulk, 16 B) from random 16-B-aligned addresses of a
// 16 GiB buffer.  Run plain for rates, under ncu for dram__bytes_read.sum:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__device__ __forceinline__ uint32_t s32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

#ifndef PROBE_U
#define PROBE_U 8
#endif
constexpr int U = PROBE_U;

// MODE 0: LDG 8 B, 1: LDG 16 B, 2: cp.async 16 B, 3: cp.async.bulk 16 B (TMA)
template <int MODE>
__global__ void __launch_bounds__(256) probe(const float4* __restrict__ x, uint64_t mask, int iters,
                                             float* __restrict__ sink, uint64_t salt) {
    __shared__ __align__(16) float4 buf[256 * U];
    __shared__ __align__(8) uint64_t bar;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    float acc = 0.f;
    if (MODE == 3) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        uint64_t idx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) idx[u] = mix(tid * 1315423911ull + (uint64_t)(it * U + u) + salt) & mask;
        if (MODE == 0) {
            float2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const float2*>(x + idx[u]));
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y;
        } else if (MODE == 1) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcs(x + idx[u]);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
        } else if (MODE == 2) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(&buf[threadIdx.x * U + u])),
                             "l"(x + idx[u]) : "memory");
            asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
            for (int u = 0; u < U; ++u) acc += buf[threadIdx.x * U + u].x;
        } else {
            if (threadIdx.x == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)),
                             "r"(256 * U * 16) : "memory");
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];"
                    ::"r"(s32(&buf[threadIdx.x * U + u])), "l"(x + idx[u]), "r"(s32(&bar)) : "memory");
            asm volatile(
                "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra W_%=;\n}" ::"r"(s32(&bar)), "r"(phase) : "memory");
            phase ^= 1u;
#pragma unroll
            for (int u = 0; u < U; ++u) acc += buf[threadIdx.x * U + u].x;
            __syncthreads();  // buffer reuse
        }
    }
    if (acc == 1234.5f) sink[tid] = acc;
}

template <int MODE>
float run(const float4* x, uint64_t n, int blocks, int iters, float* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    probe<MODE><<<blocks, 256>>>(x, n - 1, iters, sink, 7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    probe<MODE><<<blocks, 256>>>(x, n - 1, iters, sink, 99);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char** argv) {
    const uint64_t n = 1ull << 30;  // 16 GiB of float4
    float4* x;
    CK(cudaMalloc(&x, n * sizeof(float4)));
    CK(cudaMemset(x, 0, n * sizeof(float4)));
    float* sink;
    CK(cudaMalloc(&sink, (size_t)(argc > 1 ? atoi(argv[1]) : 148 * 8) * 256 * sizeof(float)));
    const int blocks = argc > 1 ? atoi(argv[1]) : 148 * 8;
    const int iters = argc > 2 ? atoi(argv[2]) : 64;
    const double reads = (double)blocks * 256 * iters * U;
    const char* names[] = {"LDG 8B (ldcs)", "LDG 16B (ldcs)", "cp.async 16B (LDGSTS)", "cp.async.bulk 16B (TMA)"};
    float ms[4] = {run<0>(x, n, blocks, iters, sink), run<1>(x, n, blocks, iters, sink),
                   run<2>(x, n, blocks, iters, sink), run<3>(x, n, blocks, iters, sink)};
    for (int i = 0; i < 4; ++i)
        printf("%-26s %8.3f ms  %7.1f G reads/s  (%.0f M reads)\n", names[i], ms[i], reads / ms[i] / 1e6,
               reads / 1e6);
    return 0;
}
