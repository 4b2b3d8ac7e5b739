// Read-bandwidth probe for the finiteness scan (validate_kernel variants).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/validate_probe tools/validate_probe.cu
//   tools/validate_probe [GiB]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t bad4(uint4 v) {
    return ((v.x & 0x7f800000u) == 0x7f800000u) | ((v.y & 0x7f800000u) == 0x7f800000u) |
           ((v.z & 0x7f800000u) == 0x7f800000u) | ((v.w & 0x7f800000u) == 0x7f800000u);
}

__device__ __forceinline__ uint4 ld_hint(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// grid-stride, U loads of 16 B per thread per trip (the product kernel)
template <int U, int MODE>
__global__ void gs(const uint4* __restrict__ x, int64_t nv, int* bad) {
    uint32_t acc = 0;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * U;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x * U + threadIdx.x; base < nv; base += step) {
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            int64_t i = base + (int64_t)j * blockDim.x;
            if (i < nv) v[j] = MODE == 0 ? __ldcs(x + i) : MODE == 1 ? ld_hint(x + i) : __ldg(x + i);
            else v[j] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) acc |= bad4(v[j]);
    }
    if (__any_sync(0xffffffffu, acc) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

// contiguous range per block
template <int U, int MODE>
__global__ void blk(const uint4* __restrict__ x, int64_t nv, int* bad) {
    uint32_t acc = 0;
    const int64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const int64_t lo = (int64_t)blockIdx.x * per, hi = min(nv, lo + per);
    for (int64_t base = lo + threadIdx.x; base < hi; base += (int64_t)blockDim.x * U) {
        uint4 v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            int64_t i = base + (int64_t)j * blockDim.x;
            if (i < hi) v[j] = MODE == 0 ? __ldcs(x + i) : ld_hint(x + i);
            else v[j] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) acc |= bad4(v[j]);
    }
    if (__any_sync(0xffffffffu, acc) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

// TMA bulk copies (cp.async.bulk) of CH-byte chunks into a NB-deep smem ring
template <int CH, int NB>
__global__ void __launch_bounds__(256) bulk(const uint4* __restrict__ x, int64_t nv, int* bad) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[NB];
    const int64_t nch = nv * 16 / CH;
    if (threadIdx.x == 0)
        for (int i = 0; i < NB; ++i)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
    __syncthreads();
    uint32_t acc = 0;
    int64_t c0 = blockIdx.x;
    auto issue = [&](int64_t c, int slot) {
        uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[slot]);
        uint32_t d = (uint32_t)__cvta_generic_to_shared(sm + slot * CH);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(d), "l"((const char*)x + c * CH), "r"(CH), "r"(b) : "memory");
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < NB; ++i) {
            int64_t c = c0 + (int64_t)i * gridDim.x;
            if (c < nch) issue(c, i);
        }
    uint32_t phase[NB] = {};
    int it = 0;
    for (int64_t c = c0; c < nch; c += gridDim.x, ++it) {
        int slot = it % NB;
        uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[slot]);
        uint32_t ph = (it / NB) & 1;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }"
                     :: "r"(b), "r"(ph) : "memory");
        const uint4* s = reinterpret_cast<const uint4*>(sm + slot * CH);
        for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) acc |= bad4(s[i]);
        __syncthreads();
        if (threadIdx.x == 0) {
            int64_t cn = c + (int64_t)NB * gridDim.x;
            if (cn < nch) issue(cn, slot);
        }
    }
    (void)phase;
    if (__any_sync(0xffffffffu, acc) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

__global__ void fill(uint32_t* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)(i * 2654435761u) & 0x3fffffffu;  // finite floats
}

template <class F>
float timeit(F f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    double gib = argc > 1 ? atof(argv[1]) : 16.0;
    size_t bytes = (size_t)(gib * (1ull << 30));
    int64_t nv = bytes / 16;
    uint4* x; int* bad;
    CK(cudaMalloc(&x, bytes));
    CK(cudaMalloc(&bad, 4));
    CK(cudaMemset(x, 0, bytes));
    if (argc > 2) {  // non-zero data: a simple LCG pattern
        fill<<<1184, 256>>>(reinterpret_cast<uint32_t*>(x), bytes / 4);
        CK(cudaDeviceSynchronize());
    }
    CK(cudaMemset(bad, 0, 4));
    if (argc > 3) {
        CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, atoi(argv[3])));
        size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity %zu\n", v);
    }
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto rep = [&](const char* name, float ms) {
        cudaError_t e = cudaGetLastError();
        printf("%-40s %8.3f ms  %7.1f GB/s %s\n", name, ms, bytes / (ms * 1e-3) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
#define GS(U, MODE, T, BPS) rep("gs U=" #U " mode=" #MODE " thr=" #T " bps=" #BPS, \
    timeit([&] { gs<U, MODE><<<sms * BPS, T>>>(x, nv, bad); }, 5))
#define BLK(U, MODE, T, BPS) rep("blk U=" #U " mode=" #MODE " thr=" #T " bps=" #BPS, \
    timeit([&] { blk<U, MODE><<<sms * BPS, T>>>(x, nv, bad); }, 5))
    GS(8, 0, 256, 8);
    GS(8, 0, 512, 4);
#define BULK(CHB, NBB, T, BPS) { auto k = bulk<CHB, NBB>; \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CHB * NBB); \
        rep("bulk " #CHB " x" #NBB " thr=" #T " bps=" #BPS, \
            timeit([&] { k<<<sms * BPS, T, CHB * NBB>>>(x, nv, bad); }, 5)); }
    BULK(16384, 4, 128, 3);
    BULK(16384, 4, 128, 2);
    BULK(16384, 3, 128, 4);
    BULK(16384, 6, 128, 2);
    BULK(16384, 8, 128, 1);
    BULK(32768, 3, 128, 2);
    BULK(32768, 2, 128, 3);
    BULK(8192, 6, 128, 4);
    BULK(8192, 12, 128, 2);
    BULK(4096, 12, 128, 4);
    BULK(16384, 4, 256, 3);
    BULK(16384, 4, 64, 3);
    BULK(65536, 3, 128, 1);
    // device-to-device copy for reference
    uint4* y; CK(cudaMalloc(&y, bytes / 2));
    rep("memcpy d2d (bytes = read+write of half)", timeit([&] { cudaMemcpyAsync(y, x, bytes / 2, cudaMemcpyDeviceToDevice); }, 5));
    int h; cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
    printf("bad=%d\n", h);
    return 0;
}
