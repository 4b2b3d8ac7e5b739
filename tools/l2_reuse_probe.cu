// L2 reuse probe: does a random 8-B gather hit the L2 lines that a TMA bulk
// stream (the validation scan's copy) or an LDG stream brought in just
// before?  K1 streams a region of S MB (cp.async.bulk ring, optional L2
// policy); K2 gathers S/128 random 8-B samples from it.  Printed: K2's time
// after K1 (warm) and after a 512-MB flush (cold), per region size.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_reuse_probe tools/l2_reuse_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void stream_tma(const unsigned char* x, int64_t bytes, int policy, unsigned* sink) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ __align__(8) uint64_t bar[8];
    const int C = 16384;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint64_t pol = 0;
    if (policy == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    if (policy == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    const int64_t nch = bytes / C;
    auto issue = [&](int64_t c, int slot) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[slot])), "r"(C) : "memory");
        if (policy)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                         ::"r"(su32(ring + slot * C)), "l"(x + c * C), "r"(C), "r"(su32(&bar[slot])), "l"(pol) : "memory");
        else
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(ring + slot * C)), "l"(x + c * C), "r"(C), "r"(su32(&bar[slot])) : "memory");
    };
    int64_t cp = blockIdx.x;
    if (threadIdx.x == 0)
        for (int i = 0; i < 8 && cp < nch; ++i, cp += gridDim.x) issue(cp, i);
    unsigned acc = 0;
    int it = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
        const int slot = it % 8;
        const uint32_t par = (it / 8) & 1;
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                     ::"r"(su32(&bar[slot])), "r"(par) : "memory");
        acc ^= reinterpret_cast<const unsigned*>(ring + slot * C)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && cp < nch) {
            issue(cp, slot);
            cp += gridDim.x;
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void stream_ldg(const uint4* x, int64_t n16, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        acc ^= __ldg(x + i).x;
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void gather(const float2* x, int64_t nsamp, int64_t nload, unsigned mul, unsigned* sink) {
    float acc = 0;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (int64_t t = t0; t < nload; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = (static_cast<uint64_t>(t) * mul) % static_cast<uint64_t>(nsamp);
        acc += __ldg(x + idx).x;
    }
    if (acc == 1.2345f) *sink = 1;
}

int main() {
    const int64_t total = int64_t{1} << 30;
    unsigned char* buf;
    unsigned char* flush;
    unsigned* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&flush, 512 << 20);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 0, total);
    cudaMemset(flush, 1, 512 << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(stream_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[] = {"cold", "after TMA", "TMA evict_normal", "TMA evict_last", "after LDG", "after gather"};
    for (int64_t mb : {16, 32, 64, 96, 128, 192}) {
        const int64_t bytes = mb << 20;
        const int64_t nsamp = bytes / 8, nload = int64_t{1} << 23;  // 8 M random loads
        printf("region %4lld MB, %lld random 8-B loads:", (long long)mb, (long long)nload);
        for (int mode = 0; mode < 6; ++mode) {
            float best = 1e9f;
            for (int rep = 0; rep < 3; ++rep) {
                stream_ldg<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(flush), (512 << 20) / 16, sink);
                if (mode >= 1 && mode <= 3) stream_tma<<<sms, 256, 8 * 16384>>>(buf, bytes, mode - 1, sink);
                if (mode == 4) stream_ldg<<<sms * 8, 256>>>(reinterpret_cast<const uint4*>(buf), bytes / 16, sink);
                if (mode == 5) gather<<<sms * 8, 256>>>(reinterpret_cast<const float2*>(buf), nsamp, nload, 40503u, sink);
                cudaEventRecord(a);
                gather<<<sms * 8, 256>>>(reinterpret_cast<const float2*>(buf), nsamp, nload, 2654435761u, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float t;
                cudaEventElapsedTime(&t, a, b);
                best = t < best ? t : best;
            }
            printf("  %s %.1f us |", names[mode], best * 1e3);
        }
        printf("\n");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
