// gather_latency_probe.cu -- how long one batch of U independent random
// loads takes for a single CTA on an otherwise idle B200 (the single-signal
// encode's situation): each thread issues U random 16-B loads, sums them, and
// derives the next batch's addresses from the sum (batches serialise).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/gather_latency_probe tools/gather_latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U, bool CS>
__global__ void probe(const double2* __restrict__ x, unsigned mask, int batches,
                      unsigned long long* out_ns, double* sink) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    unsigned idx = (threadIdx.x * 2654435761u) & mask;
    double acc = 0.0;
    for (int b = 0; b < batches; ++b) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned a = (idx + u * 40503u * 7919u) & mask;
            v[u] = CS ? __ldcs(x + a) : x[a];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x;
        idx = (idx * 1664525u + 1013904223u + (acc != acc ? 1u : 0u)) & mask;
    }
    __syncthreads();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out_ns[blockIdx.x] = t1 - t0;
    if (acc == 12345.0) sink[0] = acc;
}

int main() {
    const size_t max_elems = size_t{1} << 27;  // 2 GiB of double2
    double2* x;
    double* sink;
    unsigned long long* ns;
    cudaMalloc(&x, max_elems * sizeof(double2));
    cudaMemset(x, 0, max_elems * sizeof(double2));
    cudaMalloc(&sink, 8);
    cudaMalloc(&ns, 8 * 1024);
    unsigned long long h[1024];
    const int batches = 64;
    for (size_t elems : {size_t{1} << 16, size_t{1} << 21, size_t{1} << 27}) {
        for (int ctas : {1, 22}) {
            for (int mode = 0; mode < 4; ++mode) {
                float best = 1e30f;
                for (int rep = 0; rep < 5; ++rep) {
                    const unsigned mask = static_cast<unsigned>(elems - 1);
                    if (mode == 0) probe<8, true><<<ctas, 256>>>(x, mask, batches, ns, sink);
                    if (mode == 1) probe<8, false><<<ctas, 256>>>(x, mask, batches, ns, sink);
                    if (mode == 2) probe<16, true><<<ctas, 256>>>(x, mask, batches, ns, sink);
                    if (mode == 3) probe<32, true><<<ctas, 256>>>(x, mask, batches, ns, sink);
                    cudaMemcpy(h, ns, 8 * ctas, cudaMemcpyDeviceToHost);
                    unsigned long long mx = 0;
                    for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
                    if (rep > 0 && mx < best) best = static_cast<float>(mx);
                }
                const int U[] = {8, 8, 16, 32};
                printf("array %6zu KB  ctas %2d  U=%2d %s : %7.1f ns per batch, %6.2f ns per load per thread\n",
                       elems * 16 / 1024, ctas, U[mode], mode == 1 ? "ld   " : "ld.cs",
                       best / batches, best / batches / U[mode]);
            }
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
