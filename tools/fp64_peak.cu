// Measured FP64 peak of this B200 (the denominator of the per-stage FP64-pipe
// rooflines, profiles/r02/): DFMA / DADD / DMUL issue rate with 8 independent
// dependency chains per thread, 2048 threads per SM, every SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) fp64_loop(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = fma(x[i], a, b);
            else if (OP == 1) x[i] = __dadd_rn(x[i], b);
            else x[i] = __dmul_rn(x[i], a);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 1 << 14, threads = 256, blocks = sms * 8;
    const char* names[3] = {"dfma", "dadd", "dmul"};
    for (int op = 0; op < 3; ++op) {
        auto launch = [&] {
            if (op == 0) fp64_loop<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
            else if (op == 1) fp64_loop<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
            else fp64_loop<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        };
        launch();
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 5.0 * blocks * threads * static_cast<double>(iters) * 8;  // thread ops
        const double s = ms * 1e-3;
        printf("{\"op\": \"%s\", \"thread_ops_per_s\": %.4e, \"warp_inst_per_s\": %.4e, "
               "\"tflops\": %.3f, \"per_sm_per_clk_at_1965MHz\": %.2f}\n",
               names[op], ops / s, ops / 32 / s, (op == 0 ? 2 : 1) * ops / s / 1e12,
               ops / s / sms / 1.965e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
