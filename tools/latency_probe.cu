// latency_probe.cu -- dependent-chain latency (cycles per op) on one warp of
// the FP64 operations in the decode's locate stage chain: DADD, DMUL, trunc
// (FRND.F64), a double __shfl_xor_sync, and a shared-memory load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o latency_probe latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void chain(double seed, double* out, long long* cycles) {
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = seed * threadIdx.x;
    __syncthreads();
    double x = seed + threadIdx.x;
    volatile double* gp = seed > 1e300 ? out : sm;  // generic: shared at run time
    int idx = threadIdx.x & 31;
    const long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < kIters; ++i) {
        if (OP == 0) x = x + 1.0000001;
        if (OP == 1) x = x * 0.99999991;
        if (OP == 2) x = trunc(x * 1.0000001) + 0.5;  // trunc + DMUL + DADD
        if (OP == 3) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
        if (OP == 4) {
            idx = static_cast<int>(sm[idx]) & 31;
        }
        if (OP == 5) x = floor(x * 0.5) + 0.25;     // floor + DMUL + DADD
        if (OP == 6) x = x < 3.0 ? x + 1.0 : x - 1.0;  // DSETP + select + DADD
        if (OP == 7) x = static_cast<double>(static_cast<long long>(x)) + 1.5;  // F2I.S64 + I2F.F64.S64
        if (OP == 8) idx = static_cast<int>(gp[idx]) & 31;  // generic load that hits shared memory
        if (OP == 9) x = static_cast<double>(static_cast<long long>(idx + i)) * x;  // I2F.F64.S64 off-chain + DMUL
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    out[threadIdx.x] = x + idx;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 64 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    const char* names[] = {"DADD", "DMUL", "trunc+DMUL+DADD", "shfl.f64+DADD", "LDS (dependent)",
                           "floor+DMUL+DADD", "DSETP+sel+DADD", "F2I.S64+I2F.F64+DADD",
                           "generic LD (shared)", "I2F(indep)+DMUL"};
    for (int op = 0; op < 10; ++op) {
        long long c = 0;
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: chain<0><<<1, 32>>>(1.5, out, cyc); break;
                case 1: chain<1><<<1, 32>>>(1.5, out, cyc); break;
                case 2: chain<2><<<1, 32>>>(1.5, out, cyc); break;
                case 3: chain<3><<<1, 32>>>(1.5, out, cyc); break;
                case 4: chain<4><<<1, 32>>>(0.0, out, cyc); break;
                case 5: chain<5><<<1, 32>>>(1.5, out, cyc); break;
                case 6: chain<6><<<1, 32>>>(1.5, out, cyc); break;
                case 7: chain<7><<<1, 32>>>(1.5, out, cyc); break;
                case 8: chain<8><<<1, 32>>>(0.0, out, cyc); break;
                case 9: chain<9><<<1, 32>>>(1.0, out, cyc); break;
            }
            cudaMemcpy(&c, cyc, sizeof c, cudaMemcpyDeviceToHost);
        }
        printf("%-20s %7.1f cycles per step\n", names[op], static_cast<double>(c) / kIters);
    }
    return 0;
}
