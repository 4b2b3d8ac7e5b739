// chain_probe.cu -- cycles per locate stage (decode K5 chain) on one warp,
// split into its parts: the phase/distance arithmetic, the 16-lane argmin
// reduction, and both, plus single-op dependent latencies.
//   nvcc -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a -o tools/chain_probe tools/chain_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr double kTwoPi = 6.283185307179586476925286766559;

__device__ __forceinline__ double circ(double a, double b) {
    double d = fabs(a - b);
    if (d >= kTwoPi) d = d - kTwoPi;
    const double e = kTwoPi - d;
    return d < e ? d : e;
}

template <int MODE>
__global__ void chain(double u0, double ton, double ph0, double rb, int stages, int gsz,
                      double* out, long long* cyc, const double* gph) {
    __shared__ double sph[256];
    const int lane = threadIdx.x & 31;
    const int glane = lane & (gsz - 1);
    const double offc = (glane + 0.5) * rb, step = (glane - 0.5) * rb;
    double u_min = u0;
    for (int i = threadIdx.x; i < 256; i += 32) sph[i] = ph0 + i * 1e-3;
    // MODE 3: the phase comes through a generic pointer into shared memory,
    // MODE 4: through a global pointer (L2), loaded one stage ahead
    const double* pp = MODE == 4 ? gph : sph;
    double ph = ph0, ph_n = pp[0];
    __syncwarp();
    const long long t0 = clock64();
    for (int s = 0; s < stages; ++s) {
        if (MODE >= 3) {
            ph = ph_n;
            ph_n = pp[(s + 1) & 255];
        }
        double best_d = INFINITY, best_step = 0.0;
        int best_j = 0x7fffffff;
        if (MODE != 1) {
            const double y = (u_min + offc) * ton;
            double f = y - trunc(y);
            if (f < 0) f += 1.0;
            const double d = circ(f * kTwoPi, ph);
            if (d < best_d) {
                best_d = d;
                best_j = glane;
                best_step = step;
            }
        } else {
            best_d = u_min * (glane + 1);  // a dependent value to reduce
            best_j = glane;
            best_step = step;
        }
        if (MODE != 2) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                if (o < gsz) {
                    const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
                    const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                    const double os = __shfl_xor_sync(0xffffffffu, best_step, o);
                    if (od < best_d || (od == best_d && oj < best_j)) {
                        best_d = od;
                        best_j = oj;
                        best_step = os;
                    }
                }
            }
        }
        u_min = u_min + best_step + (MODE == 2 ? best_d * 1e-300 : 0.0);
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = u_min;
}

template <int OP>
__global__ void lat(double a, double* out, long long* cyc) {
    double x = a + threadIdx.x;
    bool p = false;
    const long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1000; ++i) {
        if (OP == 0) x = x + 1.0;                        // DADD
        if (OP == 1) x = trunc(x * 1.0000001);           // DMUL + FRND
        if (OP == 2) { p = x < 3.0; x = p ? x + 1.0 : x * 0.5; }  // DSETP + select
        if (OP == 3) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;  // SHFL.f64 + DADD
        if (OP == 4) x = fabs(x - 2.0) >= 1.0 ? x - 1.0 : x + 0.5;
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = x + p;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    long long h;
    const int stages = 200;
    const char* names[] = {"full stage", "reduction only", "arithmetic only", "full, ph via smem*", "full, ph via global"};
    double* gph;
    cudaMalloc(&gph, 256 * 8);
    cudaMemset(gph, 0, 256 * 8);
    for (int gsz : {16, 4}) {
        for (int mode = 0; mode < 5; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) chain<0><<<1, 32>>>(1234.5, 3.0517578125e-05, 1.0, 16.0, stages, gsz, out, cyc, gph);
                if (mode == 1) chain<1><<<1, 32>>>(1234.5, 3.0517578125e-05, 1.0, 16.0, stages, gsz, out, cyc, gph);
                if (mode == 2) chain<2><<<1, 32>>>(1234.5, 3.0517578125e-05, 1.0, 16.0, stages, gsz, out, cyc, gph);
                if (mode == 3) chain<3><<<1, 32>>>(1234.5, 3.0517578125e-05, 1.0, 16.0, stages, gsz, out, cyc, gph);
                if (mode == 4) chain<4><<<1, 32>>>(1234.5, 3.0517578125e-05, 1.0, 16.0, stages, gsz, out, cyc, gph);
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            }
            printf("gsz %2d %-16s: %7.1f cycles per stage\n", gsz, names[mode], (double)h / stages);
        }
    }
    const char* ln[] = {"DADD", "DMUL+FRND", "DSETP+select", "SHFL.f64+DADD", "fabs/DSETP/sel"};
    for (int op = 0; op < 5; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) lat<0><<<1, 32>>>(1.0, out, cyc);
            if (op == 1) lat<1><<<1, 32>>>(1.0, out, cyc);
            if (op == 2) lat<2><<<1, 32>>>(1.0, out, cyc);
            if (op == 3) lat<3><<<1, 32>>>(1.0, out, cyc);
            if (op == 4) lat<4><<<1, 32>>>(1.0, out, cyc);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-16s: %6.1f cycles per step\n", ln[op], (double)h / 1000);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
