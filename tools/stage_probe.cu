// stage_probe.cu -- cycles per locate stage (decode K5, locate_step,
// proj/src/locate.cpp:63-81) for variants of the stage body: 8 lane groups
// of 16 (one bucket each), 64 dependent stages, clock64 on lane 0.
//   V0 the decode's loop form (int64 j loop, I2F per stage, 3-shuffle argmin)
//   V1 candidate offset (j + 0.5) hoisted out of the stage loop
//   V2 V1 without the argmin (cost of the shuffle tree)
//   V3 V1 with a min-then-ballot argmin (2 shuffles per level + one vote)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_2011_05698_b200/csrc -o tools/stage_probe tools/stage_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace msfft_b200;

constexpr int kStages = 64;

template <int V>
__global__ void probe(double u0, int64_t tau0, int64_t n, double inv_n, double phi0, double q,
                      double* out, long long* cycles) {
    const int lane = threadIdx.x & 31;
    const int gsz = 16, lcfg = 16;
    const int glane = lane & (gsz - 1);
    double u_min = u0 + (threadIdx.x >> 4);
    double rblk = 1024.0;
    const double jh = static_cast<double>(glane) + 0.5;
    long long t0 = clock64();
    for (int stage = 0; stage < kStages; ++stage) {
        const int64_t tau = tau0 + stage;
        const double phi = phi0 + 1e-3 * stage;
        double best_d = INFINITY;
        int best_j = 0x7fffffff;
        if (V == 0) {
            for (int64_t j = glane; j < lcfg; j += gsz) {
                const double center = u_min + (static_cast<double>(j) + 0.5) * rblk;
                const double d = circular_phase_distance(position_phase(center, tau, n, inv_n), phi);
                if (d < best_d) {
                    best_d = d;
                    best_j = static_cast<int>(j);
                }
            }
        } else {
            const double center = u_min + jh * rblk;
            const double d = circular_phase_distance(position_phase(center, tau, n, inv_n), phi);
            if (d < best_d) {
                best_d = d;
                best_j = glane;
            }
        }
        if (V == 0 || V == 1) {
            for (int o = gsz >> 1; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
                const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                if (od < best_d || (od == best_d && oj < best_j)) {
                    best_d = od;
                    best_j = oj;
                }
            }
        } else if (V == 3) {
            double m = best_d;  // NaN-free here: +inf for "no candidate"
            for (int o = gsz >> 1; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, m, o);
                m = od < m ? od : m;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, best_d == m);
            const unsigned grp = (hit >> (lane & ~(gsz - 1))) & ((1u << gsz) - 1);
            best_j = grp ? __ffs(grp) - 1 : 0x7fffffff;
        }
        if (best_j == 0x7fffffff) best_j = 0;
        u_min = u_min + (static_cast<double>(best_j) - q / 2.0) * rblk;
        rblk = rblk * 0.125;
        if (rblk < 1.0) rblk = 1024.0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cycles = t1 - t0;
    out[threadIdx.x] = u_min;
}

template <int V>
void run(const char* name, double* out, long long* cyc) {
    const int64_t n = int64_t{1} << 22;
    for (int rep = 0; rep < 3; ++rep) {
        probe<V><<<1, 128>>>(12345.5, 4096, n, 1.0 / n, 1.25, 1.0, out, cyc);
        cudaDeviceSynchronize();
    }
    long long h = 0;
    double o[128];
    cudaMemcpy(&h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    printf("%-44s %7.1f cycles/stage   (u_min lane0 %.6f)\n", name, double(h) / kStages, o[0]);
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 128 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    run<0>("V0 decode loop form", out, cyc);
    run<1>("V1 hoisted j + 0.5", out, cyc);
    run<2>("V2 V1 without argmin", out, cyc);
    run<3>("V3 V1 with min + ballot argmin", out, cyc);
    return 0;
}
