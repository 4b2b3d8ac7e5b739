// barrier_probe.cu -- what a phase boundary costs on this B200: a dependent
// kernel boundary inside a CUDA graph (plain edges / programmatic edges)
// against a grid barrier inside one persistent kernel.  Each phase reads a
// word the previous phase wrote (so the dependency is real) and writes one.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/barrier_probe tools/barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));       \
            return 1;                                                               \
        }                                                                           \
    } while (0)

__global__ void phase_kernel(int* buf, int i, int pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int v = buf[(i & 1) * 4096 + blockIdx.x];
    if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) buf[((i + 1) & 1) * 4096 + blockIdx.x] = v + 1;
}

__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen,
                                             unsigned nblocks, unsigned& my_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned g = my_gen;
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicExch(const_cast<unsigned*>(gen), g + 1);
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    ++my_gen;
    __syncthreads();
}

// red.release + ld.acquire polling variant
__device__ __forceinline__ void grid_barrier2(unsigned* count, unsigned nblocks, unsigned& target) {
    __syncthreads();
    target += nblocks;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__global__ void persistent_kernel(int* buf, int phases, unsigned* count, unsigned* gen, int mode) {
    unsigned my_gen = 0, target = 0;
    for (int i = 0; i < phases; ++i) {
        const int v = buf[(i & 1) * 4096 + blockIdx.x];
        if (threadIdx.x == 0) buf[((i + 1) & 1) * 4096 + blockIdx.x] = v + 1;
        if (mode == 0)
            grid_barrier(count, gen, gridDim.x, my_gen);
        else
            grid_barrier2(count + 1, gridDim.x, target);
    }
}

int main() {
    int* buf;
    unsigned *count, *gen;
    CK(cudaMalloc(&buf, 8192 * sizeof(int)));
    CK(cudaMalloc(&count, 64));
    CK(cudaMalloc(&gen, 64));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int N = 300;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int blocks : {1, 8, sms, 2 * sms}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
            for (int i = 0; i < N; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(256);
                cfg.stream = st;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = pdl;
                CK(cudaLaunchKernelEx(&cfg, phase_kernel, buf, i, pdl));
            }
            CK(cudaStreamEndCapture(st, &g));
            cudaGraphExec_t ge;
            CK(cudaGraphInstantiate(&ge, g, 0));
            float best = 1e30f;
            for (int rep = 0; rep < 6; ++rep) {
                CK(cudaEventRecord(e0, st));
                CK(cudaGraphLaunch(ge, st));
                CK(cudaEventRecord(e1, st));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (rep > 0 && ms < best) best = ms;
            }
            printf("graph  blocks=%4d pdl=%d : %.3f us per kernel boundary\n", blocks, pdl,
                   best * 1000.f / N);
            CK(cudaGraphExecDestroy(ge));
            CK(cudaGraphDestroy(g));
        }
    }
    for (int mode = 0; mode < 2; ++mode)
        for (int blocks : {sms, 2 * sms}) {
            float best = 1e30f;
            for (int rep = 0; rep < 6; ++rep) {
                CK(cudaMemsetAsync(count, 0, 64, st));
                CK(cudaMemsetAsync(gen, 0, 64, st));
                int phases = N;
                void* args[] = {&buf, &phases, &count, &gen, &mode};
                CK(cudaEventRecord(e0, st));
                CK(cudaLaunchCooperativeKernel((void*)persistent_kernel, dim3(blocks), dim3(256),
                                               args, 0, st));
                CK(cudaEventRecord(e1, st));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                if (rep > 0 && ms < best) best = ms;
            }
            printf("persistent mode=%d blocks=%4d : %.3f us per grid barrier\n", mode, blocks,
                   best * 1000.f / N);
        }
    return 0;
}
