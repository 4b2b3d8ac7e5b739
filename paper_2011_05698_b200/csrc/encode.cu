// encode.cu -- K1+K2 as a standalone launch: one encode task per CTA (the
// task list covers every round of every iteration of the whole batch).
// The task body is encode_body.cuh.  Compiled with --fmad=false.
#include <cuda_runtime.h>

#include "encode.hpp"
#include "encode_body.cuh"

namespace msfft_b200 {

namespace {

template <class T>
__global__ void __launch_bounds__(kEncThreads, 2)
encode_kernel(const __grid_constant__ DevPlan plan, const EncTask* __restrict__ tasks,
              const T* __restrict__ x, int64_t x_stride, int64_t batch,
              const int64_t* __restrict__ sigma, double2* __restrict__ y) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    encode_barrier_init(&bar);
    uint32_t phase = 0;
    encode_task(plan, tasks[blockIdx.x], x, x_stride, batch, sigma, y, smem_raw, &bar, phase);
}

}  // namespace

void launch_encode(const DevPlan& plan, const EncTask* d_tasks, int64_t ntasks, const void* x,
                   bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                   double2* d_y, size_t smem_bytes, cudaStream_t stream) {
    if (ntasks <= 0) return;
    if (x_c128) {
        auto k = encode_kernel<double2>;
        MSFFT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        k<<<static_cast<unsigned>(ntasks), kEncThreads, smem_bytes, stream>>>(
            plan, d_tasks, static_cast<const double2*>(x), x_stride, batch, d_sigma, d_y);
    } else {
        auto k = encode_kernel<float2>;
        MSFFT_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        k<<<static_cast<unsigned>(ntasks), kEncThreads, smem_bytes, stream>>>(
            plan, d_tasks, static_cast<const float2*>(x), x_stride, batch, d_sigma, d_y);
    }
    MSFFT_LAUNCH_CHECK("encode_kernel");
}

}  // namespace msfft_b200
