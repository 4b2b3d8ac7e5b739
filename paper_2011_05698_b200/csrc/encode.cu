// encode.cu -- K1+K2 as a standalone launch: one encode task per CTA (the
// task list covers every round of every iteration of the whole batch).
// The task body is encode_body.cuh.  Compiled with --fmad=false.
#include <cuda_runtime.h>

#include "encode.hpp"

#ifdef MSFFT_TIMELINE
// diagnostic build only: per encode CTA {start ns, end ns, m}
__device__ unsigned long long g_enc_tl[8192][6];
extern "C" int msfft_debug_enc_timeline(void* dst, long long n) {
    if (n > 8192) n = 8192;
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_enc_tl, n * 48));
}
__device__ __forceinline__ unsigned long long enc_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// per gather batch of thread 0 of the first 64 CTAs: clock64
__device__ long long g_enc_batch[64][64];
__device__ int g_enc_nb[64];
extern "C" int msfft_debug_enc_batches(void* dst, void* nb) {
    int rc = static_cast<int>(cudaMemcpyFromSymbol(dst, g_enc_batch, sizeof(g_enc_batch)));
    return rc ? rc : static_cast<int>(cudaMemcpyFromSymbol(nb, g_enc_nb, sizeof(g_enc_nb)));
}
#define ENC_TL_BATCH()                                                         \
    do {                                                                       \
        if (threadIdx.x == 0 && blockIdx.x < 64) {                             \
            const int i_ = g_enc_nb[blockIdx.x];                               \
            if (i_ < 64) g_enc_batch[blockIdx.x][i_] = clock64();              \
            g_enc_nb[blockIdx.x] = i_ + 1;                                     \
        }                                                                      \
    } while (0)
// encode_body.cuh marks: 3 taps staged, 4 gather done, 5 epilogue done
#define ENC_TL_MARK(i)                                                      \
    do {                                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 8192) g_enc_tl[blockIdx.x][i] = enc_now(); \
    } while (0)
#endif
#include "encode_body.cuh"



namespace msfft_b200 {

namespace {

template <class T>
__global__ void __launch_bounds__(kEncThreads, 2)
encode_kernel(const __grid_constant__ DevPlan plan, const EncTask* __restrict__ tasks,
              const T* __restrict__ x, int64_t x_stride, int64_t batch,
              const int64_t* __restrict__ sigma, double2* __restrict__ y,
              int32_t* __restrict__ done) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t bar;
    // a gated decode launched behind this grid (programmatic dependent
    // launch) may be scheduled as soon as every task is resident: it waits
    // per iteration on `done`, not on this grid's completion
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    encode_barrier_init(&bar);
    uint32_t phase = 0;
    const EncTask& t = tasks[blockIdx.x];
#ifdef MSFFT_TIMELINE
    const unsigned long long t_start = enc_now();
    if (threadIdx.x == 0 && blockIdx.x < 64) g_enc_nb[blockIdx.x] = 0;
#endif
    encode_task(plan, t, x, x_stride, batch, sigma, y, smem_raw, &bar, phase);
    if (done) {  // release this task's buckets (or folds) to the gated consumer
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            // b <= 256: the decode waits on done[m]; b > 256: the folds go to
            // the gated bucket FFT, which waits on done[2 iters + 1 + m]
            const bool folds = plan.it[t.m].b > kEncThreads;
            atomicAdd(&done[folds ? 2 * plan.iters + 1 + t.m : t.m], 1);
        }
    }
#ifdef MSFFT_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 8192) {
        g_enc_tl[blockIdx.x][0] = t_start;
        g_enc_tl[blockIdx.x][1] = enc_now();
        g_enc_tl[blockIdx.x][2] = t.m;
    }
#endif
}

}  // namespace

void launch_encode(const DevPlan& plan, const EncTask* d_tasks, int64_t ntasks, const void* x,
                   bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                   double2* d_y, size_t smem_bytes, cudaStream_t stream, int32_t* d_done) {
    if (ntasks <= 0) return;
    if (x_c128) {
        auto k = encode_kernel<double2>;
        smem_attr(k, smem_bytes);
        k<<<static_cast<unsigned>(ntasks), kEncThreads, smem_bytes, stream>>>(
            plan, d_tasks, static_cast<const double2*>(x), x_stride, batch, d_sigma, d_y, d_done);
    } else {
        auto k = encode_kernel<float2>;
        smem_attr(k, smem_bytes);
        k<<<static_cast<unsigned>(ntasks), kEncThreads, smem_bytes, stream>>>(
            plan, d_tasks, static_cast<const float2*>(x), x_stride, batch, d_sigma, d_y, d_done);
    }
    MSFFT_LAUNCH_CHECK("encode_kernel");
}

}  // namespace msfft_b200
