// fused.cu -- one persistent launch that runs the encode (K1+K2) and the
// decode (K3..K7) of a whole batch, so the HBM-bound gather and the
// issue-bound decode share every SM instead of running back to back.
//
// CTAs pull work items from a global ticket counter.  The item list is
// E(c0) E(c1) D(c0) E(c2) D(c1) ... D(c_last): E = the encode tasks of a
// chunk of signals, D = one decode per signal of a chunk.  A decode item waits
// until its chunk's encode-completion counter reaches the chunk's task count.
// Every encode item with a smaller ticket is already held by a running CTA
// and never waits, so the spin always terminates (no deadlock), and the
// encode->decode hand-off follows the threadfence-reduction pattern
// (producer: stores, __syncthreads, __threadfence, atomicAdd; consumer: spin
// on the counter, __threadfence, __syncthreads).  Compiled with --fmad=false.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "decode_body.cuh"
#include "encode_body.cuh"
#include "fused.hpp"

#ifndef MSFFT_FUSED_MINB
#define MSFFT_FUSED_MINB 2
#endif

#ifdef MSFFT_TIMELINE
// diagnostic build only: per item {start ns, end ns, smid << 48 | m << 40 | code}
__device__ unsigned long long g_timeline[1 << 16][3];
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
extern "C" int msfft_debug_timeline(void* dst, long long n_items) {
    if (n_items > (1 << 16)) n_items = 1 << 16;
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_timeline, n_items * 24));
}
#endif

namespace msfft_b200 {

namespace {

template <class T>
__global__ void __launch_bounds__(kEncThreads, MSFFT_FUSED_MINB)
fused_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, DecArgs args,
             const EncTask* __restrict__ tasks, const int32_t* __restrict__ items,
             int32_t n_items, int64_t chunk, const int32_t* __restrict__ need,
             int32_t* __restrict__ done, int32_t* __restrict__ ticket, const T* __restrict__ x,
             int64_t x_stride, int64_t batch, unsigned char* __restrict__ work,
             int64_t n_counters) {
    int32_t* exit_count = ticket + n_counters - 1;  // the last counter slot
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ DecShared sh;
    __shared__ int s_item;
    static_assert(kEncThreads == kDecThreads, "fused CTA runs both bodies");
    // programmatic dependent launch: this grid reads the σ plan of the
    // kernel before it (wait), and the next launch may be scheduled as soon
    // as SM slots free up (launch_dependents); it uses other buffers
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    encode_barrier_init(&bar);
    uint32_t phase = 0;
    const bool bad_input = args.err[1] != 0;  // set by the validation pass
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(ticket, 1);
        __syncthreads();
        const int item = s_item;
        if (item >= n_items) break;
        const int32_t code = items[item];
#ifdef MSFFT_TIMELINE
        const unsigned long long tl_start = tl_now();
#endif
        if (code >= 0) {
            const EncTask& t = tasks[code];
            encode_task(plan, t, x, x_stride, batch, args.sigma, args.y, smem, &bar, phase);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                // done = counters + 1; the last counter is the exit count
                MSFFT_DCHECK((t.sig0 / chunk) * plan.iters + t.m + 2 < n_counters);
                atomicAdd(&done[(t.sig0 / chunk) * plan.iters + t.m], 1);
            }
        } else if (!bad_input) {
            // the decode waits per iteration (DecArgs::gate_*), so it can run
            // while the later iterations of its chunk are still being encoded
            const int64_t s0 = -static_cast<int64_t>(code) - 1;
            const int64_t c = s0 / chunk;
            MSFFT_DCHECK(s0 < batch && (c + 1) * plan.iters + 2 <= n_counters);
            DecArgs a = args;
            a.gate_done = done + c * plan.iters;
            a.gate_need = need + c * plan.iters;
            decode_signal<kDecThreads>(plan, lay, a, s0, lay.in_smem ? smem : work + s0 * lay.bytes,
                                       sh, nullptr);
        }
        __syncthreads();
#ifdef MSFFT_TIMELINE
        if (threadIdx.x == 0 && item < (1 << 16)) {
            unsigned smid;
            asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
            g_timeline[item][0] = tl_start;
            g_timeline[item][1] = tl_now();
            const unsigned m = code >= 0 ? static_cast<unsigned>(tasks[code].m) : 0xffu;
            g_timeline[item][2] = (static_cast<unsigned long long>(smid) << 48) |
                                  (static_cast<unsigned long long>(m) << 40) |
                                  static_cast<unsigned>(code);
        }
#endif
    }
    // the last CTA out resets this launch's counters (ticket, done, exit)
    // for the next launch that uses them, so no memset sits between launches
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(exit_count, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int64_t i = threadIdx.x; i < n_counters; i += blockDim.x) ticket[i] = 0;
        __threadfence();
    }
}

template <class T>
void launch_t(const DevPlan& plan, const DecLayout& lay, const FusedWork& fw, const T* x,
              int64_t x_stride, int64_t batch, const int64_t* d_sigma,
              const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work, int64_t* d_out_f,
              double2* d_out_c, int64_t* d_out_count, int32_t* d_err, size_t smem,
              cudaStream_t stream, bool programmatic) {
    auto k = fused_kernel<T>;
    smem_attr(k, smem);
    const int sms = sm_count();
    int per_sm = 0;
    {
        // occupancy per (device, kernel, shared memory), queried once
        static std::mutex mu;
        static std::map<std::tuple<int, const void*, size_t>, int> occ;
        int dev = 0;
        MSFFT_CUDA(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lock(mu);
        const auto key = std::make_tuple(dev, reinterpret_cast<const void*>(k), smem);
        auto it = occ.find(key);
        if (it == occ.end()) {
            MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kEncThreads, smem));
            occ[key] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    if (per_sm < 1) throw CudaError("fused_kernel: does not fit on an SM");
    const int64_t grid = std::min<int64_t>(static_cast<int64_t>(sms) * per_sm, fw.n_items);
    // counters are zero: from creation, then reset by the previous launch's
    // last CTA (a memset here would also serialise programmatic launches)
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 nullptr, nullptr, nullptr};
    if (programmatic) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(kEncThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MSFFT_CUDA(cudaLaunchKernelEx(&cfg, k, plan, lay, args, fw.tasks, fw.items, fw.n_items,
                                      fw.chunk, fw.need, fw.counters + 1, fw.counters, x, x_stride,
                                      batch, d_work, fw.n_counters));
    } else {
        k<<<static_cast<unsigned>(grid), kEncThreads, smem, stream>>>(
            plan, lay, args, fw.tasks, fw.items, fw.n_items, fw.chunk, fw.need, fw.counters + 1,
            fw.counters, x, x_stride, batch, d_work, fw.n_counters);
    }
    MSFFT_LAUNCH_CHECK("fused_kernel");
}

}  // namespace

int64_t fused_slots(bool x_c128, size_t smem_bytes) {
    int dev = 0, sms = 0, per_sm = 0;
    MSFFT_CUDA(cudaGetDevice(&dev));
    MSFFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (x_c128) {
        MSFFT_CUDA(cudaFuncSetAttribute(fused_kernel<double2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<double2>,
                                                                 kEncThreads, smem_bytes));
    } else {
        MSFFT_CUDA(cudaFuncSetAttribute(fused_kernel<float2>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem_bytes)));
        MSFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_kernel<float2>,
                                                                 kEncThreads, smem_bytes));
    }
    return static_cast<int64_t>(sms) * per_sm;
}

void launch_fused(const DevPlan& plan, const DecLayout& lay, const FusedWork& fw, const void* x,
                  bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                  const int64_t* d_sigma_inv, double2* d_y, unsigned char* d_work,
                  int64_t* d_out_f, double2* d_out_c, int64_t* d_out_count, int32_t* d_err,
                  size_t smem_bytes, cudaStream_t stream, bool programmatic) {
    if (fw.n_items <= 0) return;
    if (x_c128)
        launch_t(plan, lay, fw, static_cast<const double2*>(x), x_stride, batch, d_sigma,
                 d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                 stream, programmatic);
    else
        launch_t(plan, lay, fw, static_cast<const float2*>(x), x_stride, batch, d_sigma,
                 d_sigma_inv, d_y, d_work, d_out_f, d_out_c, d_out_count, d_err, smem_bytes,
                 stream, programmatic);
}

}  // namespace msfft_b200
