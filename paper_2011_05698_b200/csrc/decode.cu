// decode.cu -- K3..K7 as a standalone launch: one CTA per signal (the body
// is decode_body.cuh).  Compiled with --fmad=false.
#include <cuda_runtime.h>

#ifdef MSFFT_TIMELINE
// diagnostic build only: per decode CTA (< 64) {start, gate m passed (m < 30), end} ns
__device__ unsigned long long g_dec_tl[64][32];
__device__ __forceinline__ unsigned long long dec_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DEC_TL_MARK(m)                                                      \
    do {                                                                    \
        if (threadIdx.x == 0 && blockIdx.x < 64 && (m) < 30)                \
            g_dec_tl[blockIdx.x][1 + (m)] = dec_now();                      \
    } while (0)
#endif
#include "decode_body.cuh"
#ifdef MSFFT_TIMELINE
extern "C" int msfft_debug_dec_timeline(void* dst, long long n) {
    if (n > 64) n = 64;
    return static_cast<int>(cudaMemcpyFromSymbol(dst, g_dec_tl, n * 32 * 8));
}
#endif

#ifndef MSFFT_DEC_MINB
#define MSFFT_DEC_MINB 3  // 3 CTAs per SM: <= 85 registers, no spills
#endif

namespace msfft_b200 {

namespace {

// kMinB: CTAs per SM the register budget is sized for -- MSFFT_DEC_MINB for
// batches (one CTA per signal fills the GPU), 1 for the gated small-batch
// launch (every register for the latency chains)
template <int kMinB>
__global__ void __launch_bounds__(kDecThreads, kMinB)
decode_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, DecArgs args, int64_t batch,
              unsigned char* __restrict__ work, int32_t* __restrict__ exit_count) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ DecShared sh;
    const int64_t s = blockIdx.x;
#ifdef MSFFT_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 64) g_dec_tl[blockIdx.x][0] = dec_now();
#endif
    // err[1]: the validation pass found a non-finite sample; the call will
    // throw (ComplexSignal::validate) so there is nothing to decode.
    if (s < batch && args.err[1] == 0) {
        // two inlined copies: with the scratch in shared memory the compiler
        // sees every scratch pointer derive from `dsm` and emits LDS/STS
        // (~30 cycles) instead of generic loads (~66) on the decode's chains
        if (lay.in_smem)
            decode_signal<kDecThreads>(plan, lay, args, s, dsm, sh,
                                       lay.big ? reinterpret_cast<int*>(dsm) : nullptr);
        else
            decode_signal<kDecThreads>(plan, lay, args, s, work + s * lay.bytes, sh,
                                       lay.big ? reinterpret_cast<int*>(dsm) : nullptr);
    }
#ifdef MSFFT_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 64) g_dec_tl[blockIdx.x][31] = dec_now();
#endif
    if (!exit_count) return;
    // gated launch: the last CTA out waits for every encode task (a skipped
    // decode did not) and resets the gate counters for the next call
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(exit_count, 1) == static_cast<int>(gridDim.x) - 1) {
            int32_t* done = const_cast<int32_t*>(args.gate_done);
            int32_t* fold_done = exit_count + 1 + plan.iters;  // gated bucket FFT inputs
            for (int m = 0; m < plan.iters; ++m) {
                while (load_acquire(&done[m]) < args.gate_need[m]) __nanosleep(64);
                done[m] = 0;
                fold_done[m] = 0;  // its FFT CTAs (counted in done[m]) read it already
            }
            *exit_count = 0;
            __threadfence();
        }
    }
}

}  // namespace

DecLayout make_dec_layout(int64_t acc_cap, int64_t b_max, int64_t budget_max,
                          int64_t rounds_max) {
    DecLayout L{};
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        const int64_t o = off;
        off += (bytes + 15) & ~int64_t{15};
        return o;
    };
    const int64_t cap = std::max<int64_t>(acc_cap, 1);
    L.cap = cap;
    L.b_max = b_max;
    L.budget_max = budget_max;
    L.rounds_max = rounds_max;
    for (int p = 0; p < 2; ++p) {
        L.off_acc_f[p] = take(cap * 8);
        L.off_acc_c[p] = take(cap * 16);
    }
    L.off_tone_u = take(cap * 8);
    L.off_tone_i = take(std::max(cap, b_max) * 8);
    L.off_mag = take(std::max(cap, b_max) * 8);
    L.off_order = take(b_max * 4);
    L.off_cand_f = take(budget_max * 8);
    L.off_cand_v = take(budget_max * 16);
    L.off_cand_first = take(budget_max * 4);
    L.off_cand_sum = take(budget_max * 16);
    // rotations per (tone, round); reused for the staged rounds of the ranked
    // buckets (budget_max <= cap)
    L.off_rot = take(std::max(cap, budget_max) * rounds_max * 16);
    L.off_bstart = take((b_max + 1) * 4);
    L.off_blist = take(cap * 4);
    L.off_gc = take(cap * 3 * 16);
    L.off_phi = take(budget_max * rounds_max * 8);
    L.off_pcode = take(budget_max * rounds_max * 4);
    // large sizes (C3/C5): radix-sort scratch replaces the O(n^2) ranks
    L.big = (b_max > kSmallRank || budget_max > kSmallBudget || cap > kSmallAcc) ? 1 : 0;
    if (L.big) {
        const int64_t ncap = std::max(std::max(b_max, budget_max), cap);
        L.sort_n = ncap;
        for (int p = 0; p < 2; ++p) {
            L.off_sk[p] = take(ncap * 8);
            L.off_sv[p] = take(ncap * 4);
        }
        L.off_flag = take((ncap + kDecThreads) * 4);
        L.off_nfs = take(ncap * 8);
    }
    L.bytes = off;
    L.in_smem = (!L.big && off <= 96 * 1024) ? 1 : 0;
    return L;
}

void launch_decode(const DevPlan& plan, const DecLayout& lay, double2* d_y,
                   const int64_t* d_sigma, const int64_t* d_sigma_inv, int64_t batch,
                   unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                   int64_t* d_out_count, int32_t* d_err, cudaStream_t stream,
                   int64_t* tr_bucket, int64_t* tr_f, double2* tr_v) {
    if (batch <= 0) return;
    const size_t smem =
        lay.in_smem ? static_cast<size_t>(lay.bytes) : (lay.big ? kSortSmemBytes : 0);
    smem_attr(decode_kernel<MSFFT_DEC_MINB>, smem);
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 tr_bucket, tr_f, tr_v};
    decode_kernel<MSFFT_DEC_MINB><<<static_cast<unsigned>(batch), kDecThreads, smem, stream>>>(
        plan, lay, args, batch, d_work, nullptr);
    MSFFT_LAUNCH_CHECK("decode_kernel");
}

void launch_decode_gated(const DevPlan& plan, const DecLayout& lay, double2* d_y,
                         const int64_t* d_sigma, const int64_t* d_sigma_inv, int64_t batch,
                         unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                         int64_t* d_out_count, int32_t* d_err, const int32_t* d_need,
                         int32_t* d_done, cudaStream_t stream) {
    if (batch <= 0) return;
    const size_t smem =
        lay.in_smem ? static_cast<size_t>(lay.bytes) : (lay.big ? kSortSmemBytes : 0);
#ifndef MSFFT_GATED_MINB
#define MSFFT_GATED_MINB 1
#endif
    auto kern = decode_kernel<MSFFT_GATED_MINB>;
    smem_attr(kern, smem);
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 nullptr, nullptr, nullptr, d_done, d_need};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(batch));
    cfg.blockDim = dim3(kDecThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int32_t* exit_count = d_done + plan.iters;
    MSFFT_CUDA(cudaLaunchKernelEx(&cfg, kern, plan, lay, args, batch, d_work, exit_count));
    MSFFT_LAUNCH_CHECK("decode_kernel (gated)");
}

}  // namespace msfft_b200
