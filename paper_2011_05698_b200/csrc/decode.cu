// decode.cu -- K3..K7 as a standalone launch: one CTA per signal (the body
// is decode_body.cuh).  Compiled with --fmad=false.
#include <cuda_runtime.h>

#include "decode_body.cuh"

#ifndef MSFFT_DEC_MINB
#define MSFFT_DEC_MINB 3  // 3 CTAs per SM: <= 85 registers, no spills
#endif

namespace msfft_b200 {

namespace {

__global__ void __launch_bounds__(kDecThreads, MSFFT_DEC_MINB)
decode_kernel(const __grid_constant__ DevPlan plan, DecLayout lay, DecArgs args, int64_t batch,
              unsigned char* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ DecShared sh;
    const int64_t s = blockIdx.x;
    // err[1]: the validation pass found a non-finite sample; the call will
    // throw (ComplexSignal::validate) so there is nothing to decode.
    if (s >= batch || args.err[1] != 0) return;
    decode_signal<kDecThreads>(plan, lay, args, s, lay.in_smem ? dsm : work + s * lay.bytes, sh,
                               lay.big ? reinterpret_cast<int*>(dsm) : nullptr);
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
    MSFFT_CUDA(cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    DecArgs args{d_y, d_sigma, d_sigma_inv, d_out_f, d_out_c, d_out_count, d_err,
                 tr_bucket, tr_f, tr_v};
    decode_kernel<<<static_cast<unsigned>(batch), kDecThreads, smem, stream>>>(
        plan, lay, args, batch, d_work);
    MSFFT_LAUNCH_CHECK("decode_kernel");
}

}  // namespace msfft_b200
