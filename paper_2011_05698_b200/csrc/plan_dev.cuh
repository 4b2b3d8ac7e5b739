// plan_dev.cuh -- the per-transform plan as the kernels see it.
//
// HBM layout of one batch:
//   x      [batch][x_stride] complex64 (float2) or complex128 (double2)
//   sigma  [batch][iters]    int64      (sigma_m, drawn on the host)
//   y      [batch][values_per_signal] double2, iteration-major then
//          round-major: y[s][yoff_m + r*b_m + j] is bucket j of round r
//          of iteration m (BucketSet::values, proj/include/msfft/bucketize.hpp:24-30)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace msfft_b200 {

constexpr int kMaxIters = 40;
constexpr int kMaxTaus = 1024;
constexpr int kEncRounds = 8;       // rounds fused into one gather pass
constexpr int kEncThreads = 256;    // encode CTA size
constexpr int kMaxPack = 8;         // sub-tasks of a packed encode item
constexpr int kDecThreads = 256;    // decode CTA size
constexpr int kMaxStageTable = 64;  // locate stages the decode keeps in shared memory
constexpr int kMaxStages = 4096;    // longest precomputed locate stage table

struct DevIter {
    // Locate region lengths of every stage, len_0 = L, len_{k+1} =
    // len_k*(q+1)/l, and block widths len_k/l (locate.cpp:64, 78), computed on
    // the host with the same IEEE operations; nstage_tab = stages the locate
    // loop runs (len_k > 1 + 1e-9), or -1 if it exceeds kMaxStages.
    // (device arrays owned by the plan: nstage_tab + 1 lengths, nstage_tab
    // block widths)
    const double* stage_len;
    const double* stage_blk;
    int32_t nstage_tab, pad0_;
    int64_t b, l_width, w, h;
    int64_t budget, k_m;
    int64_t yoff;            // offset of round 0 of this iteration in a signal's y block
    int64_t gmax;            // response table covers d in [-gmax, gmax]
    const double* taps;      // w + 1 doubles (zero pad)
    const double* ghat;      // 2*gmax + 1 doubles, index d + gmax
    const double2* tw;       // b/2 forward twiddles for the b-point transform
    int32_t log2b, nrounds;
    int32_t tau_off;         // first tau of this iteration in DevPlan::taus
    int32_t taps_in_smem;    // taps staged in shared memory by a TMA bulk copy
};

struct DevPlan {
    int64_t n, k, l;
    // the samples this encode may read: x holds x[x_lo, x_hi) (index-range
    // sharding of one signal across GPUs; [0, n) otherwise)
    int64_t x_lo, x_hi;
    double q, inv_n;
    int64_t values_per_signal, acc_cap;
    int32_t iters;
    // 1: x rows hold the compact samples of sparse host ingest (ingest.hpp):
    // the sample of t' is x[task.seg_cpos[seg] + (t' - seg_lo[seg])]
    int32_t x_compact;
    int64_t x_row;  // compact mode: samples per compact row (bounds checks)
    DevIter it[kMaxIters];
    int64_t taus[kMaxTaus];
};

// One CTA of the encode kernel.
struct EncTask {
    int32_t m;               // iteration
    int32_t r0, nr;          // rounds [r0, r0 + nr) of that iteration
    int32_t fused;           // 1: CTA holds all b lanes -> fused b-point FFT
    int64_t sig0;            // first signal
    int32_t nsig;            // signals handled (fused: 256/b)
    int32_t lane0;           // first residue class (non-fused: 256-wide slice)
    int32_t nseg;
    // packed tasks (validating fused kernel, fused.cu): this sub-task's
    // threads are [tid0, tid0 + b) of the CTA; its taps sit at byte taps_off
    // of the shared staging area (-1: read from global) and are copied there
    // by this sub-task if stage_taps; its b-point arrays at double2 f_off
    int32_t tid0;
    int32_t taps_off, f_off, stage_taps, pad_;
    int32_t seg_lo[kEncRounds], seg_hi[kEncRounds];  // merged t' intervals
    int32_t seg_cpos[kEncRounds];  // compact position of seg_lo (sparse ingest)
};

}  // namespace msfft_b200

namespace msfft_b200 {
static_assert(sizeof(DevPlan) <= 31 * 1024, "DevPlan must fit the 32 KB kernel-parameter limit");
}  // namespace msfft_b200
