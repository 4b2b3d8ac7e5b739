// encode.hpp / decode.hpp launch interfaces (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "cuda_check.hpp"
#include "plan_dev.cuh"

namespace msfft_b200 {

// K1+K2 (encode.cu).  smem_bytes >= max(staged taps, 256*kEncRounds*16).
void launch_encode(const DevPlan& plan, const EncTask* d_tasks, int64_t ntasks, const void* x,
                   bool x_c128, int64_t x_stride, int64_t batch, const int64_t* d_sigma,
                   double2* d_y, size_t smem_bytes, cudaStream_t stream,
                   int32_t* d_done = nullptr);
// d_done (optional, gated launches): each task adds 1 to d_done[task.m] once
// its buckets are written, or to d_done[2 iters + 1 + task.m] once its folds
// are (b > 256: the gated bucket FFT consumes them).  Layout of the gate
// words: [need iters][done iters][exit 1][fold need iters][fold done iters],
// d_done pointing at "done".

// Per-signal decode scratch, carved from shared memory when it fits,
// otherwise from a global workspace of `stride_bytes` per signal.
struct DecLayout {
    int64_t off_acc_f[2], off_acc_c[2];
    int64_t off_tone_u, off_tone_i;
    int64_t off_mag, off_order;
    int64_t off_cand_f, off_cand_v, off_cand_first, off_cand_sum, off_rot;
    int64_t off_bstart, off_blist, off_gc, off_phi, off_pcode;
    // large-size scratch (radix sorts), present when big != 0
    int64_t off_sk[2], off_sv[2], off_flag, off_nfs, sort_n;
    int64_t bytes;      // per signal
    int64_t cap, b_max, budget_max, rounds_max;  // the sizes above (checked builds)
    int32_t in_smem;
    int32_t big;        // large-size paths: sort counters live in shared memory
};

// Above these sizes the decode switches from O(n^2) rank counting to
// block-wide radix sorts (cta_sort.cuh).
constexpr int64_t kSmallRank = 1024;    // buckets (selection order, K4)
constexpr int64_t kSmallBudget = 512;   // ranked buckets (found-map merge, K6)
constexpr int64_t kSmallAcc = 2048;     // accumulated tones (K-prune, K7)
constexpr size_t kSortSmemBytes = (16 * 256 + 32) * sizeof(int);

DecLayout make_dec_layout(int64_t acc_cap, int64_t b_max, int64_t budget_max,
                          int64_t rounds_max);

// K3..K7 (decode.cu).  out_f/out_c are [batch][k]; out_count [batch].
void launch_decode(const DevPlan& plan, const DecLayout& lay, double2* d_y,
                   const int64_t* d_sigma, const int64_t* d_sigma_inv, int64_t batch,
                   unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                   int64_t* d_out_count, int32_t* d_err, cudaStream_t stream,
                   int64_t* tr_bucket = nullptr, int64_t* tr_f = nullptr,
                   double2* tr_v = nullptr);

// The decode as a programmatic dependent launch behind an encode launched
// with d_done: it starts while the encode runs and waits, per iteration m,
// until d_done[m] reaches d_need[m] (that iteration's encode tasks).
// d_done: the gate words above (zero between calls); the last decode CTA
// out waits for every producer and resets them.
void launch_decode_gated(const DevPlan& plan, const DecLayout& lay, double2* d_y,
                         const int64_t* d_sigma, const int64_t* d_sigma_inv, int64_t batch,
                         unsigned char* d_work, int64_t* d_out_f, double2* d_out_c,
                         int64_t* d_out_count, int32_t* d_err, const int32_t* d_need,
                         int32_t* d_done, cudaStream_t stream);

// Error flags raised by the decode (mirrors exceptions that escape sfft4).
enum : int32_t { kDecErrNone = 0, kDecErrPhaseZero = 1, kDecErrRounds = 2 };

}  // namespace msfft_b200
