// wide_decode.hpp -- K3..K7 for ONE large signal spread over the whole GPU.
//
// decode_kernel runs a signal's decode in one CTA: right for batches (C4:
// 1024 independent decodes fill the GPU) but a single large signal (C5:
// N=2^27, K=10^4, b up to 65536, ~16k accumulated tones) then runs on one SM.
// The wide decode issues every phase of an iteration as grid-wide kernels
// with the same arithmetic in the same order, so results are bit-identical
// to decode_kernel:
//   K3  tones (u, home bucket, G*c) and their rotations; an event list
//       (target bucket, tone) built by counting sort and ordered by tone per
//       bucket; one warp per (round, bucket) sums the predictions in
//       ascending-f order and subtracts;
//   K4  |y0| keys, device-side radix select of the budget-th largest,
//       ordered compaction, all-pairs rank (ties: lower bucket) -> order;
//   K5  staged round values and y0/y_tau phases per (rank, stage), then one
//       lane group per ranked bucket for the multiscale locate + estimate;
//   K6  accepted candidates ranked by (f, rank), found-map sums in rank
//       order, merge into the ascending accumulated list by binary search;
//   K7  radix select of the K-th largest |c| and ordered compaction in f.
// Data-dependent sizes (accumulated count, new tones) stay on the device: the
// host issues a fixed kernel sequence sized for the plan's maxima.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <tuple>

#include "cuda_check.hpp"
#include "plan_dev.cuh"

namespace msfft_b200 {

class WideDecoder {
public:
    WideDecoder(const DevPlan& plan, int64_t acc_cap, int64_t b_max, int64_t budget_max,
                int64_t rounds_max);
    // Decodes one signal: y = its bucket values (consumed), sigma / sigma_inv
    // its per-iteration plan (device), outputs out_f[k], out_c[k],
    // *out_count; decode errors go to err[0] (as decode_kernel).
    void run(double2* y, const int64_t* sigma, const int64_t* sigma_inv, int64_t* out_f,
             double2* out_c, int64_t* out_count, int32_t* err, cudaStream_t st) {
        run_range(y, sigma, sigma_inv, out_f, out_c, out_count, err, st, 0, hplan_.iters);
    }
    // Iterations [m0, m1) only (m1 == iters also runs K7): consecutive ranges
    // on one stream make one decode, so a caller can start the decode of the
    // early iterations while the later iterations are still being encoded.
    void run_range(double2* y, const int64_t* sigma, const int64_t* sigma_inv, int64_t* out_f,
                   double2* out_c, int64_t* out_count, int32_t* err, cudaStream_t st, int m0,
                   int m1);

    ~WideDecoder();

private:
    // the fixed kernel sequence of one decode (K7 writes out_f/out_c/out_count)
    void enqueue(double2* y, const int64_t* sigma, const int64_t* sigma_inv, int32_t* err,
                 int64_t* out_f, double2* out_c, int64_t* out_count, cudaStream_t st, int m0,
                 int m1);
    void select_kth(const uint64_t* key, int64_t n_max, const int32_t* n_dev, cudaStream_t st);
    void compact_selected(const uint64_t* key, int64_t n_max, const int32_t* n_dev,
                          int32_t* out_idx, cudaStream_t st);

    DevPlan hplan_;
    DeviceBuffer<DevPlan> dplan_;
    int64_t acc_cap_, b_max_, budget_max_, rounds_max_;
    // state
    DeviceBuffer<int64_t> acc_f_[2];
    DeviceBuffer<double2> acc_c_[2];
    DeviceBuffer<int32_t> scal_;  // [0] acc_n, [1] new_n, [2] kth, [3] need_eq, [4..] misc
    DeviceBuffer<uint64_t> sel_;  // [0] prefix, [1] mask, [2] remaining
    DeviceBuffer<double> thr_;
    // K3
    DeviceBuffer<int64_t> tone_u_, tone_i_;
    DeviceBuffer<double2> gc_, rot_;
    DeviceBuffer<int32_t> cnt_, start_, cursor_, ev_, ev2_;
    DeviceBuffer<int32_t> long_;  // {count, buckets...} of event segments > kLongSeg
    // K4 / K7
    DeviceBuffer<uint64_t> key_;
    DeviceBuffer<uint32_t> hist_;
    DeviceBuffer<int32_t> cctl_, sel_idx_, order_;
    DeviceBuffer<unsigned long long> cpub_;
    DeviceBuffer<double> mag_;
    // K5 / K6
    DeviceBuffer<double2> yr_, cand_v_, cand_sum_;
    DeviceBuffer<double> phi_;
    DeviceBuffer<int32_t> pcode_, pos_, byf_, newflag_, newpos_, hit_;
    DeviceBuffer<int64_t> cand_f_, newf_;
    DeviceBuffer<int32_t> f6cnt_, f6cur_, f6start_;  // K6 bucket sort of large budgets
    // outputs, copied to the caller's buffers after the graph
    // one instantiated CUDA graph per (y, sigma, sigma_inv, err) tuple: the
    // ~40 launches per iteration replay without per-launch host overhead
    using GraphKey = std::tuple<const void*, const void*, const void*, const void*, const void*,
                                const void*, const void*, int, int>;
    std::map<GraphKey, cudaGraphExec_t> graphs_;
    int64_t k6_stage_cap_ = 0;  // k6_small: accumulated f staged in shared memory
    bool use_graphs_ = true;  // MSFFT_WIDE_GRAPH=0 launches eagerly
    bool pdl_ = true;         // MSFFT_WIDE_PDL=0: plain stream order between the kernels
};

}  // namespace msfft_b200
