// ingest.hpp -- sparse host ingest: move to the device only the samples the
// transform reads.
//
// The reference reads x[sigma_m * (t - tau) mod n] for the taps t of every
// round (bucketize_fn, proj/include/msfft/bucketize.hpp:63-86): per signal
// about 2.5% of the samples at C4.  The t' = t - tau intervals of an
// iteration depend only on the plan (w_m, tau plan), so the samples of one
// signal can be listed as
//     compact[base_m + pos] = x[sigma_m * t' mod n],  t' ascending over the
//     union U_m of the rounds' intervals,
// and gathered on the host (random reads, many threads, software prefetch)
// into pinned staging; the H2D copy then carries |compact| samples instead of
// n, and the encode reads them coalesced (EncTask::seg_cpos).  Summation
// order is unchanged, so the result is bit-identical to the dense path.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "host_plan.hpp"

namespace msfft_b200 {

struct IngestMap {
    std::vector<std::vector<std::pair<int64_t, int64_t>>> uni;  // per iteration, ascending
    std::vector<std::vector<int64_t>> pos;  // compact position of each interval's first t'
    int64_t per_signal = 0;                 // compact samples per signal
    // compact position of t' (inside U_m)
    int64_t position(int m, int64_t t) const;
};

IngestMap make_ingest_map(const SchedulePlan& plan);

// A fixed set of worker threads; run() executes fn(0..items-1) on the
// workers and the calling thread and returns when all items are done.
class HostPool {
public:
    explicit HostPool(int threads);
    ~HostPool();
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;
    int threads() const { return static_cast<int>(workers_.size()) + 1; }
    void run(int64_t items, const std::function<void(int64_t)>& fn);

private:
    void work();
    void drain();
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    std::atomic<const std::function<void(int64_t)>*> fn_{nullptr};
    std::atomic<int64_t> items_{0};
    std::atomic<int64_t> next_{0};
    int active_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// Threads for host ingest: MSFFT_INGEST_THREADS, else the hardware threads.
int ingest_threads();

// Gathers the compact samples of `count` signals (rows x + s * x_stride) into
// out[s * per_signal ..]; sigma is [count][iterations].  elem_bytes 8
// (complex64) or 16 (complex128).  If `validate`, also scans every sample of
// rows [scan_from, count) and returns true iff a non-finite value was seen
// (rows below scan_from are validated elsewhere, e.g. on the device).
bool gather_compact(HostPool& pool, const IngestMap& map, int64_t n, int iterations,
                    const void* x, int64_t x_stride, int elem_bytes, int64_t count,
                    const int64_t* sigma, void* out, bool validate, int64_t scan_from = 0);

}  // namespace msfft_b200
