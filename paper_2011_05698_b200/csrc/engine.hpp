// engine.hpp -- host orchestration of one sfft4 plan on one B200.
//
// A Plan resolves everything that does not depend on the signal (windows,
// response tables, halving schedule, tau plans, encode task list), keeps the
// device workspaces, and executes batches:
//   [H2D chunk] -> validate -> encode (K1+K2, one launch for all rounds of all
//   iterations) -> batched FFT for b > 256 -> decode (K3..K7, one CTA per
//   signal) -> outputs.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "cuda_check.hpp"
#include "encode.hpp"
#include "fft.hpp"
#include "fused.hpp"
#include "host_plan.hpp"
#include "ingest.hpp"
#include "plan_dev.cuh"
#include "wide_decode.hpp"
#include "window.hpp"

namespace msfft_b200 {

// one interval of an iteration's t' union and its compact position
struct GatherIv {
    int32_t m, pad_;
    int64_t lo, len, cpos;
};

struct ExecOptions {
    bool x_on_device = false;
    bool out_on_device = false;
    bool assume_valid = false;
    bool stage_times = false;  // CUDA events around encode / fft / decode (or fused)
    bool force_serial = false; // separate encode and decode launches (diagnostics)
    // return after enqueueing (device input and output only): outputs are
    // complete when the stream reaches them; decode errors are raised by sync()
    bool async_call = false;
    cudaStream_t stream = nullptr;
    double* pre = nullptr;   // trace: encode output (batch must be 1, host)
    double* post = nullptr;  // trace: post-subtract values
    int64_t* sel_bucket = nullptr;  // trace: per ranked bucket (sum of budgets)
    int64_t* sel_f = nullptr;
    double* sel_value = nullptr;
};

class Plan {
public:
    Plan(int64_t n, int64_t k, int64_t l, double q, double delta, bool c128, int device);
    ~Plan();
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    const SchedulePlan& schedule() const { return sched_; }
    int device() const { return device_; }
    bool c128() const { return c128_; }

    // out_c: interleaved (re, im) doubles, [batch][k].
    void execute(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                 int64_t* out_f, double* out_c, int64_t* out_count, const ExecOptions& opt,
                 double* device_ms);

    // Split phases for index-range sharding of one signal over several GPUs
    // (DESIGN.md "Multi-GPU").  encode_values: the bucket values of every
    // round of every iteration, reading only x[x_lo, x_hi) (d_x points at
    // x_lo); samples outside contribute 0, so the partial vectors of ranks
    // holding disjoint ranges sum to the full vector.  decode_values: the
    // selection/locate/estimate of each iteration on a summed vector (d_y is
    // consumed: subtraction happens in place).  All pointers are device
    // pointers; seeds are host values.
    void encode_values(int64_t batch, const void* d_x, int64_t x_stride, int64_t x_lo,
                       int64_t x_hi, const uint64_t* seeds, double2* d_y, bool validate,
                       cudaStream_t stream);
    // Tap-range sharding of one signal (x replicated on every rank): rank
    // `part` of `parts` walks only its share of every task's t' segments
    // and writes PARTIAL bucket values of every round; the partial vectors
    // of parts 0..parts-1 sum to the full vector (bucketize is a sum over
    // taps).  Per-rank encode work is 1/parts of the transform's.  The
    // finiteness check covers the part-th slice of each signal.
    void encode_values_part(int64_t batch, const void* d_x, int64_t x_stride, int64_t part,
                            int64_t parts, const uint64_t* seeds, double2* d_y, bool validate,
                            cudaStream_t stream);
    // folds: d_y holds encode_values_part's sums, whose b > 256 iterations
    // are still folds; their bucket FFTs run first.
    void decode_values(int64_t batch, double2* d_y, const uint64_t* seeds, int64_t* d_out_f,
                       double2* d_out_c, int64_t* d_out_count, cudaStream_t stream,
                       bool folds = false);
    int64_t values_per_signal() const { return dplan_.values_per_signal; }

    int64_t launches(int64_t batch, bool validate, bool serial = false) const;

    // Waits for the plan's work on `stream` (nullptr: its own stream) and
    // raises the errors of asynchronous calls since the last sync.
    void sync(cudaStream_t stream);

    // compact samples per signal moved by sparse host ingest (0 if the plan
    // uses the dense H2D path for host inputs)
    int64_t ingest_samples_per_signal() const { return sparse_ingest() ? imap_.per_signal : 0; }
    double dma_validate_share() const { return dma_share_; }
    bool sparse_ingest() const { return ingest_enabled_ && imap_.per_signal * 4 <= sched_.n; }

    // [encode, bucket fft (b > 256), decode] ms of the last execute run with
    // stage_times (summed over chunks).
    const double* stage_ms() const { return stage_ms_; }
    // bytes the last execute moved host->device (signal data, compact rows,
    // rows copied for device validation, seeds) and device->host (results,
    // status flags)
    int64_t last_h2d_bytes() const { return h2d_bytes_; }
    int64_t last_d2h_bytes() const { return d2h_bytes_; }

    std::mutex& mutex() { return mu_; }

private:
    struct TaskSet {
        DeviceBuffer<EncTask> d;
        int64_t count = 0;
        std::vector<EncTask> host;
        // gated decode (launch_decode_gated): [need per iteration][done per
        // iteration][exit count]; done/exit are zero between calls
        DeviceBuffer<int32_t> gate;
    };
    struct FusedSet {
        DeviceBuffer<EncTask> tasks;
        DeviceBuffer<int32_t> items, need, counters;
        FusedWork fw;
    };
    const TaskSet& tasks_for(int64_t batch);
    // tasks_for(batch) with every task's t' segments cut to the part-th of
    // `parts` equal contiguous pieces (tap-range sharding)
    const TaskSet& tasks_for_part(int64_t batch, int64_t part, int64_t parts);
    // slot 0: synchronous launches; 1, 2: the two alternating buffer sets of
    // programmatic (PDL) asynchronous launches
    const FusedSet& fused_for(int64_t batch, int slot = 0);
    // validating fused launch (fused.cu fused_val_kernel): chunks of signals
    // whose rows fit in L2, each V(c) E(c) D(c - lag)
    struct ValSet {
        DeviceBuffer<EncTask> tasks;
        DeviceBuffer<int32_t> items, need, counters, vneed;
        DeviceBuffer<int2> packs;
        ValWork vw;
        size_t smem = 0;
        int64_t n_packs = 0, n_vitems = 0;
    };
    const ValSet& val_for(int64_t batch, int64_t x_stride);
    bool val_fused_ok(const void* d_x, int64_t x_stride) const;
    // split: one task per merged t' segment (more CTAs for small batches)
    void append_tasks(std::vector<EncTask>& v, int64_t s_begin, int64_t s_end, bool split) const;
    bool split_tasks(int64_t n_tasks) const;
    void launch_compact_gather(int64_t batch, const void* d_x, int64_t x_stride,
                               const int64_t* d_sig, void* out, cudaStream_t st) const;
    // iterations [m0, m1) only (m1 < 0: to the end)
    void bucket_ffts(double2* y, int64_t batch, cudaStream_t st, const FftGate* gate = nullptr,
                     int m0 = 0, int m1 = -1) const;
    void run_wide_overlapped(int64_t batch, const void* d_x, int64_t x_stride,
                             const int64_t* d_sig, const int64_t* d_sig_inv, int64_t* d_out_f,
                             double2* d_out_c, int64_t* d_out_count, bool validate,
                             const DevPlan& P, cudaStream_t st);
    void upload_sigmas(int64_t batch, const uint64_t* seeds, cudaStream_t st);
    void check_flags(cudaStream_t st);
    void run_chunk(int64_t batch, const void* d_x, int64_t x_stride, const int64_t* d_sig,
                   const int64_t* d_sig_inv, int64_t* d_out_f, double2* d_out_c,
                   int64_t* d_out_count, bool validate, cudaStream_t st,
                   const ExecOptions& opt, bool compact = false);
    // host input, sparse ingest (ingest.hpp); returns true if the host scan
    // saw a non-finite sample
    // asynchronous fused launches chained with programmatic dependent launch:
    // step i+1's σ plan and encode start on the SMs step i's CTAs free while
    // its last decodes finish (buffers alternate between two sets)
    void execute_pdl(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                     int64_t* d_of, double2* d_oc, int64_t* d_ocnt, cudaStream_t st);
    bool execute_sparse(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                        int64_t* d_of, double2* d_oc, int64_t* d_ocnt, bool validate,
                        cudaStream_t st, const ExecOptions& opt);

    int device_;
    bool c128_;
    SchedulePlan sched_;
    std::vector<std::shared_ptr<const DeviceWindow>> windows_;
    DevPlan dplan_{};
    DevPlan dplan_compact_{};  // dplan_ with x_compact = 1
    DecLayout lay_{};
    DecLayout lay_dec_{};  // the standalone decode kernel's (larger shared-memory cap)
    size_t enc_smem_ = 0;
    int64_t b_max_ = 0, budget_max_ = 0;
    std::vector<int> big_b_iters_;  // iterations needing the separate FFT
    std::map<int64_t, TaskSet> tasks_;
    std::map<std::tuple<int64_t, int64_t, int64_t>, TaskSet> part_tasks_;
    std::map<int64_t, FusedSet> fused_;
    std::map<std::pair<int64_t, int64_t>, ValSet> val_;
    bool val_fused_enabled_ = true;             // MSFFT_VAL_FUSED
    int64_t val_chunk_bytes_ = int64_t{32} << 20;  // MSFFT_VAL_CHUNK_MB: x bytes per chunk
    int64_t val_item_bytes_ = int64_t{1024} << 10;  // MSFFT_VAL_ITEM_KB: one validation item
    int64_t val_dlag_ = 8;                      // MSFFT_VAL_DLAG: chunks a decode trails
    int64_t val_elag_ = 0;                      // MSFFT_VAL_ELAG: chunks an encode trails its scan
    int64_t val_smem_kb_ = 64;                  // MSFFT_VAL_SMEM_KB: dynamic smem floor
    bool val_ok_ = false;                       // every b in [32, 256], one-CTA decode
    bool fused_enabled_ = true;   // persistent encode+decode launch when all b <= 256
    int64_t fused_chunk_ = 64;    // signals per fused chunk
    int64_t fused_lag_ = 2;       // chunks a decode trails its encode by
    int64_t fused_tail_ = 0;      // last chunks whose decodes follow their encodes at once
    bool split_enabled_ = true;   // split encode tasks per segment when a launch is small
    // batches up to this size run the encode and a gated decode launch behind
    // it (the decode starts while the encode runs, one CTA per signal with
    // the standalone decode's scratch) instead of the fused kernel
    int64_t gated_max_batch_ = 16;
    bool gated_ok_ = false;
    // small launches gather their samples over every SM into compact rows
    // first (compact_gather_kernel), then encode from those (coalesced)
    bool compact_gather_ = true;
    DeviceBuffer<GatherIv> givs_;
    DeviceBuffer<double> stage_tab_;  // locate stage tables (DevIter::stage_len/blk)
    int n_givs_ = 0;
    int64_t giv_max_len_ = 0;
    mutable DeviceBuffer<unsigned char> xcompact_;
    // CUDA graphs of the small-batch sequence, per buffer set (bounded)
    struct GatedKey {
        int64_t batch;
        const void* x;
        int64_t x_stride;
        const void *sig, *sig_inv, *out_f, *out_c, *out_count, *y, *work, *xc;
        bool validate, compact;
        bool operator<(const GatedKey& o) const {
            return std::tie(batch, x, x_stride, sig, sig_inv, out_f, out_c, out_count, y, work, xc,
                            validate, compact) <
                   std::tie(o.batch, o.x, o.x_stride, o.sig, o.sig_inv, o.out_f, o.out_c,
                            o.out_count, o.y, o.work, o.xc, o.validate, o.compact);
        }
    };
    bool gated_graphs_ = true;
    std::map<GatedKey, cudaGraphExec_t> gated_graphs_map_;
    void enqueue_gated(int64_t batch, const void* d_x, int64_t x_stride, const int64_t* d_sig,
                       const int64_t* d_sig_inv, int64_t* d_out_f, double2* d_out_c,
                       int64_t* d_out_count, bool validate, bool compact, cudaStream_t st);
    size_t fused_smem_ = 0;
    size_t enc_smem_pad_ = 0;     // diagnostics: extra encode smem (lowers occupancy)

    cudaStream_t own_stream_ = nullptr, copy_stream_ = nullptr;
    cudaEvent_t ev_start_ = nullptr, ev_end_ = nullptr;
    cudaEvent_t ev_copied_[2] = {nullptr, nullptr}, ev_free_[2] = {nullptr, nullptr};
    cudaEvent_t ev_stage_[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t dec_stream_ = nullptr;  // high-priority decode stream (overlap)
    cudaEvent_t ev_chunk_ = nullptr, ev_dec_done_ = nullptr;
    // wide decode overlapped with the encode: iteration groups (MSFFT_WIDE_GROUPS,
    // 1 = encode everything first)
    static constexpr int kMaxWideGroups = 8;
    int wide_groups_ = 5;
    // ... only when the encode has this many samples to gather (C5: 18.7 M;
    // C3's 1.2 M encode is too short to pay for the extra graph launches)
    int64_t wide_overlap_min_ = int64_t{1} << 22;
    // bucket FFTs above 4096 points: two launches over all sets (fft.hpp)
    bool fft_two_pass_ = true;
    mutable DeviceBuffer<double2> fft_scratch_;
    cudaEvent_t ev_group_[kMaxWideGroups] = {};
    int64_t overlap_chunk_ = 0;          // signals per encode/decode sub-chunk (0 = serial)
    double stage_ms_[3] = {0, 0, 0};
    int64_t h2d_bytes_ = 0, d2h_bytes_ = 0;

    DeviceBuffer<double2> y_;
    DeviceBuffer<int64_t> sig_, sig_inv_;
    DeviceBuffer<unsigned char> dec_work_;
    DeviceBuffer<int64_t> out_f_, out_count_;
    DeviceBuffer<double2> out_c_;
    DeviceBuffer<int32_t> flags_;  // [0] decode error, [1] non-finite input
    DeviceBuffer<unsigned char> xstage_[2];
    // sparse host ingest
    IngestMap imap_;
    bool ingest_enabled_ = true;     // MSFFT_SPARSE_INGEST=0 forces dense H2D
    int64_t ingest_chunk_ = 128;     // signals per gather / H2D chunk
    std::unique_ptr<HostPool> pool_;
    void* gstage_[2] = {nullptr, nullptr};  // pinned compact staging
    size_t gstage_cap_ = 0;
    std::vector<int64_t> hsig_, hsig_inv_;
    // grid-wide decode of large single signals (wide_decode.hpp): used in the
    // serial path when the decode needs the large-size layout and the batch
    // is too small to fill the GPU with one CTA per signal
    std::unique_ptr<WideDecoder> wide_;
    int64_t wide_max_batch_ = 8;     // MSFFT_WIDE_MAX_BATCH (0 disables)
    int64_t rounds_max_ = 0;
    // validation split: the first dma_share_ of a validating host batch is
    // copied whole by the copy engine and checked by validate_kernel while
    // host threads scan the rest; the share adapts so both finish together
    double dma_share_ = 0.3;
    bool dma_share_fixed_ = false;      // MSFFT_DMA_VALIDATE_SHARE given
    bool dma_pending_ = false;          // timings of the last split to read
    double last_host_ms_ = 0.0;
    cudaStream_t vstream_ = nullptr;
    cudaEvent_t ev_vbeg_ = nullptr, ev_vend_ = nullptr;
    DeviceBuffer<unsigned char> vstage_;
    DeviceBuffer<uint64_t> seeds_;
    // pinned seed staging, two slots so an asynchronous call never waits for
    // the previous call's copy; the σ plan is reused while the seeds repeat
    uint64_t* h_seeds_[2] = {nullptr, nullptr};
    cudaEvent_t ev_seeds_[2] = {nullptr, nullptr};
    int64_t h_seeds_cap_ = 0;
    int seed_slot_ = 0;
    std::vector<uint64_t> last_seeds_;
    // PDL launch sets (execute_pdl)
    // opt-in (MSFFT_PDL=1): measured +1.2% per step on C4 (1.982 vs 2.007 ms,
    // tools/pdl_probe.py) -- the decode tail overlaps little
    bool pdl_enabled_ = false;
    int64_t pdl_count_ = 0;
    // stream and outputs of the previous execute (PDL chaining guard)
    cudaStream_t last_stream_ = nullptr;
    const void* last_out_[3] = {nullptr, nullptr, nullptr};
    DeviceBuffer<double2> y_pdl_[2];
    DeviceBuffer<int64_t> sig_pdl_[2], sig_inv_pdl_[2];
    uint64_t* h_pdl_seeds_[2] = {nullptr, nullptr};  // pinned, read by sigma_kernel
    int64_t h_pdl_cap_ = 0;
    std::vector<uint64_t> pdl_seeds_[2];
    std::mutex mu_;
};

// Process-wide plan cache for the one-shot API (keyed by device and all
// plan parameters), with up to kPlansPerKey plans per key so concurrent
// same-geometry calls (the reference's run_sweep threads, bench.cpp:242-280)
// run side by side instead of queueing on one plan.  The lease holds the
// plan's mutex; plans are built outside the cache lock.
constexpr int kPlansPerKey = 4;
struct PlanLease {
    std::shared_ptr<Plan> plan;
    std::unique_lock<std::mutex> lock;
};
PlanLease lease_plan(int64_t n, int64_t k, int64_t l, double q, double delta, bool c128,
                     int device);

// ComplexSignal::validate's finiteness scan on the device: `batch` rows of
// `span` samples, `x_stride` samples apart; sets *bad to 1 if any is
// non-finite.  HBM-bound streaming kernel (engine.cu).
void launch_validate(const void* d_x, bool c128, int64_t span, int64_t x_stride, int64_t batch,
                     int32_t* bad, cudaStream_t st);

}  // namespace msfft_b200
