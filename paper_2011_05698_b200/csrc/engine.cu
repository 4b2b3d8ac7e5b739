// engine.cu -- see engine.hpp.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <tuple>

#include "engine.hpp"
#include "fft.hpp"
#include "sigma.hpp"

namespace msfft_b200 {

namespace {

constexpr size_t kTapsSmemMax = 96 * 1024;
constexpr int64_t kDecSmemMax = 200 * 1024;
constexpr size_t kChunkBytes = size_t{1} << 30;  // host-input pipeline chunk

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        MSFFT_CUDA(cudaGetDevice(&prev));
        if (prev != dev) MSFFT_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

// ComplexSignal::validate's finiteness scan (proj/src/signal.cpp:22-25),
// HBM-bound.  The rows (one per signal, or the whole batch as one row when it
// is contiguous) are cut into 16-KB chunks; each CTA (one per SM) streams its
// chunks through an 8-deep shared-memory ring filled by TMA bulk copies
// (cp.async.bulk + mbarrier) -- 128 KB in flight per SM, which reads HBM at
// ~7.4 TB/s where 16-B LDGs top out at ~6.3 TB/s (tools/validate_probe.cu,
// profiles/r02/validate_probe.log).  A non-finite value is an all-ones
// exponent field: integer tests on the staged words, no FP.
__device__ __forceinline__ uint32_t val_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kValChunk = 16384;
constexpr int kValRing = 8;
constexpr int kValThreads = 256;

template <bool C128>
__device__ __forceinline__ uint32_t non_finite4(uint4 v) {
    if (C128)  // high words of the two doubles
        return ((v.y & 0x7ff00000u) == 0x7ff00000u) | ((v.w & 0x7ff00000u) == 0x7ff00000u);
    return ((v.x & 0x7f800000u) == 0x7f800000u) | ((v.y & 0x7f800000u) == 0x7f800000u) |
           ((v.z & 0x7f800000u) == 0x7f800000u) | ((v.w & 0x7f800000u) == 0x7f800000u);
}

// Chunk cursor: (row, chunk within the row) of chunk index c, advanced by
// the grid stride without 64-bit divisions (the consumer loop must stay far
// below the ~650 cycles one 16-KB chunk takes to arrive at HBM speed).
struct ChunkCursor {
    int64_t row, cir;
    __device__ void advance(int64_t q, int64_t r, int64_t cpr) {
        row += q;
        cir += r;
        if (cir >= cpr) {
            cir -= cpr;
            ++row;
        }
    }
};

template <bool C128>
__global__ void __launch_bounds__(kValThreads)
validate_kernel(const unsigned char* __restrict__ x, int64_t row_bytes, int64_t stride_bytes,
                int64_t rows, int32_t* __restrict__ bad) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ __align__(8) uint64_t bar[kValRing];
    const int64_t cpr = (row_bytes + kValChunk - 1) / kValChunk;  // chunks per row
    const int64_t nch = cpr * rows;
    const int64_t q = gridDim.x / cpr, r = gridDim.x % cpr;       // grid stride in (row, cir)
    if (threadIdx.x == 0) {
        for (int i = 0; i < kValRing; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(val_smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](const ChunkCursor& cc, int slot) {
        const int64_t off = cc.cir * kValChunk;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kValChunk), row_bytes - off));
        const uint32_t b = val_smem_u32(&bar[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(val_smem_u32(ring + slot * kValChunk)), "l"(x + cc.row * stride_bytes + off),
            "r"(bytes), "r"(b)
            : "memory");
    };
    ChunkCursor cons{blockIdx.x / cpr, blockIdx.x % cpr};  // the chunk being scanned
    ChunkCursor prod = cons;                                // the next chunk to request
    int64_t c_prod = blockIdx.x;
    if (threadIdx.x == 0)
        for (int i = 0; i < kValRing && c_prod < nch; ++i) {
            issue(prod, i);
            prod.advance(q, r, cpr);
            c_prod += gridDim.x;
        }
    uint32_t acc = 0;
    int it = 0;
    for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
        const int slot = it % kValRing;
        const uint32_t parity = static_cast<uint32_t>(it / kValRing) & 1u;
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(val_smem_u32(&bar[slot])),
            "r"(parity)
            : "memory");
        const uint4* v = reinterpret_cast<const uint4*>(ring + slot * kValChunk);
        const int64_t rem = row_bytes - cons.cir * kValChunk;
        if (rem >= kValChunk) {
#pragma unroll
            for (int i = 0; i < kValChunk / 16 / kValThreads; ++i)
                acc |= non_finite4<C128>(v[threadIdx.x + i * kValThreads]);
        } else {
            const int nv = static_cast<int>(rem / 16);
            for (int i = threadIdx.x; i < nv; i += kValThreads) acc |= non_finite4<C128>(v[i]);
        }
        cons.advance(q, r, cpr);
        __syncthreads();  // the slot is consumed before it is refilled
        if (threadIdx.x == 0 && c_prod < nch) {
            issue(prod, slot);
            prod.advance(q, r, cpr);
            c_prod += gridDim.x;
        }
    }
    if (__any_sync(0xffffffffu, acc != 0) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

// Element-wise fallback for rows that are not 16-B vectors (odd shard spans).
template <class T>
__global__ void validate_scalar_kernel(const T* __restrict__ x, int64_t n, int64_t x_stride,
                                       int64_t batch, int32_t* __restrict__ bad) {
    bool ok = true;
    for (int64_t s = blockIdx.y; s < batch; s += gridDim.y)
        for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const T v = __ldcs(x + s * x_stride + e);
            ok &= isfinite(static_cast<double>(v.x)) && isfinite(static_cast<double>(v.y));
        }
    if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}

}  // namespace

void launch_validate(const void* d_x, bool c128, int64_t span, int64_t x_stride, int64_t batch,
                     int32_t* bad, cudaStream_t st) {
    if (span <= 0 || batch <= 0) return;
    const int64_t elem = c128 ? 16 : 8;
    const int sms = sm_count();
    const bool vec = (reinterpret_cast<uintptr_t>(d_x) % 16 == 0) && (span * elem) % 16 == 0 &&
                     (x_stride * elem) % 16 == 0;
    if (vec) {
        int64_t row_bytes = span * elem, rows = batch;
        if (x_stride == span) {  // one flat row
            row_bytes *= batch;
            rows = 1;
        }
        const int64_t nch = (row_bytes + kValChunk - 1) / kValChunk * rows;
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(nch, sms)));
        const size_t smem = static_cast<size_t>(kValChunk) * kValRing;
        if (c128)
            smem_attr(validate_kernel<true>, smem);
        else
            smem_attr(validate_kernel<false>, smem);
        if (c128)
            validate_kernel<true><<<grid, kValThreads, smem, st>>>(
                static_cast<const unsigned char*>(d_x), row_bytes, x_stride * elem, rows, bad);
        else
            validate_kernel<false><<<grid, kValThreads, smem, st>>>(
                static_cast<const unsigned char*>(d_x), row_bytes, x_stride * elem, rows, bad);
    } else {
        const int64_t blocks_total = static_cast<int64_t>(sms) * 8;
        const int64_t gy = std::min<int64_t>(batch, 65535);
        const int64_t gx = std::max<int64_t>(
            1, std::min<int64_t>((span + 255) / 256, (blocks_total + gy - 1) / gy));
        const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
        if (c128)
            validate_scalar_kernel<double2><<<grid, 256, 0, st>>>(static_cast<const double2*>(d_x),
                                                                 span, x_stride, batch, bad);
        else
            validate_scalar_kernel<float2><<<grid, 256, 0, st>>>(static_cast<const float2*>(d_x),
                                                                span, x_stride, batch, bad);
    }
    MSFFT_LAUNCH_CHECK("validate_kernel");
}

namespace {

// Device twin of the host ingest gather (ingest.hpp): compact[s][cpos + i] =
// x[s][sigma_m * (lo + i) mod n] for every interval of the iterations'
// t' unions.  Small launches gather through it so the random reads of one
// signal are spread over every SM (an SM serves ~1 random access per clock,
// so a single-signal encode task reading them itself is bound by its own
// SM's L1), and the encode then reads its samples coalesced.
template <class T>
__global__ void __launch_bounds__(256)
compact_gather_kernel(const GatherIv* __restrict__ ivs, const T* __restrict__ x, int64_t x_stride,
                      const int64_t* __restrict__ sigma, int iters, uint64_t mask,
                      int64_t per_signal, T* __restrict__ out) {
    const GatherIv iv = ivs[blockIdx.y];
    const int64_t s = blockIdx.z;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= iv.len) return;
    const uint64_t sg = static_cast<uint64_t>(sigma[s * iters + iv.m]);
    const uint64_t t = static_cast<uint64_t>(iv.lo + i);
    out[s * per_signal + iv.cpos + i] = x[s * x_stride + static_cast<int64_t>((sg * t) & mask)];
}

}  // namespace

void Plan::launch_compact_gather(int64_t batch, const void* d_x, int64_t x_stride,
                                 const int64_t* d_sig, void* out, cudaStream_t st) const {
    const dim3 grid(static_cast<unsigned>((giv_max_len_ + 255) / 256),
                    static_cast<unsigned>(n_givs_), static_cast<unsigned>(batch));
    const uint64_t mask = static_cast<uint64_t>(sched_.n - 1);
    if (c128_)
        compact_gather_kernel<double2><<<grid, 256, 0, st>>>(
            givs_.get(), static_cast<const double2*>(d_x), x_stride, d_sig, sched_.iterations,
            mask, imap_.per_signal, static_cast<double2*>(out));
    else
        compact_gather_kernel<float2><<<grid, 256, 0, st>>>(
            givs_.get(), static_cast<const float2*>(d_x), x_stride, d_sig, sched_.iterations,
            mask, imap_.per_signal, static_cast<float2*>(out));
    MSFFT_LAUNCH_CHECK("compact_gather_kernel");
}

Plan::Plan(int64_t n, int64_t k, int64_t l, double q, double delta, bool c128, int device)
    : device_(device), c128_(c128) {
    DeviceGuard dg(device);
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
    sched_ = build_schedule(n, k, l, q, delta, [](int64_t nn, int64_t bb, double dd) {
        return window_support(nn, bb, dd);
    });
    if (sched_.iterations > kMaxIters)
        throw std::invalid_argument("sfft4: iteration count exceeds the device plan limit");
    // MSFFT_L2_FETCH (bytes, diagnostics): cudaLimitMaxL2FetchGranularity.
    // Not set by default: the random gather fills whole 128-B lines whatever
    // it says, and 32 B slows the streaming validation scan by a third.
    if (const char* e = std::getenv("MSFFT_L2_FETCH"))
        cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, std::atoi(e));

    size_t taps_smem_max = kTapsSmemMax;  // MSFFT_TAPS_SMEM_MAX (bytes): diagnostics
    if (const char* e = std::getenv("MSFFT_TAPS_SMEM_MAX")) taps_smem_max = std::atoll(e);
    DevPlan& P = dplan_;
    std::memset(&P, 0, sizeof(P));
    P.n = n;
    P.k = k;
    P.l = l;
    P.q = q;
    P.inv_n = 1.0 / static_cast<double>(n);
    P.x_lo = 0;
    P.x_hi = n;
    P.iters = sched_.iterations;
    P.values_per_signal = sched_.values_per_signal;
    P.acc_cap = sched_.acc_cap;
    int tau_off = 0;
    int64_t yoff = 0;
    std::vector<double> stab_len, stab_blk;  // locate stage tables of every iteration
    std::vector<std::array<int64_t, 2>> stage_off(static_cast<size_t>(sched_.iterations));
    for (int m = 0; m < sched_.iterations; ++m) {
        const IterationPlan& ip = sched_.iters[m];
        auto win = get_device_window(n, ip.b, delta);
        windows_.push_back(win);
        DevIter& it = P.it[m];
        it.b = ip.b;
        it.l_width = ip.l_width;
        it.w = win->w;
        it.h = win->h;
        it.budget = ip.budget;
        it.k_m = ip.k_m;
        it.yoff = yoff;
        it.gmax = win->gmax;
        it.taps = win->d_taps;
        it.ghat = win->d_ghat;
        it.tw = device_twiddles(ip.b);
        int lb = 0;
        while ((int64_t{1} << lb) < ip.b) ++lb;
        it.log2b = lb;
        it.nrounds = static_cast<int32_t>(ip.taus.size());
        it.tau_off = tau_off;
        {
            // locate stage lengths, same IEEE operations as locate_step
            double len = static_cast<double>(ip.l_width);
            int st = 0;
            stage_off[m][0] = static_cast<int64_t>(stab_len.size());
            stage_off[m][1] = static_cast<int64_t>(stab_blk.size());
            while (len > 1.0 + 1e-9 && st < kMaxStages - 1) {
                stab_len.push_back(len);
                stab_blk.push_back(len / static_cast<double>(l));
                len = len * (q + 1.0) / static_cast<double>(l);
                ++st;
            }
            stab_len.push_back(len);
            it.nstage_tab = (len > 1.0 + 1e-9) ? -1 : st;
        }
        const size_t taps_bytes = static_cast<size_t>(win->w + 1) * sizeof(double);
        it.taps_in_smem = taps_bytes <= taps_smem_max ? 1 : 0;
        if (tau_off + it.nrounds > kMaxTaus)
            throw std::invalid_argument("sfft4: tau plan exceeds the device plan limit");
        for (int r = 0; r < it.nrounds; ++r) P.taus[tau_off + r] = ip.taus[r];
        tau_off += it.nrounds;
        yoff += static_cast<int64_t>(it.nrounds) * ip.b;
        if (it.taps_in_smem) enc_smem_ = std::max(enc_smem_, taps_bytes);
        if (ip.b <= kEncThreads)
            enc_smem_ = std::max(enc_smem_, static_cast<size_t>(kEncThreads) *
                                                std::min(it.nrounds, kEncRounds) * sizeof(double2));
        else
            big_b_iters_.push_back(m);
        b_max_ = std::max(b_max_, ip.b);
        budget_max_ = std::max(budget_max_, ip.budget);
    }
    stage_tab_.reset(stab_len.size() + stab_blk.size() + 1);
    std::vector<double> stab(stab_len);
    stab.insert(stab.end(), stab_blk.begin(), stab_blk.end());
    stab.push_back(0.0);
    MSFFT_CUDA(cudaMemcpy(stage_tab_.get(), stab.data(), stab.size() * sizeof(double),
                          cudaMemcpyHostToDevice));
    for (int m = 0; m < sched_.iterations; ++m) {
        P.it[m].stage_len = stage_tab_.get() + stage_off[m][0];
        P.it[m].stage_blk = stage_tab_.get() + stab_len.size() + stage_off[m][1];
    }
    int64_t rounds_max = 0;
    for (const auto& ip : sched_.iters)
        rounds_max = std::max<int64_t>(rounds_max, static_cast<int64_t>(ip.taus.size()));
    lay_ = make_dec_layout(sched_.acc_cap, b_max_, budget_max_, rounds_max);
    // the standalone decode kernel may keep a larger scratch in shared
    // memory than the fused kernel (which must keep 2 CTAs per SM): up to
    // kDecSmemMax, one CTA per SM, instead of L2 round trips per access
    lay_dec_ = lay_;
    if (!lay_dec_.big && lay_dec_.bytes <= kDecSmemMax) lay_dec_.in_smem = 1;
    rounds_max_ = rounds_max;
    // Blocking streams: ordered after work on the legacy default stream, so
    // callers that pass no stream (e.g. torch default-stream producers) are safe.
    MSFFT_CUDA(cudaStreamCreateWithFlags(&own_stream_, cudaStreamDefault));
    MSFFT_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamDefault));
    MSFFT_CUDA(cudaEventCreate(&ev_start_));
    MSFFT_CUDA(cudaEventCreate(&ev_end_));
    for (int i = 0; i < 2; ++i) {
        MSFFT_CUDA(cudaEventCreateWithFlags(&ev_copied_[i], cudaEventDisableTiming));
        MSFFT_CUDA(cudaEventCreateWithFlags(&ev_free_[i], cudaEventDisableTiming));
    }
    for (int i = 0; i < 4; ++i) MSFFT_CUDA(cudaEventCreate(&ev_stage_[i]));
    int lo_prio = 0, hi_prio = 0;
    MSFFT_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    MSFFT_CUDA(cudaStreamCreateWithPriority(&dec_stream_, cudaStreamDefault, hi_prio));
    MSFFT_CUDA(cudaEventCreateWithFlags(&ev_chunk_, cudaEventDisableTiming));
    MSFFT_CUDA(cudaEventCreateWithFlags(&ev_dec_done_, cudaEventDisableTiming));
    for (auto& e : ev_group_) MSFFT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (const char* e = std::getenv("MSFFT_WIDE_OVERLAP_MIN")) wide_overlap_min_ = std::atoll(e);
    if (const char* e = std::getenv("MSFFT_FFT_TWO_PASS")) fft_two_pass_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_WIDE_GROUPS"))
        wide_groups_ = std::max(1, std::min(kMaxWideGroups, std::atoi(e)));
    if (const char* e = std::getenv("MSFFT_OVERLAP_CHUNK")) overlap_chunk_ = std::atoll(e);
    if (const char* e = std::getenv("MSFFT_FUSED")) fused_enabled_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_FUSED_CHUNK")) fused_chunk_ = std::max(1LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_FUSED_LAG")) fused_lag_ = std::max(1LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_FUSED_TAIL")) fused_tail_ = std::max(0LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_ENC_SMEM_PAD")) enc_smem_pad_ = std::atoll(e);
    fused_smem_ = std::max(enc_smem_, lay_.in_smem ? static_cast<size_t>(lay_.bytes) : size_t{0});
    if (const char* e = std::getenv("MSFFT_ENC_SPLIT")) split_enabled_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_GATED_MAX_BATCH")) gated_max_batch_ = std::atoll(e);
    if (const char* e = std::getenv("MSFFT_GATED_GRAPH")) gated_graphs_ = std::atoi(e) != 0;
    // gated launches need the one-CTA decode and every bucket FFT in one
    // shared-memory launch
    gated_ok_ = !lay_.big && big_b_iters_.size() <= static_cast<size_t>(kMaxFftSets);
    for (int m : big_b_iters_) gated_ok_ = gated_ok_ && dplan_.it[m].b <= kSmemFftMax;
    if (const char* e = std::getenv("MSFFT_FUSED_SMEM_PAD"))  // diagnostic: L1 carve-out experiments
        fused_smem_ += static_cast<size_t>(std::max(0LL, std::atoll(e)));
    // the validating fused launch packs iterations of one signal per CTA on
    // warp-aligned lanes: every b in [32, 256], the one-CTA decode
    val_ok_ = big_b_iters_.empty() && !lay_.big;
    for (int m = 0; m < sched_.iterations; ++m)
        val_ok_ = val_ok_ && dplan_.it[m].b >= 32 && dplan_.it[m].b <= kEncThreads;
    if (const char* e = std::getenv("MSFFT_VAL_FUSED")) val_fused_enabled_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_VAL_CHUNK_MB"))
        val_chunk_bytes_ = std::max(1LL, std::atoll(e)) << 20;
    if (const char* e = std::getenv("MSFFT_VAL_ITEM_KB"))
        val_item_bytes_ = std::max(16LL, std::atoll(e)) << 10;
    if (const char* e = std::getenv("MSFFT_VAL_DLAG")) val_dlag_ = std::max(0LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_VAL_SMEM_KB")) val_smem_kb_ = std::max(16LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_VAL_ELAG")) val_elag_ = std::max(0LL, std::atoll(e));
    flags_.reset(2);
    MSFFT_CUDA(cudaMemset(flags_.get(), 0, 2 * sizeof(int32_t)));
    for (int i = 0; i < 2; ++i)
        MSFFT_CUDA(cudaEventCreateWithFlags(&ev_seeds_[i], cudaEventDisableTiming));
    imap_ = make_ingest_map(sched_);
    {
        std::vector<GatherIv> iv;
        for (int m = 0; m < sched_.iterations; ++m)
            for (size_t j = 0; j < imap_.uni[m].size(); ++j) {
                const auto& u = imap_.uni[m][j];
                iv.push_back(GatherIv{m, 0, u.first, u.second - u.first + 1, imap_.pos[m][j]});
                giv_max_len_ = std::max(giv_max_len_, u.second - u.first + 1);
            }
        n_givs_ = static_cast<int>(iv.size());
        givs_.reset(iv.size());
        MSFFT_CUDA(cudaMemcpy(givs_.get(), iv.data(), iv.size() * sizeof(GatherIv),
                              cudaMemcpyHostToDevice));
    }
    if (const char* e = std::getenv("MSFFT_COMPACT_GATHER")) compact_gather_ = std::atoi(e) != 0;
    dplan_compact_ = dplan_;
    dplan_compact_.x_compact = 1;
    dplan_compact_.x_row = imap_.per_signal;
    if (const char* e = std::getenv("MSFFT_SPARSE_INGEST")) ingest_enabled_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_INGEST_CHUNK")) ingest_chunk_ = std::max(1LL, std::atoll(e));
    if (const char* e = std::getenv("MSFFT_WIDE_MAX_BATCH")) wide_max_batch_ = std::atoll(e);
    if (const char* e = std::getenv("MSFFT_PDL")) pdl_enabled_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_DMA_VALIDATE_SHARE")) {
        dma_share_ = std::min(1.0, std::max(0.0, std::atof(e)));
        dma_share_fixed_ = true;
    }
    MSFFT_CUDA(cudaStreamCreateWithFlags(&vstream_, cudaStreamNonBlocking));
    MSFFT_CUDA(cudaEventCreate(&ev_vbeg_));
    MSFFT_CUDA(cudaEventCreate(&ev_vend_));
}

Plan::~Plan() {
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    cudaSetDevice(device_);
    for (auto& kv : gated_graphs_map_)
        if (kv.second) cudaGraphExecDestroy(kv.second);
    for (auto& e : ev_group_)
        if (e) cudaEventDestroy(e);
    if (own_stream_) cudaStreamDestroy(own_stream_);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (ev_start_) cudaEventDestroy(ev_start_);
    if (ev_end_) cudaEventDestroy(ev_end_);
    for (int i = 0; i < 2; ++i) {
        if (ev_copied_[i]) cudaEventDestroy(ev_copied_[i]);
        if (ev_free_[i]) cudaEventDestroy(ev_free_[i]);
    }
    for (int i = 0; i < 4; ++i)
        if (ev_stage_[i]) cudaEventDestroy(ev_stage_[i]);
    if (dec_stream_) cudaStreamDestroy(dec_stream_);
    if (ev_chunk_) cudaEventDestroy(ev_chunk_);
    if (ev_dec_done_) cudaEventDestroy(ev_dec_done_);
    for (int i = 0; i < 2; ++i) {
        if (h_seeds_[i]) cudaFreeHost(h_seeds_[i]);
        if (ev_seeds_[i]) cudaEventDestroy(ev_seeds_[i]);
        if (h_pdl_seeds_[i]) cudaFreeHost(h_pdl_seeds_[i]);
    }
    for (int i = 0; i < 2; ++i)
        if (gstage_[i]) cudaFreeHost(gstage_[i]);
    if (vstream_) cudaStreamDestroy(vstream_);
    if (ev_vbeg_) cudaEventDestroy(ev_vbeg_);
    if (ev_vend_) cudaEventDestroy(ev_vend_);
    cudaSetDevice(cur);
}

const Plan::TaskSet& Plan::tasks_for(int64_t batch) {
    auto it = tasks_.find(batch);
    if (it != tasks_.end()) return it->second;
    std::vector<EncTask> v;
    append_tasks(v, 0, batch, false);
    if (split_tasks(static_cast<int64_t>(v.size()))) {
        v.clear();
        append_tasks(v, 0, batch, true);
    }
    TaskSet ts;
    ts.count = static_cast<int64_t>(v.size());
    ts.d.reset(v.size());
    MSFFT_CUDA(cudaMemcpy(ts.d.get(), v.data(), v.size() * sizeof(EncTask),
                          cudaMemcpyHostToDevice));
    // gate words (encode.hpp): decode need per iteration -- its encode tasks
    // (b <= 256) or its bucket-FFT CTAs (b > 256) --, done, exit, the folds'
    // encode tasks per iteration, their done
    const int iters = sched_.iterations;
    std::vector<int32_t> gate(static_cast<size_t>(4 * iters + 1), 0);
    for (const EncTask& t : v) {
        if (dplan_.it[t.m].b > kEncThreads)
            ++gate[2 * iters + 1 + t.m];
        else
            ++gate[t.m];
    }
    for (int m : big_b_iters_) gate[m] = static_cast<int32_t>(batch * dplan_.it[m].nrounds);
    ts.gate.reset(gate.size());
    MSFFT_CUDA(cudaMemcpy(ts.gate.get(), gate.data(), gate.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    ts.host = std::move(v);
    return tasks_.emplace(batch, std::move(ts)).first->second;
}

const Plan::TaskSet& Plan::tasks_for_part(int64_t batch, int64_t part, int64_t parts) {
    const auto key = std::make_tuple(batch, part, parts);
    auto it = part_tasks_.find(key);
    if (it != part_tasks_.end()) return it->second;
    std::vector<EncTask> v = tasks_for(batch).host;
    for (EncTask& t : v)
        for (int i = 0; i < t.nseg; ++i) {
            // piece `part` of [lo, hi]: every t' of the segment lands in
            // exactly one piece; an empty piece has hi < lo (no trips)
            const int64_t lo = t.seg_lo[i], len = static_cast<int64_t>(t.seg_hi[i]) - lo + 1;
            const int64_t a = lo + len * part / parts, e = lo + len * (part + 1) / parts;
            t.seg_cpos[i] += static_cast<int32_t>(a - lo);
            t.seg_lo[i] = static_cast<int32_t>(a);
            t.seg_hi[i] = static_cast<int32_t>(e - 1);
        }
    TaskSet ts;
    ts.count = static_cast<int64_t>(v.size());
    ts.d.reset(v.size());
    MSFFT_CUDA(cudaMemcpy(ts.d.get(), v.data(), v.size() * sizeof(EncTask),
                          cudaMemcpyHostToDevice));
    ts.host = std::move(v);
    return part_tasks_.emplace(key, std::move(ts)).first->second;
}

const Plan::FusedSet& Plan::fused_for(int64_t batch, int slot) {
    const int64_t key = batch * 4 + slot;
    auto it = fused_.find(key);
    if (it != fused_.end()) return it->second;
    // chunk: a multiple of the largest signal group of a fused encode task
    int64_t group = 1;
    for (int m = 0; m < sched_.iterations; ++m)
        group = std::max<int64_t>(group, kEncThreads / dplan_.it[m].b);
    const int64_t chunk = std::max<int64_t>(group, (fused_chunk_ + group - 1) / group * group);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    std::vector<EncTask> tasks;
    append_tasks(tasks, 0, batch, false);
    const bool split = split_tasks(static_cast<int64_t>(tasks.size()));
    tasks.clear();
    std::vector<std::vector<int32_t>> enc(nchunks);
    // need[c * iters + m]: encode tasks of chunk c and iteration m
    const int iters = sched_.iterations;
    std::vector<int32_t> need(static_cast<size_t>(nchunks * iters), 0);
    for (int64_t c = 0; c < nchunks; ++c) {
        const size_t before = tasks.size();
        append_tasks(tasks, c * chunk, std::min(batch, (c + 1) * chunk), split);
        for (size_t i = before; i < tasks.size(); ++i) {
            enc[c].push_back(static_cast<int32_t>(i));
            ++need[c * iters + tasks[i].m];
        }
    }
    // E(0) .. E(lag) D(0) E(lag+1) D(1) ...: decodes trail their encodes by
    // `lag` chunks so they rarely wait.  The last `tail` chunks get lag 0:
    // their decodes are claimed right after their encode tasks and run the
    // early iterations (gated per iteration) while the later iterations'
    // encodes finish, so less decode work is left after the last encode.
    std::vector<int32_t> items;
    auto decodes = [&](int64_t c) {
        for (int64_t s = c * chunk; s < std::min(batch, (c + 1) * chunk); ++s)
            items.push_back(static_cast<int32_t>(-(s + 1)));
    };
    const int64_t tail_from = std::max<int64_t>(0, nchunks - fused_tail_);
    int64_t next_dec = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        items.insert(items.end(), enc[c].begin(), enc[c].end());
        const int64_t upto = c >= tail_from ? c : c - fused_lag_;  // decode chunks <= upto
        for (; next_dec <= upto; ++next_dec) decodes(next_dec);
    }
    for (; next_dec < nchunks; ++next_dec) decodes(next_dec);
    FusedSet fs;
    fs.tasks.reset(tasks.size());
    fs.items.reset(items.size());
    fs.need.reset(need.size());
    fs.counters.reset(need.size() + 2);  // ticket, done[], exit count
    MSFFT_CUDA(cudaMemcpy(fs.tasks.get(), tasks.data(), tasks.size() * sizeof(EncTask),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(fs.items.get(), items.data(), items.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(fs.need.get(), need.data(), need.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    fs.fw.tasks = fs.tasks.get();
    fs.fw.items = fs.items.get();
    fs.fw.n_items = static_cast<int32_t>(items.size());
    fs.fw.chunk = chunk;
    fs.fw.need = fs.need.get();
    fs.fw.counters = fs.counters.get();
    fs.fw.n_chunks = nchunks;
    fs.fw.n_counters = static_cast<int64_t>(need.size()) + 2;
    MSFFT_CUDA(cudaMemset(fs.counters.get(), 0, sizeof(int32_t) * fs.fw.n_counters));
    return fused_.emplace(key, std::move(fs)).first->second;
}

bool Plan::val_fused_ok(const void* d_x, int64_t x_stride) const {
    const int64_t elem = c128_ ? 16 : 8;
    return val_ok_ && val_fused_enabled_ && fused_enabled_ &&
           reinterpret_cast<uintptr_t>(d_x) % 16 == 0 && (x_stride * elem) % 16 == 0 &&
           (sched_.n * elem) % 16 == 0;
}

// Item list of the validating fused launch (fused.cu fused_val_kernel).
// Chunk = the signals whose rows fill val_chunk_bytes_ (default 32 MB: one
// C4 signal).  Per chunk: its validation items, then its packed encode items
// (val_elag_ chunks later), then the decodes of the chunk val_dlag_ chunks
// before.  Packing: the chunk's (signal, iteration, round-group) sub-tasks,
// first-fit decreasing on b into CTAs of 256 threads (<= kMaxPack each, their
// b-point arrays within the shared memory); each distinct iteration's taps
// staged once per pack while they fit, read from global otherwise.
const Plan::ValSet& Plan::val_for(int64_t batch, int64_t x_stride) {
    const auto key = std::make_pair(batch, x_stride);
    auto found = val_.find(key);
    if (found != val_.end()) return found->second;
    const int64_t elem = c128_ ? 16 : 8;
    const int64_t row_bytes = sched_.n * elem;
    const int64_t chunk = std::max<int64_t>(1, val_chunk_bytes_ / (x_stride * elem));
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    const int iters = sched_.iterations;
    const int64_t item_bytes = std::min(row_bytes, (val_item_bytes_ + 15) / 16 * 16);
    const int64_t ipr = (row_bytes + item_bytes - 1) / item_bytes;
    if (batch * ipr >= static_cast<int64_t>(kValItemBase))
        throw std::invalid_argument("sfft4: validation item index exceeds the item code range");
    // dynamic shared memory: the encode's taps/arrays, the decode scratch,
    // and the scan's ring of 16-KB slots -- as large as two CTAs per SM allow
    size_t smem = std::max(fused_smem_, static_cast<size_t>(val_smem_kb_) << 10);
    std::vector<EncTask> proto;
    // one sub-task per merged t' segment (MSFFT_VAL_SPLIT=0: per round group):
    // 3-4x shorter gather chains per item, so an item's loads finish before
    // the scan reaches its signal (a late gather misses: the scan's lines are
    // evict_first) -- DRAM bytes per step and the step time both drop
    bool vsplit = true;
    if (const char* e = std::getenv("MSFFT_VAL_SPLIT")) vsplit = std::atoi(e) != 0;
    append_tasks(proto, 0, 1, vsplit);
    struct Bin {
        std::vector<EncTask> subs;
        int threads = 0;
        size_t f_bytes = 0;
    };
    std::vector<EncTask> tasks;
    std::vector<int2> packs;
    std::vector<std::vector<int32_t>> enc(nchunks);
    std::vector<int32_t> need(static_cast<size_t>(nchunks * iters), 0);
    for (int64_t c = 0; c < nchunks; ++c) {
        std::vector<EncTask> subs;
        for (int64_t s = c * chunk; s < std::min(batch, (c + 1) * chunk); ++s)
            for (EncTask t : proto) {
                t.sig0 = s;
                t.nsig = 1;
                t.fused = 1;
                t.lane0 = 0;
                subs.push_back(t);
                ++need[c * iters + t.m];
            }
        std::stable_sort(subs.begin(), subs.end(), [&](const EncTask& a, const EncTask& b) {
            return dplan_.it[a.m].b > dplan_.it[b.m].b;
        });
        std::vector<Bin> bins;
        for (const EncTask& t : subs) {
            const int b = static_cast<int>(dplan_.it[t.m].b);
            const size_t fb = static_cast<size_t>(t.nr) * b * sizeof(double2);
            Bin* dst = nullptr;
            for (Bin& bn : bins)
                if (bn.threads + b <= kEncThreads && static_cast<int>(bn.subs.size()) < kMaxPack &&
                    bn.f_bytes + fb <= smem) {
                    dst = &bn;
                    break;
                }
            if (!dst) {
                bins.emplace_back();
                dst = &bins.back();
            }
            dst->subs.push_back(t);
            dst->threads += b;
            dst->f_bytes += fb;
        }
        for (Bin& bn : bins) {
            int tid0 = 0;
            int32_t f_off = 0;
            size_t taps_used = 0;
            for (size_t j = 0; j < bn.subs.size(); ++j) {
                EncTask& t = bn.subs[j];
                const DevIter& di = dplan_.it[t.m];
                t.tid0 = tid0;
                tid0 += static_cast<int>(di.b);
                t.f_off = f_off;
                f_off += static_cast<int32_t>(t.nr * di.b);
                t.stage_taps = 0;
                t.taps_off = -1;
                for (size_t q = 0; q < j; ++q)
                    if (bn.subs[q].m == t.m && bn.subs[q].taps_off >= 0) t.taps_off = bn.subs[q].taps_off;
                if (t.taps_off < 0) {
                    const size_t tb = (static_cast<size_t>(di.w + 1) * sizeof(double) + 127) / 128 * 128;
                    if (taps_used + tb <= smem) {
                        t.taps_off = static_cast<int32_t>(taps_used);
                        t.stage_taps = 1;
                        taps_used += tb;
                    }
                }
            }
            enc[c].push_back(static_cast<int32_t>(packs.size()));
            packs.push_back(make_int2(static_cast<int>(tasks.size()), static_cast<int>(bn.subs.size())));
            tasks.insert(tasks.end(), bn.subs.begin(), bn.subs.end());
        }
    }
    std::vector<int32_t> items, vneed(static_cast<size_t>(nchunks), 0);
    auto vitems = [&](int64_t c) {
        for (int64_t s = c * chunk; s < std::min(batch, (c + 1) * chunk); ++s)
            for (int64_t p = 0; p < ipr; ++p) {
                items.push_back(static_cast<int32_t>(kValItemBase + s * ipr + p));
                ++vneed[c];
            }
    };
    auto decodes = [&](int64_t c) {
        for (int64_t s = c * chunk; s < std::min(batch, (c + 1) * chunk); ++s)
            items.push_back(static_cast<int32_t>(-(s + 1)));
    };
    // diagnostics (MSFFT_VAL_DEBUG): 1 = validation items only, 2 = no
    // validation items (the encode and decode alone, reading x from HBM)
    int debug = 0;
    if (const char* e = std::getenv("MSFFT_VAL_DEBUG")) debug = std::atoi(e);
    if (debug == 1)
        for (auto& e : enc) e.clear();
    // E(c) goes right before V(c + eoff): eoff = 1 after its own scan, 0
    // before it, < 0 that many chunks ahead of it (MSFFT_VAL_EOFF).  Default
    // -4 with policy 7 (gather loads evict_last, scan copies evict_first):
    // the gathers fetch their lines 4 chunks (4 signals at C4, ~20 us) before
    // the scan passes them, the scan hits those lines and its own lines do not push them out.
    // The scan-first order (eoff >= 1) gets no L2 hits on B200 at all: the
    // latency-bound gathers of a chunk run long after the scan's lines are
    // evicted (profiles/r02c).
    int64_t eoff = val_elag_ ? 1 + val_elag_ : -4;
    int policy = 7;
    if (const char* e = std::getenv("MSFFT_VAL_EOFF")) eoff = std::atoll(e);
    if (const char* e = std::getenv("MSFFT_VAL_POLICY")) policy = std::atoi(e);
    int64_t next_enc = 0, next_dec = 0, next_v = 0;
    for (int64_t t = std::min<int64_t>(0, eoff); t < nchunks + std::max<int64_t>(0, eoff); ++t) {
        const int64_t ce = t - eoff;
        if (ce >= 0 && ce < nchunks) {
            items.insert(items.end(), enc[ce].begin(), enc[ce].end());
            next_enc = ce + 1;
        }
        if (t >= 0 && t < nchunks) {
            if (debug != 2) vitems(t);
            next_v = t + 1;
        }
        for (; next_dec < std::min(next_enc, next_v) - val_dlag_; ++next_dec) decodes(next_dec);
    }
    for (; next_enc < nchunks; ++next_enc)
        items.insert(items.end(), enc[next_enc].begin(), enc[next_enc].end());
    for (; next_dec < nchunks; ++next_dec) decodes(next_dec);
    if (debug == 1) items.erase(std::remove_if(items.begin(), items.end(),
                                               [](int32_t v) { return v < 0; }),
                                items.end());

    ValSet vs;
    vs.tasks.reset(tasks.size());
    vs.items.reset(items.size());
    vs.need.reset(need.size());
    vs.vneed.reset(vneed.size());
    vs.packs.reset(packs.size());
    const int64_t n_counters = nchunks * iters + nchunks + 2;
    vs.counters.reset(static_cast<size_t>(n_counters));
    MSFFT_CUDA(cudaMemcpy(vs.tasks.get(), tasks.data(), tasks.size() * sizeof(EncTask),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(vs.items.get(), items.data(), items.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(vs.need.get(), need.data(), need.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(vs.vneed.get(), vneed.data(), vneed.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemcpy(vs.packs.get(), packs.data(), packs.size() * sizeof(int2),
                          cudaMemcpyHostToDevice));
    MSFFT_CUDA(cudaMemset(vs.counters.get(), 0, sizeof(int32_t) * n_counters));
    vs.vw.fw.tasks = vs.tasks.get();
    vs.vw.fw.items = vs.items.get();
    vs.vw.fw.n_items = static_cast<int32_t>(items.size());
    vs.vw.fw.chunk = chunk;
    vs.vw.fw.need = vs.need.get();
    vs.vw.fw.counters = vs.counters.get();
    vs.vw.fw.n_chunks = nchunks;
    vs.vw.fw.n_counters = n_counters;
    vs.vw.packs = vs.packs.get();
    vs.vw.vneed = vs.vneed.get();
    vs.vw.row_bytes = row_bytes;
    vs.vw.stride_bytes = x_stride * elem;
    vs.vw.item_bytes = item_bytes;
    vs.vw.items_per_row = ipr;
    vs.vw.policy = policy;
    vs.smem = smem;
    vs.n_packs = static_cast<int64_t>(packs.size());
    vs.n_vitems = batch * ipr;
    return val_.emplace(key, std::move(vs)).first->second;
}

// K2 for the iterations with b > 256 (the encode's fused epilogue does the
// rest): their b-point transforms and the 1/n scale, as few launches as the
// sizes allow.
void Plan::bucket_ffts(double2* y, int64_t batch, cudaStream_t st, const FftGate* gate, int m0,
                       int m1) const {
    std::vector<FftSet> sets;
    for (int m : big_b_iters_) {
        if (m < m0 || (m1 >= 0 && m >= m1)) continue;
        const DevIter& di = dplan_.it[m];
        sets.push_back(FftSet{di.yoff, di.b, di.nrounds, m});
    }
    // arrays above 4096 points go through the two-pass path, which needs a
    // scratch copy laid out like y
    bool big = false;
    for (const FftSet& f : sets) big = big || f.size > kSmemFftMax;
    if (big && !gate)
        fft_scratch_.ensure(static_cast<size_t>(batch * dplan_.values_per_signal));
    double2* scratch = big && !gate && fft_two_pass_ ? fft_scratch_.get() : nullptr;
    for (size_t i = 0; i < sets.size(); i += kMaxFftSets)
        fft_radix2_sets(y, sets.data() + i,
                        static_cast<int>(std::min<size_t>(kMaxFftSets, sets.size() - i)), batch,
                        dplan_.values_per_signal, -1, dplan_.inv_n, st, gate, scratch);
}

bool Plan::split_tasks(int64_t n_tasks) const {
    if (!split_enabled_) return false;
    int sms = 0;  // this plan's device (called once per new batch size)
    MSFFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_));
    return n_tasks < 8 * static_cast<int64_t>(sms);
}

void Plan::append_tasks(std::vector<EncTask>& v, int64_t s_begin, int64_t s_end,
                        bool split) const {
    for (int m = 0; m < sched_.iterations; ++m) {
        const DevIter& di = dplan_.it[m];
        const IterationPlan& ip = sched_.iters[m];
        for (int r0 = 0; r0 < di.nrounds; r0 += kEncRounds) {
            EncTask t{};
            t.m = m;
            t.r0 = r0;
            t.nr = std::min(kEncRounds, di.nrounds - r0);
            // merged t' intervals [-h - tau, h - tau] of the chunk's rounds
            std::vector<std::pair<int64_t, int64_t>> iv;
            for (int r = r0; r < r0 + t.nr; ++r) iv.emplace_back(-di.h - ip.taus[r], di.h - ip.taus[r]);
            std::sort(iv.begin(), iv.end());
            std::vector<std::pair<int64_t, int64_t>> merged;
            for (const auto& s : iv) {
                if (!merged.empty() && s.first <= merged.back().second + 1)
                    merged.back().second = std::max(merged.back().second, s.second);
                else
                    merged.push_back(s);
            }
            const auto emit = [&](EncTask t) {
                if (di.b <= kEncThreads) {
                    t.fused = 1;
                    t.nsig = static_cast<int32_t>(kEncThreads / di.b);
                    t.lane0 = 0;
                    for (int64_t s0 = s_begin; s0 < s_end; s0 += t.nsig) {
                        t.sig0 = s0;
                        v.push_back(t);
                    }
                } else {
                    t.fused = 0;
                    t.nsig = 1;
                    for (int64_t s0 = s_begin; s0 < s_end; ++s0)
                        for (int64_t lane0 = 0; lane0 < di.b; lane0 += kEncThreads) {
                            t.sig0 = s0;
                            t.lane0 = static_cast<int32_t>(lane0);
                            v.push_back(t);
                        }
                }
            };
            const auto seg = [&](EncTask& t, int i, size_t j) {
                t.seg_lo[i] = static_cast<int32_t>(merged[j].first);
                t.seg_hi[i] = static_cast<int32_t>(merged[j].second);
                t.seg_cpos[i] = static_cast<int32_t>(imap_.position(m, merged[j].first));
            };
            if (!split) {
                t.nseg = static_cast<int32_t>(merged.size());
                for (size_t i = 0; i < merged.size(); ++i) seg(t, static_cast<int>(i), i);
                emit(t);
            } else {
                // small launches: one task per merged segment, which covers
                // a contiguous run of rounds (the intervals shift with tau,
                // which grows with r), so no sample is loaded twice
                for (size_t j = 0; j < merged.size(); ++j) {
                    EncTask ts = t;
                    int ra = t.r0 + t.nr, rb = t.r0 - 1;
                    for (int r = t.r0; r < t.r0 + t.nr; ++r)
                        if (-di.h - ip.taus[r] >= merged[j].first && di.h - ip.taus[r] <= merged[j].second) {
                            ra = std::min(ra, r);
                            rb = std::max(rb, r);
                        }
                    ts.r0 = ra;
                    ts.nr = rb - ra + 1;
                    ts.nseg = 1;
                    seg(ts, 0, j);
                    emit(ts);
                }
            }
        }
    }
}

int64_t Plan::launches(int64_t batch, bool validate, bool serial) const {
    if (!serial && gated_ok_ && batch <= gated_max_batch_)  // sigma (+ gather) + encode
        return 3 + (compact_gather_ ? 1 : 0) + (big_b_iters_.empty() ? 0 : 1) +
               (validate ? 1 : 0);  // (+ bucket FFTs) + decode (+ validate)
    if (!serial && validate && val_ok_ && val_fused_enabled_ && fused_enabled_)
        return 2;  // sigma + validating fused (device rows, 16-B aligned)
    if (!serial && fused_enabled_ && big_b_iters_.empty() && !lay_.big)
        return 2 + (validate ? 1 : 0);  // sigma + fused (+ validate)
    // per (sub-)chunk: encode + bucket FFTs for b > 256 + decode
    int64_t per_chunk = 2;
    for (int m : big_b_iters_) {
        int lb = dplan_.it[m].log2b;
        int64_t passes = 0, s0 = 0;
        while (s0 < lb) {
            s0 += (s0 == 0) ? std::min(lb, 11) : std::min<int64_t>(lb - s0, 7);
            ++passes;
        }
        per_chunk += 1 + passes;  // bitrev + stage passes
    }
    const int64_t chunks =
        (overlap_chunk_ > 0 && batch > overlap_chunk_) ? (batch + overlap_chunk_ - 1) / overlap_chunk_
                                                       : 1;
    return 1 + (validate ? 1 : 0) + chunks * per_chunk;  // + sigma (+ validate)
}

// The small-batch launch sequence: [validate] [compact gather] encode
// [gated bucket FFTs] gated decode.  The decode is a programmatic dependent
// launch that starts while the encode runs and waits per iteration for that
// iteration's tasks (one CTA per signal, the standalone decode's registers
// and shared-memory scratch).
void Plan::enqueue_gated(int64_t batch, const void* d_x, int64_t x_stride, const int64_t* d_sig,
                         const int64_t* d_sig_inv, int64_t* d_out_f, double2* d_out_c,
                         int64_t* d_out_count, bool validate, bool compact, cudaStream_t st) {
    if (validate) launch_validate(d_x, c128_, sched_.n, x_stride, batch, flags_.get() + 1, st);
    const TaskSet& ts = tasks_for(batch);
    int32_t* gate = const_cast<int32_t*>(ts.gate.get());
    const int iters = sched_.iterations;
    const DevPlan* EP = compact ? &dplan_compact_ : &dplan_;
    const void* ex = d_x;
    int64_t es = x_stride;
    if (compact_gather_ && !compact && n_givs_ <= 65535) {
        // the samples of every iteration, gathered over all SMs first
        launch_compact_gather(batch, d_x, x_stride, d_sig, xcompact_.get(), st);
        EP = &dplan_compact_;
        ex = xcompact_.get();
        es = imap_.per_signal;
    }
    launch_encode(*EP, ts.d.get(), ts.count, ex, c128_, es, batch, d_sig, y_.get(),
                  enc_smem_ + enc_smem_pad_, st, gate + iters);
    if (!big_b_iters_.empty()) {
        // b > 256: the bucket FFTs as a gated launch between the two
        const FftGate g{gate + 3 * iters + 1, gate + 2 * iters + 1, gate + iters};
        bucket_ffts(y_.get(), batch, st, &g);
    }
    launch_decode_gated(dplan_, lay_dec_, y_.get(), d_sig, d_sig_inv, batch, dec_work_.get(),
                        d_out_f, d_out_c, d_out_count, flags_.get(), gate, gate + iters, st);
}

// Large single signals (wide decode): the encode and the bucket FFTs go out
// in iteration groups [0,1), [1,2), [2,4), [4,8), ... (the early iterations
// have the large b and the small windows, so they encode fastest), each
// group ending in an event; the wide decode of a group's iterations runs on
// the high-priority decode stream once its event fires, so the decode of
// the early iterations overlaps the encode of the later ones.
void Plan::run_wide_overlapped(int64_t batch, const void* d_x, int64_t x_stride,
                               const int64_t* d_sig, const int64_t* d_sig_inv, int64_t* d_out_f,
                               double2* d_out_c, int64_t* d_out_count, bool validate,
                               const DevPlan& P, cudaStream_t st) {
    if (validate) {
        // a non-finite sample makes the call throw: nothing to decode (the
        // scan was launched by run_chunk; this waits for it alone)
        int32_t bad = 0;
        MSFFT_CUDA(cudaMemcpyAsync(&bad, flags_.get() + 1, sizeof(bad), cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        if (bad) return;
    }
    if (!wide_)
        wide_ = std::make_unique<WideDecoder>(dplan_, sched_.acc_cap, b_max_, budget_max_,
                                              rounds_max_);
    const TaskSet& ts = tasks_for(batch);
    const int iters = sched_.iterations;
    const int64_t k = sched_.k, vps = dplan_.values_per_signal;
    std::vector<std::pair<int, int>> groups;
    for (int m0 = 0; m0 < iters;) {
        const int m1 = static_cast<int>(groups.size()) + 1 >= wide_groups_
                           ? iters
                           : std::min(iters, m0 == 0 ? 1 : 2 * m0);
        groups.emplace_back(m0, m1);
        m0 = m1;
    }
    // tasks are iteration-major (append_tasks)
    int64_t t0 = 0;
    for (size_t g = 0; g < groups.size(); ++g) {
        const auto [m0, m1] = groups[g];
        int64_t t1 = t0;
        while (t1 < ts.count && ts.host[t1].m < m1) ++t1;
        launch_encode(P, ts.d.get() + t0, t1 - t0, d_x, c128_, x_stride, batch, d_sig, y_.get(),
                      enc_smem_ + enc_smem_pad_, st);
        bucket_ffts(y_.get(), batch, st, nullptr, m0, m1);
        MSFFT_CUDA(cudaEventRecord(ev_group_[g], st));
        t0 = t1;
    }
    for (int64_t s = 0; s < batch; ++s)
        for (size_t g = 0; g < groups.size(); ++g) {
            if (s == 0) MSFFT_CUDA(cudaStreamWaitEvent(dec_stream_, ev_group_[g], 0));
            wide_->run_range(y_.get() + s * vps, d_sig + s * iters, d_sig_inv + s * iters,
                             d_out_f + s * k, d_out_c + s * k, d_out_count + s, flags_.get(),
                             dec_stream_, groups[g].first, groups[g].second);
        }
    MSFFT_CUDA(cudaEventRecord(ev_dec_done_, dec_stream_));
    MSFFT_CUDA(cudaStreamWaitEvent(st, ev_dec_done_, 0));
}

void Plan::run_chunk(int64_t batch, const void* d_x, int64_t x_stride, const int64_t* d_sig,
                     const int64_t* d_sig_inv, int64_t* d_out_f, double2* d_out_c,
                     int64_t* d_out_count, bool validate, cudaStream_t st,
                     const ExecOptions& opt, bool compact) {
    const int64_t n = sched_.n;
    const DevPlan& P = compact ? dplan_compact_ : dplan_;
    const bool traced = opt.pre || opt.post || opt.sel_bucket;
    if (!traced && !opt.stage_times && !opt.force_serial && gated_ok_ && batch <= gated_max_batch_) {
        // small batches: a latency path, so the launch sequence is replayed
        // from a CUDA graph once it has run eagerly for these buffers
        const bool use_gather = compact_gather_ && !compact && n_givs_ <= 65535;
        if (use_gather) {
            const size_t elem = c128_ ? sizeof(double2) : sizeof(float2);
            xcompact_.ensure(static_cast<size_t>(batch * imap_.per_signal) * elem);
        }
        const GatedKey key{batch, d_x, x_stride, d_sig, d_sig_inv, d_out_f, d_out_c, d_out_count,
                           y_.get(), dec_work_.get(), xcompact_.get(), validate, compact};
        if (!gated_graphs_) {
            enqueue_gated(batch, d_x, x_stride, d_sig, d_sig_inv, d_out_f, d_out_c, d_out_count,
                          validate, compact, st);
            return;
        }
        auto it = gated_graphs_map_.find(key);
        if (it == gated_graphs_map_.end()) {
            // first use of these buffers: eager (allocates lazily built
            // tables), and remembered so the next call captures
            if (gated_graphs_map_.size() >= 8) {
                MSFFT_CUDA(cudaStreamSynchronize(st));
                for (auto& kv : gated_graphs_map_)
                    if (kv.second) cudaGraphExecDestroy(kv.second);
                gated_graphs_map_.clear();
            }
            gated_graphs_map_.emplace(key, nullptr);
            enqueue_gated(batch, d_x, x_stride, d_sig, d_sig_inv, d_out_f, d_out_c, d_out_count,
                          validate, compact, st);
            return;
        }
        if (!it->second) {
            cudaStream_t cap = nullptr;
            MSFFT_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            MSFFT_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_gated(batch, d_x, x_stride, d_sig, d_sig_inv, d_out_f, d_out_c,
                              d_out_count, validate, compact, cap);
            } catch (...) {
                cudaStreamEndCapture(cap, &g);
                if (g) cudaGraphDestroy(g);
                cudaStreamDestroy(cap);
                throw;
            }
            MSFFT_CUDA(cudaStreamEndCapture(cap, &g));
            cudaGraphExec_t ex = nullptr;
            MSFFT_CUDA(cudaGraphInstantiate(&ex, g, 0));
            cudaGraphDestroy(g);
            cudaStreamDestroy(cap);
            it->second = ex;
        }
        MSFFT_CUDA(cudaGraphLaunch(it->second, st));
        return;
    }
    if (validate && !traced && !opt.force_serial && !compact && val_fused_ok(d_x, x_stride)) {
        // one persistent launch: the validation scan, the encode and the
        // decode, the encode's random reads served from the L2 lines the scan
        // of the same signals brings in
        const ValSet& vs = val_for(batch, x_stride);
        if (opt.stage_times) MSFFT_CUDA(cudaEventRecord(ev_stage_[0], st));
        launch_fused_validating(P, lay_, vs.vw, d_x, c128_, x_stride, batch, d_sig, d_sig_inv,
                                y_.get(), dec_work_.get(), d_out_f, d_out_c, d_out_count,
                                flags_.get(), vs.smem, st);
        if (opt.stage_times) {
            MSFFT_CUDA(cudaEventRecord(ev_stage_[1], st));
            MSFFT_CUDA(cudaEventSynchronize(ev_stage_[1]));
            float ms = 0.f;
            MSFFT_CUDA(cudaEventElapsedTime(&ms, ev_stage_[0], ev_stage_[1]));
            stage_ms_[0] += ms;
        }
        return;
    }
    if (validate) launch_validate(d_x, c128_, n, x_stride, batch, flags_.get() + 1, st);
    if (!traced && !opt.force_serial && fused_enabled_ && big_b_iters_.empty() && !lay_.big) {
        // one persistent launch: encode and decode share the SMs
        const FusedSet& fs = fused_for(batch);
        if (opt.stage_times) MSFFT_CUDA(cudaEventRecord(ev_stage_[0], st));
        launch_fused(P, lay_, fs.fw, d_x, c128_, x_stride, batch, d_sig, d_sig_inv,
                     y_.get(), dec_work_.get(), d_out_f, d_out_c, d_out_count, flags_.get(),
                     fused_smem_, st);
        if (opt.stage_times) {
            MSFFT_CUDA(cudaEventRecord(ev_stage_[1], st));
            MSFFT_CUDA(cudaEventSynchronize(ev_stage_[1]));
            float ms = 0.f;
            MSFFT_CUDA(cudaEventElapsedTime(&ms, ev_stage_[0], ev_stage_[1]));
            stage_ms_[0] += ms;  // fused encode+decode
        }
        return;
    }
    if (!traced && !opt.stage_times && !opt.force_serial && overlap_chunk_ > 0 &&
        batch > overlap_chunk_) {
        // Overlapped pipeline: the encode of sub-chunk c+1 (HBM-bound) runs
        // while the decode of sub-chunk c (SM-bound) runs on a higher-priority
        // stream; an event per sub-chunk orders decode after its encode.
        const size_t elem = c128_ ? sizeof(double2) : sizeof(float2);
        const int iters = sched_.iterations;
        const int64_t k = sched_.k, vps = dplan_.values_per_signal;
        for (int64_t c0 = 0; c0 < batch; c0 += overlap_chunk_) {
            const int64_t cb = std::min(overlap_chunk_, batch - c0);
            const TaskSet& tsc = tasks_for(cb);
            const void* xc = static_cast<const unsigned char*>(d_x) + c0 * x_stride * elem;
            double2* yc = y_.get() + c0 * vps;
            launch_encode(P, tsc.d.get(), tsc.count, xc, c128_, x_stride, cb,
                          d_sig + c0 * iters, yc, enc_smem_, st);
            bucket_ffts(yc, cb, st);
            MSFFT_CUDA(cudaEventRecord(ev_chunk_, st));
            MSFFT_CUDA(cudaStreamWaitEvent(dec_stream_, ev_chunk_, 0));
            launch_decode(dplan_, lay_dec_, yc, d_sig + c0 * iters, d_sig_inv + c0 * iters, cb,
                          lay_.in_smem ? nullptr : dec_work_.get() + c0 * lay_.bytes,
                          d_out_f + c0 * k, d_out_c + c0 * k, d_out_count + c0, flags_.get(),
                          dec_stream_);
        }
        MSFFT_CUDA(cudaEventRecord(ev_dec_done_, dec_stream_));
        MSFFT_CUDA(cudaStreamWaitEvent(st, ev_dec_done_, 0));
        return;
    }
    if (!traced && !opt.stage_times && !opt.force_serial && lay_.big && batch <= wide_max_batch_ &&
        wide_groups_ > 1 && batch * imap_.per_signal >= wide_overlap_min_) {
        run_wide_overlapped(batch, d_x, x_stride, d_sig, d_sig_inv, d_out_f, d_out_c, d_out_count,
                            validate, P, st);
        return;
    }
    const TaskSet& ts = tasks_for(batch);
    if (opt.stage_times) MSFFT_CUDA(cudaEventRecord(ev_stage_[0], st));
    launch_encode(P, ts.d.get(), ts.count, d_x, c128_, x_stride, batch, d_sig, y_.get(),
                  enc_smem_ + enc_smem_pad_, st);
    if (opt.stage_times) MSFFT_CUDA(cudaEventRecord(ev_stage_[1], st));
    bucket_ffts(y_.get(), batch, st);
    if (opt.stage_times) MSFFT_CUDA(cudaEventRecord(ev_stage_[2], st));
    const size_t ybytes = sizeof(double2) * static_cast<size_t>(dplan_.values_per_signal);
    if (opt.pre) {
        MSFFT_CUDA(cudaMemcpyAsync(opt.pre, y_.get(), ybytes, cudaMemcpyDeviceToHost, st));
    }
    DeviceBuffer<int64_t> tb, tf;
    DeviceBuffer<double2> tv;
    if (opt.sel_bucket) {
        tb.reset(static_cast<size_t>(sched_.acc_cap));
        tf.reset(static_cast<size_t>(sched_.acc_cap));
        tv.reset(static_cast<size_t>(sched_.acc_cap));
    }
    if (!traced && lay_.big && batch <= wide_max_batch_) {
        // large single signals: every phase of the decode over the whole GPU
        if (!wide_)
            wide_ = std::make_unique<WideDecoder>(dplan_, sched_.acc_cap, b_max_, budget_max_,
                                                  rounds_max_);
        // a non-finite sample found by this call's validation makes the call
        // throw: skip the decode (without validation the flag is clear --
        // check_flags resets it after every call -- and the decode is
        // enqueued without waiting for the encode)
        int32_t bad = 0;
        if (validate) {
            MSFFT_CUDA(cudaMemcpyAsync(&bad, flags_.get() + 1, sizeof(bad), cudaMemcpyDeviceToHost, st));
            MSFFT_CUDA(cudaStreamSynchronize(st));
        }
        if (!bad) {
            const int iters = sched_.iterations;
            const int64_t k = sched_.k, vps = dplan_.values_per_signal;
            for (int64_t s = 0; s < batch; ++s)
                wide_->run(y_.get() + s * vps, d_sig + s * iters, d_sig_inv + s * iters,
                           d_out_f + s * k, d_out_c + s * k, d_out_count + s, flags_.get(), st);
        }
    } else {
        launch_decode(dplan_, lay_dec_, y_.get(), d_sig, d_sig_inv, batch, dec_work_.get(), d_out_f,
                      d_out_c, d_out_count, flags_.get(), st, tb.get(), tf.get(), tv.get());
    }
    if (opt.stage_times) {
        MSFFT_CUDA(cudaEventRecord(ev_stage_[3], st));
        MSFFT_CUDA(cudaEventSynchronize(ev_stage_[3]));
        for (int i = 0; i < 3; ++i) {
            float ms = 0.f;
            MSFFT_CUDA(cudaEventElapsedTime(&ms, ev_stage_[i], ev_stage_[i + 1]));
            stage_ms_[i] += ms;
        }
    }
    if (opt.post) {
        MSFFT_CUDA(cudaMemcpyAsync(opt.post, y_.get(), ybytes, cudaMemcpyDeviceToHost, st));
    }
    if (opt.sel_bucket) {
        const size_t nb = static_cast<size_t>(sched_.acc_cap);
        MSFFT_CUDA(cudaMemcpyAsync(opt.sel_bucket, tb.get(), nb * 8, cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaMemcpyAsync(opt.sel_f, tf.get(), nb * 8, cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaMemcpyAsync(opt.sel_value, tv.get(), nb * 16, cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
    }
}

void Plan::execute(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                   int64_t* out_f, double* out_c, int64_t* out_count, const ExecOptions& opt,
                   double* device_ms) {
    DeviceGuard dg(device_);
    if (batch <= 0) return;
    const int64_t n = sched_.n, k = sched_.k;
    const int iters = sched_.iterations;
    if (x_stride < n) throw std::invalid_argument("msfft_execute: x_stride < n");
    cudaStream_t st = opt.stream ? opt.stream : own_stream_;
    const size_t elem = c128_ ? sizeof(double2) : sizeof(float2);
    const bool async_call = opt.async_call && !opt.stage_times && !opt.pre && !opt.post &&
                            !opt.sel_bucket;
    if (async_call && !(opt.x_on_device && opt.out_on_device))
        throw std::invalid_argument("msfft_execute: MSFFT_FLAG_ASYNC needs device input and output");
    // A PDL launch may overlap the previous one's last decodes, so it must not
    // write the outputs that launch writes, and the two-set buffer rotation
    // assumes one stream: otherwise launch stream-ordered.
    const bool pdl_safe = last_out_[0] == nullptr ||
                          (st == last_stream_ && out_f != last_out_[0] && out_c != last_out_[1] &&
                           out_count != last_out_[2]);
    last_stream_ = st;
    last_out_[0] = out_f;
    last_out_[1] = out_c;
    last_out_[2] = out_count;
    if (async_call && pdl_enabled_ && fused_enabled_ && !opt.force_serial && big_b_iters_.empty() &&
        !lay_.big && lay_.in_smem && pdl_safe &&
        fused_for(batch).fw.n_items >= fused_slots(c128_, fused_smem_)) {
        // PDL needs a grid that fills every CTA slot (see execute_pdl)
        execute_pdl(batch, x, x_stride, seeds, out_f, reinterpret_cast<double2*>(out_c), out_count,
                    st);
        if (device_ms) *device_ms = 0.0;
        return;
    }

    // chunking: device inputs run as one chunk; host inputs stream through
    // two staging buffers overlapped with compute
    const int64_t sig_bytes = static_cast<int64_t>(elem) * n;
    const bool sparse = !opt.x_on_device && sparse_ingest();
    const int64_t chunk =
        opt.x_on_device ? batch
        : sparse        ? std::min(batch, ingest_chunk_)
                        : std::max<int64_t>(1, std::min<int64_t>(batch, kChunkBytes / sig_bytes));
    y_.ensure(static_cast<size_t>(chunk * dplan_.values_per_signal));
    if (!lay_.in_smem) dec_work_.ensure(static_cast<size_t>(chunk * lay_.bytes));
    if (!opt.out_on_device) {
        out_f_.ensure(static_cast<size_t>(batch * k));
        out_c_.ensure(static_cast<size_t>(batch * k));
        out_count_.ensure(static_cast<size_t>(batch));
    }
    if (!opt.x_on_device && !sparse)
        for (int i = 0; i < 2; ++i) xstage_[i].ensure(static_cast<size_t>(chunk * sig_bytes));

    int64_t* d_of = opt.out_on_device ? out_f : out_f_.get();
    double2* d_oc = opt.out_on_device ? reinterpret_cast<double2*>(out_c) : out_c_.get();
    int64_t* d_ocnt = opt.out_on_device ? out_count : out_count_.get();

    pdl_count_ = 0;  // a stream-ordered call ends any PDL chain
    stage_ms_[0] = stage_ms_[1] = stage_ms_[2] = 0.0;
    h2d_bytes_ = 0;
    d2h_bytes_ = 0;
    MSFFT_CUDA(cudaEventRecord(ev_start_, st));
    upload_sigmas(batch, seeds, st);
    const bool validate = !opt.assume_valid;
    bool host_bad = false;
    if (opt.x_on_device) {
        run_chunk(batch, x, x_stride, sig_.get(), sig_inv_.get(), d_of, d_oc, d_ocnt, validate,
                  st, opt);
    } else if (sparse) {
        host_bad = execute_sparse(batch, x, x_stride, seeds, d_of, d_oc, d_ocnt, validate, st, opt);
    } else {
        MSFFT_CUDA(cudaStreamWaitEvent(copy_stream_, ev_start_, 0));
        const unsigned char* hx = static_cast<const unsigned char*>(x);
        int64_t idx = 0;
        for (int64_t s0 = 0; s0 < batch; s0 += chunk, ++idx) {
            const int64_t cb = std::min(chunk, batch - s0);
            const int slot = static_cast<int>(idx & 1);
            if (idx >= 2) MSFFT_CUDA(cudaStreamWaitEvent(copy_stream_, ev_free_[slot], 0));
            unsigned char* dst = xstage_[slot].get();
            if (x_stride == n) {
                MSFFT_CUDA(cudaMemcpyAsync(dst, hx + s0 * x_stride * elem, cb * sig_bytes,
                                           cudaMemcpyHostToDevice, copy_stream_));
            } else {
                MSFFT_CUDA(cudaMemcpy2DAsync(dst, sig_bytes, hx + s0 * x_stride * elem,
                                             x_stride * elem, sig_bytes, cb,
                                             cudaMemcpyHostToDevice, copy_stream_));
            }
            h2d_bytes_ += cb * sig_bytes;
            MSFFT_CUDA(cudaEventRecord(ev_copied_[slot], copy_stream_));
            MSFFT_CUDA(cudaStreamWaitEvent(st, ev_copied_[slot], 0));
            run_chunk(cb, dst, n, sig_.get() + s0 * iters, sig_inv_.get() + s0 * iters,
                      d_of + s0 * k, d_oc + s0 * k, d_ocnt + s0, validate, st, opt);
            MSFFT_CUDA(cudaEventRecord(ev_free_[slot], st));
        }
    }
    if (!opt.out_on_device) {
        MSFFT_CUDA(cudaMemcpyAsync(out_f, d_of, sizeof(int64_t) * batch * k,
                                   cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaMemcpyAsync(out_c, d_oc, sizeof(double2) * batch * k,
                                   cudaMemcpyDeviceToHost, st));
        MSFFT_CUDA(cudaMemcpyAsync(out_count, d_ocnt, sizeof(int64_t) * batch,
                                   cudaMemcpyDeviceToHost, st));
        d2h_bytes_ += static_cast<int64_t>(sizeof(int64_t) + sizeof(double2)) * batch * k +
                      static_cast<int64_t>(sizeof(int64_t)) * batch;
    }
    MSFFT_CUDA(cudaEventRecord(ev_end_, st));
    if (async_call) {
        if (device_ms) *device_ms = 0.0;  // not measured: the call did not wait
        return;
    }
    if (device_ms) {
        MSFFT_CUDA(cudaEventSynchronize(ev_end_));
        float ms = 0.f;
        MSFFT_CUDA(cudaEventElapsedTime(&ms, ev_start_, ev_end_));
        *device_ms = ms;
    }
    if (host_bad) {
        MSFFT_CUDA(cudaMemsetAsync(flags_.get(), 0, 2 * sizeof(int32_t), st));
        MSFFT_CUDA(cudaStreamSynchronize(st));
        throw std::invalid_argument("ComplexSignal: non-finite sample");
    }
    check_flags(st);
}

bool Plan::execute_sparse(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                          int64_t* d_of, double2* d_oc, int64_t* d_ocnt, bool validate,
                          cudaStream_t st, const ExecOptions& opt) {
    const int64_t n = sched_.n, k = sched_.k, C = imap_.per_signal;
    const int iters = sched_.iterations;
    const size_t elem = c128_ ? sizeof(double2) : sizeof(float2);
    const int64_t chunk = std::min(batch, ingest_chunk_);
    const size_t stage_bytes = static_cast<size_t>(chunk * C) * elem;
    if (!pool_) pool_ = std::make_unique<HostPool>(ingest_threads());
    if (gstage_cap_ < stage_bytes) {
        MSFFT_CUDA(cudaStreamSynchronize(copy_stream_));
        for (int i = 0; i < 2; ++i) {
            if (gstage_[i]) cudaFreeHost(gstage_[i]);
            gstage_[i] = nullptr;
            MSFFT_CUDA(cudaHostAlloc(&gstage_[i], stage_bytes, cudaHostAllocDefault));
        }
        gstage_cap_ = stage_bytes;
    }
    for (int i = 0; i < 2; ++i) xstage_[i].ensure(stage_bytes);
    // the host's copy of the sigma plan (the device draws the same values)
    hsig_.resize(static_cast<size_t>(batch * iters));
    hsig_inv_.resize(static_cast<size_t>(batch * iters));
    pool_->run(batch, [&](int64_t s) {
        draw_sigmas(seeds[s], n, iters, hsig_.data() + s * iters, hsig_inv_.data() + s * iters);
    });
    const unsigned char* hx = static_cast<const unsigned char*>(x);
    bool bad = false;
    // validation split (see engine.hpp): rebalance from the last split's
    // timings, then queue the DMA + device check of rows [0, n_dma)
    if (dma_pending_) {
        float dma_ms = 0.f;
        if (cudaEventElapsedTime(&dma_ms, ev_vbeg_, ev_vend_) == cudaSuccess && dma_ms > 0.f &&
            last_host_ms_ > 0.0 && !dma_share_fixed_) {
            const double gap = (last_host_ms_ - dma_ms) / (last_host_ms_ + dma_ms);
            dma_share_ = std::min(0.9, std::max(0.0, dma_share_ + 0.5 * gap * (1.0 - dma_share_)));
        }
        dma_pending_ = false;
    }
    // the copy engine only runs asynchronously from page-locked memory
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, x) == cudaSuccess &&
                        pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const int64_t n_dma =
        validate && pinned ? static_cast<int64_t>(dma_share_ * static_cast<double>(batch)) : 0;
    if (n_dma > 0) {
        const size_t sig_bytes = static_cast<size_t>(n) * elem;
        const int64_t vchunk = std::max<int64_t>(1, static_cast<int64_t>((size_t{256} << 20) / sig_bytes));
        vstage_.ensure(static_cast<size_t>(vchunk) * sig_bytes);
        MSFFT_CUDA(cudaEventRecord(ev_chunk_, st));  // after the flag reset
        MSFFT_CUDA(cudaStreamWaitEvent(vstream_, ev_chunk_, 0));
        MSFFT_CUDA(cudaEventRecord(ev_vbeg_, vstream_));
        for (int64_t s0 = 0; s0 < n_dma; s0 += vchunk) {
            const int64_t cb = std::min(vchunk, n_dma - s0);
            if (x_stride == n)
                MSFFT_CUDA(cudaMemcpyAsync(vstage_.get(), hx + s0 * x_stride * elem, cb * sig_bytes,
                                           cudaMemcpyHostToDevice, vstream_));
            else
                MSFFT_CUDA(cudaMemcpy2DAsync(vstage_.get(), sig_bytes, hx + s0 * x_stride * elem,
                                             x_stride * elem, sig_bytes, cb,
                                             cudaMemcpyHostToDevice, vstream_));
            launch_validate(vstage_.get(), c128_, n, n, cb, flags_.get() + 1, vstream_);
            h2d_bytes_ += static_cast<int64_t>(cb * sig_bytes);
        }
        MSFFT_CUDA(cudaEventRecord(ev_vend_, vstream_));
    }
    const auto host_t0 = std::chrono::steady_clock::now();
    MSFFT_CUDA(cudaStreamWaitEvent(copy_stream_, ev_start_, 0));
    int64_t idx = 0;
    for (int64_t s0 = 0; s0 < batch; s0 += chunk, ++idx) {
        const int64_t cb = std::min(chunk, batch - s0);
        const int slot = static_cast<int>(idx & 1);
        // the pinned slot's previous H2D must be done before it is refilled
        if (idx >= 2) MSFFT_CUDA(cudaEventSynchronize(ev_copied_[slot]));
        bad |= gather_compact(*pool_, imap_, n, iters, hx + s0 * x_stride * elem, x_stride,
                              static_cast<int>(elem), cb, hsig_.data() + s0 * iters, gstage_[slot],
                              validate, n_dma - s0);
        if (idx >= 2) MSFFT_CUDA(cudaStreamWaitEvent(copy_stream_, ev_free_[slot], 0));
        MSFFT_CUDA(cudaMemcpyAsync(xstage_[slot].get(), gstage_[slot],
                                   static_cast<size_t>(cb * C) * elem, cudaMemcpyHostToDevice,
                                   copy_stream_));
        h2d_bytes_ += cb * C * static_cast<int64_t>(elem);
        MSFFT_CUDA(cudaEventRecord(ev_copied_[slot], copy_stream_));
        MSFFT_CUDA(cudaStreamWaitEvent(st, ev_copied_[slot], 0));
        run_chunk(cb, xstage_[slot].get(), C, sig_.get() + s0 * iters, sig_inv_.get() + s0 * iters,
                  d_of + s0 * k, d_oc + s0 * k, d_ocnt + s0, false, st, opt, true);
        MSFFT_CUDA(cudaEventRecord(ev_free_[slot], st));
    }
    if (n_dma > 0) {
        last_host_ms_ = std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now() - host_t0).count();
        dma_pending_ = true;
        MSFFT_CUDA(cudaStreamWaitEvent(st, ev_vend_, 0));  // flags_[1] complete before the check
    }
    return bad;
}

void Plan::upload_sigmas(int64_t batch, const uint64_t* seeds, cudaStream_t st) {
    // sigma plan: exact mt19937_64 draws on the device, one thread per signal
    const int iters = sched_.iterations;
    if (static_cast<int64_t>(last_seeds_.size()) == batch &&
        std::equal(seeds, seeds + batch, last_seeds_.begin()))
        return;  // sig_ / sig_inv_ already hold this batch's plan (stream-ordered)
    if (h_seeds_cap_ < batch) {
        MSFFT_CUDA(cudaStreamSynchronize(st));
        for (int i = 0; i < 2; ++i) {
            if (h_seeds_[i]) cudaFreeHost(h_seeds_[i]);
            h_seeds_[i] = nullptr;
            MSFFT_CUDA(cudaMallocHost(&h_seeds_[i], sizeof(uint64_t) * batch));
        }
        h_seeds_cap_ = batch;
    }
    sig_.ensure(static_cast<size_t>(batch * iters));
    sig_inv_.ensure(static_cast<size_t>(batch * iters));
    seeds_.ensure(static_cast<size_t>(batch));
    seed_slot_ ^= 1;
    MSFFT_CUDA(cudaEventSynchronize(ev_seeds_[seed_slot_]));  // this slot's last copy is done
    std::memcpy(h_seeds_[seed_slot_], seeds, sizeof(uint64_t) * batch);
    MSFFT_CUDA(cudaMemcpyAsync(seeds_.get(), h_seeds_[seed_slot_], sizeof(uint64_t) * batch,
                               cudaMemcpyHostToDevice, st));
    h2d_bytes_ += static_cast<int64_t>(sizeof(uint64_t)) * batch;
    MSFFT_CUDA(cudaEventRecord(ev_seeds_[seed_slot_], st));
    launch_sigma(seeds_.get(), batch, iters, sched_.n, sig_.get(), sig_inv_.get(), st);
    last_seeds_.assign(seeds, seeds + batch);
}

void Plan::execute_pdl(int64_t batch, const void* x, int64_t x_stride, const uint64_t* seeds,
                       int64_t* d_of, double2* d_oc, int64_t* d_ocnt, cudaStream_t st) {
    const int iters = sched_.iterations;
    const int p = static_cast<int>(pdl_count_++ & 1);
    y_pdl_[p].ensure(static_cast<size_t>(batch * dplan_.values_per_signal));
    sig_pdl_[p].ensure(static_cast<size_t>(batch * iters));
    sig_inv_pdl_[p].ensure(static_cast<size_t>(batch * iters));
    if (h_pdl_cap_ < batch) {
        MSFFT_CUDA(cudaStreamSynchronize(st));
        for (int i = 0; i < 2; ++i) {
            if (h_pdl_seeds_[i]) cudaFreeHost(h_pdl_seeds_[i]);
            h_pdl_seeds_[i] = nullptr;
            MSFFT_CUDA(cudaMallocHost(&h_pdl_seeds_[i], sizeof(uint64_t) * batch));
            pdl_seeds_[i].clear();
        }
        h_pdl_cap_ = batch;
    }
    // set p's seed slot is rewritten only when its seeds change (and only
    // after the work that read it is done)
    if (static_cast<int64_t>(pdl_seeds_[p].size()) != batch ||
        !std::equal(seeds, seeds + batch, pdl_seeds_[p].begin())) {
        MSFFT_CUDA(cudaStreamSynchronize(st));
        std::memcpy(h_pdl_seeds_[p], seeds, sizeof(uint64_t) * batch);
        pdl_seeds_[p].assign(seeds, seeds + batch);
    }
    // Both launches may start while the previous fused launch (set p^1) is
    // finishing.  They touch only set p, whose last user (two launches back)
    // has exited: the previous launch fills every CTA slot and could only
    // become fully resident after it did.
    launch_sigma(h_pdl_seeds_[p], batch, iters, sched_.n, sig_pdl_[p].get(), sig_inv_pdl_[p].get(),
                 st, true);
    const FusedSet& fs = fused_for(batch, 1 + p);
    launch_fused(dplan_, lay_, fs.fw, x, c128_, x_stride, batch, sig_pdl_[p].get(),
                 sig_inv_pdl_[p].get(), y_pdl_[p].get(), dec_work_.get(), d_of, d_oc, d_ocnt,
                 flags_.get(), fused_smem_, st, true);
}

void Plan::sync(cudaStream_t stream) {
    DeviceGuard dg(device_);
    check_flags(stream ? stream : own_stream_);
}

void Plan::check_flags(cudaStream_t st) {
    int32_t hflags[2] = {0, 0};
    MSFFT_CUDA(cudaMemcpyAsync(hflags, flags_.get(), sizeof(hflags), cudaMemcpyDeviceToHost, st));
    d2h_bytes_ += static_cast<int64_t>(sizeof(hflags));
    MSFFT_CUDA(cudaMemsetAsync(flags_.get(), 0, 2 * sizeof(int32_t), st));
    MSFFT_CUDA(cudaStreamSynchronize(st));
    if (hflags[1]) throw std::invalid_argument("ComplexSignal: non-finite sample");
    if (hflags[0] == kDecErrPhaseZero) throw std::domain_error("phase_of: zero value");
    if (hflags[0] == kDecErrRounds)
        throw std::invalid_argument("locate_frequency: not enough rounds for the schedule");
}

void Plan::encode_values(int64_t batch, const void* d_x, int64_t x_stride, int64_t x_lo,
                         int64_t x_hi, const uint64_t* seeds, double2* d_y, bool validate,
                         cudaStream_t stream) {
    DeviceGuard dg(device_);
    if (batch <= 0) return;
    const int64_t n = sched_.n;
    if (x_lo < 0 || x_hi > n || x_lo >= x_hi)
        throw std::invalid_argument("msfft_encode_values: need 0 <= x_lo < x_hi <= n");
    if (x_stride < x_hi - x_lo) throw std::invalid_argument("msfft_encode_values: x_stride < x_hi - x_lo");
    cudaStream_t st = stream ? stream : own_stream_;
    MSFFT_CUDA(cudaMemsetAsync(flags_.get(), 0, 2 * sizeof(int32_t), st));
    upload_sigmas(batch, seeds, st);
    if (validate) launch_validate(d_x, c128_, x_hi - x_lo, x_stride, batch, flags_.get() + 1, st);
    DevPlan p = dplan_;
    p.x_lo = x_lo;
    p.x_hi = x_hi;
    const TaskSet& ts = tasks_for(batch);
    launch_encode(p, ts.d.get(), ts.count, d_x, c128_, x_stride, batch, sig_.get(), d_y,
                  enc_smem_, st);
    bucket_ffts(d_y, batch, st);
    check_flags(st);
}

void Plan::encode_values_part(int64_t batch, const void* d_x, int64_t x_stride, int64_t part,
                              int64_t parts, const uint64_t* seeds, double2* d_y, bool validate,
                              cudaStream_t stream) {
    DeviceGuard dg(device_);
    if (batch <= 0) return;
    const int64_t n = sched_.n;
    if (parts < 1 || part < 0 || part >= parts)
        throw std::invalid_argument("msfft_encode_values_part: need 0 <= part < parts");
    if (x_stride < n) throw std::invalid_argument("msfft_encode_values_part: x_stride < n");
    cudaStream_t st = stream ? stream : own_stream_;
    MSFFT_CUDA(cudaMemsetAsync(flags_.get(), 0, 2 * sizeof(int32_t), st));
    upload_sigmas(batch, seeds, st);
    if (validate) {  // this rank checks its slice of every signal
        const int64_t lo = n * part / parts, hi = n * (part + 1) / parts;
        const size_t elem = c128_ ? sizeof(double2) : sizeof(float2);
        launch_validate(static_cast<const unsigned char*>(d_x) + lo * elem, c128_, hi - lo,
                        x_stride, batch, flags_.get() + 1, st);
    }
    const TaskSet& ts = tasks_for_part(batch, part, parts);
    launch_encode(dplan_, ts.d.get(), ts.count, d_x, c128_, x_stride, batch, sig_.get(), d_y,
                  enc_smem_, st);
    // iterations with b > 256 stay folds: their b-point FFTs (linear) run
    // once on the summed vector (decode_values with folds = true), not per rank
    check_flags(st);
}

void Plan::decode_values(int64_t batch, double2* d_y, const uint64_t* seeds, int64_t* d_out_f,
                         double2* d_out_c, int64_t* d_out_count, cudaStream_t stream,
                         bool folds) {
    DeviceGuard dg(device_);
    if (batch <= 0) return;
    cudaStream_t st = stream ? stream : own_stream_;
    if (folds) bucket_ffts(d_y, batch, st);
    if (!lay_.in_smem) dec_work_.ensure(static_cast<size_t>(batch * lay_.bytes));
    MSFFT_CUDA(cudaMemsetAsync(flags_.get(), 0, 2 * sizeof(int32_t), st));
    upload_sigmas(batch, seeds, st);
    if (lay_.big && batch <= wide_max_batch_) {
        if (!wide_)
            wide_ = std::make_unique<WideDecoder>(dplan_, sched_.acc_cap, b_max_, budget_max_,
                                                  rounds_max_);
        const int iters = sched_.iterations;
        const int64_t k = sched_.k, vps = dplan_.values_per_signal;
        // decode from the plan's own bucket buffer: the caller's vector stays
        // untouched and the captured graphs are keyed on a stable address
        y_.ensure(static_cast<size_t>(batch * vps));
        MSFFT_CUDA(cudaMemcpyAsync(y_.get(), d_y, sizeof(double2) * batch * vps,
                                   cudaMemcpyDeviceToDevice, st));
        d_y = y_.get();
        for (int64_t s = 0; s < batch; ++s)
            wide_->run(d_y + s * vps, sig_.get() + s * iters, sig_inv_.get() + s * iters,
                       d_out_f + s * k, d_out_c + s * k, d_out_count + s, flags_.get(), st);
    } else {
        launch_decode(dplan_, lay_dec_, d_y, sig_.get(), sig_inv_.get(), batch, dec_work_.get(),
                      d_out_f, d_out_c, d_out_count, flags_.get(), st);
    }
    check_flags(st);
}

PlanLease lease_plan(int64_t n, int64_t k, int64_t l, double q, double delta, bool c128,
                     int device) {
    using Key = std::tuple<int, int64_t, int64_t, int64_t, double, double, bool>;
    static std::mutex mu;
    static std::map<Key, std::vector<std::shared_ptr<Plan>>> cache;
    const Key key{device, n, k, l, q, delta, c128};
    std::vector<std::shared_ptr<Plan>> have;
    {
        std::lock_guard<std::mutex> g(mu);
        have = cache[key];
    }
    // an idle plan of this geometry, if any
    for (auto& p : have) {
        std::unique_lock<std::mutex> lk(p->mutex(), std::try_to_lock);
        if (lk.owns_lock()) return PlanLease{p, std::move(lk)};
    }
    if (have.size() < static_cast<size_t>(kPlansPerKey)) {
        // construct outside the cache lock: window design can take seconds and
        // must not block other geometries (as get_flat_window, window.cpp:179-193)
        auto p = std::make_shared<Plan>(n, k, l, q, delta, c128, device);
        std::unique_lock<std::mutex> lk(p->mutex());
        std::lock_guard<std::mutex> g(mu);
        cache[key].push_back(p);
        return PlanLease{p, std::move(lk)};
    }
    std::unique_lock<std::mutex> lk(have.front()->mutex());  // all busy: wait for one
    return PlanLease{have.front(), std::move(lk)};
}

}  // namespace msfft_b200
