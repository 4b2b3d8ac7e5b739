// encode_body.cuh -- K1+K2 for one encode task, shared by encode_kernel
// (one task per CTA) and fused_kernel (persistent CTAs pulling tasks).
// Compiled with --fmad=false.
//
// Reference semantics (bucketize_fn, proj/include/msfft/bucketize.hpp:63-86),
// per round (sigma, tau):
//     for t = -h..h:  fold[t mod b] += g[h+t] * x[sigma*(t - tau) mod n]
//     values = FFT_b(fold) / n
// Rewritten in t' = t - tau: round r reads x[sigma*t'] for t' in
// [-h - tau_r, h - tau_r].  All rounds of one iteration share sigma, so a
// sample needed by several rounds is loaded ONCE: a thread owns the residue
// class t' = c (mod b), walks the union of the rounds' intervals in
// increasing t', and for each covering round r adds g[h + t' + tau_r] * x into
// that round's accumulator, which is bin (c + tau_r) mod b.  Each (round,
// bin) therefore accumulates exactly the reference's terms in exactly the
// reference's order (increasing t), without FMA: the folds are bit-identical
// to the CPU's.  The b-point transform is the reference's radix-2 DIT in
// shared memory (bit-identical as well).
//
// Work split: a task (256 threads) takes one iteration m, a chunk of <= 8
// rounds, and either 256/b whole signals (b <= 256: fused FFT epilogue) or a
// 256-lane slice of one signal (b > 256: folds go to HBM and the batched FFT
// in fft.cu finishes them).  The iteration's window taps are staged into
// shared memory with one TMA bulk copy (cp.async.bulk + mbarrier).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"
#include "plan_dev.cuh"

#ifndef ENC_TL_MARK
#define ENC_TL_MARK(i) do { } while (0)
#endif
#ifndef ENC_TL_BATCH
#define ENC_TL_BATCH() do { } while (0)
#endif

namespace msfft_b200 {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// kKeep: the validating fused kernel streams every sample of the signal
// next to its encode: the gather's load carries an L2 eviction policy
// (createpolicy: evict_last keeps the lines it fetches for the scan)
template <bool kKeep = false>
__device__ __forceinline__ float2 ld_sample(const float2* p, uint64_t pol = 0) {
    if (!kKeep) return __ldcs(p);
    float2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
    return v;
}
template <bool kKeep = false>
__device__ __forceinline__ double2 ld_sample(const double2* p, uint64_t pol = 0) {
    if (!kKeep) return __ldcs(p);
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

// Once per CTA before the first encode_task.
__device__ __forceinline__ void encode_barrier_init(uint64_t* bar) {
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
}

// Sample sources of the gather: the whole signal (x[sigma t' mod n]), an
// index-range shard of it (x holds x[x_lo, x_hi); other samples count as 0),
// or the compact rows of sparse host ingest (x[seg_cpos + t' - seg_lo]).
enum LoadMode { kLoadFull = 0, kLoadShard = 1, kLoadCompact = 2 };

// Walks the task's merged t' segments for residue class c (t' = c mod b) in
// increasing t' and adds g[h + t' + tau_r] * x into acc[r] for every round r
// whose tap interval covers t'.
// kSmemTaps: `taps` points into shared memory (the staged window), so the
// per-(sample, round) tap reads are LDS; otherwise read-only global loads.
// Per batch of U samples the rounds go outermost (nr is uniform, one branch
// per round) and each round's U tap reads are issued together from clamped,
// always-valid indices; only the adds are predicated on the tap interval.
// acc[r] still receives its terms in increasing t' (u ascending within a
// batch, batches ascending), the reference's order.
template <class T, int kMode, bool kSmemTaps, bool kKeep = false>
__device__ __forceinline__ void gather_accumulate(const DevPlan& plan, const EncTask& task,
                                                  const T* __restrict__ xs, uint32_t sg,
                                                  const double* __restrict__ taps, int64_t h,
                                                  uint32_t wu,
                                                  const int64_t* taus, int nr, int64_t b, int c,
                                                  double2 (&acc)[kEncRounds], uint64_t pol = 0) {
    const uint32_t mask = static_cast<uint32_t>(plan.n - 1);
    const uint32_t lo = static_cast<uint32_t>(plan.x_lo);
    const uint32_t span = static_cast<uint32_t>(plan.x_hi - plan.x_lo);
    uint32_t th[kEncRounds];  // tau_r + h: tap index = t' + tau_r + h (mod 2^32)
#pragma unroll
    for (int r = 0; r < kEncRounds; ++r)
        th[r] = r < nr ? static_cast<uint32_t>(taus[r] + h) : 0u;
    const int32_t bm = static_cast<int32_t>(b - 1);
    for (int sgi = 0; sgi < task.nseg; ++sgi) {
        const int32_t A = task.seg_lo[sgi], B = task.seg_hi[sgi];
        const T* cbase = xs + task.seg_cpos[sgi] - A;  // compact: sample of t' at cbase[t']
        int64_t t = A + ((c - A) & bm);
        constexpr int U = 8;
        const int64_t stride = b;
        for (; t <= B; t += U * stride) {
            ENC_TL_BATCH();
            T v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t tt = t + u * stride;
                v[u].x = 0;
                v[u].y = 0;
                if (tt <= B) {
                    if (kMode == kLoadCompact) {
                        MSFFT_DCHECK(task.seg_cpos[sgi] + (tt - A) >= 0 &&
                                     task.seg_cpos[sgi] + (tt - A) < plan.x_row);
                        v[u] = ld_sample<kKeep>(cbase + tt, pol);
                    } else {
                        const uint32_t src = (sg * static_cast<uint32_t>(tt)) & mask;
                        if (kMode == kLoadFull) {
                            v[u] = ld_sample<kKeep>(xs + src, pol);
                        } else {
                            v[u].x = 0;
                            v[u].y = 0;
                            if (src - lo < span) v[u] = ld_sample<kKeep>(xs + (src - lo), pol);
                        }
                    }
                }
            }
            double xr[U], xi[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                xr[u] = static_cast<double>(v[u].x);
                xi[u] = static_cast<double>(v[u].y);
            }
#pragma unroll
            for (int r = 0; r < kEncRounds; ++r) {
                // skip a round whose tap interval misses the whole batch
                const int64_t a = t + static_cast<int64_t>(th[r]);
                if (r < nr && a + (U - 1) * stride >= 0 && a < static_cast<int64_t>(wu)) {
                    double g[U];
                    bool in[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int64_t tt = t + u * stride;
                        const uint32_t idx = static_cast<uint32_t>(tt) + th[r];
                        in[u] = tt <= B && idx < wu;
                        const uint32_t ci = in[u] ? idx : 0u;
                        g[u] = kSmemTaps ? taps[ci] : __ldg(taps + ci);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (in[u]) {
                            acc[r].x += g[u] * xr[u];
                            acc[r].y += g[u] * xi[u];
                        }
                }
            }
        }
    }
}

// One encode task with the whole CTA.  The caller guarantees that no thread
// still uses smem_raw from a previous item (a __syncthreads before).
// `phase` is the mbarrier parity to wait on next; it flips once per staged
// copy.
template <class T>
__device__ __forceinline__ void encode_task(const DevPlan& plan, const EncTask& task,
                                            const T* __restrict__ x, int64_t x_stride,
                                            int64_t batch, const int64_t* __restrict__ sigma,
                                            double2* __restrict__ y, unsigned char* smem_raw,
                                            uint64_t* bar, uint32_t& phase) {
    const DevIter& it = plan.it[task.m];
    const int tid = threadIdx.x;
    const int64_t b = it.b;
    const int log2b = it.log2b;
    const int nr = task.nr;
    const int64_t h = it.h;
    const uint32_t wu = static_cast<uint32_t>(it.w);
    const int64_t* taus = plan.taus + it.tau_off + task.r0;

    // ---- stage the window taps: one TMA bulk copy, completion on an mbarrier
    if (it.taps_in_smem) {
        const uint32_t bytes = static_cast<uint32_t>((it.w + 1) * sizeof(double));
        if (tid == 0) {
            // order earlier generic-proxy use of this smem before the async copy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
            const uint32_t chunk = 32768;
            for (uint32_t off = 0; off < bytes; off += chunk) {
                const uint32_t len = bytes - off < chunk ? bytes - off : chunk;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                    "[%0], [%1], %2, [%3];"
                    ::"r"(smem_u32(smem_raw + off)),
                    "l"(reinterpret_cast<const unsigned char*>(it.taps) + off), "r"(len),
                    "r"(smem_u32(bar))
                    : "memory");
            }
        }
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase)
            : "memory");
        phase ^= 1u;
    }
    ENC_TL_MARK(3);

    // ---- thread -> (signal, residue class)
    int sl, c;
    if (task.fused) {
        sl = tid >> log2b;
        c = tid & static_cast<int>(b - 1);
    } else {
        sl = 0;
        c = task.lane0 + tid;
    }
    const int64_t s = task.sig0 + sl;
    const bool active = sl < task.nsig && s < batch;

    double2 acc[kEncRounds];
#pragma unroll
    for (int r = 0; r < kEncRounds; ++r) acc[r] = make_double2(0.0, 0.0);

    if (active) {
        const uint32_t sg = static_cast<uint32_t>(sigma[s * plan.iters + task.m]);
        const T* xs = x + s * x_stride;
        // the load mode and the tap source are uniform per task: branch once,
        // not per sample
        const double* st = reinterpret_cast<const double*>(smem_raw);
        if (it.taps_in_smem) {
            if (plan.x_compact)
                gather_accumulate<T, kLoadCompact, true>(plan, task, xs, sg, st, h, wu, taus, nr, b, c, acc);
            else if (plan.x_lo == 0 && plan.x_hi == plan.n)
                gather_accumulate<T, kLoadFull, true>(plan, task, xs, sg, st, h, wu, taus, nr, b, c, acc);
            else
                gather_accumulate<T, kLoadShard, true>(plan, task, xs, sg, st, h, wu, taus, nr, b, c, acc);
        } else {
            if (plan.x_compact)
                gather_accumulate<T, kLoadCompact, false>(plan, task, xs, sg, it.taps, h, wu, taus, nr, b, c, acc);
            else if (plan.x_lo == 0 && plan.x_hi == plan.n)
                gather_accumulate<T, kLoadFull, false>(plan, task, xs, sg, it.taps, h, wu, taus, nr, b, c, acc);
            else
                gather_accumulate<T, kLoadShard, false>(plan, task, xs, sg, it.taps, h, wu, taus, nr, b, c, acc);
        }
    }

    ENC_TL_MARK(4);
    const double inv_n = plan.inv_n;
    const int64_t vps = plan.values_per_signal;
    if (!task.fused) {
        if (active) {
            double2* ys = y + s * vps + it.yoff + static_cast<int64_t>(task.r0) * b;
#pragma unroll
            for (int r = 0; r < kEncRounds; ++r)
                if (r < nr) {
                    MSFFT_DCHECK(it.yoff + (task.r0 + r + 1) * b <= vps);
                    ys[static_cast<int64_t>(r) * b + ((c + taus[r]) & (b - 1))] = acc[r];
                }
        }
        return;
    }

    // ---- fused epilogue: b-point radix-2 DIT of every (signal, round) in smem
    __syncthreads();  // taps region is reused for the folds
    double2* F = reinterpret_cast<double2*>(smem_raw);
    const int nsig_cta = kEncThreads >> log2b;
    const int per_sig = nr << log2b;  // nr * b
#pragma unroll
    for (int r = 0; r < kEncRounds; ++r) {
        if (r < nr) {
            const unsigned bin = static_cast<unsigned>((c + taus[r]) & (b - 1));
            F[sl * per_sig + (r << log2b) + bitrev_bits(bin, log2b)] = acc[r];
        }
    }
    __syncthreads();
    const int nbf = (nsig_cta * per_sig) >> 1;
    for (int st = 1; st <= log2b; ++st) {
        const int half = 1 << (st - 1);
        const int step_sh = log2b - st;  // twiddle stride b / 2^st
        for (int bf = tid; bf < nbf; bf += kEncThreads) {
            const int arr = bf >> (log2b - 1);
            const int p = bf & ((1 << (log2b - 1)) - 1);
            const int blk = p >> (st - 1);
            const int off = p & (half - 1);
            const int j = (arr << log2b) + (blk << st) + off;
            const double2 w = it.tw[off << step_sh];
            const double2 x0 = F[j];
            const double2 tv = cmul(F[j + half], w);
            F[j + half] = make_double2(x0.x - tv.x, x0.y - tv.y);
            F[j] = make_double2(x0.x + tv.x, x0.y + tv.y);
        }
        __syncthreads();
    }
    const int total = nsig_cta * per_sig;
    for (int e = tid; e < total; e += kEncThreads) {
        const int es = e / per_sig;
        const int rem = e - es * per_sig;
        const int64_t sig = task.sig0 + es;
        if (es < task.nsig && sig < batch) {
            const double2 v = F[e];
            y[sig * vps + it.yoff + static_cast<int64_t>(task.r0) * b + rem] =
                make_double2(v.x * inv_n, v.y * inv_n);
        }
    }
}

// A packed encode item (validating fused kernel): up to kMaxPack sub-tasks,
// each ONE signal and one iteration with 32 <= b <= 256, side by side on
// warp-aligned thread ranges [tid0, tid0 + b).  Packing iterations of the
// same signal (instead of 256/b signals of one iteration) keeps a CTA's
// random reads inside one or two signals, so they hit the L2 lines the
// validation stream of those signals brings in.  Per sub-task the arithmetic
// is encode_task's (same union walk, same radix-2 DIT), so the folds and
// bucket values are bit-identical to it (kMaxPack sub-tasks at most).

template <class T>
__device__ __forceinline__ void encode_pack(const DevPlan& plan, const EncTask* __restrict__ sub,
                                            int nsub, const T* __restrict__ x, int64_t x_stride,
                                            const int64_t* __restrict__ sigma,
                                            double2* __restrict__ y, unsigned char* smem_raw,
                                            uint64_t* bar, uint32_t& phase, uint64_t pol) {
    const int tid = threadIdx.x;
    // ---- stage the distinct iterations' taps with one mbarrier transaction
    uint32_t bytes_total = 0;
    for (int j = 0; j < nsub; ++j)
        if (sub[j].stage_taps)
            bytes_total += static_cast<uint32_t>((plan.it[sub[j].m].w + 1) * sizeof(double));
    if (bytes_total) {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(smem_u32(bar)), "r"(bytes_total) : "memory");
            for (int j = 0; j < nsub; ++j) {
                if (!sub[j].stage_taps) continue;
                const DevIter& it = plan.it[sub[j].m];
                const uint32_t bytes = static_cast<uint32_t>((it.w + 1) * sizeof(double));
                unsigned char* dst = smem_raw + sub[j].taps_off;
                for (uint32_t off = 0; off < bytes; off += 32768) {
                    const uint32_t len = bytes - off < 32768 ? bytes - off : 32768;
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                        "[%0], [%1], %2, [%3];"
                        ::"r"(smem_u32(dst + off)),
                        "l"(reinterpret_cast<const unsigned char*>(it.taps) + off), "r"(len),
                        "r"(smem_u32(bar))
                        : "memory");
                }
            }
        }
        asm volatile(
            "{\n .reg .pred p;\n WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(phase)
            : "memory");
        phase ^= 1u;
    }

    // ---- thread -> sub-task (warp-uniform: tid0 and b are multiples of 32)
    int j = -1, max_log2b = 0;
    for (int q = 0; q < nsub; ++q) {
        const DevIter& iq = plan.it[sub[q].m];
        max_log2b = iq.log2b > max_log2b ? iq.log2b : max_log2b;
        if (tid >= sub[q].tid0 && tid < sub[q].tid0 + iq.b) j = q;
    }
    const bool active = j >= 0;
    const EncTask& task = sub[active ? j : 0];
    const DevIter& it = plan.it[task.m];
    const int64_t b = it.b;
    const int log2b = it.log2b;
    const int nr = task.nr;
    const int c = tid - task.tid0;
    const int64_t s = task.sig0;
    const int64_t* taus = plan.taus + it.tau_off + task.r0;

    double2 acc[kEncRounds];
#pragma unroll
    for (int r = 0; r < kEncRounds; ++r) acc[r] = make_double2(0.0, 0.0);
    if (active) {
        const uint32_t sg = static_cast<uint32_t>(sigma[s * plan.iters + task.m]);
        const T* xs = x + s * x_stride;
        const int64_t h = it.h;
        const uint32_t wu = static_cast<uint32_t>(it.w);
        if (task.taps_off >= 0)
            gather_accumulate<T, kLoadFull, true, true>(
                plan, task, xs, sg, reinterpret_cast<const double*>(smem_raw + task.taps_off), h,
                wu, taus, nr, b, c, acc, pol);
        else
            gather_accumulate<T, kLoadFull, false, true>(plan, task, xs, sg, it.taps, h, wu, taus,
                                                         nr, b, c, acc, pol);
    }

    // ---- b-point radix-2 DIT of every (sub-task, round) in smem
    __syncthreads();  // the taps region is reused for the arrays
    double2* F = reinterpret_cast<double2*>(smem_raw) + (active ? task.f_off : 0);
    if (active) {
#pragma unroll
        for (int r = 0; r < kEncRounds; ++r)
            if (r < nr) {
                const unsigned bin = static_cast<unsigned>((c + taus[r]) & (b - 1));
                F[(r << log2b) + bitrev_bits(bin, log2b)] = acc[r];
            }
    }
    __syncthreads();
    const int nbf = (nr << log2b) >> 1;
    for (int st = 1; st <= max_log2b; ++st) {
        if (active && st <= log2b) {
            const int half = 1 << (st - 1);
            const int step_sh = log2b - st;
            for (int bf = c; bf < nbf; bf += static_cast<int>(b)) {
                const int arr = bf >> (log2b - 1);
                const int p = bf & ((1 << (log2b - 1)) - 1);
                const int blk = p >> (st - 1);
                const int off = p & (half - 1);
                const int jj = (arr << log2b) + (blk << st) + off;
                const double2 w = it.tw[off << step_sh];
                const double2 x0 = F[jj];
                const double2 tv = cmul(F[jj + half], w);
                F[jj + half] = make_double2(x0.x - tv.x, x0.y - tv.y);
                F[jj] = make_double2(x0.x + tv.x, x0.y + tv.y);
            }
        }
        __syncthreads();
    }
    if (active) {
        const double inv_n = plan.inv_n;
        double2* ys = y + s * plan.values_per_signal + it.yoff + static_cast<int64_t>(task.r0) * b;
        for (int e = c; e < (nr << log2b); e += static_cast<int>(b)) {
            const double2 v = F[e];
            ys[e] = make_double2(v.x * inv_n, v.y * inv_n);
        }
    }
}

}  // namespace
}  // namespace msfft_b200
