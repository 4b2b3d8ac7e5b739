// wide_decode.cu -- see wide_decode.hpp.  Compiled with --fmad=false; every
// value is computed with decode_body.cuh's operations in its order.
#include <algorithm>
#include <cstdlib>
#include <utility>

#include "decode_body.cuh"
#include "wide_decode.hpp"

namespace msfft_b200 {

namespace {

constexpr int kT = 256;               // threads per CTA of the grid kernels
constexpr int kSelBits = 12;           // radix-select digit (last digit: 4 bits)
constexpr int kSelBins = 1 << kSelBits;
constexpr int kScanT = 1024;
constexpr int kLongSeg = 64;          // longer event segments sort with a whole CTA
constexpr int kLongSmem = 8192;

unsigned grid_of(int64_t work) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((work + kT - 1) / kT, 148 * 16)));
}

__device__ __forceinline__ int64_t n_or(const int32_t* n_dev, int64_t n_max) {
    return n_dev ? static_cast<int64_t>(*n_dev) : n_max;
}

// Programmatic dependent launch: every kernel of the decode sequence waits
// for its predecessor's completion (and memory) before touching anything,
// then lets its successor be scheduled, so a kernel's launch overlaps the
// one before it instead of following its completion -- in the stream and in
// the captured graph (programmatic edges).
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <class... KArgs, class... Args>
void launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MSFFT_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

#define GRID_LOOP(i, n) \
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (n); \
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)

__global__ void zero_words(uint32_t* p, int64_t n) {
    pdl_entry();
    GRID_LOOP(i, n) p[i] = 0u;
}

// cudaMemsetAsync(p, 0, bytes) as a kernel of the programmatic chain
void zero_async(bool pdl, void* p, size_t bytes, cudaStream_t st) {
    const int64_t words = static_cast<int64_t>(bytes / 4);
    launch_pdl(pdl, zero_words, grid_of(words), kT, 0, st, static_cast<uint32_t*>(p), words);
}

// ---------------------------------------------------------------- scans
// Exclusive scan of in[0..len) into out (may alias); total -> *total.
// long_list (K3's bucket counts): the indices with more than kLongSeg entries
// are listed as {count, indices...} for the CTA sorter.
// Each warp owns a contiguous segment and walks it in coalesced 32-element
// tiles (warp shuffles scan a tile); a block scan of the warp totals gives
// each segment its offset.
__global__ void __launch_bounds__(kScanT)
scan_kernel(const int32_t* in, int64_t len_max, const int32_t* len_dev, int32_t* out,
            int32_t* total, int32_t* long_list) {
    pdl_entry();
    constexpr int kWarps = kScanT / 32;
    __shared__ int32_t wsum[kWarps];
    const int64_t len = n_or(len_dev, len_max);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t seg = (len + kWarps - 1) / kWarps;
    const int64_t lo = w * seg, hi = std::min<int64_t>(lo + seg, len);
    int32_t s = 0;
#pragma unroll 8
    for (int64_t i = lo + lane; i < hi; i += 32) s += in[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) wsum[w] = s;
    __syncthreads();
    if (w == 0) {
        const int32_t v = wsum[lane];
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        wsum[lane] = x - v;  // exclusive
        if (lane == 31 && total) *total = x;
    }
    __syncthreads();
    int32_t carry = wsum[w];
    for (int64_t t0 = lo; t0 < hi; t0 += 32) {
        const int64_t i = t0 + lane;
        const int32_t v = i < hi ? in[i] : 0;
        int32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (i < hi) out[i] = carry + x - v;
        if (long_list && v > kLongSeg)
            long_list[1 + atomicAdd(&long_list[0], 1)] = static_cast<int32_t>(i);
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
}

// ---------------------------------------------------------------- K3
__global__ void k3_tones(const DevPlan* __restrict__ P, int m, const int64_t* __restrict__ sigma,
                         const int64_t* __restrict__ AF, const double2* __restrict__ AC,
                         const int32_t* __restrict__ acc_n, int64_t* __restrict__ tone_u,
                         int64_t* __restrict__ tone_i, double2* __restrict__ gc,
                         int32_t* __restrict__ cnt, int32_t* __restrict__ cursor,
                         int32_t* __restrict__ long_list, double2* __restrict__ rot) {
    pdl_entry();
    const DevIter& it = P->it[m];
    const int64_t n = acc_n[0];
    const int64_t b = it.b, L = it.l_width, nmask = P->n - 1;
    // clear what k3_scatter / k3_segsort count into (not used before them)
    GRID_LOOP(z, b) cursor[z] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) long_list[0] = 0;
    const double invL = 1.0 / static_cast<double>(L);
    const int64_t sg = sigma[m];
    GRID_LOOP(j, n) {
        const int64_t u = (sg * AF[j]) & nmask;
        const int64_t i = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
        tone_u[j] = u;
        tone_i[j] = i;
        const double2 c = AC[j];
        const unsigned act = __activemask();
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double g = ghat_at(it, (i - 1 + d) * L - u);
            gc[j * 3 + d] = make_double2(g * c.x, g * c.y);
            // lanes with the same target bucket add once (small b: every
            // tone of the warp hits one of a few counters)
            const int bk = static_cast<int>((i - 1 + d) & (b - 1));
            const unsigned same = __match_any_sync(act, bk);
            if ((same & ((1u << lane) - 1u)) == 0) atomicAdd(&cnt[bk], __popc(same));
        }
    }
    // the rotation per (tone, round), u recomputed (k3_rot's values)
    const int nr = it.nrounds;
    const int64_t* taus = P->taus + it.tau_off;
    GRID_LOOP(e, n * nr) {
        const int64_t j = e / nr, r = e - j * nr;
        const int64_t u = (sg * AF[j]) & nmask;
        rot[e] = unit_root(P->n, P->inv_n, taus[r] * u);
    }
}

__global__ void k3_scatter(const DevPlan* __restrict__ P, int m, const int32_t* __restrict__ acc_n,
                           const int64_t* __restrict__ tone_i, const int32_t* __restrict__ start,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ ev) {
    pdl_entry();
    const int64_t b = P->it[m].b;
    const int64_t total = static_cast<int64_t>(acc_n[0]) * 3;
    GRID_LOOP(e, total) {
        const int64_t j = e / 3;
        const int d = static_cast<int>(e - j * 3);
        const int64_t beta = (tone_i[j] - 1 + d) & (b - 1);
        // one atomic per distinct bucket of the warp (the in-bucket order is
        // irrelevant: k3_segsort orders each bucket's events by key)
        const unsigned act = __activemask();
        const int lane = threadIdx.x & 31;
        const unsigned same = __match_any_sync(act, static_cast<int>(beta));
        const int leader = __ffs(same) - 1;
        int32_t base = 0;
        if (lane == leader) base = atomicAdd(&cursor[beta], __popc(same));
        base = __shfl_sync(same, base, leader);
        const int32_t pos = start[beta] + base + __popc(same & ((1u << lane) - 1u));
        MSFFT_DCHECK(pos >= 0 && pos < total && total <= 3 * P->acc_cap);
        ev[pos] = static_cast<int32_t>(j * 4 + d);
    }
}

// Each bucket's events in ascending tone order (keys j*4+d are unique per
// bucket).  One launch, two block roles: the first `long_blocks` CTAs take
// the long segments the scan listed (small b) and the warps of the other CTAs
// take one short segment each by rank counting.  A long segment's keys are
// distinct integers below 4 * acc_n, so they sort through a bitmap in shared
// memory (set a bit per key, popcount prefix over the words, emit the set
// bits in order: five barriers whatever the length); when the key range does
// not fit the buffer, a bitonic network, and rank counting for segments
// beyond the buffer.
constexpr int kLongT = 1024;
__global__ void __launch_bounds__(kLongT)
k3_segsort(const DevPlan* __restrict__ P, int m, const int32_t* __restrict__ start,
           const int32_t* __restrict__ cnt, const int32_t* __restrict__ ev,
           int32_t* __restrict__ ev2, const int32_t* __restrict__ long_list, int long_blocks,
           const int32_t* __restrict__ acc_n) {
    pdl_entry();
    __shared__ int32_t ks[kLongSmem];
    __shared__ int32_t wtot[kLongT / 32];
    if (static_cast<int>(blockIdx.x) >= long_blocks) {
        const int64_t b = P->it[m].b;
        const int lane = threadIdx.x & 31;
        const int64_t warp =
            (static_cast<int64_t>(blockIdx.x - long_blocks) * blockDim.x + threadIdx.x) >> 5;
        const int64_t nwarps = (static_cast<int64_t>(gridDim.x - long_blocks) * blockDim.x) >> 5;
        for (int64_t beta = warp; beta < b; beta += nwarps) {
            const int32_t s0 = start[beta], len = cnt[beta];
            if (len > kLongSeg) continue;  // a long-role CTA sorts it
            for (int32_t e = lane; e < len; e += 32) {
                const int32_t key = ev[s0 + e];
                int32_t rank = 0;
                for (int32_t o = 0; o < len; ++o) rank += ev[s0 + o] < key;
                ev2[s0 + rank] = key;
            }
        }
        return;
    }
    const int32_t nlong = long_list[0];
    const int32_t nwords = (4 * acc_n[0] + 31) >> 5;  // bitmap over the key range
    for (int32_t li = blockIdx.x; li < nlong; li += long_blocks) {
        const int64_t beta = long_list[1 + li];
        const int32_t s0 = start[beta], len = cnt[beta];
        if (nwords <= kLongSmem) {
            uint32_t* bm = reinterpret_cast<uint32_t*>(ks);
            const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
            __syncthreads();  // the previous segment's emit is done
            for (int32_t w = tid; w < nwords; w += kLongT) bm[w] = 0u;
            __syncthreads();
            for (int32_t e = tid; e < len; e += kLongT) {
                const int32_t key = ev[s0 + e];
                MSFFT_DCHECK(key >= 0 && (key >> 5) < nwords);
                atomicOr(&bm[key >> 5], 1u << (key & 31));
            }
            __syncthreads();
            // thread t owns words [t * per, (t + 1) * per)
            const int32_t per = (nwords + kLongT - 1) / kLongT;
            const int32_t w0 = tid * per, w1 = min(nwords, w0 + per);
            int32_t mine = 0;
            for (int32_t w = w0; w < w1; ++w) mine += __popc(bm[w]);
            int32_t x = mine;
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wtot[wid] = x;
            __syncthreads();
            if (wid == 0) {
                const int32_t v = wtot[lane];
                int32_t t = v;
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
                    if (lane >= o) t += y;
                }
                wtot[lane] = t - v;  // exclusive
            }
            __syncthreads();
            int32_t off = s0 + wtot[wid] + x - mine;
            for (int32_t w = w0; w < w1; ++w) {
                uint32_t bits = bm[w];
                while (bits) {
                    const int bpos = __ffs(bits) - 1;
                    bits &= bits - 1;
                    ev2[off++] = (w << 5) + bpos;
                }
            }
            continue;
        }
        if (len > kLongSmem) {
            for (int32_t e = threadIdx.x; e < len; e += kLongT) {
                const int32_t key = ev[s0 + e];
                int32_t rank = 0;
                for (int32_t o = 0; o < len; ++o) rank += ev[s0 + o] < key;
                ev2[s0 + rank] = key;
            }
            continue;
        }
        int32_t pw = 1;
        while (pw < len) pw <<= 1;
        __syncthreads();
        for (int32_t e = threadIdx.x; e < pw; e += kLongT) ks[e] = e < len ? ev[s0 + e] : 0x7fffffff;
        __syncthreads();
        for (int32_t k = 2; k <= pw; k <<= 1) {
            for (int32_t j = k >> 1; j > 0; j >>= 1) {
                // one compare-exchange pair (i, i + j), bit j of i clear, per thread
                for (int32_t t = threadIdx.x; t < (pw >> 1); t += kLongT) {
                    const int32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                    const int32_t l = i + j;
                    const int32_t a = ks[i], c = ks[l];
                    const bool up = (i & k) == 0;
                    if ((a > c) == up) {
                        ks[i] = c;
                        ks[l] = a;
                    }
                }
                __syncthreads();
            }
        }
        for (int32_t e = threadIdx.x; e < len; e += kLongT) ev2[s0 + e] = ks[e];
    }
}

// The prediction of every (round, bucket), summed in ascending-f order
// (decode_body.cuh K3).  A warp takes up to 32 consecutive (round, bucket)
// pairs, one per lane: a lane sums a short event list (<= kK3Short events, the
// sparse iterations) by itself; the long lists (small b) are then summed by
// the whole warp one after another -- lanes stage 32 contributions at a time,
// lane 0 adds them in order, and the next chunk's operands load meanwhile.
constexpr int kK3Short = 8;
__global__ void __launch_bounds__(kT)
k3_sum(const DevPlan* __restrict__ P, int m, const int32_t* __restrict__ start,
       const int32_t* __restrict__ cnt, const int32_t* __restrict__ ev2,
       const double2* __restrict__ gc, const double2* __restrict__ rot, double2* __restrict__ Y) {
    pdl_entry();
    __shared__ double2 stage[kT];
    const DevIter& it = P->it[m];
    const int64_t b = it.b;
    const int nr = it.nrounds;
    const int64_t total = static_cast<int64_t>(nr) * b;
    const int lane = threadIdx.x & 31;
    const int wslot = threadIdx.x & ~31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    // pairs per warp: as few as the grid allows (one when warps >= pairs,
    // so the long lists of small b run one per warp in parallel)
    const int64_t per = std::min<int64_t>(32, (total + nwarps - 1) / nwarps);
    for (int64_t base = warp * per; base < total; base += nwarps * per) {
        const int64_t e = base + lane;
        int32_t s0 = 0, len = 0;
        int r = 0;
        if (lane < per && e < total) {
            r = static_cast<int>(e / b);
            const int64_t beta = e - static_cast<int64_t>(r) * b;
            s0 = start[beta];
            len = cnt[beta];
        }
        if (len > 0 && len <= kK3Short) {
            double2 pred = make_double2(0.0, 0.0);
            for (int32_t q = 0; q < len; ++q) {
                const int32_t key = ev2[s0 + q];
                const double2 v = cmul(gc[(key >> 2) * 3 + (key & 3)],
                                       rot[static_cast<int64_t>(key >> 2) * nr + r]);
                pred.x += v.x;
                pred.y += v.y;
            }
            const double2 o = Y[e];
            Y[e] = make_double2(o.x - pred.x, o.y - pred.y);
        }
        unsigned long_mask = __ballot_sync(0xffffffffu, len > kK3Short);
        while (long_mask) {
            const int src = __ffs(long_mask) - 1;
            long_mask &= long_mask - 1;
            const int32_t ls0 = __shfl_sync(0xffffffffu, s0, src);
            const int32_t llen = __shfl_sync(0xffffffffu, len, src);
            const int lr = __shfl_sync(0xffffffffu, r, src);
            double2 pred = make_double2(0.0, 0.0);
            // software-pipelined: while lane 0 adds chunk c, the lanes' loads of
            // the operands of chunks c+1 and c+2 and of chunk c+3's event keys
            // are in flight (an operand load follows its key load, two L2
            // round trips; one chunk of adds covers about one)
            const auto key_at = [&](int32_t c) { return c + lane < llen ? ev2[ls0 + c + lane] : -1; };
            const auto operands = [&](int32_t key, double2& g, double2& rr) {
                g = make_double2(0.0, 0.0);
                rr = g;
                if (key >= 0) {
                    g = gc[(key >> 2) * 3 + (key & 3)];
                    rr = rot[static_cast<int64_t>(key >> 2) * nr + lr];
                }
            };
            double2 g0, r0, g1, r1;
            int32_t key2 = key_at(64);
            operands(key_at(0), g0, r0);
            operands(key_at(32), g1, r1);
            for (int32_t c0 = 0; c0 < llen; c0 += 32) {
                const int32_t take = min(32, llen - c0);
                const int32_t key3 = key_at(c0 + 96);
                double2 g2, r2;
                operands(key2, g2, r2);
                if (lane < take) stage[threadIdx.x] = cmul(g0, r0);
                __syncwarp();
                if (lane == 0)
                    for (int l = 0; l < take; ++l) {
                        const double2 v = stage[wslot + l];
                        pred.x += v.x;
                        pred.y += v.y;
                    }
                __syncwarp();
                g0 = g1;
                r0 = r1;
                g1 = g2;
                r1 = r2;
                key2 = key3;
            }
            if (lane == 0) {
                const int64_t le = base + src;
                const double2 o = Y[le];
                Y[le] = make_double2(o.x - pred.x, o.y - pred.y);
            }
        }
    }
}

// ---------------------------------------------------------------- select
// keys: value bits + 1 for |.| >= 0 (NaN -> 0, ranks last); larger = earlier.
// The launch also prepares what the kernels after it need, so no launch is
// spent on it: (zero_p, zero_n) words cleared (the K4 rank counters), and the
// radix select's state -- sel = {prefix, prefix mask, rank remaining, blocks
// done} with rank = min(kth_dev ? *kth_dev : unbounded, kth_host, cap_kth),
// also stored to *kth_out (K7's keep count), and a clear digit histogram
// (each select pass's last block clears it again for the next).
__global__ void keys_from_values(const double2* __restrict__ v, int64_t n_max,
                                 const int32_t* __restrict__ n_dev, double* __restrict__ mag,
                                 uint64_t* __restrict__ key, uint32_t* __restrict__ zero_p,
                                 int64_t zero_n, uint64_t* __restrict__ sel,
                                 uint32_t* __restrict__ hist, int64_t kth_host,
                                 const int32_t* __restrict__ kth_dev, int64_t cap_kth,
                                 int32_t* __restrict__ kth_out) {
    pdl_entry();
    GRID_LOOP(i, zero_n) zero_p[i] = 0u;
    GRID_LOOP(i, kSelBins) hist[i] = 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        int64_t kth = kth_host;
        if (kth_dev && *kth_dev < kth) kth = *kth_dev;
        if (kth > cap_kth) kth = cap_kth;
        if (kth_out) *kth_out = static_cast<int32_t>(kth);
        sel[0] = 0;
        sel[1] = 0;
        sel[2] = static_cast<uint64_t>(kth);
        sel[3] = 0;
    }
    const int64_t n = n_or(n_dev, n_max);
    GRID_LOOP(j, n) {
        const double2 x = v[j];
        const double mg = cabs_ref(x.x, x.y);
        if (mag) mag[j] = mg == mg ? mg : -1.0;
        key[j] = mg == mg ? static_cast<uint64_t>(__double_as_longlong(mg)) + 1ull : 0ull;
    }
}

// One radix-select digit in one launch: every block histograms its keys
// (those matching the prefix) into the global histogram; the last block to
// finish picks the digit of the kth largest (suffix counts over the bins), updates sel,
// and clears the histogram and the block count for the next digit.
__global__ void __launch_bounds__(kT)
sel_digit(const uint64_t* __restrict__ key, int64_t n_max, const int32_t* __restrict__ n_dev,
          uint64_t* sel, int shift, int width, uint32_t* hist) {
    pdl_entry();
    __shared__ uint32_t h[kSelBins];
    __shared__ uint64_t part[kT];
    __shared__ int last;
    const int64_t n = n_or(n_dev, n_max);
    const uint64_t prefix = sel[0], mask = sel[1], remaining = sel[2];
    if (remaining == 0) return;  // uniform: every block returns, hist stays clear
    const uint64_t dmask = (uint64_t{1} << width) - 1;
    for (int i = threadIdx.x; i < kSelBins; i += kT) h[i] = 0;
    __syncthreads();
    GRID_LOOP(j, n) {
        const uint64_t k = key[j];
        if ((k & mask) == prefix) atomicAdd(&h[(k >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSelBins; i += kT)
        if (h[i]) atomicAdd(&hist[i], h[i]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(reinterpret_cast<unsigned long long*>(&sel[3]), 1ull) ==
               static_cast<unsigned long long>(gridDim.x) - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    constexpr int per = kSelBins / kT;
    const int t = threadIdx.x;
    uint32_t hv[per];
    uint64_t s = 0;
#pragma unroll
    for (int i = 0; i < per; ++i) {
        hv[i] = __ldcg(&hist[t * per + i]);
        s += hv[i];
    }
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < kT; o <<= 1) {  // suffix sums over threads >= t
        const uint64_t v = t + o < kT ? part[t + o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    const uint64_t above = part[t] - s;  // keys in higher bins
    if (above < remaining && remaining <= above + s) {
        uint64_t cum = above;
#pragma unroll
        for (int i = per - 1; i >= 0; --i) {
            if (cum + hv[i] >= remaining && cum < remaining) {
                sel[0] = prefix | static_cast<uint64_t>(t * per + i) << shift;
                sel[1] = mask | ((uint64_t{1} << width) - 1) << shift;
                sel[2] = remaining - cum;
            }
            cum += hv[i];
        }
    }
    for (int i = t; i < kSelBins; i += kT) hist[i] = 0u;
    if (t == 0) sel[3] = 0;
}

// The low 40 bits of the selection in one CTA: the keys matching the
// 24-bit prefix of the first two digits are gathered into shared memory
// (read from global memory each pass if they do not fit), then four 10-bit
// digits are picked with sel_digit's rule.  The final sel (full key, full
// mask, rank among equal keys) is the one the remaining 12-bit digits give.
constexpr int kFinT = 1024;
constexpr int kFinCap = 4096;
__global__ void __launch_bounds__(kFinT)
sel_finish(const uint64_t* __restrict__ key, int64_t n_max, const int32_t* __restrict__ n_dev,
           uint64_t* sel) {
    pdl_entry();
    __shared__ uint64_t cand[kFinCap];
    __shared__ uint32_t hist[kFinT];
    __shared__ uint32_t part[kFinT];
    __shared__ int cnt;
    __shared__ uint64_t s_prefix, s_mask, s_rem;
    const int t = threadIdx.x;
    if (t == 0) {
        cnt = 0;
        s_prefix = sel[0];
        s_mask = sel[1];
        s_rem = sel[2];
    }
    __syncthreads();
    if (s_rem == 0) return;  // uniform
    const int64_t n = n_or(n_dev, n_max);
    {
        const uint64_t pf = s_prefix, mk = s_mask;
        for (int64_t j = t; j < n; j += kFinT) {
            const uint64_t k = key[j];
            if ((k & mk) == pf) {
                const int p = atomicAdd(&cnt, 1);
                if (p < kFinCap) cand[p] = k;
            }
        }
    }
    __syncthreads();
    const int c = cnt;
    const bool in_smem = c <= kFinCap;
    for (int shift = 30; shift >= 0; shift -= 10) {
        hist[t] = 0;
        __syncthreads();
        const uint64_t pf = s_prefix, mk = s_mask;
        if (in_smem) {
            for (int i = t; i < c; i += kFinT) {
                const uint64_t k = cand[i];
                if ((k & mk) == pf) atomicAdd(&hist[(k >> shift) & 1023u], 1u);
            }
        } else {
            for (int64_t j = t; j < n; j += kFinT) {
                const uint64_t k = key[j];
                if ((k & mk) == pf) atomicAdd(&hist[(k >> shift) & 1023u], 1u);
            }
        }
        __syncthreads();
        const uint32_t hv = hist[t];
        part[t] = hv;
        __syncthreads();
        for (int o = 1; o < kFinT; o <<= 1) {  // suffix sums over bins >= t
            const uint32_t v = t + o < kFinT ? part[t + o] : 0u;
            __syncthreads();
            part[t] += v;
            __syncthreads();
        }
        const uint64_t above = part[t] - hv;  // keys in higher bins
        const uint64_t rem = s_rem;
        __syncthreads();  // every thread has read s_rem before it changes
        if (above < rem && rem <= above + hv) {
            s_prefix = pf | static_cast<uint64_t>(t) << shift;
            s_mask = mk | uint64_t{1023} << shift;
            s_rem = rem - above;
        }
        __syncthreads();
    }
    if (t == 0) {
        sel[0] = s_prefix;
        sel[1] = s_mask;
        sel[2] = s_rem;
    }
}

// Ordered compaction in one launch: indices of the keys > thr and of the
// first need_eq keys == thr (sel = {thr, mask, need_eq, ...} after the
// select), in index order.  Blocks draw their chunk from a ticket, publish
// the chunk's (> thr, == thr) counts in one flagged word, and sum the words
// of the chunks before theirs -- published by blocks that drew earlier
// tickets, so they are running or done and the wait cannot deadlock -- then
// write their own slice.  The last block out clears the words and the ticket
// for the next use.
constexpr int kCChunk = 1024;
__global__ void __launch_bounds__(kT)
sel_compact(const uint64_t* __restrict__ key, int64_t n_max, const int32_t* __restrict__ n_dev,
            const uint64_t* __restrict__ sel, unsigned long long* __restrict__ pub,
            int32_t* __restrict__ ctl, int32_t* __restrict__ out_idx) {
    pdl_entry();
    __shared__ int warp_sel[kT / 32], warp_eq[kT / 32];
    __shared__ int64_t run_sel, run_eq;
    __shared__ int s_bid, gt_s, eq_s, s_last;
    const int64_t n = n_or(n_dev, n_max);
    const uint64_t thr = sel[0];
    const int64_t need_eq = static_cast<int64_t>(sel[2]);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        s_bid = atomicAdd(&ctl[0], 1);
        gt_s = eq_s = 0;
    }
    __syncthreads();
    const int bid = s_bid;
    const int64_t base = static_cast<int64_t>(bid) * kCChunk;
    constexpr int kR = kCChunk / kT;
    uint64_t kreg[kR];
    int gt = 0, eq = 0;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const int64_t j = base + static_cast<int64_t>(r) * kT + threadIdx.x;
        kreg[r] = j < n ? key[j] : 0ull;
        gt += j < n && kreg[r] > thr;
        eq += j < n && kreg[r] == thr;
    }
    for (int o = 16; o > 0; o >>= 1) {
        gt += __shfl_xor_sync(0xffffffffu, gt, o);
        eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    if (lane == 0) {
        atomicAdd(&gt_s, gt);
        atomicAdd(&eq_s, eq);
    }
    __syncthreads();
    if (threadIdx.x == 0)
        *reinterpret_cast<volatile unsigned long long*>(&pub[bid]) =
            (1ull << 63) | (static_cast<unsigned long long>(gt_s) << 31) |
            static_cast<unsigned long long>(eq_s);
    if (wid == 0) {
        int64_t g = 0, e = 0;
        for (int q = lane; q < bid; q += 32) {
            unsigned long long w;
            do {
                w = *reinterpret_cast<volatile unsigned long long*>(&pub[q]);
            } while (!(w >> 63));
            g += static_cast<int64_t>((w >> 31) & 0x7fffffffull);
            e += static_cast<int64_t>(w & 0x7fffffffull);
        }
        for (int o = 16; o > 0; o >>= 1) {
            g += __shfl_xor_sync(0xffffffffu, g, o);
            e += __shfl_xor_sync(0xffffffffu, e, o);
        }
        if (lane == 0) {
            run_sel = g + std::min<int64_t>(e, need_eq);
            run_eq = e;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const int64_t j = base + static_cast<int64_t>(r) * kT + threadIdx.x;
        const uint64_t k = kreg[r];
        const bool is_eq = j < n && k == thr;
        const bool is_gt = j < n && k > thr;
        const unsigned eq_mask = __ballot_sync(0xffffffffu, is_eq);
        if (lane == 0) warp_eq[wid] = __popc(eq_mask);
        __syncthreads();
        int eq_before = __popc(eq_mask & ((1u << lane) - 1u)), eq_total = 0;
        for (int w = 0; w < kT / 32; ++w) {
            if (w < wid) eq_before += warp_eq[w];
            eq_total += warp_eq[w];
        }
        const bool take = is_gt || (is_eq && run_eq + eq_before < need_eq);
        const unsigned sel_mask = __ballot_sync(0xffffffffu, take);
        if (lane == 0) warp_sel[wid] = __popc(sel_mask);
        __syncthreads();
        int sel_before = __popc(sel_mask & ((1u << lane) - 1u)), sel_total = 0;
        for (int w = 0; w < kT / 32; ++w) {
            if (w < wid) sel_before += warp_sel[w];
            sel_total += warp_sel[w];
        }
        if (take) out_idx[run_sel + sel_before] = static_cast<int32_t>(j);
        __syncthreads();
        if (threadIdx.x == 0) {
            run_sel += sel_total;
            run_eq += eq_total;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ctl[1], 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (s_last) {
        for (int q = threadIdx.x; q < static_cast<int>(gridDim.x); q += kT) pub[q] = 0ull;
        if (threadIdx.x == 0) {
            ctl[0] = 0;
            ctl[1] = 0;
        }
    }
}

// ---------------------------------------------------------------- K4
// rank among the selected buckets by (|y0| desc, bucket asc): blockIdx.x
// tiles the elements, blockIdx.y the comparison range; partial ranks add up.
// Compared through the select keys (the magnitude's bit pattern + 1, NaN -> 0:
// the same order as the magnitudes with NaN as -1), high words first: almost
// every pair is decided by one 32-bit integer compare instead of two FP64
// compares on the half-rate pipe.
__global__ void __launch_bounds__(kT)
k4_rank(const int32_t* __restrict__ sel_idx, int64_t budget, const uint64_t* __restrict__ key,
        int32_t* __restrict__ rank_out) {
    pdl_entry();
    __shared__ uint32_t th[kT], tl[kT];
    __shared__ int32_t ti[kT];
    const int64_t e = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int32_t idx = e < budget ? sel_idx[e] : 0;
    const uint64_t kj = e < budget ? key[idx] : 0ull;
    const uint32_t hj = static_cast<uint32_t>(kj >> 32), lj = static_cast<uint32_t>(kj);
    const int64_t span = (budget + gridDim.y - 1) / gridDim.y;
    const int64_t c0 = blockIdx.y * span, c1 = std::min<int64_t>(c0 + span, budget);
    int32_t rank = 0;
    for (int64_t t0 = c0; t0 < c1; t0 += kT) {
        __syncthreads();
        if (t0 + threadIdx.x < c1) {
            const int32_t o = sel_idx[t0 + threadIdx.x];
            const uint64_t ko = key[o];
            ti[threadIdx.x] = o;
            th[threadIdx.x] = static_cast<uint32_t>(ko >> 32);
            tl[threadIdx.x] = static_cast<uint32_t>(ko);
        }
        __syncthreads();
        const int lim = static_cast<int>(std::min<int64_t>(kT, c1 - t0));
#pragma unroll 8
        for (int q = 0; q < lim; ++q) {
            const uint32_t hq = th[q];
            rank += hq > hj;
            if (hq == hj) {
                const uint32_t lq = tl[q];
                rank += (lq > lj) || (lq == lj && ti[q] < idx);
            }
        }
    }
    if (e < budget && rank) atomicAdd(&rank_out[e], rank);
}

// The last-ranked selection also gives the 0.2 * kth threshold.
__global__ void k4_scatter(const int32_t* __restrict__ sel_idx, const int32_t* __restrict__ rank,
                           int64_t budget, int32_t* __restrict__ order,
                           const double* __restrict__ mag, double* __restrict__ thr) {
    pdl_entry();
    GRID_LOOP(e, budget) {
        MSFFT_DCHECK(rank[e] >= 0 && rank[e] < budget);
        const int32_t r = rank[e], idx = sel_idx[e];
        order[r] = idx;
        if (r == budget - 1) *thr = 0.2 * mag[idx];
    }
}

// b <= 1024: the whole selection in one CTA -- |y0| (NaN -> -1), stable rank
// by (|y0| desc, bucket asc) of every bucket, order[rank] for the ranked
// ones and the 0.2 * kth threshold (decode_body.cuh K4, small path).
constexpr int kSmallK4 = 1024;
__global__ void __launch_bounds__(kSmallK4)
k4_small(const DevPlan* __restrict__ P, int m, const double2* __restrict__ Y,
         double* __restrict__ mag, int32_t* __restrict__ order, double* __restrict__ thr) {
    pdl_entry();
    __shared__ double sm[kSmallK4];
    const DevIter& it = P->it[m];
    const int b = static_cast<int>(it.b);
    const int64_t budget = it.budget;
    const int j = threadIdx.x;
    double mj = 0.0;
    if (j < b) {
        const double2 v = Y[j];
        const double mg = cabs_ref(v.x, v.y);
        mj = mg == mg ? mg : -1.0;
        sm[j] = mj;
        mag[j] = mj;
    }
    // rank order (|y0| desc, bucket asc) by a bitonic sort of (magnitude,
    // bucket) pairs; padding (-2 < every magnitude and the NaN sentinel -1)
    // sorts last
    static_assert((kSmallK4 & (kSmallK4 - 1)) == 0, "bitonic size");
    __shared__ int32_t si[kSmallK4];
    if (j >= b) sm[j] = -2.0;
    si[j] = j;
    __syncthreads();
    int pw = 2;
    while (pw < b) pw <<= 1;
    for (int k = 2; k <= pw; k <<= 1) {
        for (int h = k >> 1; h > 0; h >>= 1) {
            const int p = j ^ h;
            if (p > j && p < pw) {
                const double ma = sm[j], mb = sm[p];
                const int ia = si[j], ib = si[p];
                const bool p_first = (mb > ma) || (mb == ma && ib < ia);
                if (p_first == ((j & k) == 0)) {
                    sm[j] = mb;
                    sm[p] = ma;
                    si[j] = ib;
                    si[p] = ia;
                }
            }
            __syncthreads();
        }
    }
    if (j < budget) order[j] = si[j];
    if (j == budget - 1) *thr = 0.2 * sm[j];
}

// ---------------------------------------------------------------- K5
// Every ranked bucket's round values staged in rank order, and the phases
// of y0 / y_tau per (rank, stage) -- both read Y directly, so one launch.
__global__ void k5_stage_phase(const DevPlan* __restrict__ P, int m,
                               const int32_t* __restrict__ order, const double2* __restrict__ Y,
                               double2* __restrict__ yr, double* __restrict__ phi,
                               int32_t* __restrict__ pcode, uint32_t* __restrict__ zero_a,
                               int64_t zero_an, uint32_t* __restrict__ zero_b, int64_t zero_bn) {
    pdl_entry();
    // counters of later kernels of the chain, free by now: this iteration's
    // K6 order counters and the next iteration's K3 bucket counts
    GRID_LOOP(i, zero_an) zero_a[i] = 0u;
    GRID_LOOP(i, zero_bn) zero_b[i] = 0u;
    const DevIter& it = P->it[m];
    const int nr = it.nrounds, ns = nr - 1;
    const int64_t total = it.budget * nr;
    GRID_LOOP(e, total) {
        const int64_t rk = e / nr, st = e - rk * nr;
        const int64_t beta = order[rk];
        const double2 yt = Y[st * it.b + beta];
        yr[e] = yt;
        if (st == 0) continue;
        const double2 y0e = Y[beta];
        int code = 0;
        double ph = 0.0;
        if (yt.x == 0.0 && yt.y == 0.0) {
            code = 1;
        } else {
            const double2 z = cdiv_ref(y0e.x, y0e.y, yt.x, yt.y);
            if (z.x == 0.0 && z.y == 0.0) code = 2;
            ph = atan2(z.y, z.x);
            if (ph < 0.0) ph += kTwoPi;
            ph = ph + 0.0;
        }
        const int64_t pe = rk * ns + (st - 1);
        phi[pe] = ph;
        pcode[pe] = code;
    }
}

// One lane group per ranked bucket (decode_body.cuh K5 + K6 estimate).
constexpr int kK5Stage = 1024;  // (lane groups per CTA) x (stages) staged in shared memory
__global__ void __launch_bounds__(kT)
k5_locate(const DevPlan* __restrict__ P, int m, const int64_t* __restrict__ sigma_inv,
          const int32_t* __restrict__ order, const double* __restrict__ mag,
          const double* __restrict__ thr_p, const double2* __restrict__ yr,
          const double* __restrict__ phi_t, const int32_t* __restrict__ pcode,
          int64_t* __restrict__ cand_f, double2* __restrict__ cand_v, int32_t* __restrict__ err,
          const double2* __restrict__ Y, uint32_t* __restrict__ zero_a, int64_t zero_an,
          uint32_t* __restrict__ zero_b, int64_t zero_bn) {
    pdl_entry();
    // Y != nullptr: no k5_stage_phase launch ran -- each lane group computes
    // its bucket's stage phases into shared memory itself (k5_stage_phase's
    // arithmetic), and this launch clears the counters that kernel would
    GRID_LOOP(i, zero_an) zero_a[i] = 0u;
    GRID_LOOP(i, zero_bn) zero_b[i] = 0u;
    __shared__ double s_phi[kK5Stage];
    __shared__ int32_t s_code[kK5Stage];
    const DevIter& it = P->it[m];
    const int64_t n = P->n, nmask = n - 1;
    const double inv_n = P->inv_n;
    const int64_t L = it.l_width;
    const double Ld = static_cast<double>(L), invL = 1.0 / Ld;
    const int nr = it.nrounds, ns = nr - 1;
    const int64_t* taus = P->taus + it.tau_off;
    const int64_t budget = it.budget;
    const int64_t lcfg = P->l;
    const double q = P->q;
    const double thr = *thr_p;
    const int64_t sgi = sigma_inv[m];
    const int gsz = lcfg > 16 ? 32 : (lcfg > 8 ? 16 : (lcfg > 4 ? 8 : 4));
    const int lane = threadIdx.x & 31;
    const int glane = lane & (gsz - 1);
    // stage tables in shared memory for the short chain (decode_body.cuh
    // locate_stages), when the schedule fits them
    __shared__ double s_blk[kMaxStageTable];
    __shared__ int64_t s_tau[kMaxStageTable + 1];
    const int nst_all = it.nstage_tab;
    const int64_t jpl = (lcfg + gsz - 1) / gsz;
    const bool fast = nst_all >= 0 && nst_all < kMaxStageTable && nst_all < nr &&
                      locate_fast_ok(gsz, jpl);
    if (fast) {
        if (threadIdx.x < nst_all) s_blk[threadIdx.x] = it.stage_blk[threadIdx.x];
        if (threadIdx.x <= nst_all) s_tau[threadIdx.x] = taus[threadIdx.x];
        __syncthreads();
    }
    const int64_t gid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / gsz;
    const int64_t ngroups = (static_cast<int64_t>(gridDim.x) * blockDim.x) / gsz;
    const int64_t rounds_up = (budget + ngroups - 1) / ngroups * ngroups;
    for (int64_t rank = gid; rank < rounds_up; rank += ngroups) {
        // whole warp past the budget: skip (warp-uniform)
        const int64_t warp_first = rank - (lane / gsz);
        if (warp_first >= budget) continue;
        const bool live = rank < budget;
        const int64_t beta = live ? order[rank] : 0;
        int64_t f_out = -1;
        double2 v_out = make_double2(0.0, 0.0);
        double2 y0 = make_double2(0.0, 0.0);
        const double* phi_r = phi_t + rank * ns;
        const int32_t* code_r = pcode + rank * ns;
        if (Y) {
            double* my_phi = s_phi + (threadIdx.x / gsz) * ns;
            int32_t* my_code = s_code + (threadIdx.x / gsz) * ns;
            __syncwarp();  // the previous rank's chain is done with the slices
            if (live) {
                y0 = Y[beta];
                for (int st = 1 + glane; st < nr; st += gsz) {
                    const double2 yt = Y[st * it.b + beta];
                    int code = 0;
                    double ph = 0.0;
                    if (yt.x == 0.0 && yt.y == 0.0) {
                        code = 1;
                    } else {
                        const double2 z = cdiv_ref(y0.x, y0.y, yt.x, yt.y);
                        if (z.x == 0.0 && z.y == 0.0) code = 2;
                        ph = atan2(z.y, z.x);
                        if (ph < 0.0) ph += kTwoPi;
                        ph = ph + 0.0;
                    }
                    my_phi[st - 1] = ph;
                    my_code[st - 1] = code;
                }
            }
            __syncwarp();
            phi_r = my_phi;
            code_r = my_code;
        } else if (live) {
            y0 = yr[rank * nr];
        }
        bool ok = live && mag[beta] > thr;
        if (ok && y0.x == 0.0 && y0.y == 0.0) ok = false;
        double u_min = (2.0 * static_cast<double>(beta) - 1.0) * Ld / 2.0;
        double len = Ld;
        int stage = 0;
        const int nst = it.nstage_tab;
        if (fast) {
            u_min = locate_stages_dispatch(gsz, jpl, u_min, nst, live, ok, glane, lcfg, q / 2.0,
                                           inv_n, phi_r, code_r, s_blk, s_tau, err);
            if (nst > 0) len = it.stage_len[nst];
            stage = nst;  // the loop below has nothing left
        }
        while (!fast && (nst >= 0 ? stage < nst : len > 1.0 + 1e-9)) {
            ++stage;
            if (stage >= nr) {
                if (ok && glane == 0) atomicCAS(err, 0, kDecErrRounds);
                ok = false;
                break;
            }
            double ph = 0.0;
            if (ok) {
                const int pe = stage - 1;
                const int code = code_r[pe];
                if (code == 1) {
                    ok = false;
                } else {
                    if (code == 2) {
                        if (glane == 0) atomicCAS(err, 0, kDecErrPhaseZero);
                        ok = false;
                    }
                    ph = phi_r[pe];
                }
            }
            const int64_t tau = taus[stage];
            const double rblk = nst >= 0 ? it.stage_blk[stage - 1] : len / static_cast<double>(lcfg);
            double best_d = INFINITY;
            int best_j = 0x7fffffff;
            for (int64_t j = glane; j < lcfg; j += gsz) {
                const double center = u_min + (static_cast<double>(j) + 0.5) * rblk;
                const double d = circular_phase_distance(position_phase(center, tau, n, inv_n), ph);
                if (d < best_d) {
                    best_d = d;
                    best_j = static_cast<int>(j);
                }
            }
            for (int o = gsz >> 1; o > 0; o >>= 1) {
                const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
                const int oj = __shfl_xor_sync(0xffffffffu, best_j, o);
                if (od < best_d || (od == best_d && oj < best_j)) {
                    best_d = od;
                    best_j = oj;
                }
            }
            if (best_j == 0x7fffffff) best_j = 0;
            u_min = u_min + (static_cast<double>(best_j) - q / 2.0) * rblk;
            len = nst >= 0 ? it.stage_len[stage] : len * (q + 1.0) / static_cast<double>(lcfg);
        }
        if (ok) {
            const double lo = u_min, hi = u_min + len;
            int64_t u = static_cast<int64_t>(ceil(lo));
            if (!(static_cast<double>(u) < hi)) u = llround(0.5 * (lo + hi));
            u &= nmask;  // u mod n (n is a power of two): locate.cpp:120-121
            const int64_t i = static_cast<int64_t>(floor(static_cast<double>(u) * invL + 0.5));
            const double g = ghat_at(it, i * L - u);
            if (!(fabs(g) < 0.5)) {
                v_out = make_double2(y0.x / g, y0.y / g);
                f_out = (sgi * u) & nmask;
            }
        }
        if (live && glane == 0) {
            cand_f[rank] = f_out;
            cand_v[rank] = v_out;
        }
    }
}

// ---------------------------------------------------------------- K6
// position of each accepted candidate in (f, rank) order (2-D split as
// k4_rank), then byf[pos] = rank.
__global__ void __launch_bounds__(kT)
k6_sortf(const int64_t* __restrict__ cand_f, int64_t budget, int32_t* __restrict__ pos_out) {
    pdl_entry();
    __shared__ int64_t tf[kT];
    const int64_t r = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int64_t fr = r < budget ? cand_f[r] : -1;
    const int64_t span = (budget + gridDim.y - 1) / gridDim.y;
    const int64_t c0 = blockIdx.y * span, c1 = std::min<int64_t>(c0 + span, budget);
    int32_t pos = 0;
    for (int64_t t0 = c0; t0 < c1; t0 += kT) {
        __syncthreads();
        if (t0 + threadIdx.x < c1) tf[threadIdx.x] = cand_f[t0 + threadIdx.x];
        __syncthreads();
        const int lim = static_cast<int>(std::min<int64_t>(kT, c1 - t0));
        for (int qq = 0; qq < lim; ++qq) {
            const int64_t fo = tf[qq];
            pos += fo >= 0 && (fo < fr || (fo == fr && t0 + qq < r));
        }
    }
    if (r < budget && fr >= 0 && pos) atomicAdd(&pos_out[r], pos);
}

// Large budgets: (f, rank) order by a bucket sort on the top 12 bits of f
// (the f are near-uniform on [0, n)): counts, a scan, a scatter, then each
// bucket's few entries ranked by (f, rank).  Buckets ascend in f, so byf is
// exactly the order k6_sortf + k6_scatter give.
constexpr int kF6B = 4096;
constexpr int64_t kF6BucketMin = 2048;  // budgets from here use the bucket sort

__global__ void k6b_count(const int64_t* __restrict__ cand_f, int64_t budget, int shift,
                          int32_t* __restrict__ cnt, int32_t* __restrict__ cursor,
                          int32_t* __restrict__ naccepted) {
    pdl_entry();
    GRID_LOOP(z, kF6B) cursor[z] = 0;  // used from k6b_scatter on
    GRID_LOOP(r, budget) {
        const int64_t f = cand_f[r];
        const unsigned act = __activemask();
        const unsigned acc = __ballot_sync(act, f >= 0);
        if (f >= 0) atomicAdd(&cnt[f >> shift], 1);
        if ((threadIdx.x & 31) == __ffs(act) - 1 && acc) atomicAdd(naccepted, __popc(acc));
    }
}

__global__ void k6b_scatter(const int64_t* __restrict__ cand_f, int64_t budget, int shift,
                            const int32_t* __restrict__ start, int32_t* __restrict__ cursor,
                            int32_t* __restrict__ tmp, int64_t* __restrict__ tmpf) {
    pdl_entry();
    GRID_LOOP(r, budget) {
        const int64_t f = cand_f[r];
        if (f < 0) continue;
        const int64_t bk = f >> shift;
        const int32_t q = start[bk] + atomicAdd(&cursor[bk], 1);
        tmp[q] = static_cast<int32_t>(r);
        tmpf[q] = f;  // the key beside the rank: k6b_sort streams (f, rank) pairs
    }
}

__global__ void k6b_sort(int shift, const int32_t* __restrict__ start,
                         const int32_t* __restrict__ cnt, const int32_t* __restrict__ tmp,
                         const int64_t* __restrict__ tmpf, int32_t* __restrict__ byf) {
    pdl_entry();
    // one thread per accepted entry (start[kF6B] of them), ranked within its
    // bucket by streaming the bucket's (f, rank) pairs: entries are laid out
    // bucket by bucket, so the lanes of a warp mostly scan the same bucket and
    // each pair is one broadcast load -- a spectrum clustered into one bucket
    // costs O(len) coalesced steps per warp, not O(len) dependent
    // random loads per thread
    GRID_LOOP(p, static_cast<int64_t>(start[kF6B])) {
        const int32_t ri = tmp[p];
        const int64_t fi = tmpf[p];
        const int64_t bk = fi >> shift;
        const int32_t s0 = start[bk], len = cnt[bk];
        int32_t rank = 0;
#pragma unroll 4
        for (int32_t j = 0; j < len; ++j) {
            const int64_t fj = tmpf[s0 + j];
            const int32_t rj = tmp[s0 + j];
            rank += fj < fi || (fj == fi && rj < ri);
        }
        byf[s0 + rank] = ri;
    }
}

__global__ void k6_scatter(const int64_t* __restrict__ cand_f, const int32_t* __restrict__ pos,
                           int64_t budget, int32_t* __restrict__ byf,
                           int32_t* __restrict__ naccepted) {
    pdl_entry();
    GRID_LOOP(r, budget) {
        if (cand_f[r] >= 0) {
            byf[pos[r]] = static_cast<int32_t>(r);
            atomicAdd(naccepted, 1);
        }
    }
}

// Run starts: the found-map sum in rank order, presence in the accumulated
// list, and the "new f" flag.  The one binary search over the accumulated
// list serves the whole merge: apos[p] = the run's insertion point (read by
// k6_merge_new) and hit[j] = p for an f already at position j (read, and
// reset to -1, by k6_merge_acc), so neither searches again.
__global__ void k6_runs(const int64_t* __restrict__ cand_f, const double2* __restrict__ cand_v,
                        const int32_t* __restrict__ byf, const int32_t* __restrict__ naccepted,
                        const int64_t* __restrict__ AF, const int32_t* __restrict__ acc_n,
                        double2* __restrict__ run_sum, int32_t* __restrict__ newflag,
                        int32_t* __restrict__ apos, int32_t* __restrict__ hit) {
    pdl_entry();
    const int64_t A = naccepted[0];
    const int an = acc_n[0];
    GRID_LOOP(p, A) {
        const int64_t f = cand_f[byf[p]];
        const bool start = p == 0 || cand_f[byf[p - 1]] != f;
        int32_t flag = 0;
        if (start) {
            double2 sum = make_double2(0.0, 0.0);
            for (int64_t p2 = p; p2 < A && cand_f[byf[p2]] == f; ++p2) {
                const double2 v = cand_v[byf[p2]];
                sum.x += v.x;
                sum.y += v.y;
            }
            run_sum[p] = sum;
            int lo = 0, hi = an;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (AF[mid] < f) lo = mid + 1; else hi = mid;
            }
            flag = (lo < an && AF[lo] == f) ? 0 : 1;
            apos[p] = lo;
            if (!flag) hit[lo] = static_cast<int32_t>(p);
        }
        newflag[p] = flag;
    }
}

__global__ void k6_merge_acc(const int64_t* __restrict__ AF, const double2* __restrict__ AC,
                             const int32_t* __restrict__ acc_n, const int64_t* __restrict__ newf,
                             const int32_t* __restrict__ nnew_p, int32_t* __restrict__ hit,
                             const double2* __restrict__ run_sum, int64_t* __restrict__ NF,
                             double2* __restrict__ NC) {
    pdl_entry();
    const int64_t an = acc_n[0];
    const int nnew = nnew_p[0];
    GRID_LOOP(j, an) {
        const int64_t fj = AF[j];
        int lo = 0, hi = nnew;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (newf[mid] < fj) lo = mid + 1; else hi = mid;
        }
        const int before = lo;
        double2 c = AC[j];
        const int32_t p = hit[j];  // the accepted run with this f (k6_runs), or -1
        if (p >= 0) {
            const double2 add = run_sum[p];
            c = make_double2(c.x + add.x, c.y + add.y);
            hit[j] = -1;
        }
        NF[j + before] = fj;
        NC[j + before] = c;
    }
}

__global__ void k6_merge_new(const int64_t* __restrict__ AF, const int32_t* __restrict__ acc_n,
                             const int64_t* __restrict__ cand_f, const int32_t* __restrict__ byf,
                             const int32_t* __restrict__ naccepted,
                             const int32_t* __restrict__ newflag, const int32_t* __restrict__ newpos,
                             const double2* __restrict__ run_sum, int64_t* __restrict__ NF,
                             double2* __restrict__ NC, const int32_t* __restrict__ new_n,
                             int32_t* __restrict__ acc_n_next, int32_t* __restrict__ nacc_next,
                             int64_t acc_cap, int64_t* __restrict__ newf,
                             const int32_t* __restrict__ apos) {
    pdl_entry();
    const int64_t A = naccepted[0];
    const int an = acc_n[0];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // the next iteration's slots (the counters alternate per iteration, so
        // nothing of this launch reads them): acc_n += new_n, accepted = 0
        MSFFT_DCHECK(an + new_n[0] <= acc_cap);
        acc_n_next[0] = an + new_n[0];
        nacc_next[0] = 0;
    }
    GRID_LOOP(p, A) {
        if (!newflag[p]) continue;
        const int64_t fr = cand_f[byf[p]];
        const int lo = apos[p];  // lower bound of fr in the accumulated list (k6_runs)
        MSFFT_DCHECK(lo >= 0 && lo <= an && (lo == an || AF[lo] > fr) && (lo == 0 || AF[lo - 1] < fr));
        const double2 sum = run_sum[p];
        newf[newpos[p]] = fr;  // the ascending new-f list k6_merge_acc searches
        NF[lo + newpos[p]] = fr;
        NC[lo + newpos[p]] = make_double2(0.0 + sum.x, 0.0 + sum.y);
    }
}

// budget <= 1024: the whole found-map merge in one CTA (same ordering rules
// and arithmetic as k6_sortf .. k6_merge_acc): accepted candidates ranked by
// (f, rank) in shared memory, run sums in rank order, block scan of the "new
// f" flags, then the merge into the ascending accumulated list.
constexpr int kSmallK6 = 1024;
constexpr int64_t kSmallK6Acc = 16384;  // accumulated-list cap for the one-CTA merge
constexpr int64_t kK6StageMax = 8192;   // accumulated f staged in its shared memory
__global__ void __launch_bounds__(kSmallK6)
k6_small(const DevPlan* __restrict__ P, int m, const int64_t* __restrict__ cand_f,
         const double2* __restrict__ cand_v, const int64_t* __restrict__ AF_g,
         const double2* __restrict__ AC, const int32_t* __restrict__ acc_n,
         int32_t* __restrict__ acc_n_next, int32_t* __restrict__ nacc_next,
         int64_t* __restrict__ NF, double2* __restrict__ NC, int32_t stage_cap) {
    pdl_entry();
    // the accumulated f list is binary-searched per accepted f: staged in
    // shared memory (dynamic, stage_cap entries) when it fits, so the
    // searches are ~30-cycle steps instead of L2 round trips
    extern __shared__ int64_t s_af[];
    __shared__ int64_t sf[kSmallK6];     // f by rank, then f at sorted position
    __shared__ int32_t byf[kSmallK6];    // rank at sorted position
    __shared__ double2 rsum[kSmallK6];   // run sums at run starts
    __shared__ int32_t nflag[kSmallK6];  // new-f flag -> exclusive prefix
    __shared__ int64_t newf[kSmallK6];
    __shared__ int32_t wsum[kSmallK6 / 32];
    __shared__ int32_t s_acc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t budget = P->it[m].budget;
    if (tid == 0) s_acc = acc_n[0];
    const int64_t fr = tid < budget ? cand_f[tid] : -1;
    __syncthreads();
    const int an = s_acc;
    const bool staged = an <= stage_cap;
    if (staged)
        for (int j = tid; j < an; j += kSmallK6) s_af[j] = AF_g[j];
    const int64_t* AF = staged ? s_af : AF_g;
    // accepted ranks in (f, rank) order: a bitonic sort of the unique keys
    // f * 1024 + rank (rejected ranks sort last); newf is free until later
    static_assert(kSmallK6 == 1024, "one key per thread, rank in 10 bits");
    uint64_t* key = reinterpret_cast<uint64_t*>(newf);
    key[tid] = fr >= 0 ? (static_cast<uint64_t>(fr) << 10) | static_cast<uint64_t>(tid)
                       : ~uint64_t{0};
    const int A = __syncthreads_count(fr >= 0);
    int pw = 2;
    while (pw < budget) pw <<= 1;
    for (int k = 2; k <= pw; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            const int p = tid ^ j;
            if (p > tid && p < pw) {
                const uint64_t a = key[tid], c = key[p];
                if ((a > c) == ((tid & k) == 0)) {
                    key[tid] = c;
                    key[p] = a;
                }
            }
            __syncthreads();
        }
    }
    if (tid < A) byf[tid] = static_cast<int32_t>(key[tid] & 1023u);
    sf[tid] = tid < A ? static_cast<int64_t>(key[tid] >> 10) : -1;
    __syncthreads();
    int flag = 0;
    if (tid < A) {
        const int64_t f = sf[tid];
        if (tid == 0 || sf[tid - 1] != f) {
            double2 sum = make_double2(0.0, 0.0);
            for (int p2 = tid; p2 < A && sf[p2] == f; ++p2) {
                const double2 v = cand_v[byf[p2]];
                sum.x += v.x;
                sum.y += v.y;
            }
            rsum[tid] = sum;
            int lo = 0, hi = an;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (AF[mid] < f) lo = mid + 1; else hi = mid;
            }
            flag = (lo < an && AF[lo] == f) ? 0 : 1;
        }
    }
    // exclusive scan of the flags over the block
    int v = flag;
    for (int o = 1; o < 32; o <<= 1) {
        const int w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int wv = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int w = __shfl_up_sync(0xffffffffu, wv, o);
            if (lane >= o) wv += w;
        }
        wsum[lane] = wv;
    }
    __syncthreads();
    const int npos = v - flag + (warp ? wsum[warp - 1] : 0);
    const int nnew = wsum[kSmallK6 / 32 - 1];
    nflag[tid] = flag;
    if (flag) newf[npos] = sf[tid];
    __syncthreads();
    for (int j = tid; j < an; j += kSmallK6) {
        const int64_t fj = AF[j];
        int lo = 0, hi = nnew;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (newf[mid] < fj) lo = mid + 1; else hi = mid;
        }
        const int before = lo;
        int plo = 0, phi2 = A;
        while (plo < phi2) {
            const int mid = (plo + phi2) >> 1;
            if (sf[mid] < fj) plo = mid + 1; else phi2 = mid;
        }
        double2 c = AC[j];
        if (plo < A && sf[plo] == fj) {
            const double2 add = rsum[plo];
            c = make_double2(c.x + add.x, c.y + add.y);
        }
        NF[j + before] = fj;
        NC[j + before] = c;
    }
    if (tid < A && nflag[tid]) {
        const int64_t f = sf[tid];
        int lo = 0, hi = an;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (AF[mid] < f) lo = mid + 1; else hi = mid;
        }
        const double2 sum = rsum[tid];
        NF[lo + npos] = f;
        NC[lo + npos] = make_double2(0.0 + sum.x, 0.0 + sum.y);
    }
    __syncthreads();
    if (tid == 0) {
        MSFFT_DCHECK(an + nnew <= P->acc_cap);
        acc_n_next[0] = an + nnew;
        nacc_next[0] = 0;
    }
}

// ---------------------------------------------------------------- K7
__global__ void k7_emit(const int32_t* __restrict__ sel_idx, const int32_t* __restrict__ scal,
                        const int64_t* __restrict__ AF, const double2* __restrict__ AC,
                        int64_t* __restrict__ out_f, double2* __restrict__ out_c,
                        int64_t* __restrict__ out_count) {
    pdl_entry();
    const int64_t keep = scal[2];
    GRID_LOOP(p, keep) {
        const int32_t j = sel_idx[p];
        MSFFT_DCHECK(j >= 0);
        out_f[p] = AF[j];
        out_c[p] = AC[j];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out_count = keep;
}

}  // namespace

WideDecoder::WideDecoder(const DevPlan& plan, int64_t acc_cap, int64_t b_max, int64_t budget_max,
                         int64_t rounds_max)
    : hplan_(plan),
      acc_cap_(std::max<int64_t>(acc_cap, 1)),
      b_max_(b_max),
      budget_max_(std::max<int64_t>(budget_max, 1)),
      rounds_max_(rounds_max) {
    dplan_.reset(1);
    MSFFT_CUDA(cudaMemcpy(dplan_.get(), &plan, sizeof(DevPlan), cudaMemcpyHostToDevice));
    const int64_t A = acc_cap_, B = b_max_, Q = budget_max_, R = rounds_max_;
    for (int p = 0; p < 2; ++p) {
        acc_f_[p].reset(A);
        acc_c_[p].reset(A);
    }
    scal_.reset(8);
    sel_.reset(4);
    thr_.reset(1);
    tone_u_.reset(A);
    tone_i_.reset(A);
    gc_.reset(3 * A);
    rot_.reset(A * R);
    cnt_.reset(B);
    start_.reset(B + 1);
    cursor_.reset(B);
    long_.reset(B + 1);
    ev_.reset(3 * A);
    ev2_.reset(3 * A);
    const int64_t NK = std::max(B, A);
    key_.reset(NK);
    mag_.reset(B);
    hist_.reset(kSelBins);
    // sel_compact: a flagged count word per chunk and {ticket, blocks done},
    // zero between launches (its last block clears them)
    const int64_t ncc = (NK + kCChunk - 1) / kCChunk;
    cpub_.reset(static_cast<size_t>(ncc));
    cctl_.reset(2);
    MSFFT_CUDA(cudaMemset(cpub_.get(), 0, static_cast<size_t>(ncc) * sizeof(unsigned long long)));
    MSFFT_CUDA(cudaMemset(cctl_.get(), 0, 2 * sizeof(int32_t)));
    sel_idx_.reset(std::max(Q, A));
    order_.reset(Q);
    yr_.reset(Q * R);
    phi_.reset(Q * R);
    pcode_.reset(Q * R);
    cand_f_.reset(Q);
    cand_v_.reset(Q);
    cand_sum_.reset(Q);
    pos_.reset(Q);
    byf_.reset(Q);
    f6cnt_.reset(kF6B);
    f6cur_.reset(kF6B);
    f6start_.reset(kF6B + 1);
    newflag_.reset(Q);
    newpos_.reset(Q);
    newf_.reset(Q);
    // hit_[j] = accepted run whose f is already at accumulated position j; -1
    // between iterations (k6_merge_acc resets what k6_runs set)
    hit_.reset(static_cast<size_t>(acc_cap_));
    MSFFT_CUDA(cudaMemset(hit_.get(), 0xff, static_cast<size_t>(acc_cap_) * sizeof(int32_t)));
    if (const char* e = std::getenv("MSFFT_WIDE_GRAPH")) use_graphs_ = std::atoi(e) != 0;
    if (const char* e = std::getenv("MSFFT_WIDE_PDL")) pdl_ = std::atoi(e) != 0;
    // kernel attributes are set before any capture
    k6_stage_cap_ = std::min<int64_t>(acc_cap_, kK6StageMax);
    smem_attr(k6_small, static_cast<size_t>(k6_stage_cap_) * sizeof(int64_t));
}

// sel_ and hist_ were prepared by the keys_from_values launch before it.
void WideDecoder::select_kth(const uint64_t* key, int64_t n_max, const int32_t* n_dev,
                             cudaStream_t st) {
    // the top 24 bits over the whole grid, the low 40 in one CTA
    for (int top = 64; top > 40;) {
        const int width = std::min(kSelBits, top);
        const int shift = top - width;
        launch_pdl(pdl_, sel_digit, std::min<unsigned>(grid_of(n_max), 148), kT, 0, st, key, n_max, n_dev,
                   sel_.get(), shift, width, hist_.get());
        top = shift;
    }
    launch_pdl(pdl_, sel_finish, 1, kFinT, 0, st, key, n_max, n_dev, sel_.get());
    MSFFT_LAUNCH_CHECK("wide select");
}

void WideDecoder::compact_selected(const uint64_t* key, int64_t n_max, const int32_t* n_dev,
                                   int32_t* out_idx, cudaStream_t st) {
    const int64_t nch = (n_max + kCChunk - 1) / kCChunk;
    launch_pdl(pdl_, sel_compact, static_cast<unsigned>(nch), kT, 0, st, key, n_max, n_dev, sel_.get(),
               cpub_.get(), cctl_.get(), out_idx);
    MSFFT_LAUNCH_CHECK("wide compaction");
}

WideDecoder::~WideDecoder() {
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
}

void WideDecoder::run_range(double2* y, const int64_t* sigma, const int64_t* sigma_inv,
                            int64_t* out_f, double2* out_c, int64_t* out_count, int32_t* err,
                            cudaStream_t st, int m0, int m1) {
    if (!use_graphs_) {
        enqueue(y, sigma, sigma_inv, err, out_f, out_c, out_count, st, m0, m1);
    } else {
        // K7 writes the caller's outputs directly, so they are part of the key
        const GraphKey key{y, sigma, sigma_inv, err, out_f, out_c, out_count, m0, m1};
        auto it = graphs_.find(key);
        if (it == graphs_.end() && graphs_.size() >= 16) {
            // bounded: callers that pass fresh buffers every call
            // recapture instead of accumulating executable graphs
            MSFFT_CUDA(cudaStreamSynchronize(st));
            for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second);
            graphs_.clear();
        }
        if (it == graphs_.end()) {
            cudaStream_t cap = nullptr;
            MSFFT_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            cudaGraph_t g = nullptr;
            MSFFT_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
            enqueue(y, sigma, sigma_inv, err, out_f, out_c, out_count, cap, m0, m1);
            MSFFT_CUDA(cudaStreamEndCapture(cap, &g));
            cudaGraphExec_t ex = nullptr;
            MSFFT_CUDA(cudaGraphInstantiate(&ex, g, 0));
            cudaGraphDestroy(g);
            cudaStreamDestroy(cap);
            it = graphs_.emplace(key, ex).first;
        }
        MSFFT_CUDA(cudaGraphLaunch(it->second, st));
    }
}

void WideDecoder::enqueue(double2* y, const int64_t* sigma, const int64_t* sigma_inv, int32_t* err,
                          int64_t* out_f, double2* out_c, int64_t* out_count, cudaStream_t st,
                          int m0, int m1) {
    const DevPlan& H = hplan_;
    const DevPlan* P = dplan_.get();
    // scal_: [1] new_n, [2] kth; the accumulated count and the accepted
    // counter alternate between two slots per iteration ([0]/[5], [4]/[6]),
    // so an iteration's last kernel can publish the next iteration's values
    // while its own blocks still read the current ones
    int32_t* new_n = scal_.get() + 1;
    int32_t* kth = scal_.get() + 2;
    auto acc_slot = [&](int par) { return scal_.get() + (par ? 5 : 0); };
    auto nacc_slot = [&](int par) { return scal_.get() + (par ? 6 : 4); };
    if (m0 == 0) zero_async(pdl_, scal_.get(), 8 * sizeof(int32_t), st);
    const unsigned gA = grid_of(acc_cap_ * 3);
    for (int m = m0; m < m1; ++m) {
        const DevIter& it = H.it[m];
        const int64_t b = it.b, nr = it.nrounds, budget = it.budget;
        double2* Y = y + it.yoff;
        const int cur = m & 1, nxt = cur ^ 1;
        const int64_t* AF = acc_f_[cur].get();
        const double2* AC = acc_c_[cur].get();
        const int32_t* acc_n = acc_slot(cur);
        int32_t* naccepted = nacc_slot(cur);
        if (m > 0) {
            // ---- K3 (cnt_ was cleared by the previous iteration's k5_stage_phase)
            launch_pdl(pdl_, k3_tones, grid_of(acc_cap_ * nr), kT, 0, st, P, m, sigma, AF, AC, acc_n, tone_u_.get(),
                                                      tone_i_.get(), gc_.get(), cnt_.get(), cursor_.get(),
                                                      long_.get(), rot_.get());
            launch_pdl(pdl_, scan_kernel, 1, kScanT, 0, st, cnt_.get(), b, nullptr, start_.get(), nullptr,
                       long_.get());
            launch_pdl(pdl_, k3_scatter, gA, kT, 0, st, P, m, acc_n, tone_i_.get(), start_.get(), cursor_.get(),
                                          ev_.get());
            {
                const int long_blocks = static_cast<int>(std::min<int64_t>(b, 148 * 2));
                const int short_blocks = static_cast<int>(
                    std::max<int64_t>(1, std::min<int64_t>((b * 32 + kLongT - 1) / kLongT, 148 * 4)));
                launch_pdl(pdl_, k3_segsort, static_cast<unsigned>(long_blocks + short_blocks), kLongT, 0, st,
                           P, m, start_.get(), cnt_.get(), ev_.get(), ev2_.get(), long_.get(), long_blocks,
                           acc_n);
            }
            launch_pdl(pdl_, k3_sum, grid_of(nr * b * 32), kT, 0, st, P, m, start_.get(), cnt_.get(), ev2_.get(),
                                                        gc_.get(), rot_.get(), Y);
            MSFFT_LAUNCH_CHECK("wide K3");
        }
        // ---- K4
        if (b <= kSmallK4) {
            launch_pdl(pdl_, k4_small, 1, kSmallK4, 0, st, P, m, Y, mag_.get(), order_.get(), thr_.get());
        } else {
            // also clears the K4 rank counters (pos_)
            launch_pdl(pdl_, keys_from_values, grid_of(b), kT, 0, st, Y, b, nullptr, mag_.get(), key_.get(),
                       reinterpret_cast<uint32_t*>(pos_.get()), budget, sel_.get(), hist_.get(), budget,
                       nullptr, b, nullptr);
            select_kth(key_.get(), b, nullptr, st);
            compact_selected(key_.get(), b, nullptr, sel_idx_.get(), st);
            {
                const unsigned tiles = static_cast<unsigned>((budget + kT - 1) / kT);
                const unsigned split = std::max(1u, std::min(64u, 1184u / tiles));
                launch_pdl(pdl_, k4_rank, dim3(tiles, split), kT, 0, st, sel_idx_.get(), budget, key_.get(), pos_.get());
                launch_pdl(pdl_, k4_scatter, grid_of(budget), kT, 0, st, sel_idx_.get(), pos_.get(), budget,
                                                           order_.get(), mag_.get(), thr_.get());
            }
        }
        // ---- K5
        // k5_stage_phase also clears the counters of kernels further down the
        // chain: the K6 order counters of this iteration (the f-bucket counts
        // or the all-pairs positions; pos_ is free once K4 has scattered) and
        // the next iteration's K3 bucket counts
        const bool k6_small_path = budget <= kSmallK6 && acc_cap_ <= kSmallK6Acc;
        uint32_t* zero_a = nullptr;
        int64_t zero_an = 0;
        if (!k6_small_path) {
            zero_a = reinterpret_cast<uint32_t*>(budget >= kF6BucketMin ? f6cnt_.get() : pos_.get());
            zero_an = budget >= kF6BucketMin ? int64_t{kF6B} : budget;
        }
        const int64_t zero_bn = m + 1 < H.iters ? H.it[m + 1].b : 0;
        // stage phases inside k5_locate (one launch) when its lane groups'
        // slices fit the shared staging; else the separate kernel first
        const int gsz = H.l > 16 ? 32 : (H.l > 8 ? 16 : (H.l > 4 ? 8 : 4));
        const bool k5_one = static_cast<int64_t>(kT / gsz) * (nr - 1) <= kK5Stage;
        if (!k5_one)
            launch_pdl(pdl_, k5_stage_phase, grid_of(std::max(budget * nr, std::max(zero_an, zero_bn))), kT, 0,
                       st, P, m, order_.get(), Y, yr_.get(), phi_.get(), pcode_.get(), zero_a, zero_an,
                       reinterpret_cast<uint32_t*>(cnt_.get()), zero_bn);
        launch_pdl(pdl_, k5_locate, grid_of(std::max(budget * 32, k5_one ? std::max(zero_an, zero_bn) : int64_t{0})),
                   kT, 0, st, P, m, sigma_inv, order_.get(), mag_.get(), thr_.get(), yr_.get(), phi_.get(),
                   pcode_.get(), cand_f_.get(), cand_v_.get(), err,
                   k5_one ? static_cast<const double2*>(Y) : nullptr, k5_one ? zero_a : nullptr,
                   k5_one ? zero_an : int64_t{0},
                   k5_one ? reinterpret_cast<uint32_t*>(cnt_.get()) : nullptr, k5_one ? zero_bn : int64_t{0});
        MSFFT_LAUNCH_CHECK("wide K4/K5");
        // ---- K6
        if (k6_small_path) {
            launch_pdl(pdl_, k6_small, 1, kSmallK6, k6_stage_cap_ * sizeof(int64_t), st, P, m,
                       cand_f_.get(), cand_v_.get(), AF, AC, acc_n, acc_slot(nxt), nacc_slot(nxt),
                       acc_f_[nxt].get(), acc_c_[nxt].get(), static_cast<int32_t>(k6_stage_cap_));
        } else {
            if (budget >= kF6BucketMin) {
                int nbits = 0;
                while ((int64_t{1} << nbits) < H.n) ++nbits;
                const int shift = std::max(0, nbits - 12);  // f >> shift < 4096
                launch_pdl(pdl_, k6b_count, grid_of(std::max<int64_t>(budget, kF6B)), kT, 0, st,
                           cand_f_.get(), budget, shift, f6cnt_.get(), f6cur_.get(), naccepted);
                launch_pdl(pdl_, scan_kernel, 1, kScanT, 0, st, f6cnt_.get(), int64_t{kF6B}, nullptr,
                           f6start_.get(), f6start_.get() + kF6B, nullptr);
                // newf_ is free until k6_merge_new: it holds the keys of the bucket sort
                launch_pdl(pdl_, k6b_scatter, grid_of(budget), kT, 0, st, cand_f_.get(), budget, shift,
                           f6start_.get(), f6cur_.get(), pos_.get(), newf_.get());
                launch_pdl(pdl_, k6b_sort, grid_of(budget), kT, 0, st, shift, f6start_.get(),
                           f6cnt_.get(), pos_.get(), newf_.get(), byf_.get());
            } else {
                const unsigned tiles = static_cast<unsigned>((budget + kT - 1) / kT);
                const unsigned split = std::max(1u, std::min(64u, 1184u / tiles));
                launch_pdl(pdl_, k6_sortf, dim3(tiles, split), kT, 0, st, cand_f_.get(), budget, pos_.get());
                launch_pdl(pdl_, k6_scatter, grid_of(budget), kT, 0, st, cand_f_.get(), pos_.get(), budget, byf_.get(),
                                                           naccepted);
            }
            launch_pdl(pdl_, k6_runs, grid_of(budget), kT, 0, st, cand_f_.get(), cand_v_.get(), byf_.get(),
                                                    naccepted, AF, acc_n, cand_sum_.get(),
                                                    newflag_.get(), pos_.get(), hit_.get());
            launch_pdl(pdl_, scan_kernel, 1, kScanT, 0, st, newflag_.get(), budget, naccepted, newpos_.get(), new_n,
                       nullptr);
            // new entries first (they also list the new f for the accumulated
            // entries' offsets and publish the next iteration's counters)
            launch_pdl(pdl_, k6_merge_new, grid_of(budget), kT, 0, st, AF, acc_n, cand_f_.get(), byf_.get(),
                                                         naccepted, newflag_.get(), newpos_.get(),
                                                         cand_sum_.get(), acc_f_[nxt].get(),
                                                         acc_c_[nxt].get(), new_n, acc_slot(nxt),
                                                         nacc_slot(nxt), acc_cap_, newf_.get(), pos_.get());
            launch_pdl(pdl_, k6_merge_acc, grid_of(acc_cap_), kT, 0, st, AF, AC, acc_n, newf_.get(), new_n,
                                                           hit_.get(), cand_sum_.get(), acc_f_[nxt].get(),
                                                           acc_c_[nxt].get());
        }
        MSFFT_LAUNCH_CHECK("wide K6");
    }
    if (m1 < H.iters) return;
    // ---- K7: the K largest |c| (stable over ascending f), emitted in f order
    const int fin = H.iters & 1;
    const int32_t* acc_n = acc_slot(fin);
    launch_pdl(pdl_, keys_from_values, grid_of(acc_cap_), kT, 0, st, acc_c_[fin].get(), acc_cap_, acc_n, nullptr,
                                                       key_.get(), nullptr, int64_t{0}, sel_.get(), hist_.get(),
                                                       int64_t{H.k}, acc_n, acc_cap_, kth);
    select_kth(key_.get(), acc_cap_, acc_n, st);
    compact_selected(key_.get(), acc_cap_, acc_n, sel_idx_.get(), st);
    launch_pdl(pdl_, k7_emit, grid_of(H.k), kT, 0, st, sel_idx_.get(), scal_.get(), acc_f_[fin].get(),
                                         acc_c_[fin].get(), out_f, out_c, out_count);
    MSFFT_LAUNCH_CHECK("wide K7");
}

}  // namespace msfft_b200
