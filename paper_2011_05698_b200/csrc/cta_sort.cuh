// cta_sort.cuh -- block-wide primitives for the decode's large-size paths
// (C3/C5: b up to 65536 buckets, budgets up to 10^4, ~2*10^4 accumulated
// tones), where the O(n^2) rank counting of the small-size path would take
// seconds on one CTA.
//
// cta_radix_sort: stable ascending LSD radix sort of (u64 key, i32 value)
// pairs with 4-bit digits.  Thread t owns a contiguous tile, counts digits
// into its own column of a [16][threads] table (no atomics), the table is
// scanned digit-major, and each thread scatters its tile in order, so equal
// keys keep their input order (the std::stable_sort ties of the reference).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace msfft_b200 {
namespace {

// Exclusive scan of cnt[0..count) in place by a CTA of T threads; returns the
// total to every thread.  count must be a multiple of T.
template <int T>
__device__ __forceinline__ int cta_exclusive_scan(int* cnt, int count, int* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = count / T;
    int local = 0;
    for (int i = 0; i < per; ++i) local += cnt[tid * per + i];
    int v = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
    }
    if (lane == 31) warp_tot[warp] = v;
    __syncthreads();
    if (warp == 0) {
        int wv = lane < T / 32 ? warp_tot[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int w = __shfl_up_sync(0xffffffffu, wv, o);
            if (lane >= o) wv += w;
        }
        if (lane < T / 32) warp_tot[lane] = wv;  // inclusive warp prefix
    }
    __syncthreads();
    int run = v - local + (warp ? warp_tot[warp - 1] : 0);  // exclusive start
    for (int i = 0; i < per; ++i) {
        const int c = cnt[tid * per + i];
        cnt[tid * per + i] = run;
        run += c;
    }
    const int total = warp_tot[T / 32 - 1];
    __syncthreads();
    return total;
}

// Sorts n pairs; (k0, v0) in, (k1, v1) scratch.  Returns true when the
// result ended in (k1, v1).  cnt: 16*T ints of scratch (shared memory
// preferred), warp_tot: T/32 ints of shared memory.  Only the low key_bits
// bits of the keys are examined.
template <int T>
__device__ bool cta_radix_sort(uint64_t* k0, int32_t* v0, uint64_t* k1, int32_t* v1, int n,
                               int key_bits, int* cnt, int* warp_tot) {
    const int tid = threadIdx.x;
    const int tile = (n + T - 1) / T;
    const int lo = min(n, tid * tile), hi = min(n, lo + tile);
    bool flipped = false;
    for (int shift = 0; shift < key_bits; shift += 4) {
        uint64_t* ks = flipped ? k1 : k0;
        int32_t* vs = flipped ? v1 : v0;
        uint64_t* kd = flipped ? k0 : k1;
        int32_t* vd = flipped ? v0 : v1;
        // counts: column tid of a digit-major [16][T] table
        for (int d = 0; d < 16; ++d) cnt[d * T + tid] = 0;
        for (int i = lo; i < hi; ++i) ++cnt[static_cast<int>((ks[i] >> shift) & 15u) * T + tid];
        __syncthreads();
        // scan in (digit, thread) order: each thread scans 16 consecutive
        // entries of the table, which is exactly the digit-major order
        cta_exclusive_scan<T>(cnt, 16 * T, warp_tot);
        for (int i = lo; i < hi; ++i) {
            const uint64_t key = ks[i];
            int& slot = cnt[static_cast<int>((key >> shift) & 15u) * T + tid];
            kd[slot] = key;
            vd[slot] = vs[i];
            ++slot;
        }
        __syncthreads();
        flipped = !flipped;
    }
    return flipped;
}

// Key that sorts non-negative doubles descending (NaN and negative markers
// last), for the std::stable_sort(..., |a| > |b|) orders of the reference.
__device__ __forceinline__ uint64_t desc_key(double v) {
    if (!(v >= 0.0)) return ~uint64_t{0};
    return ~static_cast<uint64_t>(__double_as_longlong(v));
}

}  // namespace
}  // namespace msfft_b200
