// fft.hpp -- batched power-of-two FFT on the device whose every butterfly
// performs the same IEEE operations, on the same operands and twiddles, as
// the reference's radix-2 DIT (proj/src/fft.cpp:32-66), so results are
// bit-identical to it.  Used by the window designer (n-point, cold path) and
// for bucket transforms too large for one CTA's shared memory.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace msfft_b200 {

// Twiddles e^{-2 pi i k/n}, k < n/2, evaluated on the host with the same libm
// calls as twiddle_table (proj/src/fft.cpp:14-28) and cached on the current
// device per size.  Returned pointer stays valid for the process lifetime.
const double2* device_twiddles(int64_t n);

// Host copy of the same table (for tests / host-side use).
const double* host_twiddles(int64_t n);

// In-place transform of `batch` arrays of `size` complex doubles.  Array i
// starts at data + (i / inner) * outer_stride + (i % inner) * size.
// sign < 0: forward kernel; sign > 0: conjugated twiddles (fft_radix2 sign).
// After the last butterfly every value is multiplied by `scale` (component
// wise, as `v *= scale` in the reference) unless scale == 1.
void fft_radix2_batched(double2* data, int64_t size, int64_t batch, int64_t inner,
                        int64_t outer_stride, int sign, double scale, cudaStream_t stream);

// One set of equally sized arrays for fft_radix2_sets: for each of `batch`
// rows (row stride outer_stride), `inner` arrays of `size` starting at
// data + off + row * outer_stride.
struct FftSet {
    int64_t off, size, inner;
    int m = 0;  // iteration (gated launches: the counter slot of the set)
};
constexpr int kMaxFftSets = 16;
constexpr int64_t kSmemFftMax = 4096;  // largest array transformed in one CTA

// Gated launch of fft_radix2_sets (every set <= kSmemFftMax): a programmatic
// dependent launch behind the encode whose CTA for a set of iteration m
// starts once wait_done[m] reaches wait_need[m], and adds 1 to post_done[m]
// when its array is transformed.
struct FftGate {
    const int32_t* wait_done;
    const int32_t* wait_need;
    int32_t* post_done;
};

// fft_radix2_batched of several sets: the sets with size <= 4096 go into ONE
// launch (one CTA per array, shared memory), larger ones through the
// multi-pass path.  Bit-identical to transforming each set separately.
// scratch (optional): a buffer laid out like data (rows of outer_stride):
// sets with 4096 < size <= 2^18 then take two launches in all (a gathered
// bit-reversal + stages 1..11, then the remaining stages) instead of three
// per size.
void fft_radix2_sets(double2* data, const FftSet* sets, int nsets, int64_t batch,
                     int64_t outer_stride, int sign, double scale, cudaStream_t stream,
                     const FftGate* gate = nullptr, double2* scratch = nullptr);

}  // namespace msfft_b200
