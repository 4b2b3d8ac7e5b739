// signal_ops.hpp -- device versions of the reference's signal helpers
// (SURVEY.md 8(f) rows 2-3): the steps either side of the hot path.
//
//   synthesize / generate_test_signal   proj/src/signal.cpp:76-121
//   add_awgn                            proj/src/signal.cpp:123-152
//   dft_dense / idft_dense              proj/src/signal.cpp:37-54
//   top_k_spectrum                      proj/src/bench.cpp:33-46
//
// All pointers named d_* are device pointers.  Errors are thrown with the
// reference's exception types and messages.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host_plan.hpp"

namespace msfft_b200 {

// Truth of generate_test_signal (random_sparse_spectrum with the reference's
// Rng: Floyd sampling + uniform phases, signal.cpp:100-121), ascending f.
void random_sparse_spectrum(int64_t n, int64_t k, uint64_t seed, std::vector<int64_t>& f,
                            std::vector<double>& c);
// Same draws from a caller's stream (random_sparse_spectrum(n, k, rng)).
void random_sparse_spectrum(int64_t n, int64_t k, HostRng& rng, std::vector<int64_t>& f,
                            std::vector<double>& c);

// synthesize (signal.cpp:76-98) of `count` tones (f ascending, c interleaved)
// into d_x (n samples, complex128 or complex64).  The per-tone phasor
// recurrence and the per-sample sum over tones in ascending f run on the
// device with the reference's operation order and no FMA; the cos/sin seeds
// (every 1024 samples) and step phasors come from host libm, so the samples
// are bit-identical to the reference while count * ceil(n/1024) <= 2^23
// (the seed table); beyond that the seeds use device sincos (ulp-level).
// Returns true if the bit-identical path was used.
bool synthesize_device(int64_t n, const int64_t* f, const double* c, int64_t count, bool c128,
                       void* d_x, cudaStream_t st);

// add_awgn (signal.cpp:123-152) in place on d_x: the same validation, +inf
// sentinel and realised-power scaling (scale = sqrt(P_sig 10^(-snr/10) /
// P_noise)); the complex Gaussian noise is Box-Muller over Philox4x32-10
// counters (sample index, seed) instead of the reference's sequential
// mt19937_64 stream, so the noise has the same law but not the same samples.
void awgn_device(void* d_x, bool c128, int64_t n, double snr_db, uint64_t seed, cudaStream_t st);

// dft_dense (sign < 0: forward, x validated, times 1/n) or idft_dense (sign >
// 0: unnormalised inverse) of `batch` contiguous signals; d_in complex128 or
// complex64 (exact upcast), d_out complex128.  Bit-identical to the
// reference (the same radix-2 butterflies and host-libm twiddles).
void dense_dft_device(const void* d_in, bool in_c128, int64_t n, int64_t batch, double2* d_out,
                      int sign, cudaStream_t st);

// top_k_spectrum: the k largest |X| (glibc hypot restated) of d_spec (n
// values), returned in ascending f.  Ties at the k-th magnitude keep the
// lowest indices (nth_element leaves that choice unspecified).
int64_t top_k_device(const double2* d_spec, int64_t n, int64_t k, int64_t* f, double* c,
                     cudaStream_t st);

}  // namespace msfft_b200
