// components.hpp -- the reference's secondary public entry points on the
// sfft4 path, batched on the device.  sfft4 itself never
// calls these (its encode/decode run fused, engine.cu); they exist so a
// caller of the reference's component API finds the same functions:
//
//   bucketize        proj/src/bucketize.cpp:50-61, bucketize.hpp:63-86
//   predict_buckets  proj/src/bucketize.cpp:70-95
//   locate_frequency proj/src/locate.cpp:83-123 (locate_step :63-81)
//   estimate_value   proj/src/sfft4.cpp:27-36
//
// (subtract, bucketize.cpp:97-104, is elementwise and lives in the C++
// header.)  All d_* pointers are device pointers; the window (n, b, delta)
// comes from the process cache (window.hpp).  Errors are thrown with the
// reference's exception types and messages.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace msfft_b200 {

// `rounds` bucketizations of one signal d_x (n samples, complex64 upcast
// exactly or complex128) under (sigma[r], tau[r]) (host arrays): d_out is
// [rounds][b] complex128.  Per bin, the taps are summed in ascending t as the
// reference's fold loop does (no FMA), then the radix-2 DIT and * 1/n:
// bit-identical to bucketize.  Returns w (BucketSet::samples_read).
int64_t bucketize_device(const void* d_x, bool c128, int64_t n, int64_t b, double delta,
                         const int64_t* sigma, const int64_t* tau, int64_t rounds, double2* d_out,
                         cudaStream_t st);

// predict_buckets of `count` known tones (d_f ascending, d_c) for each of the
// `rounds` (sigma, tau) pairs: d_out [rounds][b].  Contributions enter each
// bucket in ascending f with the reference's operands (G * c) * rot; G from
// the window's device response table, rot by sincos (ulp-level vs libm).
void predict_buckets_device(int64_t n, int64_t b, double delta, const int64_t* d_f,
                            const double2* d_c, int64_t count, const int64_t* sigma,
                            const int64_t* tau, int64_t rounds, double2* d_out, cudaStream_t st);

// locate_frequency for `count` buckets d_bucket against one round set
// d_rounds [nrounds][b] with tau[r] (host); round 0 must have tau 0.
// Outputs per bucket: d_u, d_stages, d_status (0 located, 1 nullopt, 2
// phase_of(0) -> the caller throws std::domain_error "phase_of: zero value",
// 3 the region needed more rounds than given, 4 bucket outside [0, b)).  Decisions are the
// reference's FP64 operations in its order (same as the fused decode).
void locate_frequency_device(int64_t n, int64_t b, int64_t l, double q, const int64_t* d_bucket,
                             int64_t count, const double2* d_rounds, const int64_t* tau,
                             int64_t nrounds, int64_t* d_u, int32_t* d_stages, int32_t* d_status,
                             cudaStream_t st);

// estimate_value for `count` (y0, u) pairs: d_out = y0 / G_{iL-u}, or
// d_status = 1 where |G| < 0.5 (the reference throws std::domain_error).
void estimate_values_device(int64_t n, int64_t b, double delta, const double2* d_y0,
                            const int64_t* d_u, int64_t count, double2* d_out, int32_t* d_status,
                            cudaStream_t st);

// ---- scalar locate helpers and the sampler-driven fold (locate_ops.cu) ----
// Batched over host arrays; each evaluates the device functions the decodes
// use.  LocateRegionDev mirrors LocateRegion (locate.hpp:23-32).
struct LocateRegionDev {
    double u_min;
    double length;
    int32_t stage;
    int32_t reserved;
};

// phase_of (locate.cpp:32-37) of z[k] (interleaved complex128): phase in
// [0, 2pi), status 1 where z == 0 (the reference throws domain_error).
void phase_of_host(const double* z, int64_t count, double* phase, int32_t* status,
                   cudaStream_t st);
// position_phase(u[k], tau[k], n) (locate.cpp:19-23).
void position_phase_host(const double* u, const int64_t* tau, int64_t count, int64_t n,
                         double* out, cudaStream_t st);
// circular_phase_distance(a[k], b[k]) (locate.cpp:14-17).
void circular_phase_distance_host(const double* a, const double* b, int64_t count, double* out,
                                  cudaStream_t st);
// locate_step({phi[k], tau[k]}, region[k], {l, q}, n) (locate.cpp:63-81).
void locate_step_host(const double* phi, const int64_t* tau, const LocateRegionDev* region,
                      int64_t count, int64_t l, double q, int64_t n, LocateRegionDev* out,
                      cudaStream_t st);
// bucketize_fn (bucketize.hpp:63-86) for `rounds` sample sequences the caller
// evaluated in tap order: values [rounds][w] complex128, values[r][h + t] =
// sample(src_t); out [rounds][b].  Returns w.
int64_t bucketize_taps_host(int64_t n, int64_t b, double delta, const double* values,
                            int64_t rounds, double* out, cudaStream_t st);

}  // namespace msfft_b200
