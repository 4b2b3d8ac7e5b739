/*
 * msfft_b200.h -- C ABI of the B200-native sFFT4.0 hot path.
 *
 * Drop-in boundary for
 *     msfft::SfftResult msfft::sfft4(const ComplexSignal& x, int64_t k,
 *                                    const MultiscaleConfig& cfg,
 *                                    uint64_t seed, double delta = 1e-8);
 * (reference: proj/include/msfft/sfft4.hpp:64-65, result/stat types :32-45,
 * implementation proj/src/sfft4.cpp:131-187).  Plain pointers and sizes only;
 * no torch or C++ types cross this boundary.  A C++ wrapper with the
 * reference's exact signature and exception types is include/msfft_b200.hpp.
 *
 * Errors: every entry point returns an msfft_status.  MSFFT_ERR_INVALID_ARGUMENT
 * and MSFFT_ERR_DOMAIN carry the reference's std::invalid_argument /
 * std::domain_error messages verbatim in err[errlen] (e.g. "sfft4: need 1 <= K
 * <= n/8", proj/src/sfft4.cpp:135; "MultiscaleConfig: l/(q+1) must exceed 1",
 * proj/src/locate.cpp:29).  There is no CPU fallback: without a usable CUDA
 * device every call fails with MSFFT_ERR_CUDA.
 *
 * Thread safety: all entry points are reentrant.  Windows and response tables
 * live in a process-wide cache keyed (device, n, b, delta) like
 * get_flat_window (proj/src/window.cpp:179-193).  A plan handle may be used by
 * one thread at a time.
 */
#ifndef MSFFT_B200_H
#define MSFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSFFT_B200_ABI_VERSION 1
#define MSFFT_MAX_ITERATIONS 64

typedef enum msfft_status {
    MSFFT_OK = 0,
    MSFFT_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    MSFFT_ERR_DOMAIN = 2,           /* std::domain_error escaping sfft4       */
    MSFFT_ERR_CUDA = 3,             /* no device / CUDA failure               */
    MSFFT_ERR_RUNTIME = 4           /* anything else                          */
} msfft_status;

typedef enum msfft_dtype {
    MSFFT_C128 = 0, /* interleaved (re, im) float64: cplx, proj/include/msfft/fft.hpp:9 */
    MSFFT_C64 = 1   /* interleaved (re, im) float32, upcast exactly to float64            */
} msfft_dtype;

typedef enum msfft_location { MSFFT_HOST = 0, MSFFT_DEVICE = 1 } msfft_location;

enum msfft_flags {
    /* Skip the O(n) finiteness scan of x (ComplexSignal::validate,
     * proj/src/signal.cpp:18-26) because the caller validated at ingest. */
    MSFFT_FLAG_ASSUME_VALID = 1u << 0,
    /* Record CUDA events around each stage on the execution stream; read
     * them back with msfft_plan_stage_times. */
    MSFFT_FLAG_STAGE_TIMES = 1u << 1,
    /* Run the encode and the decode as separate launches instead of the
     * persistent fused kernel (diagnostics: per-kernel rooflines). */
    MSFFT_FLAG_SERIAL = 1u << 2,
    /* msfft_execute returns once the work is enqueued on the stream (device
     * input and output only): outputs are complete when the stream reaches
     * them, decode errors are reported by the next msfft_plan_sync.  Calls
     * that repeat the previous seeds reuse the σ plan on the device. */
    MSFFT_FLAG_ASYNC = 1u << 3
};

/* TransformStats (proj/include/msfft/sfft4.hpp:32-40). */
typedef struct msfft_stats {
    int64_t samples_used;      /* distinct time indices read            */
    int64_t samples_round_sum; /* sum_m (R_m + 1) * w_m                 */
    double sample_fraction;    /* samples_used / n                      */
    double runtime_ms;         /* device time of the transform          */
    int32_t iterations;
    int32_t reserved;
    int64_t b_first;
    int32_t stage_counts[MSFFT_MAX_ITERATIONS]; /* R_m per iteration */
} msfft_stats;

typedef struct msfft_plan_s* msfft_plan;

const char* msfft_version(void);
int msfft_device_count(void);

/* ---- one-shot drop-in: msfft::sfft4 ----------------------------------------
 * x: n complex samples (dtype) in host or device memory.  Output: at most
 * `cap` entries in ascending frequency (the std::map order of SparseSpectrum);
 * *out_count is the entry count (<= k).  stats may be NULL. */
int msfft_sfft4(const void* x, int64_t n, int32_t dtype, int32_t x_location, int64_t k,
                int64_t l, double q, uint64_t seed, double delta, int64_t cap, int64_t* out_f,
                double* out_c, int64_t* out_count, msfft_stats* stats, char* err, size_t errlen);

/* ---- plans: batches of independent signals sharing (n, k, l, q, delta) ----
 * Creating a plan designs every window of the halving schedule on `device`
 * (the reference resolves them before its timer too, sfft4.cpp:146-154). */
int msfft_plan_create(int64_t n, int64_t k, int64_t l, double q, double delta, int32_t dtype,
                      int32_t device, msfft_plan* out, char* err, size_t errlen);
void msfft_plan_destroy(msfft_plan plan);

/* Data-independent stats of the plan (samples_used/runtime left 0). */
int msfft_plan_stats(msfft_plan plan, msfft_stats* stats);

/* Transforms `batch` signals x[s * x_stride .. + n), s < batch, with seeds
 * seeds[s] (host array).  Outputs are [batch][k] (out_f int64, out_c
 * interleaved float64) and out_count[batch], in host or device memory per
 * out_location.  Host inputs are streamed to the device in chunks overlapped
 * with compute.  stream: cudaStream_t (NULL = the plan's own stream); the
 * call returns after the outputs are complete.  *device_ms (optional): CUDA
 * event time from the first device operation to the last. */
int msfft_execute(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                  int32_t x_location, const uint64_t* seeds, int64_t* out_f, double* out_c,
                  int64_t* out_count, int32_t out_location, uint32_t flags, void* stream,
                  double* device_ms, char* err, size_t errlen);

/* Waits for the plan's work on `stream` (NULL: the plan's own stream) and
 * returns the first error raised by asynchronous msfft_execute calls since
 * the last sync (then clears it). */
int msfft_plan_sync(msfft_plan plan, void* stream, char* err, size_t errlen);

/* Algorithmic traffic of the fused gather for `batch` signals with these
 * seeds (host computation from the plan, data independent): *loads = samples
 * loaded (each distinct t' of an iteration once), *sectors = distinct 32-byte
 * sectors they touch, summed over iterations and signals. */
int msfft_plan_gather_traffic(msfft_plan plan, int64_t batch, const uint64_t* seeds,
                              int64_t* loads, int64_t* sectors);

/* [encode, bucket FFT for b > 256, decode] milliseconds of the last
 * msfft_execute issued with MSFFT_FLAG_STAGE_TIMES (summed over chunks). */
int msfft_plan_stage_times(msfft_plan plan, double* ms3);

/* Number of device kernel launches one msfft_execute of `batch` device-
 * resident signals issues (for bench accounting). */
int64_t msfft_plan_launches(msfft_plan plan, int64_t batch, uint32_t flags);

/* Samples per signal that msfft_execute moves host->device for HOST inputs:
 * with sparse ingest, only the samples the transform reads (gathered on the
 * host by all its threads into pinned staging; the finiteness scan of the
 * whole signal also runs on the host); 0 = dense path (whole signals are
 * copied).  Sparse ingest is used when it moves at most n/4 samples per
 * signal and the environment does not set MSFFT_SPARSE_INGEST=0. */
int64_t msfft_plan_ingest_samples(msfft_plan plan);

/* ComplexSignal::validate (proj/src/signal.cpp:18-26; decl
 * proj/include/msfft/signal.hpp:13-18) for `batch` signals of n samples,
 * x_stride samples apart: n a power of two >= 4, sample_count == n, every
 * sample finite -- checked in that order, with the reference's messages
 * (MSFFT_ERR_INVALID_ARGUMENT).  Device input: one HBM-bound scan on
 * `stream` (NULL = legacy default), synchronous; *device_ms (optional)
 * receives the scan kernel's CUDA-event time.  Host input: scanned on the
 * calling thread. */
int msfft_validate_signal(const void* x, int64_t n, int64_t sample_count, int64_t batch,
                          int64_t x_stride, int32_t dtype, int32_t x_location, void* stream,
                          double* device_ms, char* err, size_t errlen);

/* Bytes the plan's last msfft_execute moved host->device (whole signals or
 * compact ingest rows, rows copied whole for device-side validation, seeds)
 * and device->host (results, status flags).  No reference counterpart: the
 * e2e accounting of bench.py. */
int msfft_plan_copy_bytes(msfft_plan plan, int64_t* h2d, int64_t* d2h);

/* ---- split phases: one signal sharded by index range over several GPUs ----
 * No reference counterpart (the reference transforms one signal on one host,
 * sfft4.cpp:133-200); this is the SURVEY §8(e) multi-GPU path.  A rank holding
 * x[x_lo, x_hi) of each signal calls msfft_encode_values to get PARTIAL
 * bucket values (every round of every iteration; the samples it does not hold
 * count as 0).  Bucketize is linear in x, so summing the partial vectors of
 * ranks whose ranges tile [0, n) (one all-reduce) gives the full vector, up to
 * the order of that final sum.  msfft_decode_values then runs selection,
 * locate and estimate on it exactly as msfft_execute does after its encode.
 * x (x_stride >= x_hi - x_lo samples per signal), y ([batch][values_per_signal]
 * complex128), out_f/out_c/out_count ([batch][k], [batch]) are DEVICE
 * pointers; seeds is a host array.  decode consumes y (subtraction happens in
 * place).  flags: MSFFT_FLAG_ASSUME_VALID skips the finite check of the slice. */
int64_t msfft_plan_values_per_signal(msfft_plan plan);
int msfft_encode_values(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                        int64_t x_lo, int64_t x_hi, const uint64_t* seeds, double* y,
                        uint32_t flags, void* stream, char* err, size_t errlen);
/* Tap-range sharding (x replicated on every rank): part `part` of `parts`
 * walks only its contiguous share of every encode task's t' segments (all
 * rounds, all iterations) and writes PARTIAL bucket values; the parts' vectors
 * sum to the full vector.  Per-rank encode work is 1/parts of the whole
 * (msfft_encode_values' index-range split walks every tap on every rank).
 * x holds whole signals (x_stride >= n); the finiteness check covers the
 * part-th slice of each signal.  Iterations with b > 256 are written as FOLDS
 * (before their b-point FFT, which is linear): decode the summed vector with
 * msfft_decode_folds, which runs those FFTs once and then decodes. */
int msfft_encode_values_part(msfft_plan plan, int64_t batch, const void* x, int64_t x_stride,
                             int64_t part, int64_t parts, const uint64_t* seeds, double* y,
                             uint32_t flags, void* stream, char* err, size_t errlen);
int msfft_decode_values(msfft_plan plan, int64_t batch, double* y, const uint64_t* seeds,
                        int64_t* out_f, double* out_c, int64_t* out_count, void* stream,
                        char* err, size_t errlen);

int msfft_decode_folds(msfft_plan plan, int64_t batch, double* y, const uint64_t* seeds,
                       int64_t* out_f, double* out_c, int64_t* out_count, void* stream,
                       char* err, size_t errlen);

/* ---- signal helpers: the steps either side of the path -------
 * Reference: proj/src/signal.cpp, proj/src/io.cpp, proj/src/bench.cpp:33-46.
 * `location` says where x / spec / out live (MSFFT_HOST or MSFFT_DEVICE); the
 * work runs on the current device either way. */

/* error_metrics (signal.cpp:154-184 / signal.hpp:31-38). */
typedef struct msfft_eval_metrics {
    int64_t l0_err; /* coefficients off by more than 1e-6 */
    double l1_err;  /* (1/k) sum |d|                       */
    double l2_err;  /* sqrt((1/k) sum |d|^2)               */
} msfft_eval_metrics;

/* generate_test_signal (signal.cpp:116-121): the truth (k distinct positions
 * by Floyd sampling, unit coefficients with uniform phase) is drawn with the
 * reference's mt19937_64 sampler, so truth_f (ascending) / truth_c
 * (interleaved) are identical to the reference's; x (n samples, dtype) is
 * synthesized on the device -- bit-identical to synthesize() when
 * k * ceil(n/1024) <= 2^23 (*bit_exact = 1), else within ulps (device seeds). */
int msfft_generate_test_signal(int64_t n, int64_t k, uint64_t seed, int32_t dtype,
                               int32_t location, void* x, int64_t* truth_f, double* truth_c,
                               int32_t* bit_exact, char* err, size_t errlen);

/* synthesize (signal.cpp:76-98) of `count` entries (f strictly ascending,
 * c interleaved, host arrays) into x. */
int msfft_synthesize(int64_t n, const int64_t* f, const double* c, int64_t count, int32_t dtype,
                     int32_t location, void* x, int32_t* bit_exact, char* err, size_t errlen);

/* add_awgn (signal.cpp:123-152) in place: same validation, +infinity
 * sentinel and realised-power scaling; the complex Gaussian noise comes from
 * Philox4x32-10 counters (seed, sample index) on the device -- the same law,
 * not the reference's sample sequence. */
int msfft_add_awgn(void* x, int64_t n, int32_t dtype, int32_t location, double snr_db,
                   uint64_t seed, char* err, size_t errlen);

/* dft_dense (signal.cpp:37-44): out[s][i] = (1/n) sum_j x[s][j] e^{-2 pi i ij/n}
 * for `batch` contiguous signals; out is complex128 in the same location.
 * Bit-identical to the reference.  idft_dense (signal.cpp:46-54): the
 * unnormalised inverse of complex128 spectra. */
int msfft_dft_dense(const void* x, int64_t n, int64_t batch, int32_t dtype, int32_t location,
                    double* out, char* err, size_t errlen);
int msfft_idft_dense(const double* spec, int64_t n, int64_t batch, int32_t location, double* out,
                     char* err, size_t errlen);

/* top_k_spectrum (bench.cpp:33-46): the k largest |spec[i]| of a complex128
 * spectrum as (f ascending, c) in host arrays of capacity k; ties at the k-th
 * magnitude keep the lowest indices. */
int msfft_top_k_spectrum(const double* spec, int64_t n, int64_t k, int32_t location,
                         int64_t* out_f, double* out_c, int64_t* out_count, char* err,
                         size_t errlen);

/* error_metrics over host (f, c) lists; duplicate positions: the last wins
 * (std::map assignment). */
int msfft_error_metrics(int64_t truth_n, const int64_t* truth_f, const double* truth_c,
                        int64_t truth_count, int64_t est_n, const int64_t* est_f,
                        const double* est_c, int64_t est_count, int64_t k,
                        msfft_eval_metrics* out, char* err, size_t errlen);

/* MSFT signal files (io.cpp:17-55): 8-byte magic "MSFT\0\0\0\0", u64 n, n
 * little-endian float64 (re, im) pairs.  Errors are MSFFT_ERR_RUNTIME with the
 * reference's messages ("read_signal_file: bad magic in <path>", ...);
 * non-finite samples MSFFT_ERR_INVALID_ARGUMENT.  Reading into complex64
 * rounds each component. */
int msfft_signal_file_length(const char* path, int64_t* n, char* err, size_t errlen);
int msfft_read_signal_file(const char* path, int32_t dtype, int32_t location, void* x,
                           int64_t cap, int64_t* n, char* err, size_t errlen);
int msfft_write_signal_file(const char* path, const void* x, int64_t n, int32_t dtype,
                            int32_t location, char* err, size_t errlen);

/* Truth CSV (io.cpp:57-92): "position,re,im" then rows "%lld,%.17g,%.17g". */
int msfft_write_truth_csv(const char* path, const int64_t* f, const double* c, int64_t count,
                          char* err, size_t errlen);
int msfft_read_truth_csv(const char* path, int64_t n, int64_t* f, double* c, int64_t cap,
                         int64_t* count, char* err, size_t errlen);

/* ---- phase-error Monte Carlo (phase_mc.hpp:14-56, paper Fig. 5) ---------------
 * run_phase_experiment: per SNR, the accepted-trial histogram of the
 * locator's phase error.  The attempts (spectra, sigma, noise seeds, bucket
 * picks) replay the reference's Rng streams exactly on the host; the two
 * lazy-source bucketizations of every trial run on the device.  trials_out
 * (nullable) receives [nsnr][trials] accepted trials in order. */
#define MSFFT_PHASE_BINS 70
typedef struct msfft_phase_histogram {
    double snr_db;
    int64_t n, k, l_width, trials;
    double bin_mass[MSFFT_PHASE_BINS]; /* 0.1-wide log10 bins over [-6, 1) */
    double p50, p99, max;
} msfft_phase_histogram;
typedef struct msfft_phase_trial {
    double dphi;
    int64_t u, bucket, tau;
    double y0[2], y_tau[2];
    double measured_phi, true_phi;
} msfft_phase_trial;
int msfft_phase_experiment(int64_t n, int64_t k, int64_t b, const double* snr_list, int64_t nsnr,
                           int64_t trials, uint64_t seed, msfft_phase_histogram* out,
                           msfft_phase_trial* trials_out, char* err, size_t errlen);

/* ---- host-only plan pieces (no device needed) -------------------------------
 * sigma_m, sigma^-1_m for the first `iterations` iterations of a transform
 * seeded `seed`: random_params(n, Rng(seed), 0) per iteration
 * (proj/src/bucketize.cpp:39-48, proj/src/sfft4.cpp:48). */
int msfft_sigma_plan(uint64_t seed, int64_t n, int32_t iterations, int64_t* sigma,
                     int64_t* sigma_inv, char* err, size_t errlen);
/* The tau plan {0, tau_1..tau_R} of an iteration with bucket width l_width
 * (stage_count + tau_schedule, proj/src/sfft4.cpp:49-55, locate.cpp:39-53). */
int msfft_tau_plan(double l_width, int64_t n, int64_t l, double q, int64_t* taus, int32_t cap,
                   int32_t* rounds, char* err, size_t errlen);

/* ---- the reference's scalar plan helpers (host; same code the plan uses) -----
 * mod_inverse      proj/src/bucketize.cpp:21-37 (errors: even sigma, bad n)
 * bucket_of        proj/src/bucketize.cpp:63-68 (returns -1 for l_width/b <= 0)
 * stage_count      proj/src/locate.cpp:44-53 (the reference loops forever when
 *                  l/(q+1) <= 1; here that is the MultiscaleConfig error)
 * tau_schedule     proj/src/locate.cpp:39-42
 * config_validate  MultiscaleConfig::validate, proj/src/locate.cpp:25-30
 * check_parameter_bounds  proj/src/locate.cpp:125-132 (q unused, as there)
 * initial_bucket_count    proj/src/sfft4.cpp:115-129 (windows designed on the
 *                  GPU, so it needs a device) */
int msfft_mod_inverse(int64_t sigma, int64_t n, int64_t* out, char* err, size_t errlen);
int64_t msfft_bucket_of(int64_t u, int64_t l_width, int64_t b);
int msfft_stage_count(double region_length, int64_t l, double q, int32_t* out, char* err,
                      size_t errlen);
int msfft_tau_schedule(double region_length, int64_t n, int64_t* out, char* err, size_t errlen);
int msfft_config_validate(int64_t l, double q, char* err, size_t errlen);
int msfft_check_parameter_bounds(double max_dphi, int64_t l, double q, int32_t* l_ok,
                                 double* q_min, char* err, size_t errlen);
int msfft_initial_bucket_count(int64_t n, int64_t k, double delta, int64_t* out, char* err,
                               size_t errlen);

/* ---- the locate arithmetic, batched on the device ---------------------------
 * Each evaluates, for `count` host-array entries, the same device functions
 * the fused / wide decodes run (so callers and tests see the GPU's
 * arithmetic):
 * phase_of                 proj/src/locate.cpp:32-37: z interleaved complex128,
 *                          status[k] = 1 where z == 0 (the reference throws
 *                          std::domain_error "phase_of: zero value")
 * position_phase           proj/src/locate.cpp:19-23 (n a power of two)
 * circular_phase_distance  proj/src/locate.cpp:14-17
 * locate_step              proj/src/locate.cpp:63-81: measurement (phi[k],
 *                          tau[k]), region[k] -> out[k] */
typedef struct msfft_locate_region {  /* LocateRegion, locate.hpp:23-32 */
    double u_min;
    double length;
    int32_t stage;
    int32_t reserved;
} msfft_locate_region;
int msfft_phase_of(const double* z, int64_t count, double* phase, int32_t* status, char* err,
                   size_t errlen);
int msfft_position_phase(const double* u, const int64_t* tau, int64_t count, int64_t n,
                         double* out, char* err, size_t errlen);
int msfft_circular_phase_distance(const double* a, const double* b, int64_t count, double* out,
                                  char* err, size_t errlen);
int msfft_locate_step(const double* phi, const int64_t* tau, const msfft_locate_region* region,
                      int64_t count, int64_t l, double q, int64_t n, msfft_locate_region* out,
                      char* err, size_t errlen);

/* bucketize_fn<Sampler> (proj/include/msfft/bucketize.hpp:63-86): the caller
 * evaluates its sampler once per tap in increasing tap order (the reference's
 * contract) into values[r][h + t], t = -h..h (w = window support, complex128,
 * host); the GPU folds per bin in ascending t, runs the radix-2 DIT and
 * scales by 1/n: out [rounds][b] complex128 (host), bit-identical to the
 * reference's fold.  *samples_read (optional) = w. */
int msfft_bucketize_taps(int64_t n, int64_t b, double delta, const double* values, int64_t rounds,
                         double* out, int64_t* samples_read, char* err, size_t errlen);

/* ---- kernel-level entry points (parity tests) ------------------------------
 * Window taps/support exactly as design_flat_window (window.cpp:105-177). */
int msfft_window(int64_t n, int64_t b, double delta, int32_t device, int64_t* w, double* taps,
                 int64_t taps_cap, char* err, size_t errlen);
/* FlatWindow::response_at (window.cpp:89-99) at any integer offsets idx[k]
 * (reduced mod n), evaluated on the device with the series the decode's
 * response table uses (for |idx| <= 3L/2 + 1 exactly the table's values). */
int msfft_window_response(int64_t n, int64_t b, double delta, int32_t device,
                          const int64_t* idx, int64_t count, double* out, char* err,
                          size_t errlen);
/* One signal (host memory), returning every iteration's bucket vectors before
 * (pre: encode output, BucketSet::values of bucketize) and after (post) the
 * subtraction of known tones, iteration-major then round-major, plus the
 * final spectrum.  pre/post hold the plan's sum_m rounds_m*b_m complex
 * values.  sel_* (optional, sum_m budget_m slots, iteration-major then by
 * rank of |y0|): bucket id, located frequency f (-1 when below threshold,
 * not located or rejected by the estimate) and the estimate value
 * (run_iteration, proj/src/sfft4.cpp:75-103). */
int msfft_trace(const void* x, int64_t n, int32_t dtype, int64_t k, int64_t l, double q,
                uint64_t seed, double delta, double* pre, double* post, int64_t* sel_bucket,
                int64_t* sel_f, double* sel_value, int64_t cap, int64_t* out_f, double* out_c,
                int64_t* out_count, char* err, size_t errlen);

/* ---- the reference's component API on the path --------------
 * Batched device versions of the functions the reference's own tests call
 * directly.  `location` flags say where each array lives (MSFFT_HOST or
 * MSFFT_DEVICE); complex arrays are interleaved (re, im) doubles.
 *
 * bucketize (proj/src/bucketize.cpp:50-61, bucketize.hpp:63-86) of one
 * signal x (n samples, dtype) under `rounds` permutations (sigma[r], tau[r])
 * (host arrays) with the window (n, b, delta): values [rounds][b], bit-equal
 * to the reference; *samples_read = w. */
int msfft_bucketize(const void* x, int64_t n, int32_t dtype, int32_t x_location, int64_t b,
                    double delta, const int64_t* sigma, const int64_t* tau, int64_t rounds,
                    double* values, int32_t values_location, int64_t* samples_read, char* err,
                    size_t errlen);
/* predict_buckets (bucketize.cpp:70-95) of `count` known tones (f strictly
 * ascending in [0, n), c) for each (sigma[r], tau[r]): values [rounds][b].
 * f, c and values are in `location`. */
int msfft_predict_buckets(int64_t n, int64_t b, double delta, const int64_t* f, const double* c,
                          int64_t count, const int64_t* sigma, const int64_t* tau,
                          int64_t rounds, double* values, int32_t location, char* err,
                          size_t errlen);
/* locate_frequency (proj/src/locate.cpp:83-123) of `count` buckets against
 * one round set: rounds [nrounds][b] (round r bucketized with tau[r], host
 * array; tau[0] must be 0), config (l, q).  Per bucket: u, stages and status
 * (0 located, 1 nullopt: a needed bucket value is exactly zero).  A zero
 * quotient raises MSFFT_ERR_DOMAIN "phase_of: zero value" as the
 * reference's phase_of throws.  buckets/rounds/u/stages/status in
 * `location`. */
int msfft_locate_frequency(int64_t n, int64_t b, int64_t l, double q, const int64_t* buckets,
                           int64_t count, const double* rounds, const int64_t* tau,
                           int64_t nrounds, int64_t* u, int32_t* stages, int32_t* status,
                           int32_t location, char* err, size_t errlen);
/* estimate_value (proj/src/sfft4.cpp:27-36) of `count` (y0, u) pairs with the
 * window (n, b, delta): out = y0 / G_{iL-u}; status 1 where |G| < 0.5 (the
 * reference throws std::domain_error "estimate_value: located position
 * outside the pass region").  y0/u/out/status in `location`. */
int msfft_estimate_values(int64_t n, int64_t b, double delta, const double* y0, const int64_t* u,
                          int64_t count, double* out, int32_t* status, int32_t location,
                          char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif /* MSFFT_B200_H */
