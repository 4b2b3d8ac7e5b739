/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The C ABI that both CPU oracles implement:
 *   - oracle/ref_shim.cpp      wraps the reference library's own public API
 *                              (compiled from /root/reference/proj/src into
 *                              oracle/_ref/libmsfft_ref.so by oracle/Makefile);
 *   - oracle/port/msfft_port.cpp  is an independent CPU restatement of the same
 *                              algorithm (oracle/_port/libmsfft_port.so).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load these libraries, and only as the checker or the CPU baseline.
 * The product (paper_2011_05698_b200/) never links or calls anything here.
 *
 * Conventions
 *   - complex buffers are interleaved (re, im) float64;
 *   - every function returning int uses ORC_OK / ORC_INVALID_ARGUMENT /
 *     ORC_DOMAIN_ERROR / ORC_OTHER and copies exception text into err[errlen];
 *   - ORC_INVALID_ARGUMENT mirrors std::invalid_argument in the reference,
 *     ORC_DOMAIN_ERROR mirrors std::domain_error.
 */
#ifndef MSFFT_ORACLE_API_H
#define MSFFT_ORACLE_API_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_INVALID_ARGUMENT = 1, ORC_DOMAIN_ERROR = 2, ORC_OTHER = 3 };

#define ORC_MAX_ITERS 64
#define ORC_MAX_ROUNDS 512

/* Which implementation this library is: "reference" or "port". */
const char* orc_kind(void);

/* ---- scalars / plan pieces (proj/src/locate.cpp, bucketize.cpp, sfft4.cpp) ---- */
uint64_t orc_splitmix64(uint64_t x);
int orc_mod_inverse(int64_t sigma, int64_t n, int64_t* out, char* err, int64_t errlen);
int64_t orc_bucket_of(int64_t u, int64_t l_width, int64_t b);
int64_t orc_tau_schedule(double region_length, int64_t n);
int orc_stage_count(double region_length, int64_t l, double q);
int orc_check_parameter_bounds(double max_dphi, int64_t l, double q, int* l_ok, double* q_min,
                               char* err, int64_t errlen);
int orc_cfg_validate(int64_t l, double q, char* err, int64_t errlen);
/* random_params with tau_override = 0 (as sfft4 uses it), `count` successive
 * draws from Rng(seed). */
int orc_random_params(int64_t n, uint64_t seed, int64_t count, int64_t* sigma, int64_t* sigma_inv,
                      char* err, int64_t errlen);
int orc_initial_bucket_count(int64_t n, int64_t k, double delta, int64_t* out, char* err,
                             int64_t errlen);

/* Data-independent plan of sfft4(n, k, {l,q}, seed, delta): iterations, b_m,
 * w_m, rounds (R_m + 1), the tau plan (flattened, rounds[m] entries each),
 * sigma_m, sigma_inv_m, budget_m = min(k_m, b_m).  Arrays have room for
 * ORC_MAX_ITERS iterations and ORC_MAX_ROUNDS taus in total. */
typedef struct orc_plan {
    int32_t iterations;
    int64_t b_first;
    int64_t b[ORC_MAX_ITERS];
    int64_t w[ORC_MAX_ITERS];
    int32_t rounds[ORC_MAX_ITERS];
    int64_t k_m[ORC_MAX_ITERS];
    int64_t budget[ORC_MAX_ITERS];
    int64_t sigma[ORC_MAX_ITERS];
    int64_t sigma_inv[ORC_MAX_ITERS];
    int64_t taus[ORC_MAX_ROUNDS];
} orc_plan;
int orc_plan_build(int64_t n, int64_t k, int64_t l, double q, uint64_t seed, double delta,
                   orc_plan* plan, char* err, int64_t errlen);

/* ---- flat window (proj/src/window.cpp) ---- */
/* Designs (or fetches from the process cache) the window; writes w and, if
 * taps_cap >= w, the w taps g_time[0..w). */
int orc_window(int64_t n, int64_t b, double delta, int64_t* w, double* taps, int64_t taps_cap,
               char* err, int64_t errlen);
int orc_response_at(int64_t n, int64_t b, double delta, const int64_t* idx, int64_t count,
                    double* out, char* err, int64_t errlen);

/* ---- bucketization (proj/src/bucketize.cpp) ---- */
int orc_bucketize(int64_t n, const double* x, int64_t b, double delta, int64_t sigma, int64_t tau,
                  double* out, char* err, int64_t errlen);
int orc_predict(int64_t n, int64_t b, double delta, int64_t nk, const int64_t* f, const double* c,
                int64_t sigma, int64_t tau, double* out, char* err, int64_t errlen);

/* locate_frequency (proj/src/locate.cpp:83-123).  round_vals holds nrounds
 * rounds of b interleaved values; taus their offsets (taus[0] must be 0).
 * *u = -1 when the reference returns nullopt. */
int orc_locate(int64_t n, int64_t b, double delta, int64_t l, double q, int64_t bucket,
               int64_t nrounds, const int64_t* taus, const double* round_vals, int64_t* u,
               int* stages, char* err, int64_t errlen);
int orc_estimate_value(int64_t n, int64_t b, double delta, double y_re, double y_im, int64_t u,
                       double* out, char* err, int64_t errlen);

/* ---- full transform (proj/src/sfft4.cpp:131-187) ----
 * x: n interleaved complex128.  Output entries in ascending f (map order).
 * stats_i: [samples_used, samples_round_sum, iterations, b_first,
 *           stage_counts[0..iterations)]  (room for 4 + ORC_MAX_ITERS)
 * stats_d: [sample_fraction, runtime_ms] */
int orc_sfft4(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
              double delta, int64_t cap, int64_t* out_f, double* out_c, int64_t* out_count,
              int64_t* stats_i, double* stats_d, char* err, int64_t errlen);

/* Per-iteration intermediates of the same transform (a replay of
 * run_iteration through the public calls).  Buffer sizes follow the plan:
 *   pre/post: sum_m rounds[m]*b[m] complex values (bucket vectors before and
 *             after subtracting the known tones), iteration-major;
 *   sel_*:    sum_m budget[m] slots; per selected rank: bucket id (-1 if the
 *             rank was below threshold), located u (-1 nullopt), status
 *             (0 = accepted, 1 = below threshold, 2 = locate nullopt,
 *             3 = estimate rejected), value (2 doubles), f.
 * Returns the final spectrum like orc_sfft4. */
int orc_sfft4_trace(int64_t n, const double* x, int64_t k, int64_t l, double q, uint64_t seed,
                    double delta, double* pre, double* post, int64_t* sel_bucket, int64_t* sel_u,
                    int32_t* sel_status, double* sel_value, int64_t* sel_f, int64_t cap,
                    int64_t* out_f, double* out_c, int64_t* out_count, char* err,
                    int64_t errlen);

/* Threaded batch of independent transforms over complex64 signals (upcast
 * exactly to complex128), one std::thread worker per `threads`, like the
 * reference's run_sweep pool (proj/src/bench.cpp:242-280).  out_* are
 * [nsig][cap].  *wall_ms is the wall time of the whole batch (windows are
 * pre-resolved before the clock starts). */
int orc_sfft4_batch_c64(int64_t nsig, int64_t n, const float* x, int64_t k, int64_t l, double q,
                        const uint64_t* seeds, double delta, int threads, int64_t cap,
                        int64_t* out_f, double* out_c, int64_t* out_count, double* wall_ms,
                        char* err, int64_t errlen);

/* ---- signal model (proj/src/signal.cpp) ---- */
int orc_generate_test_signal(int64_t n, int64_t k, uint64_t seed, double* x, int64_t* f,
                             double* c, char* err, int64_t errlen);
int orc_add_awgn(int64_t n, double* x, double snr_db, uint64_t seed, char* err, int64_t errlen);

/* ---- signal helpers, SURVEY 8(f) rows 2-3 (signal.cpp, io.cpp, bench.cpp) ---- */
/* dft_dense (signal.cpp:37-44) / idft_dense (:46-54); x, out: n complex. */
int orc_dft_dense(int64_t n, const double* x, double* out, char* err, int64_t errlen);
int orc_idft_dense(int64_t n, const double* spec, double* out, char* err, int64_t errlen);
/* synthesize (signal.cpp:76-98) of `count` entries (f ascending). */
int orc_synthesize(int64_t n, int64_t count, const int64_t* f, const double* c, double* x,
                   char* err, int64_t errlen);
/* error_metrics (signal.cpp:154-184): out_l0, out_l1, out_l2. */
int orc_error_metrics(int64_t n, int64_t tcount, const int64_t* tf, const double* tc,
                      int64_t ecount, const int64_t* ef, const double* ec, int64_t k,
                      int64_t* out_l0, double* out_l1, double* out_l2, char* err,
                      int64_t errlen);
/* top_k_spectrum (bench.cpp:33-46): k largest |spec| as ascending (f, c). */
int orc_top_k_spectrum(int64_t n, const double* spec, int64_t k, int64_t* out_f, double* out_c,
                       int64_t* out_count, char* err, int64_t errlen);
/* MSFT signal files and truth CSV (io.cpp:17-92). */
int orc_write_signal_file(const char* path, int64_t n, const double* x, char* err,
                          int64_t errlen);
int orc_read_signal_file(const char* path, int64_t cap, double* x, int64_t* n, char* err,
                         int64_t errlen);
int orc_write_truth_csv(const char* path, int64_t n, int64_t count, const int64_t* f,
                        const double* c, char* err, int64_t errlen);
int orc_read_truth_csv(const char* path, int64_t n, int64_t cap, int64_t* f, double* c,
                       int64_t* count, char* err, int64_t errlen);

/* ---- phase-error Monte Carlo (phase_mc.cpp:94-212) ----
 * run_phase_experiment: per SNR, bin_mass[70], p50, p99, max (out_hist is
 * [nsnr][73]: 70 masses then p50, p99, max). */
int orc_phase_experiment(int64_t n, int64_t k, int64_t b, const double* snr, int64_t nsnr,
                         int64_t trials, uint64_t seed, double* out_hist, char* err,
                         int64_t errlen);
/* The accepted trials of SNR index si of the same experiment, in order:
 * out_i [trials][3] = u, bucket, tau; out_d [trials][7] = y0 (re, im),
 * y_tau (re, im), measured_phi, true_phi, dphi. */
int orc_phase_trials(int64_t n, int64_t k, int64_t b, double snr, int64_t si, int64_t trials,
                     uint64_t seed, int64_t* out_i, double* out_d, char* err, int64_t errlen);

#ifdef __cplusplus
}
#endif
#endif
