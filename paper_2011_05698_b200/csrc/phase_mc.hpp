// phase_mc.hpp -- the phase-error Monte Carlo of the reference
// (proj/src/phase_mc.cpp:94-212, paper Fig. 5) on the GPU: SURVEY.md 8(f)
// row 4.
//
// Per SNR the reference draws attempts from one Rng stream; each attempt
// draws a K-tone spectrum, sigma, a noise seed and up to b bucket picks, then
// bucketizes a lazily evaluated, permuted, noisy signal at tau = 0 and
// tau = round(n/L) and measures the phase error of the chosen isolated tone.
// Here the RNG replay (everything that decides WHICH trials exist) runs on
// the host with the reference's exact draws; the two O(w K) bucketizations
// of every candidate run on the device, one CTA per (trial, round).  Tone
// phasors use exact angles and device libm (the reference steps a phasor
// recurrence re-synced every 512 taps), so y0 / y_tau agree to ~1e-13
// relative and dphi to ~1e-13 absolute.
#pragma once

#include <cstdint>
#include <vector>

namespace msfft_b200 {

constexpr int kPhaseBins = 70;  // PhaseErrorHistogram::kBinCount (phase_mc.hpp:25-29)

struct PhaseTrialOut {
    double dphi = 0.0;
    int64_t u = 0, bucket = 0, tau = 0;
    double y0[2] = {0, 0}, y_tau[2] = {0, 0};
    double measured_phi = 0.0, true_phi = 0.0;
};

struct PhaseHistogramOut {
    double snr_db = 0.0;
    int64_t n = 0, k = 0, l_width = 0, trials = 0;
    double bin_mass[kPhaseBins] = {};
    double p50 = 0.0, p99 = 0.0, max = 0.0;
};

// run_phase_experiment (phase_mc.cpp:166-212).  If `trials_out` is given it
// receives, per SNR, the accepted trials in acceptance order.
std::vector<PhaseHistogramOut> phase_experiment(int64_t n, int64_t k, int64_t b,
                                                const std::vector<double>& snr_list,
                                                int64_t trials, uint64_t seed,
                                                std::vector<std::vector<PhaseTrialOut>>* trials_out);

}  // namespace msfft_b200
