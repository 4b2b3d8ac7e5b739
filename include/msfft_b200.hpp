// msfft_b200.hpp -- header-only C++ drop-in over the C ABI (msfft_b200.h).
//
// Mirrors the reference's public types and entry point
//   SfftResult sfft4(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
//                    uint64_t seed, double delta = 1e-8);
// (proj/include/msfft/sfft4.hpp:32-45, 64-65; signal.hpp:13-28;
// locate.hpp:13-19) with the same field names, the same ascending std::map
// result and the same exception classes/messages.  A caller of the reference
// switches by including this header and linking libmsfft_b200.so; defining
// MSFFT_B200_AS_MSFFT before the include also makes `msfft::` name these
// types (only when the reference headers are not included in the same TU).
#pragma once

#include <complex>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "msfft_b200.h"

namespace msfft_b200 {

using cplx = std::complex<double>;

struct ComplexSignal {
    int64_t n = 0;
    std::vector<cplx> samples;
};

struct SparseSpectrum {
    int64_t n = 0;
    std::map<int64_t, cplx> entries;
};

struct MultiscaleConfig {
    int64_t l = 16;
    double q = 1.0;
    double shrink() const { return static_cast<double>(l) / (q + 1.0); }
};

struct TransformStats {
    int64_t samples_used = 0;
    int64_t samples_round_sum = 0;
    double sample_fraction = 0.0;
    double runtime_ms = 0.0;  // device time of the transform
    int iterations = 0;
    int64_t b_first = 0;
    std::vector<int> stage_counts;
};

struct SfftResult {
    SparseSpectrum spectrum;
    TransformStats stats;
};

// Thrown for device / CUDA failures (no CPU fallback exists).
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void throw_status(int status, const char* msg) {
    switch (status) {
        case MSFFT_OK: return;
        case MSFFT_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MSFFT_ERR_DOMAIN: throw std::domain_error(msg);
        case MSFFT_ERR_CUDA: throw DeviceError(msg);
        default: throw std::runtime_error(msg);
    }
}

inline SfftResult sfft4(const ComplexSignal& x, int64_t k, const MultiscaleConfig& cfg,
                        uint64_t seed, double delta = 1e-8) {
    if (static_cast<int64_t>(x.samples.size()) != x.n)
        throw std::invalid_argument("ComplexSignal: sample count != n");
    const int64_t cap = k > 0 ? k : 1;
    std::vector<int64_t> f(static_cast<size_t>(cap));
    std::vector<double> c(static_cast<size_t>(2 * cap));
    int64_t count = 0;
    msfft_stats st{};
    char err[1024] = {0};
    const int rc = msfft_sfft4(x.samples.data(), x.n, MSFFT_C128, MSFFT_HOST, k, cfg.l, cfg.q,
                               seed, delta, cap, f.data(), c.data(), &count, &st, err,
                               sizeof(err));
    throw_status(rc, err);
    SfftResult r;
    r.spectrum.n = x.n;
    for (int64_t i = 0; i < count; ++i) r.spectrum.entries[f[i]] = cplx(c[2 * i], c[2 * i + 1]);
    r.stats.samples_used = st.samples_used;
    r.stats.samples_round_sum = st.samples_round_sum;
    r.stats.sample_fraction = st.sample_fraction;
    r.stats.runtime_ms = st.runtime_ms;
    r.stats.iterations = st.iterations;
    r.stats.b_first = st.b_first;
    r.stats.stage_counts.assign(st.stage_counts, st.stage_counts + st.iterations);
    return r;
}

}  // namespace msfft_b200

#ifdef MSFFT_B200_AS_MSFFT
namespace msfft = msfft_b200;
#endif
