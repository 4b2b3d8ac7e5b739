// test_dropin.cpp -- a reference-style caller switched to the B200 drop-in.
// Mirrors run_cell (proj/src/bench.cpp:104-152): generate -> transform ->
// compare, here against the reference library's own sfft4 (oracle ABI).
// Build: g++ -std=c++17 -I include tests/cpp/test_dropin.cpp
//        -L paper_2011_05698_b200 -lmsfft_b200 -L oracle/_ref -lmsfft_ref
#define MSFFT_B200_AS_MSFFT
#include <cmath>
#include <cstdio>

#include "../../oracle/oracle_api.h"
#include "msfft_b200.hpp"

int main() {
    const int64_t n = 1 << 16, k = 50;
    const uint64_t seed = 7;
    std::vector<double> xi(2 * n), c_truth(2 * k);
    std::vector<int64_t> f_truth(k);
    char err[512];
    if (orc_generate_test_signal(n, k, orc_splitmix64(seed ^ 0x51), xi.data(), f_truth.data(),
                                 c_truth.data(), err, sizeof(err)) != 0) {
        std::printf("generate failed: %s\n", err);
        return 2;
    }
    msfft::ComplexSignal x;
    x.n = n;
    x.samples.resize(n);
    for (int64_t j = 0; j < n; ++j) x.samples[j] = msfft::cplx(xi[2 * j], xi[2 * j + 1]);
    const uint64_t algo = orc_splitmix64(seed ^ 0x53);
    const msfft::SfftResult r = msfft::sfft4(x, k, msfft::MultiscaleConfig{16, 1.0}, algo, 1e-8);

    std::vector<int64_t> rf(k);
    std::vector<double> rc(2 * k);
    int64_t cnt = 0;
    std::vector<int64_t> si(4 + ORC_MAX_ITERS);
    double sd[2];
    if (orc_sfft4(n, xi.data(), k, 16, 1.0, algo, 1e-8, k, rf.data(), rc.data(), &cnt, si.data(),
                  sd, err, sizeof(err)) != 0) {
        std::printf("reference failed: %s\n", err);
        return 2;
    }
    if (static_cast<int64_t>(r.spectrum.entries.size()) != cnt) {
        std::printf("count %zu vs %ld\n", r.spectrum.entries.size(), static_cast<long>(cnt));
        return 1;
    }
    int64_t i = 0;
    double worst = 0.0;
    for (const auto& [f, c] : r.spectrum.entries) {
        if (f != rf[i]) {
            std::printf("support differs at %ld: %ld vs %ld\n", static_cast<long>(i),
                        static_cast<long>(f), static_cast<long>(rf[i]));
            return 1;
        }
        const msfft::cplx ref(rc[2 * i], rc[2 * i + 1]);
        worst = std::max(worst, std::abs(c - ref) / std::abs(ref));
        ++i;
    }
    if (r.stats.samples_used != si[0] || r.stats.iterations != si[2] || r.stats.b_first != si[3]) {
        std::printf("stats differ\n");
        return 1;
    }
    try {
        msfft::sfft4(x, n, msfft::MultiscaleConfig{16, 1.0}, algo, 1e-8);
        std::printf("expected invalid_argument\n");
        return 1;
    } catch (const std::invalid_argument& e) {
        if (std::string(e.what()) != "sfft4: need 1 <= K <= n/8") {
            std::printf("wrong message: %s\n", e.what());
            return 1;
        }
    }
    std::printf("dropin ok: %ld entries identical support, max rel err %.3e\n",
                static_cast<long>(cnt), worst);
    return worst <= 1e-9 ? 0 : 1;
}
