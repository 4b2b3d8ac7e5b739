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
    if (worst > 1e-9) return 1;

    // ---- the reference's functions around the transform (signal.hpp, io.hpp,
    // phase_mc.hpp, bench.cpp top_k_spectrum) against the reference library
#define CHECK(cond, what)                          \
    do {                                           \
        if (!(cond)) {                             \
            std::printf("FAILED: %s\n", what);     \
            return 1;                              \
        }                                          \
    } while (0)
    {
        const int64_t n2 = 1 << 14, k2 = 30;
        const auto [gx, gt] = msfft::generate_test_signal(n2, k2, 99);
        std::vector<double> rx(2 * n2), rct(2 * k2);
        std::vector<int64_t> rft(k2);
        CHECK(orc_generate_test_signal(n2, k2, 99, rx.data(), rft.data(), rct.data(), err,
                                       sizeof(err)) == 0, "reference generate");
        for (int64_t j = 0; j < n2; ++j)
            CHECK(gx.samples[j] == msfft::cplx(rx[2 * j], rx[2 * j + 1]), "generate bit-exact");
        int64_t t = 0;
        for (const auto& [f, c] : gt.entries) {
            CHECK(f == rft[t] && c == msfft::cplx(rct[2 * t], rct[2 * t + 1]), "truth identical");
            ++t;
        }
        const std::vector<msfft::cplx> X = msfft::dft_dense(gx);
        std::vector<double> RX(2 * n2);
        CHECK(orc_dft_dense(n2, rx.data(), RX.data(), err, sizeof(err)) == 0, "reference dft");
        for (int64_t j = 0; j < n2; ++j)
            CHECK(X[j] == msfft::cplx(RX[2 * j], RX[2 * j + 1]), "dft_dense bit-exact");
        const msfft::ComplexSignal back = msfft::idft_dense(X);
        std::vector<double> RB(2 * n2);
        CHECK(orc_idft_dense(n2, RX.data(), RB.data(), err, sizeof(err)) == 0, "reference idft");
        for (int64_t j = 0; j < n2; ++j)
            CHECK(back.samples[j] == msfft::cplx(RB[2 * j], RB[2 * j + 1]), "idft_dense bit-exact");
        const msfft::SparseSpectrum top = msfft::top_k_spectrum(X, n2, k2);
        std::vector<int64_t> tf(k2);
        std::vector<double> tc(2 * k2);
        int64_t tcount = 0;
        CHECK(orc_top_k_spectrum(n2, RX.data(), k2, tf.data(), tc.data(), &tcount, err,
                                 sizeof(err)) == 0, "reference top_k");
        t = 0;
        for (const auto& [f, c] : top.entries) {
            CHECK(f == tf[t] && c == msfft::cplx(tc[2 * t], tc[2 * t + 1]), "top_k identical");
            ++t;
        }
        const msfft::EvalMetrics m = msfft::error_metrics(gt, top, k2);
        int64_t l0 = 0;
        double l1 = 0, l2 = 0;
        CHECK(orc_error_metrics(n2, k2, rft.data(), rct.data(), tcount, tf.data(), tc.data(), k2,
                                &l0, &l1, &l2, err, sizeof(err)) == 0, "reference metrics");
        CHECK(m.l0_err == l0 && m.l1_err == l1 && m.l2_err == l2, "error_metrics identical");
        // files: ours -> reference reader, byte-identical CSV
        msfft::write_signal_file("/tmp/msfft_dropin.msft", gx);
        std::vector<double> fx(2 * n2);
        int64_t fn = 0;
        CHECK(orc_read_signal_file("/tmp/msfft_dropin.msft", n2, fx.data(), &fn, err,
                                   sizeof(err)) == 0 && fn == n2, "reference reads our file");
        CHECK(fx == rx, "signal file round trip");
        CHECK(msfft::read_signal_file("/tmp/msfft_dropin.msft").samples == gx.samples,
              "our reader");
        msfft::write_truth_csv("/tmp/msfft_dropin_a.csv", gt);
        CHECK(orc_write_truth_csv("/tmp/msfft_dropin_b.csv", n2, k2, rft.data(), rct.data(), err,
                                  sizeof(err)) == 0, "reference csv");
        const msfft::SparseSpectrum ta = msfft::read_truth_csv("/tmp/msfft_dropin_a.csv", n2);
        const msfft::SparseSpectrum tb = msfft::read_truth_csv("/tmp/msfft_dropin_b.csv", n2);
        CHECK(ta.entries == gt.entries && tb.entries == gt.entries, "truth csv round trip");
        try {
            msfft::read_signal_file("/tmp/msfft_dropin_missing.msft");
            CHECK(false, "missing file must throw");
        } catch (const std::runtime_error& e) {
            CHECK(std::string(e.what()).rfind("read_signal_file: cannot open", 0) == 0,
                  "runtime_error message");
        }
        // noise: realised power ratio matches the request
        const msfft::ComplexSignal noisy = msfft::add_awgn(gx, 20.0, 5);
        double ps = 0, pn = 0;
        for (int64_t j = 0; j < n2; ++j) {
            ps += std::norm(gx.samples[j]);
            pn += std::norm(noisy.samples[j] - gx.samples[j]);
        }
        CHECK(std::abs(pn / ps / 0.01 - 1.0) < 1e-9, "add_awgn realised SNR");
    }
    {
        const std::vector<double> snr = {0.0, 20.0};
        const auto hs = msfft::run_phase_experiment(8192, 50, 256, snr, 40, 3);
        std::vector<double> ref(73 * snr.size());
        CHECK(orc_phase_experiment(8192, 50, 256, snr.data(), static_cast<int64_t>(snr.size()), 40,
                                   3, ref.data(), err, sizeof(err)) == 0, "reference phase mc");
        for (size_t i = 0; i < snr.size(); ++i) {
            CHECK(hs[i].trials == 40 && hs[i].l_width == 32, "histogram header");
            CHECK(std::abs(hs[i].p50 - ref[73 * i + 70]) <= 1e-9, "phase p50");
            CHECK(std::abs(hs[i].max - ref[73 * i + 72]) <= 1e-9, "phase max");
        }
    }
    // ---- component API on the path (bucketize.hpp, locate.hpp, sfft4.hpp:50)
    {
        const int64_t n3 = 1 << 14, b3 = 64;
        const double d3 = 1e-8;
        const auto win = msfft::get_flat_window(n3, b3, d3);
        int64_t wref = 0;
        CHECK(orc_window(n3, b3, d3, &wref, nullptr, 0, err, sizeof(err)) == 0, "reference window");
        CHECK(win->w == wref && win->l_width == n3 / b3, "window support");
        const auto [sx, st] = msfft::generate_test_signal(n3, 12, 5);
        std::vector<double> sxi(2 * n3);
        for (int64_t j = 0; j < n3; ++j) {
            sxi[2 * j] = sx.samples[j].real();
            sxi[2 * j + 1] = sx.samples[j].imag();
        }
        // taus of one iteration (sfft4.cpp:49-55) and a sigma
        int32_t nr = 0;
        std::vector<int64_t> taus(32);
        CHECK(msfft_tau_plan(static_cast<double>(n3 / b3), n3, 16, 1.0, taus.data(), 32, &nr, err,
                             sizeof(err)) == 0, "tau plan");
        std::vector<msfft::PermutationParams> ps;
        for (int r = 0; r < nr; ++r) ps.push_back({4097, 0, taus[r]});
        const auto rounds = msfft::bucketize_rounds(sx, *win, ps);
        std::vector<double> rv(2 * b3 * nr);
        for (int r = 0; r < nr; ++r) {
            std::vector<double> one(2 * b3);
            CHECK(orc_bucketize(n3, sxi.data(), b3, d3, ps[r].sigma, ps[r].tau, one.data(), err,
                                sizeof(err)) == 0, "reference bucketize");
            for (int64_t j = 0; j < b3; ++j)
                CHECK(rounds[r].values[j] == msfft::cplx(one[2 * j], one[2 * j + 1]),
                      "bucketize bit-exact");
            std::copy(one.begin(), one.end(), rv.begin() + 2 * b3 * r);
        }
        const msfft::BucketSet pred = msfft::predict_buckets(st, *win, ps[1]);
        std::vector<int64_t> pf;
        std::vector<double> pc, pref(2 * b3);
        for (const auto& [f, c] : st.entries) {
            pf.push_back(f);
            pc.push_back(c.real());
            pc.push_back(c.imag());
        }
        CHECK(orc_predict(n3, b3, d3, static_cast<int64_t>(pf.size()), pf.data(), pc.data(),
                          ps[1].sigma, ps[1].tau, pref.data(), err, sizeof(err)) == 0,
              "reference predict");
        double pmax = 0.0, perr = 0.0;
        for (int64_t j = 0; j < b3; ++j) {
            const msfft::cplx r(pref[2 * j], pref[2 * j + 1]);
            pmax = std::max(pmax, std::abs(r));
            perr = std::max(perr, std::abs(pred.values[j] - r));
        }
        CHECK(perr <= 1e-13 * pmax, "predict_buckets within ulps");
        const msfft::BucketSet resid = msfft::subtract(rounds[1], pred);
        CHECK(std::abs(resid.values[0] - (rounds[1].values[0] - pred.values[0])) == 0.0,
              "subtract");
        bool threw = false;
        try {
            msfft::subtract(rounds[0], rounds[1]);
        } catch (const std::invalid_argument& e) {
            threw = std::string(e.what()) == "subtract: bucket sets are not from the same round";
        }
        CHECK(threw, "subtract geometry check");
        std::vector<int64_t> all(b3);
        for (int64_t j = 0; j < b3; ++j) all[j] = j;
        const auto loc = msfft::locate_frequencies(all, rounds, msfft::MultiscaleConfig{16, 1.0},
                                                   *win);
        for (int64_t j = 0; j < b3; ++j) {
            int64_t u = -1;
            int stg = 0;
            CHECK(orc_locate(n3, b3, d3, 16, 1.0, j, nr, taus.data(), rv.data(), &u, &stg, err,
                             sizeof(err)) == 0, "reference locate");
            CHECK(u < 0 ? !loc[j] : (loc[j] && loc[j]->u == u && loc[j]->stages == stg),
                  "locate_frequency identical");
            if (loc[j]) {
                double ev[2];
                CHECK(orc_estimate_value(n3, b3, d3, rounds[0].values[j].real(),
                                         rounds[0].values[j].imag(), u, ev, err,
                                         sizeof(err)) == 0, "reference estimate");
                const msfft::cplx e = msfft::estimate_value(rounds[0].values[j], u, *win);
                CHECK(std::abs(e - msfft::cplx(ev[0], ev[1])) <= 1e-13 * std::abs(e),
                      "estimate_value");
            }
        }
    }
    std::printf("dropin ok: %ld entries identical support, max rel err %.3e; signal/io/phase/component API ok\n",
                static_cast<long>(cnt), worst);
    return 0;
}
