// signal_io.cpp -- see signal_io.hpp.
#include "signal_io.hpp"

#include <cuda_runtime.h>

#include <cinttypes>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuda_check.hpp"
#include "host_plan.hpp"

namespace msfft_b200 {

namespace {

constexpr char kMagic[8] = {'M', 'S', 'F', 'T', 0, 0, 0, 0};
constexpr int64_t kStage = int64_t{1} << 22;  // samples per staging piece (64 MiB c128)

struct File {
    std::FILE* f = nullptr;
    File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
    int close() {
        const int r = std::fclose(f);
        f = nullptr;
        return r;
    }
};

struct Pinned {
    void* p = nullptr;
    explicit Pinned(size_t bytes) { MSFFT_CUDA(cudaMallocHost(&p, bytes)); }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

bool finite2(double a, double b) { return std::isfinite(a) && std::isfinite(b); }

// Header of an MSFT file; returns n (io.cpp:33-42).
uint64_t read_header(std::FILE* f, const std::string& path) {
    char magic[8] = {};
    if (std::fread(magic, 1, 8, f) != 8 || std::memcmp(magic, kMagic, 4) != 0)
        throw std::runtime_error("read_signal_file: bad magic in " + path);
    uint64_t n = 0;
    if (std::fread(&n, sizeof(n), 1, f) != 1 || !is_pow2_u(n) || n < 4 || n > (uint64_t{1} << 30))
        throw std::runtime_error("read_signal_file: bad length field in " + path);
    return n;
}

}  // namespace

int64_t signal_file_length(const std::string& path) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("read_signal_file: cannot open " + path);
    return static_cast<int64_t>(read_header(in.f, path));
}

int64_t read_signal_file(const std::string& path, bool c128, bool on_device, void* x,
                         int64_t cap) {
    File in(path, "rb");
    if (!in.f) throw std::runtime_error("read_signal_file: cannot open " + path);
    const int64_t n = static_cast<int64_t>(read_header(in.f, path));
    if (n > cap) return n;
    const int64_t piece = std::min<int64_t>(n, kStage);
    std::vector<double> buf(static_cast<size_t>(2 * piece));
    std::unique_ptr<Pinned> pin;
    if (on_device) pin = std::make_unique<Pinned>(static_cast<size_t>(piece) * (c128 ? 16 : 8));
    bool finite = true;
    for (int64_t s0 = 0; s0 < n; s0 += piece) {
        const int64_t len = std::min(piece, n - s0);
        if (std::fread(buf.data(), 16, static_cast<size_t>(len), in.f) != static_cast<size_t>(len))
            throw std::runtime_error("read_signal_file: truncated file " + path);
        for (int64_t j = 0; j < len && finite; ++j) finite = finite2(buf[2 * j], buf[2 * j + 1]);
        const size_t esz = c128 ? 16 : 8;
        unsigned char* dst = on_device ? static_cast<unsigned char*>(pin->p)
                                       : static_cast<unsigned char*>(x) + s0 * esz;
        if (c128) {
            std::memcpy(dst, buf.data(), static_cast<size_t>(len) * 16);
        } else {
            float* d = reinterpret_cast<float*>(dst);
            for (int64_t j = 0; j < 2 * len; ++j) d[j] = static_cast<float>(buf[j]);
        }
        if (on_device)
            MSFFT_CUDA(cudaMemcpy(static_cast<unsigned char*>(x) + s0 * esz, pin->p,
                                  static_cast<size_t>(len) * esz, cudaMemcpyHostToDevice));
    }
    // read_signal_file validates the samples it read (io.cpp:52)
    if (!finite) throw std::invalid_argument("ComplexSignal: non-finite sample");
    return n;
}

void write_signal_file(const std::string& path, const void* x, int64_t n, bool c128,
                       bool on_device) {
    // x.validate() before anything is written (io.cpp:18)
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("ComplexSignal: n must be a power of two >= 4");
    const int64_t piece = std::min<int64_t>(n, kStage);
    const size_t esz = c128 ? 16 : 8;
    std::vector<double> buf(static_cast<size_t>(2 * piece));
    std::unique_ptr<Pinned> pin;
    if (on_device) pin = std::make_unique<Pinned>(static_cast<size_t>(piece) * esz);
    auto fetch = [&](int64_t s0, int64_t len) {
        const unsigned char* src = static_cast<const unsigned char*>(x) + s0 * esz;
        if (on_device) {
            MSFFT_CUDA(cudaMemcpy(pin->p, src, static_cast<size_t>(len) * esz,
                                  cudaMemcpyDeviceToHost));
            src = static_cast<const unsigned char*>(pin->p);
        }
        if (c128) {
            std::memcpy(buf.data(), src, static_cast<size_t>(len) * 16);
        } else {
            const float* s = reinterpret_cast<const float*>(src);
            for (int64_t j = 0; j < 2 * len; ++j) buf[j] = static_cast<double>(s[j]);
        }
    };
    for (int64_t s0 = 0; s0 < n; s0 += piece) {  // validation pass
        const int64_t len = std::min(piece, n - s0);
        fetch(s0, len);
        for (int64_t j = 0; j < len; ++j)
            if (!finite2(buf[2 * j], buf[2 * j + 1]))
                throw std::invalid_argument("ComplexSignal: non-finite sample");
    }
    File out(path, "wb");
    if (!out.f) throw std::runtime_error("write_signal_file: cannot open " + path);
    const uint64_t nn = static_cast<uint64_t>(n);
    bool ok = std::fwrite(kMagic, 1, 8, out.f) == 8 && std::fwrite(&nn, sizeof(nn), 1, out.f) == 1;
    for (int64_t s0 = 0; ok && s0 < n; s0 += piece) {
        const int64_t len = std::min(piece, n - s0);
        fetch(s0, len);
        ok = std::fwrite(buf.data(), 16, static_cast<size_t>(len), out.f) == static_cast<size_t>(len);
    }
    ok = (out.close() == 0) && ok;
    if (!ok) throw std::runtime_error("write_signal_file: write failed for " + path);
}

void write_truth_csv(const std::string& path, const int64_t* f, const double* c, int64_t count) {
    // SparseSpectrum is a std::map: rows in ascending position, later
    // duplicates win
    std::map<int64_t, std::pair<double, double>> m;
    for (int64_t i = 0; i < count; ++i) m[f[i]] = {c[2 * i], c[2 * i + 1]};
    File out(path, "w");
    if (!out.f) throw std::runtime_error("write_truth_csv: cannot open " + path);
    bool ok = std::fputs("position,re,im\n", out.f) >= 0;
    char buf[96];
    for (const auto& [pos, v] : m) {
        std::snprintf(buf, sizeof(buf), "%" PRId64 ",%.17g,%.17g\n", pos, v.first, v.second);
        ok = ok && std::fputs(buf, out.f) >= 0;
    }
    ok = (out.close() == 0) && ok;
    if (!ok) throw std::runtime_error("write_truth_csv: write failed for " + path);
}

int64_t read_truth_csv(const std::string& path, int64_t n, int64_t* f, double* c, int64_t cap) {
    File in(path, "r");
    if (!in.f) throw std::runtime_error("read_truth_csv: cannot open " + path);
    std::map<int64_t, std::pair<double, double>> m;
    std::string line;
    bool header = true;
    auto row = [&] {
        if (header) {
            header = false;
        } else if (!line.empty()) {
            // getline(row, field, ',') x3, std::stoll / std::stod (io.cpp:78-86)
            const size_t a = line.find(',');
            const size_t b = a == std::string::npos ? a : line.find(',', a + 1);
            const int64_t pos = std::stoll(line.substr(0, a));
            const double re = std::stod(a == std::string::npos ? std::string() : line.substr(a + 1, b - a - 1));
            const double im = std::stod(b == std::string::npos ? std::string() : line.substr(b + 1));
            m[pos] = {re, im};
        }
        line.clear();
    };
    int ch;
    while ((ch = std::fgetc(in.f)) != EOF) {
        if (ch == '\n')
            row();
        else
            line.push_back(static_cast<char>(ch));
    }
    if (!line.empty()) row();
    // truth.validate() (signal.cpp:28-39)
    if (n < 4 || !is_pow2_u(static_cast<uint64_t>(n)))
        throw std::invalid_argument("SparseSpectrum: n must be a power of two >= 4");
    if (static_cast<int64_t>(m.size()) > n)
        throw std::invalid_argument("SparseSpectrum: more entries than n");
    for (const auto& [pos, v] : m) {
        if (pos < 0 || pos >= n) throw std::invalid_argument("SparseSpectrum: position out of range");
        if (!finite2(v.first, v.second))
            throw std::invalid_argument("SparseSpectrum: non-finite coefficient");
    }
    int64_t i = 0;
    for (const auto& [pos, v] : m) {
        if (i < cap) {
            f[i] = pos;
            c[2 * i] = v.first;
            c[2 * i + 1] = v.second;
        }
        ++i;
    }
    return i;
}

EvalMetrics error_metrics(int64_t truth_n, const int64_t* tf, const double* tc, int64_t tcount,
                          int64_t est_n, const int64_t* ef, const double* ec, int64_t ecount,
                          int64_t k) {
    if (truth_n != est_n) throw std::invalid_argument("error_metrics: size mismatch");
    using cx = std::complex<double>;
    std::map<int64_t, cx> truth, est;
    for (int64_t i = 0; i < tcount; ++i) truth[tf[i]] = cx(tc[2 * i], tc[2 * i + 1]);
    for (int64_t i = 0; i < ecount; ++i) est[ef[i]] = cx(ec[2 * i], ec[2 * i + 1]);
    std::map<int64_t, bool> support;
    for (const auto& kv : truth) support[kv.first] = true;
    for (const auto& kv : est) support[kv.first] = true;
    if (k <= 0) {
        if (!support.empty())
            throw std::invalid_argument("error_metrics: k = 0 with nonempty support union");
        return {};
    }
    EvalMetrics m;
    double sum_abs = 0.0, sum_sq = 0.0;
    for (const auto& kv : support) {
        const auto ti = truth.find(kv.first);
        const auto ei = est.find(kv.first);
        const cx tv = ti == truth.end() ? cx(0, 0) : ti->second;
        const cx ev = ei == est.end() ? cx(0, 0) : ei->second;
        const double d = std::abs(tv - ev);
        sum_abs += d;
        sum_sq += d * d;
        if (d > 1e-6) ++m.l0;
    }
    m.l1 = sum_abs / static_cast<double>(k);
    m.l2 = std::sqrt(sum_sq / static_cast<double>(k));
    return m;
}

}  // namespace msfft_b200
