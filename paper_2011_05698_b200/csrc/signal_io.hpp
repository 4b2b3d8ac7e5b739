// signal_io.hpp -- MSFT signal files, truth CSV and error metrics (SURVEY.md
// 8(f) rows 2-3), with the reference's formats, checks and messages:
//   write_signal_file / read_signal_file   proj/src/io.cpp:17-55
//   write_truth_csv / read_truth_csv       proj/src/io.cpp:57-92
//   error_metrics                          proj/src/signal.cpp:154-184
// Signal data may live in host or device memory; device transfers stream
// through pinned staging in 64 MiB pieces.
#pragma once

#include <cstdint>
#include <string>

namespace msfft_b200 {

struct EvalMetrics {
    int64_t l0 = 0;
    double l1 = 0.0, l2 = 0.0;
};

int64_t signal_file_length(const std::string& path);

// Reads into x (cap samples; c128 or c64 = rounded), host or device memory.
// Returns n; if n > cap nothing is stored.
int64_t read_signal_file(const std::string& path, bool c128, bool on_device, void* x, int64_t cap);

void write_signal_file(const std::string& path, const void* x, int64_t n, bool c128,
                       bool on_device);

void write_truth_csv(const std::string& path, const int64_t* f, const double* c, int64_t count);

// Returns the entry count; stores min(count, cap) entries in ascending f.
int64_t read_truth_csv(const std::string& path, int64_t n, int64_t* f, double* c, int64_t cap);

EvalMetrics error_metrics(int64_t truth_n, const int64_t* tf, const double* tc, int64_t tcount,
                          int64_t est_n, const int64_t* ef, const double* ec, int64_t ecount,
                          int64_t k);

}  // namespace msfft_b200
