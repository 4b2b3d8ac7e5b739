// window.hpp -- the flat (Gaussian (*) boxcar) window on the device.
//
// design_flat_window (proj/src/window.cpp:105-177) is restated with its
// n-point transforms on the GPU (fft.hpp, bit-identical butterflies), so the
// taps and the support w equal the reference's; the process cache mirrors
// get_flat_window (window.cpp:179-193) keyed (device, n, b, delta).  Each
// cached window also carries the device table of its frequency response
// G_d = response_at(d) (window.cpp:89-99) for |d| <= 3L/2 + 1, which replaces
// the reference's O(w) cosine series per call in predict/estimate.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace msfft_b200 {

struct DeviceWindow {
    int device = 0;
    int64_t n = 0, b = 0, l_width = 0, w = 0, h = 0;
    double delta = 0.0;
    std::vector<double> taps;     // host copy of g_time[0..w)
    double* d_taps = nullptr;     // device taps, w + 1 doubles (zero pad), 16-B aligned
    double* d_ghat = nullptr;     // device G_d for d in [-gmax, gmax], index d + gmax
    int64_t gmax = 0;             // 3L/2 + 1
    ~DeviceWindow();
};

// Throws std::invalid_argument with the reference's messages for infeasible
// or out-of-range (n, b, delta).  Thread-safe.
std::shared_ptr<const DeviceWindow> get_device_window(int64_t n, int64_t b, double delta);

// w only (designs and caches the window on the current device).
int64_t window_support(int64_t n, int64_t b, double delta);

// FlatWindow::response_at (window.cpp:89-99) at arbitrary offsets idx[k]
// (any integer; reduced mod n), computed on the device exactly as the
// response table is (same series, same summation scheme): host arrays.
void window_response_list(int64_t n, int64_t b, double delta, const int64_t* idx, int64_t count,
                          double* out);

}  // namespace msfft_b200
