// common.cuh -- device-side scalar arithmetic shared by the sm_100a kernels.
//
// Every translation unit that includes this is compiled with --fmad=false:
// the reference host build has no FMA (x86-64 baseline, no -march; see
// SURVEY.md Appendix B), so any contraction would change last bits of the
// bucket values and of the decode's discrete decisions.  Helpers below
// restate the exact libm / libgcc behaviour the reference binary calls
// (objdump of the reference library shows calls to __divdc3, cabs and atan2).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace msfft_b200 {

// Checked build (-DMSFFT_CHECKED, tools/build_variant.py checked ...): every
// scratch array the kernels index through dptr<T> carries its capacity and
// traps with the file, line and thread on an out-of-range index; MSFFT_DCHECK
// guards the remaining computed indices.  Normal builds: dptr<T> is T* and
// the checks compile to nothing.
#ifdef MSFFT_CHECKED
#define MSFFT_DCHECK(c)                                                                   \
    do {                                                                                  \
        if (!(c)) {                                                                       \
            printf("MSFFT_DCHECK %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));          \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
template <class T>
struct CheckedPtr {
    T* p = nullptr;
    int64_t n = 0;
    CheckedPtr() = default;
    __host__ __device__ CheckedPtr(T* p_, int64_t n_) : p(p_), n(n_) {}
    __device__ T& operator[](int64_t i) const {
        MSFFT_DCHECK(p != nullptr && i >= 0 && i < n);
        return p[i];
    }
    __device__ operator T*() const { return p; }
};
template <class T>
using dptr = CheckedPtr<T>;
template <class T>
__device__ inline dptr<T> make_dptr(T* p, int64_t n) {
    return dptr<T>(p, n);
}
#else
#define MSFFT_DCHECK(c) \
    do {                \
    } while (0)
template <class T>
using dptr = T*;
template <class T>
__device__ __forceinline__ T* make_dptr(T* p, int64_t) {
    return p;
}
#endif

// 2*pi as in proj/src/locate.cpp:10 / window.cpp:15 (2.0 * std::numbers::pi).
constexpr double kTwoPi = 6.283185307179586476925286766559;

// |z| exactly as glibc 2.39 cabs/hypot (generic, non-FMA kernel of
// sysdeps/ieee754/dbl-64/e_hypot.c).  The reference uses std::abs(cplx) for
// the selection order (proj/src/sfft4.cpp:81-85), the K-prune
// (sfft4.cpp:172-174) and the band scan (window.cpp:58).  Checked bit-equal
// to glibc on 2e7 random pairs (tests/test_host_math.py).
__host__ __device__ inline double hypot_kernel(double ax, double ay) {
    double t1, t2;
    double h = sqrt(ax * ax + ay * ay);
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

__host__ __device__ inline double cabs_ref(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    if (isinf(x) || isinf(y)) return INFINITY;
    if (isnan(x) || isnan(y)) return x + y;
    const double ax = x < y ? y : x;
    const double ay = x < y ? x : y;
    if (ax > 0x1p511) {
        if (ay <= ax * 0x1p-54) return ax + ay;
        return hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
    }
    if (ay < 0x1p-511) {
        if (ax >= ay / 0x1p-54) return ax + ay;
        return hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
    }
    if (ay <= ax * 0x1p-54) return ax + ay;
    return hypot_kernel(ax, ay);
}

// (a+ib)/(c+id) following libgcc's __divdc3 (GCC 13 libgcc2.c: Smith's
// method with the power-of-two pre-scalings), which the reference's
// std::complex<double> division compiles to (proj/src/locate.cpp:110).
__host__ __device__ inline double2 cdiv_ref(double a, double b, double c, double d) {
    const double RBIG = 1.7976931348623157e308 / 2.0;
    const double RMIN = 2.2250738585072014e-308;
    const double RMIN2 = 2.220446049250313e-16;
    const double RMINSCAL = 1.0 / 2.220446049250313e-16;
    const double RMAX2 = RBIG * RMIN2;
    double ratio, denom, x, y;
    if (fabs(c) < fabs(d)) {
        if (fabs(d) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(d) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(d) < RMAX2)) ||
                   ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(d) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = c / d;
        denom = (c * ratio) + d;
        if (fabs(ratio) > RMIN) {
            x = ((a * ratio) + b) / denom;
            y = ((b * ratio) - a) / denom;
        } else {
            x = ((c * (a / d)) + b) / denom;
            y = ((c * (b / d)) - a) / denom;
        }
    } else {
        if (fabs(c) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (fabs(c) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(c) < RMAX2)) ||
                   ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(c) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = d / c;
        denom = (d * ratio) + c;
        if (fabs(ratio) > RMIN) {
            x = ((b * ratio) + a) / denom;
            y = (b - (a * ratio)) / denom;
        } else {
            x = (a + (d * (b / c))) / denom;
            y = (b - (d * (a / c))) / denom;
        }
    }
    return make_double2(x, y);
}

// fmod(x, n) for n a power of two: exact (x/n, trunc and the product are
// exact, and the difference is representable), equal to libm fmod.
__host__ __device__ inline double fmod_pow2(double x, double n) {
    return x - trunc(x / n) * n;
}

// position_phase (proj/src/locate.cpp:19-23).  inv_n = 1/n is exact for a
// power of two, so the multiplications below equal the reference's divisions.
__host__ __device__ inline double position_phase(double u, int64_t tau, int64_t n, double inv_n) {
    const double nd = static_cast<double>(n);
    const double p = u * static_cast<double>(tau);
    double x = p - trunc(p * inv_n) * nd;  // fmod(p, n), exact
    if (x < 0) x += nd;
    return x * kTwoPi * inv_n;
}

// The same with n and tau already converted to double (the decode's stage
// chain keeps them in registers).
__host__ __device__ inline double position_phase_d(double u, double tau, double nd, double inv_n) {
    const double p = u * tau;
    double x = p - trunc(p * inv_n) * nd;  // fmod(p, n), exact
    if (x < 0) x += nd;
    return x * kTwoPi * inv_n;
}

// circular_phase_distance (proj/src/locate.cpp:14-17).  Both phases lie in
// [0, 2pi], so |a-b| <= 2pi and fmod reduces to one exact subtraction.
__host__ __device__ inline double circular_phase_distance(double a, double b) {
    double d = fabs(a - b);
    if (d >= kTwoPi) d = d - kTwoPi;
    const double e = kTwoPi - d;
    return d < e ? d : e;
}

// Complex multiply without FMA, the finite-value path of GCC's expansion.
__host__ __device__ inline double2 cmul(double2 x, double2 y) {
    return make_double2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
}

__device__ __forceinline__ unsigned bitrev_bits(unsigned v, int bits) {
    return bits == 0 ? 0u : (__brev(v) >> (32 - bits));
}

}  // namespace msfft_b200
