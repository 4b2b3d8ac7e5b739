// locate_ops.cu -- the reference's scalar locate helpers and the
// sampler-driven fold, batched on the device (see components.hpp).  Each
// kernel evaluates exactly the __host__ __device__ functions the fused and
// wide decodes use (common.cuh), so a caller -- or a parity test -- sees the
// device's arithmetic, not a host restatement:
//
//   phase_of                 proj/src/locate.cpp:32-37
//   position_phase           proj/src/locate.cpp:19-23
//   circular_phase_distance  proj/src/locate.cpp:14-17
//   locate_step              proj/src/locate.cpp:63-81
//   bucketize_fn<Sampler>    proj/include/msfft/bucketize.hpp:63-86
#include "components.hpp"

#include <stdexcept>

#include "common.cuh"
#include "cuda_check.hpp"
#include "fft.hpp"
#include "window.hpp"

namespace msfft_b200 {
namespace {

constexpr int kT = 256;

unsigned blocks(int64_t count) { return static_cast<unsigned>((count + kT - 1) / kT); }

__global__ void phase_of_kernel(const double2* __restrict__ z, int64_t count,
                                double* __restrict__ out, int32_t* __restrict__ status) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    const double2 v = z[k];
    if (v.x == 0.0 && v.y == 0.0) {  // the reference throws domain_error
        status[k] = 1;
        out[k] = 0.0;
        return;
    }
    double a = atan2(v.y, v.x);  // the decode's phase (decode_body.cuh K5 prologue)
    if (a < 0.0) a += kTwoPi;
    out[k] = a + 0.0;
    status[k] = 0;
}

__global__ void position_phase_kernel(const double* __restrict__ u, const int64_t* __restrict__ tau,
                                      int64_t count, int64_t n, double* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    out[k] = position_phase(u[k], tau[k], n, 1.0 / static_cast<double>(n));
}

__global__ void circ_dist_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                 int64_t count, double* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    out[k] = circular_phase_distance(a[k], b[k]);
}

// locate_step: l block centres, strict < keeps the lowest block, widen by q/2
// blocks on each side, length * (q+1) / l.
__global__ void locate_step_kernel(const double* __restrict__ phi, const int64_t* __restrict__ tau,
                                   const LocateRegionDev* __restrict__ in, int64_t count,
                                   int64_t l, double q, int64_t n,
                                   LocateRegionDev* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (k >= count) return;
    const LocateRegionDev rg = in[k];
    const double inv_n = 1.0 / static_cast<double>(n);
    const double r = rg.length / static_cast<double>(l);
    int64_t best = 0;
    double best_d = INFINITY;
    for (int64_t j = 0; j < l; ++j) {
        const double center = rg.u_min + (static_cast<double>(j) + 0.5) * r;
        const double d = circular_phase_distance(position_phase(center, tau[k], n, inv_n), phi[k]);
        if (d < best_d) {
            best_d = d;
            best = j;
        }
    }
    LocateRegionDev nx;
    nx.u_min = rg.u_min + (static_cast<double>(best) - q / 2.0) * r;
    nx.length = rg.length * (q + 1.0) / static_cast<double>(l);
    nx.stage = rg.stage + 1;
    nx.reserved = 0;
    out[k] = nx;
}

// One thread per (round, bin): the fold of bucketize_fn with the sampler's
// values given in tap order (v[r][h + t] = sample(src_t)), ascending t per
// bin as the reference's loop adds them, no FMA.
__global__ void __launch_bounds__(kT)
fold_taps_kernel(const double2* __restrict__ v, int64_t b, int64_t h, int64_t w,
                 const double* __restrict__ taps, double2* __restrict__ out) {
    const int64_t bin = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    const int r = blockIdx.y;
    if (bin >= b) return;
    const double2* vr = v + static_cast<int64_t>(r) * w;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t t = -h + ((bin + h) & (b - 1)); t <= h; t += b) {
        const double g = taps[h + t];
        const double2 s = vr[h + t];
        acc.x += g * s.x;
        acc.y += g * s.y;
    }
    out[static_cast<int64_t>(r) * b + bin] = acc;
}

template <class T>
struct Scratch {
    T* p = nullptr;
    explicit Scratch(int64_t count) {
        MSFFT_CUDA(cudaMalloc(&p, sizeof(T) * static_cast<size_t>(count > 0 ? count : 1)));
    }
    ~Scratch() { cudaFree(p); }
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
};

template <class T>
void h2d(T* d, const T* h, int64_t count, cudaStream_t st) {
    MSFFT_CUDA(cudaMemcpyAsync(d, h, sizeof(T) * count, cudaMemcpyHostToDevice, st));
}
template <class T>
void d2h(T* h, const T* d, int64_t count, cudaStream_t st) {
    MSFFT_CUDA(cudaMemcpyAsync(h, d, sizeof(T) * count, cudaMemcpyDeviceToHost, st));
}

}  // namespace

void phase_of_host(const double* z, int64_t count, double* phase, int32_t* status,
                   cudaStream_t st) {
    if (count <= 0) return;
    Scratch<double2> dz(count);
    Scratch<double> dp(count);
    Scratch<int32_t> ds(count);
    h2d(dz.p, reinterpret_cast<const double2*>(z), count, st);
    phase_of_kernel<<<blocks(count), kT, 0, st>>>(dz.p, count, dp.p, ds.p);
    MSFFT_LAUNCH_CHECK("phase_of_kernel");
    d2h(phase, dp.p, count, st);
    d2h(status, ds.p, count, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void position_phase_host(const double* u, const int64_t* tau, int64_t count, int64_t n,
                         double* out, cudaStream_t st) {
    if (count <= 0) return;
    Scratch<double> du(count), dout(count);
    Scratch<int64_t> dt(count);
    h2d(du.p, u, count, st);
    h2d(dt.p, tau, count, st);
    position_phase_kernel<<<blocks(count), kT, 0, st>>>(du.p, dt.p, count, n, dout.p);
    MSFFT_LAUNCH_CHECK("position_phase_kernel");
    d2h(out, dout.p, count, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void circular_phase_distance_host(const double* a, const double* b, int64_t count, double* out,
                                  cudaStream_t st) {
    if (count <= 0) return;
    Scratch<double> da(count), db(count), dout(count);
    h2d(da.p, a, count, st);
    h2d(db.p, b, count, st);
    circ_dist_kernel<<<blocks(count), kT, 0, st>>>(da.p, db.p, count, dout.p);
    MSFFT_LAUNCH_CHECK("circ_dist_kernel");
    d2h(out, dout.p, count, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

void locate_step_host(const double* phi, const int64_t* tau, const LocateRegionDev* region,
                      int64_t count, int64_t l, double q, int64_t n, LocateRegionDev* out,
                      cudaStream_t st) {
    if (count <= 0) return;
    Scratch<double> dphi(count);
    Scratch<int64_t> dt(count);
    Scratch<LocateRegionDev> din(count), dout(count);
    h2d(dphi.p, phi, count, st);
    h2d(dt.p, tau, count, st);
    h2d(din.p, region, count, st);
    locate_step_kernel<<<blocks(count), kT, 0, st>>>(dphi.p, dt.p, din.p, count, l, q, n, dout.p);
    MSFFT_LAUNCH_CHECK("locate_step_kernel");
    d2h(out, dout.p, count, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
}

int64_t bucketize_taps_host(int64_t n, int64_t b, double delta, const double* values,
                            int64_t rounds, double* out, cudaStream_t st) {
    if (rounds < 1 || rounds > 65535)
        throw std::invalid_argument("msfft: rounds must be in [1, 65535]");
    auto win = get_device_window(n, b, delta);
    const int64_t w = win->w;
    Scratch<double2> dv(rounds * w), dout(rounds * b);
    h2d(dv.p, reinterpret_cast<const double2*>(values), rounds * w, st);
    fold_taps_kernel<<<dim3(blocks(b), static_cast<unsigned>(rounds)), kT, 0, st>>>(
        dv.p, b, win->h, w, win->d_taps, dout.p);
    MSFFT_LAUNCH_CHECK("fold_taps_kernel");
    fft_radix2_batched(dout.p, b, rounds, rounds, 0, -1, 1.0 / static_cast<double>(n), st);
    d2h(reinterpret_cast<double2*>(out), dout.p, rounds * b, st);
    MSFFT_CUDA(cudaStreamSynchronize(st));
    return w;
}

}  // namespace msfft_b200
