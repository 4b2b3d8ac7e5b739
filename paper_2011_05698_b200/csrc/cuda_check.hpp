// cuda_check.hpp -- CUDA error to C++ exception plumbing (host only).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace msfft_b200 {

// Distinct type so the C ABI can map device failures to MSFFT_CUDA_ERROR.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                        cudaGetErrorString(e) + ")");
}

#define MSFFT_CUDA(call) ::msfft_b200::cuda_check((call), #call)
#define MSFFT_LAUNCH_CHECK(name) ::msfft_b200::cuda_check(cudaGetLastError(), name)

// RAII device buffer.
template <class T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t count) { reset(count); }
    ~DeviceBuffer() { release(); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    void reset(size_t count) {
        release();
        if (count) MSFFT_CUDA(cudaMalloc(reinterpret_cast<void**>(&p_), count * sizeof(T)));
        n_ = count;
    }
    void ensure(size_t count) {
        if (count > n_) reset(count);
    }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

}  // namespace msfft_b200
