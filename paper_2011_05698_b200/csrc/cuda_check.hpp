// cuda_check.hpp -- CUDA error to C++ exception plumbing (host only).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

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

// cudaFuncSetAttribute(fn, MaxDynamicSharedMemorySize, bytes) on the current
// device, issued only when the kernel's limit must grow: the driver call
// costs microseconds, which small launches would pay on every call.
inline void smem_attr(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> set;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set[{dev, fn}];
    if (bytes > cur) {
        cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(bytes)),
                   "cudaFuncSetAttribute");
        cur = bytes;
    }
}
template <class F>
inline void smem_attr(F* fn, size_t bytes) {
    smem_attr(reinterpret_cast<const void*>(fn), bytes);
}

// SM count of the current device (cached per device).
inline int sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev),
               "cudaDeviceGetAttribute");
    cache[dev] = sms;
    return sms;
}

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
