// Shared host/device plumbing: status codes as C++ exceptions, CUDA checks,
// device buffers, launch accounting.
#pragma once

#include <cuda_runtime.h>

#include <new>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "walkforge_b200.h"

namespace wf {

// One exception type carrying a wf_status; the ABI layer turns it into the
// return code + wf_last_error() (error.hpp:8-48 hierarchy, by code).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }
[[noreturn]] inline void config_error(const std::string& msg) { raise(WF_ERR_CONFIG, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        raise(e == cudaErrorMemoryAllocation ? WF_ERR_OOM : WF_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define WF_CUDA(call) ::wf::cuda_check((call), #call)

extern std::atomic<uint64_t> g_kernel_launches;
inline void count_launch(uint64_t n = 1) { g_kernel_launches.fetch_add(n, std::memory_order_relaxed); }
#define WF_LAUNCHED() do { ::wf::count_launch(); WF_CUDA(cudaGetLastError()); } while (0)

// Owning device allocation.
template <typename T>
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(size_t n) { allocate(n); }
    ~DeviceBuffer() { release(); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(o.ptr_), n_(o.n_) { o.ptr_ = nullptr; o.n_ = 0; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) { release(); ptr_ = o.ptr_; n_ = o.n_; o.ptr_ = nullptr; o.n_ = 0; }
        return *this;
    }
    void allocate(size_t n) {
        release();
        if (n == 0) return;
        WF_CUDA(cudaMalloc(&ptr_, n * sizeof(T)));
        n_ = n;
    }
    void release() {
        if (ptr_) cudaFree(ptr_);
        ptr_ = nullptr;
        n_ = 0;
    }
    T* get() const { return ptr_; }
    size_t size() const { return n_; }
    size_t bytes() const { return n_ * sizeof(T); }

private:
    T* ptr_ = nullptr;
    size_t n_ = 0;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        WF_CUDA(cudaGetDevice(&prev));
        if (prev != dev) WF_CUDA(cudaSetDevice(dev));
    }
    // For destructors and the *_destroy entry points, which must not throw: at
    // interpreter / process shutdown the runtime may already be torn down.
    DeviceGuard(int dev, std::nothrow_t) noexcept {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
            return;
        }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) cudaGetLastError();
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline bool is_device_pointer(const void* p) {
    if (p == nullptr) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline int sm_count(int dev) {
    int n = 0;
    WF_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

}  // namespace wf
