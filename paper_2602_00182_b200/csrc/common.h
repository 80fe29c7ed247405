// Host-side shared helpers: error capture for the C-ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

namespace detgpu {

void set_global_error(const std::string& msg);
const std::string& global_error();

#define DETGPU_CUDA_TRY(expr)                                                                   \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            ::detgpu::set_global_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
            return DETGPU_ECUDA;                                                                \
        }                                                                                       \
    } while (0)

// Kernel attributes (cudaFuncSetAttribute) are per device: `mask` records the devices on which a
// kernel's attributes are already set. Returns true when they must be set on the current device.
inline bool attrs_needed(const std::atomic<uint64_t>& mask, int* dev_out) {
    int dev = 0;
    cudaGetDevice(&dev);
    *dev_out = dev;
    return dev >= 64 || !(mask.load(std::memory_order_acquire) & (1ull << dev));
}
inline void attrs_done(std::atomic<uint64_t>& mask, int dev) {
    if (dev < 64) mask.fetch_or(1ull << dev, std::memory_order_release);
}

}  // namespace detgpu
