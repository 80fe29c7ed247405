// Host-side shared helpers: error capture for the C-ABI.
#pragma once
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

}  // namespace detgpu
