// Receipt v2 digest: per-step Merkle roots of the logits trace on the GPU (digest.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace detgpu {

constexpr int kLeafBytes = 4096;   // v2 leaf size: 4 KiB of f32 logits (1024 values)

// roots_dev[(slot * tcap + t) * 32 ..] = Merkle root of step t of slot (t < steps_dev[slot]) over
// the trace rows trace + slot * slot_stride + t * V.
cudaError_t launch_receipt_roots(const float* trace, int64_t slot_stride, const int* steps_dev, int n_slots, int tmax,
                                 int V, uint8_t* roots_dev, int tcap, cudaStream_t stream);

}  // namespace detgpu
