// The reference ToyModel (reference proj/include/verinf/detcore.hpp:139-149) on the GPU, bit-exact
// with the reference's infer() under its archA / archB profiles (detcore.cpp:12-20).
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "detgpu.h"

namespace detgpu {

constexpr uint32_t kToyVocab = 32;
constexpr uint32_t kToyDim = 16;

struct ToyWeights {
    float* w = nullptr;   // embed[32x16] | recur[16x16] | hidden[16x16] | project[32x16]
    int arch = 0;         // 0 archA (canonical tree), 1 archB (sequential, split)
};

int toy_init(ToyWeights& tw, const char* model_id, int arch, cudaStream_t stream);
void toy_free(ToyWeights& tw);
int toy_generate(ToyWeights& tw, uint32_t n, const uint32_t* const* prompts, const uint32_t* lens,
                 const detgpu_policy* pols, const uint64_t* seeds, uint32_t batch_size, uint32_t* const* tokens_out,
                 float* const* logits_out, uint8_t* out_hash, uint32_t flags, detgpu_stats* stats, cudaStream_t stream,
                 std::string* err);

}  // namespace detgpu
