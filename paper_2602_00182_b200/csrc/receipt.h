// Host SHA-256 and canonical-output hashing (receipt path).
#pragma once
#include <cstddef>
#include <cstdint>

namespace detgpu {

class Sha256 {
public:
    Sha256();
    void update(const void* data, size_t n);
    void final(uint8_t out[32]);

private:
    void compress(const uint8_t* p, size_t nblocks);
    uint32_t h_[8];
    uint8_t buf_[64];
    uint64_t total_ = 0;
    size_t fill_ = 0;
};

bool sha_ni_available();
void hash_canonical(const uint32_t* tokens, uint32_t T, const float* logits, uint32_t V, uint8_t out[32]);
// receipt v2
constexpr size_t kV2LeafBytes = 4096;
void merkle_leaf(const void* blob, size_t n, uint8_t out[32]);
void merkle_node(const uint8_t l[32], const uint8_t r[32], uint8_t out[32]);
void step_root(const float* logits, uint32_t V, uint8_t out[32]);
void hash_canonical_v2_roots(const uint32_t* tokens, uint32_t T, const uint8_t* roots, uint32_t V, uint8_t out[32]);

}  // namespace detgpu
