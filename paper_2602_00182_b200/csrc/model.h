// Named model shapes and the deterministic weight recipe. The CPU oracle restates
// the same table independently (oracle/oracle.cpp kConfigs).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>

namespace detgpu {

struct ModelConfig {
    const char* name;
    int L, d, hq, hkv, hd, F, V;
    double theta;
    float eps;
};

inline const ModelConfig* find_model_config(const char* model_id) {
    static const ModelConfig kConfigs[] = {
        {"llama-tiny", 2, 256, 4, 2, 64, 768, 4096, 500000.0, 1e-5f},
        {"llama3-8b", 32, 4096, 32, 8, 128, 14336, 128256, 500000.0, 1e-5f},
        {"llama-mid", 2, 1024, 8, 2, 128, 3584, 32000, 500000.0, 1e-5f},   // 8B kernel shapes (hd 128, G 4), oracle-fast
    };
    for (const auto& c : kConfigs) {
        const size_t n = std::strlen(c.name);
        if (std::strncmp(model_id, c.name, n) == 0 && (model_id[n] == 0 || model_id[n] == ':')) return &c;
    }
    return nullptr;
}

// reference detcore.cpp:266-273
inline uint64_t fnv1a64(const char* s) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (const unsigned char* c = reinterpret_cast<const unsigned char*>(s); *c; ++c) {
        h ^= *c;
        h *= 0x100000001B3ULL;
    }
    return h;
}
// reference prng.hpp:18-31
inline uint64_t splitmix64_step(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t x = a ^ (0x9E3779B97F4A7C15ULL + (b << 6) + (b >> 2));
    return splitmix64_step(x);
}
// PrngState::seeded (prng.hpp:36-44)
inline void prng_seeded(uint64_t seed, uint64_t s[4]) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) s[i] = splitmix64_step(x);
    if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 0x9E3779B97F4A7C15ULL;
}
inline int half_log2_round(int n) { return static_cast<int>(std::lround(0.5 * std::log2(static_cast<double>(n)))); }

// tensor ids: 0 embed, 1 lm_head, 2 final_norm, 16+16*l + {0 attn_norm, 1 wq, 2 wk, 3 wv, 4 wo,
// 5 ffn_norm, 6 w_gate, 7 w_up, 8 w_down}
enum TensorSlot { kAttnNorm = 0, kWq = 1, kWk = 2, kWv = 3, kWo = 4, kFfnNorm = 5, kWgate = 6, kWup = 7, kWdown = 8 };
inline int layer_tensor_id(int l, int slot) { return 16 + 16 * l + slot; }

}  // namespace detgpu
