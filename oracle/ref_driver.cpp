// C entry points over the UNMODIFIED reference detcore/codec sources (compiled by `make ref`).
// Used only to (1) generate tests/golden/toy_reference.json (tests/golden/make_toy_golden.py) and
// (2) time the reference CPU engine for bench.py's `--impl reference` / cpu_baseline legs.
// TEST / MEASUREMENT INFRASTRUCTURE ONLY.
#include <openssl/sha.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "verinf/codec.hpp"
#include "verinf/da.hpp"
#include "verinf/detcore.hpp"
#include "verinf/sha256.hpp"

using namespace verinf;
using namespace verinf::detcore;

// The reference's SHA-256 entry point (sha256.hpp; libsodium in the reference build), over OpenSSL.
namespace verinf {
Hash32 sha256(std::span<const uint8_t> data) {
    Hash32 h;
    SHA256(data.data(), data.size(), h.data());
    return h;
}
}  // namespace verinf

static DecodePolicy make_policy(int kind, int has_k, uint32_t k, int has_p, float p, uint32_t max_tokens) {
    DecodePolicy pol;
    pol.kind = DecodeKind(kind);
    if (has_k) pol.k = k;
    if (has_p) pol.p = p;
    pol.max_tokens = max_tokens;
    return pol;
}

static ExecutionTuple make_exec(const char* model_id, const uint8_t* digest, const char* arch, const char* driver,
                                const DecodePolicy& pol, uint64_t seed, const uint32_t* prompt, uint32_t plen) {
    ExecutionTuple e;
    e.model_id = model_id;
    std::memcpy(e.container_digest.data(), digest, 32);
    e.arch = arch;
    e.driver_tag = driver;
    e.decode_policy = pol;
    e.seed = seed;
    e.prompt.assign(prompt, prompt + plen);
    return e;
}

extern "C" {

// The reference's DA Merkle rules (da.cpp:27-61), for the receipt-v2 golden vectors.
void ref_leaf_hash(const uint8_t* blob, size_t n, uint8_t* out) {
    const Hash32 h = da::leaf_hash(std::span<const uint8_t>(blob, n));
    std::memcpy(out, h.data(), 32);
}
void ref_node_hash(const uint8_t* l, const uint8_t* r, uint8_t* out) {
    Hash32 a, b;
    std::memcpy(a.data(), l, 32);
    std::memcpy(b.data(), r, 32);
    const Hash32 h = da::node_hash(a, b);
    std::memcpy(out, h.data(), 32);
}
void ref_merkle_root(const uint8_t* leaf_hashes, size_t n, uint8_t* out) {
    std::vector<Hash32> v(n);
    for (size_t i = 0; i < n; ++i) std::memcpy(v[i].data(), leaf_hashes + 32 * i, 32);
    const Hash32 h = da::merkle_root(v);
    std::memcpy(out, h.data(), 32);
}

// Runs reference infer(); writes tokens (max_tokens), canonical bytes length, out_hash = SHA-256(
// canonical_bytes) and req_hash = SHA-256(encode_execution_tuple). Returns 0, or 1 on
// std::invalid_argument.
int ref_infer(const char* model_id, const uint8_t* digest, const char* arch, const char* driver, int kind, int has_k,
              uint32_t k, int has_p, float p, uint32_t max_tokens, uint64_t seed, const uint32_t* prompt,
              uint32_t plen, uint32_t* tokens_out, uint64_t* canonical_len, uint8_t* out_hash, uint8_t* req_hash,
              float* logits_out) {
    try {
        ExecutionTuple e = make_exec(model_id, digest, arch, driver, make_policy(kind, has_k, k, has_p, p, max_tokens),
                                     seed, prompt, plen);
        InferenceOutput out = infer(e);
        for (size_t i = 0; i < out.tokens.size(); ++i) tokens_out[i] = out.tokens[i];
        if (logits_out != nullptr)
            for (size_t s = 0; s < out.logits_trace.size(); ++s)
                std::memcpy(logits_out + s * ToyModel::kVocab, out.logits_trace[s].data(),
                            sizeof(float) * out.logits_trace[s].size());
        *canonical_len = out.canonical_bytes.size();
        SHA256(out.canonical_bytes.data(), out.canonical_bytes.size(), out_hash);
        Bytes req = codec::encode_execution_tuple(e);
        SHA256(req.data(), req.size(), req_hash);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// Reference infer_batch over n copies of a tuple family (seed = seed0 + i); returns 0 and writes
// out_hash for each, 1 on invalid_argument.
int ref_infer_batch(const char* model_id, const uint8_t* digest, const char* arch, int kind, int has_k, uint32_t k,
                    int has_p, float p, uint32_t max_tokens, uint64_t seed0, const uint32_t* prompt, uint32_t plen,
                    uint32_t n, uint32_t batch_size, uint8_t* out_hashes) {
    try {
        std::vector<ExecutionTuple> execs;
        for (uint32_t i = 0; i < n; ++i)
            execs.push_back(make_exec(model_id, digest, arch, "drv-1", make_policy(kind, has_k, k, has_p, p, max_tokens),
                                      seed0 + i, prompt, plen));
        auto outs = infer_batch(execs, batch_size);
        for (uint32_t i = 0; i < n; ++i)
            SHA256(outs[i].canonical_bytes.data(), outs[i].canonical_bytes.size(), out_hashes + 32 * size_t(i));
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

// CPU baseline: `threads` workers each run reference infer() + SHA-256 on independent requests
// (the engine is pure and reentrant, detcore.hpp:13-17) until `n_requests` are done.
// Returns elapsed seconds; *tokens = generated tokens.
double ref_bench(const char* model_id, const char* arch, uint32_t max_tokens, uint32_t plen, uint32_t n_requests,
                 int threads, uint64_t* tokens) {
    std::atomic<uint32_t> next{0};
    std::atomic<uint64_t> ntok{0};
    uint8_t digest[32] = {0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t)
        th.emplace_back([&] {
            for (;;) {
                const uint32_t i = next.fetch_add(1);
                if (i >= n_requests) break;
                PrngState rng = PrngState::seeded(uint64_t(i) ^ 0xABCD);
                std::vector<uint32_t> prompt(plen);
                for (auto& x : prompt) x = uint32_t(rng.next_below(ToyModel::kVocab));
                ExecutionTuple e = make_exec(model_id, digest, arch, "drv-1", DecodePolicy::greedy(max_tokens), i,
                                             prompt.data(), plen);
                InferenceOutput out = infer(e);
                uint8_t h[32];
                SHA256(out.canonical_bytes.data(), out.canonical_bytes.size(), h);
                ntok += out.tokens.size();
            }
        });
    for (auto& x : th) x.join();
    *tokens = ntok.load();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
