// Header-only C++ shim: the reference's detcore API (proj/include/verinf/detcore.hpp:21-163) on top
// of the detgpu C-ABI. A reference maintainer swaps `verinf::detcore::infer` for
// `detgpu::detcore::infer` (same types, same std::invalid_argument behaviour) and links
// libdetgpu.so; see INTEGRATION.md. Requires C++17.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "detgpu.h"

namespace detgpu::detcore {

using Bytes = std::vector<uint8_t>;
using Hash32 = std::array<uint8_t, 32>;

enum class DecodeKind : uint8_t { greedy = 0, top_k = 1, nucleus = 2 };

struct DecodePolicy {   // detcore.hpp:52-66
    DecodeKind kind = DecodeKind::greedy;
    std::optional<uint32_t> k;
    std::optional<float> p;
    uint32_t max_tokens = 0;
    static DecodePolicy greedy(uint32_t t) { return {DecodeKind::greedy, std::nullopt, std::nullopt, t}; }
    static DecodePolicy top_k(uint32_t k, uint32_t t) { return {DecodeKind::top_k, k, std::nullopt, t}; }
    static DecodePolicy nucleus(float p, uint32_t t) { return {DecodeKind::nucleus, std::nullopt, p, t}; }
    detgpu_policy to_c() const {
        detgpu_policy c{};
        c.kind = static_cast<uint8_t>(kind);
        c.has_k = k.has_value();
        c.has_p = p.has_value();
        c.k = k.value_or(0);
        c.p = p.value_or(0.0f);
        c.max_tokens = max_tokens;
        return c;
    }
};

struct ExecutionTuple {   // detcore.hpp:68-77
    std::string model_id;
    Hash32 container_digest{};
    std::string arch;   // "archA" | "archB" (reference ToyModel) | "b200" (transformer)
    std::string driver_tag;
    DecodePolicy decode_policy;
    uint64_t seed = 0;
    std::vector<uint32_t> prompt;
};

struct InferenceOutput {   // detcore.hpp:79-85, plus the receipt's out_hash
    std::vector<uint32_t> tokens;
    std::vector<std::vector<float>> logits_trace;
    Bytes canonical_bytes;
    Hash32 out_hash{};
};

namespace detail {
// One engine per (device, model_id, arch): weights are generated once and stay resident.
inline detgpu_engine* engine_for(const ExecutionTuple& e, int device) {
    static std::mutex mu;
    static std::map<std::tuple<int, std::string, std::string>, detgpu_engine*> engines;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(device, e.model_id, e.arch);
    auto it = engines.find(key);
    if (it != engines.end()) return it->second;
    detgpu_engine* h = nullptr;
    const int rc = detgpu_create(device, e.model_id.c_str(), e.arch.c_str(), 64, 2048, &h);
    if (rc == DETGPU_EINVAL) throw std::invalid_argument(detgpu_global_error());
    if (rc != DETGPU_OK) throw std::runtime_error(detgpu_global_error());
    engines[key] = h;
    return h;
}
}  // namespace detail

// detcore.cpp:387-410. Groups by (model_id, arch); per-tuple bytes equal individual infer().
inline std::vector<InferenceOutput> infer_batch(const std::vector<ExecutionTuple>& execs, size_t batch_size,
                                                int device = 0) {
    if (batch_size == 0) throw std::invalid_argument("infer_batch: batch_size must be positive");
    std::vector<InferenceOutput> out(execs.size());
    std::map<std::pair<std::string, std::string>, std::vector<size_t>> groups;
    for (size_t i = 0; i < execs.size(); ++i) groups[{execs[i].model_id, execs[i].arch}].push_back(i);
    for (auto& [key, idx] : groups) {
        if (!detgpu_arch_supported(key.second.c_str()))
            throw std::invalid_argument("infer: unknown arch profile '" + key.second + "'");
        detgpu_engine* h = detail::engine_for(execs[idx[0]], device);
        detgpu_model_info info{};
        detgpu_get_model_info(h, &info);
        const size_t n = idx.size();
        std::vector<const uint32_t*> prompts(n);
        std::vector<uint32_t> lens(n);
        std::vector<detgpu_policy> pols(n);
        std::vector<uint64_t> seeds(n);
        std::vector<std::vector<uint32_t>> toks(n);
        std::vector<std::vector<float>> logits(n);
        std::vector<uint32_t*> tok_ptrs(n);
        std::vector<float*> lg_ptrs(n);
        std::vector<uint8_t> hashes(32 * n);
        for (size_t j = 0; j < n; ++j) {
            const ExecutionTuple& e = execs[idx[j]];
            prompts[j] = e.prompt.data();
            lens[j] = static_cast<uint32_t>(e.prompt.size());
            pols[j] = e.decode_policy.to_c();
            seeds[j] = e.seed;
            toks[j].resize(e.decode_policy.max_tokens);
            logits[j].resize(size_t(e.decode_policy.max_tokens) * info.vocab);
            tok_ptrs[j] = toks[j].data();
            lg_ptrs[j] = logits[j].data();
        }
        const int rc = detgpu_generate(h, static_cast<uint32_t>(n), prompts.data(), lens.data(), pols.data(),
                                       seeds.data(), static_cast<uint32_t>(batch_size), tok_ptrs.data(),
                                       lg_ptrs.data(), hashes.data(), 0, nullptr);
        if (rc == DETGPU_EINVAL || rc == DETGPU_ENONFINITE) throw std::invalid_argument(detgpu_last_error(h));
        if (rc != DETGPU_OK) throw std::runtime_error(detgpu_last_error(h));
        for (size_t j = 0; j < n; ++j) {
            InferenceOutput& o = out[idx[j]];
            const uint32_t T = execs[idx[j]].decode_policy.max_tokens;
            o.tokens = std::move(toks[j]);
            o.logits_trace.resize(T);
            for (uint32_t t = 0; t < T; ++t)
                o.logits_trace[t].assign(logits[j].begin() + size_t(t) * info.vocab,
                                         logits[j].begin() + size_t(t + 1) * info.vocab);
            o.canonical_bytes.resize(detgpu_canonical_size(T, info.vocab));
            detgpu_encode_canonical(o.tokens.data(), T, logits[j].data(), info.vocab, o.canonical_bytes.data());
            std::copy(hashes.begin() + 32 * j, hashes.begin() + 32 * (j + 1), o.out_hash.begin());
        }
    }
    return out;
}

// detcore.cpp:380-385
inline InferenceOutput infer(const ExecutionTuple& e, int device = 0) { return infer_batch({e}, 1, device)[0]; }

// receipts.cpp:119 req_hash
inline Hash32 req_hash(const ExecutionTuple& e) {
    const detgpu_policy p = e.decode_policy.to_c();
    const size_t n = detgpu_encode_exec_tuple(e.model_id.c_str(), e.container_digest.data(), e.arch.c_str(),
                                              e.driver_tag.c_str(), &p, e.seed, e.prompt.data(),
                                              static_cast<uint32_t>(e.prompt.size()), nullptr);
    Bytes b(n);
    detgpu_encode_exec_tuple(e.model_id.c_str(), e.container_digest.data(), e.arch.c_str(), e.driver_tag.c_str(), &p,
                             e.seed, e.prompt.data(), static_cast<uint32_t>(e.prompt.size()), b.data());
    Hash32 h{};
    detgpu_sha256(b.data(), b.size(), h.data());
    return h;
}

}  // namespace detgpu::detcore
