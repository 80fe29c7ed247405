// Header-only C++ shim: the reference's detcore API (proj/include/verinf/detcore.hpp:21-163) on top
// of the detgpu C-ABI. A reference maintainer swaps `verinf::detcore::infer` for
// `detgpu::detcore::infer` (same types, same std::invalid_argument behaviour) and links
// libdetgpu.so; see INTEGRATION.md. Requires C++17.
#pragma once

#include <algorithm>
#include <array>
#include <climits>
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

// ---- approved profiles (detcore.hpp:21-45, detcore.cpp:12-26) ----
// The reference's profiles name an accumulation order; the GPU engine runs canonical_tree and
// sequential on the reference ToyModel (engine arch "archA" / "archB") and tcgen05_b200 on the
// Llama-style transformer (engine arch "b200"). A caller's registry may add more names for these
// orders, exactly as the reference's ArchRegistry::add does.
enum class ReductionOrder : uint8_t { canonical_tree = 0, sequential = 1, tcgen05_b200 = 2 };
enum class FmaEmulation : uint8_t { fused = 0, split = 1 };

struct ArchProfile {
    std::string name;
    ReductionOrder reduction_order = ReductionOrder::canonical_tree;
    FmaEmulation fma_emulation = FmaEmulation::split;
};

class ArchRegistry {
public:
    static const ArchRegistry& defaults() {
        static const ArchRegistry reg = [] {
            ArchRegistry r;
            r.add({"archA", ReductionOrder::canonical_tree, FmaEmulation::fused});
            r.add({"archB", ReductionOrder::sequential, FmaEmulation::split});
            r.add({"b200", ReductionOrder::tcgen05_b200, FmaEmulation::fused});
            return r;
        }();
        return reg;
    }
    void add(ArchProfile p) { profiles_[p.name] = std::move(p); }
    const ArchProfile* find(const std::string& name) const {
        auto it = profiles_.find(name);
        return it == profiles_.end() ? nullptr : &it->second;
    }
    bool contains(const std::string& name) const { return find(name) != nullptr; }
    std::vector<std::string> names() const {
        std::vector<std::string> v;
        for (auto& kv : profiles_) v.push_back(kv.first);
        return v;
    }

private:
    std::map<std::string, ArchProfile> profiles_;
};

// ---- engine cache ----
// One engine per (device, model_id, engine arch) holds the weights resident. Sized from the
// requests: an engine is rebuilt with a larger context when a request needs it (the reference
// accepts any length). A per-engine mutex serialises generate + copy-out (the reference's infer
// is pure and thread-safe; the handle is not). At most max_engines stay cached (least recently
// used dropped); release_engines() frees them all (an engine still in use by another thread is
// destroyed when that call returns).
struct EngineOptions {
    uint32_t max_batch = 64;       // decode slots per engine (larger batch_size runs in groups: same bytes)
    uint32_t min_context = 2048;   // initial context capacity; grown to the next power of two on demand
    size_t max_engines = 4;
};

namespace detail {
struct CachedEngine {
    detgpu_engine* h = nullptr;
    uint32_t max_context = 0;
    uint64_t last_used = 0;
    std::mutex mu;
    ~CachedEngine() {
        if (h) detgpu_destroy(h);
    }
};
struct Cache {
    std::mutex mu;
    EngineOptions opt;
    uint64_t clock = 0;
    std::map<std::tuple<int, std::string, std::string>, std::shared_ptr<CachedEngine>> engines;
};
inline Cache& cache() {
    // Never destroyed: engines still cached at process exit are reclaimed with the process. A
    // static destructor would call detgpu_destroy after the CUDA runtime's own teardown has run.
    static Cache* c = new Cache;
    return *c;
}
inline const char* engine_arch(const ArchProfile& p) {
    switch (p.reduction_order) {
        case ReductionOrder::canonical_tree: return "archA";
        case ReductionOrder::sequential: return "archB";
        default: return "b200";
    }
}
inline std::shared_ptr<CachedEngine> engine_for(const std::string& model_id, const char* arch, uint32_t need_ctx,
                                                int device) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto key = std::make_tuple(device, model_id, std::string(arch));
    auto it = c.engines.find(key);
    if (it != c.engines.end() && it->second->max_context >= need_ctx) {
        it->second->last_used = ++c.clock;
        return it->second;
    }
    uint32_t ctx = std::max<uint32_t>(1, c.opt.min_context);
    while (ctx < need_ctx) ctx *= 2;
    if (it == c.engines.end() && c.engines.size() >= std::max<size_t>(1, c.opt.max_engines)) {
        auto victim = c.engines.begin();
        for (auto v = c.engines.begin(); v != c.engines.end(); ++v)
            if (v->second->last_used < victim->second->last_used) victim = v;
        c.engines.erase(victim);
    }
    auto e = std::make_shared<CachedEngine>();
    const bool toy = std::string(arch) != "b200";
    const int rc = detgpu_create(device, model_id.c_str(), arch, c.opt.max_batch, toy ? 1 : ctx, &e->h);
    if (rc == DETGPU_EINVAL) throw std::invalid_argument(detgpu_global_error());
    if (rc != DETGPU_OK) throw std::runtime_error(detgpu_global_error());
    e->max_context = toy ? UINT32_MAX : ctx;
    e->last_used = ++c.clock;
    c.engines[key] = e;
    return e;
}
}  // namespace detail

inline void set_engine_options(const EngineOptions& o) {
    std::lock_guard<std::mutex> lk(detail::cache().mu);
    detail::cache().opt = o;
}
inline void release_engines() {
    std::lock_guard<std::mutex> lk(detail::cache().mu);
    detail::cache().engines.clear();
}

// detcore.cpp:387-410. Groups by (model_id, profile); per-tuple bytes equal individual infer().
// Validation before any work, in the reference's order (unknown arch, then policy, then tokens).
inline std::vector<InferenceOutput> infer_batch(const std::vector<ExecutionTuple>& execs, size_t batch_size,
                                                const ArchRegistry& registry = ArchRegistry::defaults(),
                                                int device = 0) {
    if (batch_size == 0) throw std::invalid_argument("infer_batch: batch_size must be positive");
    std::vector<InferenceOutput> out(execs.size());
    std::map<std::pair<std::string, std::string>, std::vector<size_t>> groups;
    for (size_t i = 0; i < execs.size(); ++i) {
        const ArchProfile* prof = registry.find(execs[i].arch);
        if (prof == nullptr) throw std::invalid_argument("infer: unknown arch profile '" + execs[i].arch + "'");
        groups[{execs[i].model_id, detail::engine_arch(*prof)}].push_back(i);
    }
    for (auto& [key, idx] : groups) {
        uint32_t need = 1;
        for (size_t i : idx)
            need = std::max<uint32_t>(need, static_cast<uint32_t>(std::max<size_t>(execs[i].prompt.size(), 1)) +
                                                execs[i].decode_policy.max_tokens);
        std::shared_ptr<detail::CachedEngine> eng = detail::engine_for(key.first, key.second.c_str(), need, device);
        std::lock_guard<std::mutex> use(eng->mu);
        detgpu_engine* h = eng->h;
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
inline InferenceOutput infer(const ExecutionTuple& e, const ArchRegistry& registry = ArchRegistry::defaults(),
                             int device = 0) {
    return infer_batch({e}, 1, registry, device)[0];
}

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
