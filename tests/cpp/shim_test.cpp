// C++ caller of the reference-shaped shim (include/detgpu_detcore.hpp), as a reference maintainer
// would call it: the SURVEY §8(c) golden cases must reproduce the reference's own hashes.
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "detgpu_detcore.hpp"

using namespace detgpu::detcore;

static std::string hex(const uint8_t* p, size_t n) {
    static const char* d = "0123456789abcdef";
    std::string s;
    for (size_t i = 0; i < n; ++i) {
        s.push_back(d[p[i] >> 4]);
        s.push_back(d[p[i] & 15]);
    }
    return s;
}

int main() {
    std::setvbuf(stdout, nullptr, _IONBF, 0);   // a crash still shows how far it got
    ExecutionTuple e;
    e.model_id = "model-a";
    const char* c = "container-a";
    detgpu_sha256(reinterpret_cast<const uint8_t*>(c), std::strlen(c), e.container_digest.data());
    e.arch = "archA";
    e.driver_tag = "drv-1";
    e.seed = 42;
    e.prompt = {1, 5, 9, 13, 2};
    e.decode_policy = DecodePolicy::top_k(4, 4);
    InferenceOutput o = infer(e);
    const std::string oh = hex(o.out_hash.data(), 32);
    const Hash32 rq = req_hash(e);
    if (oh != "0e9a353b8c5e90e25da31269140f95b3c678864efc731b914363133397e61560" ||
        hex(rq.data(), 32) != "1c5d710199bde6fabe2c664fd4e5ce09b5855cfc03c58608488956e53f1a0fe4") {
        std::printf("FAIL toy receipt %s\n", oh.c_str());
        return 1;
    }
    uint8_t again[32];
    detgpu_sha256(o.canonical_bytes.data(), o.canonical_bytes.size(), again);
    if (std::memcmp(again, o.out_hash.data(), 32) != 0) {
        std::printf("FAIL canonical bytes\n");
        return 1;
    }
    e.decode_policy = DecodePolicy::greedy(64);
    if (hex(infer(e).out_hash.data(), 32) != "8d1ffd911d4934391a909f04fcffe3d7259a8c9cce8ab241ea6f80889400caf4") {
        std::printf("FAIL toy greedy\n");
        return 1;
    }
    // transformer: batch composition never changes the bytes
    std::vector<ExecutionTuple> batch;
    for (int i = 0; i < 10; ++i) {
        ExecutionTuple t = e;
        t.arch = "b200";
        t.model_id = "llama-tiny:shim";
        t.seed = 100 + i;
        t.prompt = {uint32_t(7 * i + 1), uint32_t(3 * i + 2), 9, 10};
        t.decode_policy = i % 2 ? DecodePolicy::nucleus(0.9f, 12) : DecodePolicy::greedy(12);
        batch.push_back(t);
    }
    auto a = infer_batch(batch, 10);
    auto b = infer_batch(batch, 3);
    for (size_t i = 0; i < batch.size(); ++i) {
        if (a[i].out_hash != b[i].out_hash || a[i].out_hash != infer(batch[i]).out_hash) {
            std::printf("FAIL batch invariance at %zu\n", i);
            return 1;
        }
    }
    // a caller's registry (detcore.hpp:34-47): a new name for the canonical-tree order gives
    // archA's bytes; the default registry rejects the name
    {
        ArchRegistry reg = ArchRegistry::defaults();
        reg.add({"archC", ReductionOrder::canonical_tree, FmaEmulation::fused});
        ExecutionTuple t = e;
        t.arch = "archC";
        if (infer(t, reg).out_hash != infer(e).out_hash) {
            std::printf("FAIL custom registry\n");
            return 1;
        }
        try {
            infer(t);
            std::printf("FAIL: default registry accepted archC\n");
            return 1;
        } catch (const std::invalid_argument&) {
        }
    }
    // concurrent callers share one cached engine: bytes unchanged
    {
        std::vector<Hash32> got(8);
        std::vector<std::thread> th;
        for (int i = 0; i < 8; ++i) th.emplace_back([&, i] { got[i] = infer(batch[i % 4]).out_hash; });
        for (auto& t : th) t.join();
        for (int i = 0; i < 8; ++i)
            if (got[i] != a[i % 4].out_hash) {
                std::printf("FAIL concurrent infer at %d\n", i);
                return 1;
            }
    }
    // a request beyond the cached engine's context rebuilds it (the reference has no limit);
    // an empty prompt is accepted (BOS rule) like the reference accepts it
    {
        ExecutionTuple t = batch[0];
        t.prompt.assign(2100, 5);
        t.decode_policy = DecodePolicy::greedy(4);
        if (infer(t).tokens.size() != 4) {
            std::printf("FAIL long context\n");
            return 1;
        }
        t.prompt.clear();
        ExecutionTuple u = t;
        u.prompt = {0};
        if (infer(t).out_hash != infer(u).out_hash) {
            std::printf("FAIL empty prompt != [BOS]\n");
            return 1;
        }
        release_engines();
        if (infer(batch[1]).out_hash != a[1].out_hash) {
            std::printf("FAIL after release_engines\n");
            return 1;
        }
    }
    try {
        e.arch = "archZ";
        infer(e);
        std::printf("FAIL: no invalid_argument for unknown arch\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    std::printf("OK\n");
    std::fflush(stdout);
    return 0;
}
