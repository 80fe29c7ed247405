// C entry points over the UNMODIFIED reference receipts / codec / sign / sha256 / da sources
// (compiled by `make -C oracle ref-receipts` with libsodium from PyNaCl and nlohmann json).
// Used only to generate tests/golden/receipts_reference.json. TEST INFRASTRUCTURE ONLY.
#include <cstring>
#include <string>

#include "verinf/codec.hpp"
#include "verinf/receipts.hpp"
#include "verinf/sign.hpp"

using namespace verinf;

namespace {
size_t put(const void* src, size_t n, uint8_t* dst, size_t cap) {
    if (dst != nullptr && n <= cap) std::memcpy(dst, src, n);
    return n;
}
}  // namespace

extern "C" {

// Builds a receipt with make_receipt (receipts.cpp:107-127) for the tuple and canonical output
// bytes given, signed with Ed25519Signer::from_seed(sign_seed). Writes body / wire / JSON /
// public key into caller buffers (each returns its size in *_n; NULL buffer = size query).
int refr_make(const char* model_id, const uint8_t* digest, const char* arch, const char* driver, int kind, int has_k,
              uint32_t k, int has_p, float p, uint32_t max_tokens, uint64_t seed, const uint32_t* prompt,
              uint32_t plen, const uint8_t* canonical, size_t canonical_n, const uint8_t* sign_seed,
              const char* chain_id, const char* da_pointer, uint32_t key_epoch, uint64_t timestamp,
              const uint8_t* att_quote, size_t att_quote_n, int has_quote, uint8_t* body, size_t* body_n,
              uint8_t* wire, size_t* wire_n, char* json, size_t* json_n, uint8_t* pubkey) {
    detcore::ExecutionTuple e;
    e.model_id = model_id;
    std::memcpy(e.container_digest.data(), digest, 32);
    e.arch = arch;
    e.driver_tag = driver;
    e.decode_policy.kind = detcore::DecodeKind(kind);
    if (has_k) e.decode_policy.k = k;
    if (has_p) e.decode_policy.p = p;
    e.decode_policy.max_tokens = max_tokens;
    e.seed = seed;
    e.prompt.assign(prompt, prompt + plen);
    detcore::InferenceOutput out;
    out.canonical_bytes.assign(canonical, canonical + canonical_n);
    Hash32 sd;
    std::memcpy(sd.data(), sign_seed, 32);
    const auto signer = sign::Ed25519Signer::from_seed(sd);
    std::optional<Bytes> quote;
    if (has_quote) quote = Bytes(att_quote, att_quote + att_quote_n);
    const receipts::Receipt rc =
        receipts::make_receipt(e, out, signer, chain_id, da_pointer, key_epoch, timestamp, quote);
    const Bytes b = receipts::canonical_receipt_body(rc);
    const Bytes w = receipts::encode_receipt(rc);
    const std::string j = receipts::receipt_to_json(rc);
    const Bytes pk = signer.public_key();
    *body_n = put(b.data(), b.size(), body, *body_n);
    *wire_n = put(w.data(), w.size(), wire, *wire_n);
    *json_n = put(j.c_str(), j.size() + 1, reinterpret_cast<uint8_t*>(json), *json_n);
    std::memcpy(pubkey, pk.data(), 32);
    return 0;
}

// decode_receipt + verify_receipt (receipts.cpp:72-82, 133-149) on wire bytes; 1 verified,
// 0 rejected (why filled), -1 undecodable.
int refr_verify(const uint8_t* wire, size_t wire_n, const uint8_t* pubkey, char* why, size_t why_cap) {
    auto rc = receipts::decode_receipt(std::span<const uint8_t>(wire, wire_n));
    if (!rc) return -1;
    std::string w;
    const bool ok = receipts::verify_receipt(*rc, std::span<const uint8_t>(pubkey, 32),
                                             receipts::Registry::defaults(), &w);
    std::snprintf(why, why_cap, "%s", w.c_str());
    return ok ? 1 : 0;
}

// receipt_from_json then encode_receipt: the wire bytes of a JSON receipt (0 when rejected).
size_t refr_json_to_wire(const char* json, uint8_t* wire, size_t cap) {
    auto rc = receipts::receipt_from_json(json);
    if (!rc) return 0;
    const Bytes w = receipts::encode_receipt(*rc);
    return put(w.data(), w.size(), wire, cap);
}

// policy_to_string / policy_from_string (codec.cpp:123-190).
size_t refr_policy_to_string(int kind, int has_k, uint32_t k, int has_p, float p, uint32_t max_tokens, char* out,
                             size_t cap) {
    detcore::DecodePolicy pol;
    pol.kind = detcore::DecodeKind(kind);
    if (has_k) pol.k = k;
    if (has_p) pol.p = p;
    pol.max_tokens = max_tokens;
    const std::string s = codec::policy_to_string(pol);
    return put(s.c_str(), s.size() + 1, reinterpret_cast<uint8_t*>(out), cap);
}
int refr_policy_from_string(const char* text, int* kind, int* has_k, uint32_t* k, int* has_p, float* p,
                            uint32_t* max_tokens) {
    auto pol = codec::policy_from_string(text);
    if (!pol) return 0;
    *kind = int(pol->kind);
    *has_k = pol->k.has_value();
    *k = pol->k.value_or(0);
    *has_p = pol->p.has_value();
    *p = pol->p.value_or(0.0f);
    *max_tokens = pol->max_tokens;
    return 1;
}

}  // extern "C"
