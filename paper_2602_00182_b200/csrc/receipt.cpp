// Host side of the receipt path: SHA-256 (SHA-NI with a portable fallback), the canonical output
// layout (reference detcore.cpp:73-84) hashed without materialising it, and the ExecutionTuple
// codec (reference codec.cpp:67-170) with a strict decoder.
#include <cpuid.h>
#include <immintrin.h>

#include <cstring>
#include <string>

#include "detgpu.h"
#include "receipt.h"

#include <algorithm>
#include <array>
#include <vector>

namespace detgpu {

namespace {

const uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void blocks_portable(uint32_t* h, const uint8_t* p, size_t nblocks) {
    for (size_t blk = 0; blk < nblocks; ++blk, p += 64) {
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t(p[4 * i]) << 24) | (uint32_t(p[4 * i + 1]) << 16) | (uint32_t(p[4 * i + 2]) << 8) |
                   uint32_t(p[4 * i + 3]);
        for (int i = 16; i < 64; ++i) {
            const uint32_t s0 = ror(w[i - 15], 7) ^ ror(w[i - 15], 18) ^ (w[i - 15] >> 3);
            const uint32_t s1 = ror(w[i - 2], 17) ^ ror(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
        for (int i = 0; i < 64; ++i) {
            const uint32_t t1 = hh + (ror(e, 6) ^ ror(e, 11) ^ ror(e, 25)) + ((e & f) ^ (~e & g)) + kK[i] + w[i];
            const uint32_t t2 = (ror(a, 2) ^ ror(a, 13) ^ ror(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            hh = g;
            g = f;
            f = e;
            e = d + t1;
            d = c;
            c = b;
            b = a;
            a = t1 + t2;
        }
        h[0] += a;
        h[1] += b;
        h[2] += c;
        h[3] += d;
        h[4] += e;
        h[5] += f;
        h[6] += g;
        h[7] += hh;
    }
}

// SHA-NI compression (Intel SHA extensions): state kept as ABEF / CDGH lanes.
__attribute__((target("sha,sse4.1"))) void blocks_shani(uint32_t* h, const uint8_t* p, size_t nblocks) {
    const __m128i MASK = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&h[0]));   // DCBA
    __m128i st1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&h[4]));   // HGFE
    tmp = _mm_shuffle_epi32(tmp, 0xB1);                                       // CDAB
    st1 = _mm_shuffle_epi32(st1, 0x1B);                                       // EFGH
    __m128i st0 = _mm_alignr_epi8(tmp, st1, 8);                               // ABEF
    st1 = _mm_blend_epi16(st1, tmp, 0xF0);                                    // CDGH
    for (size_t blk = 0; blk < nblocks; ++blk, p += 64) {
        const __m128i abef = st0, cdgh = st1;
        __m128i m[4];
        for (int i = 0; i < 4; ++i)
            m[i] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * i)), MASK);
        for (int r = 0; r < 16; ++r) {
            __m128i& cur = m[r & 3];
            if (r >= 4) {
                // schedule: W[16..] from msg1/msg2 on the rolling 4-vector window
                __m128i t = _mm_sha256msg1_epu32(m[r & 3], m[(r + 1) & 3]);
                t = _mm_add_epi32(t, _mm_alignr_epi8(m[(r + 3) & 3], m[(r + 2) & 3], 4));
                cur = _mm_sha256msg2_epu32(t, m[(r + 3) & 3]);
            }
            const __m128i k = _mm_loadu_si128(reinterpret_cast<const __m128i*>(&kK[4 * r]));
            __m128i msg = _mm_add_epi32(cur, k);
            st1 = _mm_sha256rnds2_epu32(st1, st0, msg);
            msg = _mm_shuffle_epi32(msg, 0x0E);
            st0 = _mm_sha256rnds2_epu32(st0, st1, msg);
        }
        st0 = _mm_add_epi32(st0, abef);
        st1 = _mm_add_epi32(st1, cdgh);
    }
    tmp = _mm_shuffle_epi32(st0, 0x1B);   // FEBA
    st1 = _mm_shuffle_epi32(st1, 0xB1);   // DCHG
    st0 = _mm_blend_epi16(tmp, st1, 0xF0);   // DCBA
    st1 = _mm_alignr_epi8(st1, tmp, 8);      // HGFE
    _mm_storeu_si128(reinterpret_cast<__m128i*>(&h[0]), st0);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(&h[4]), st1);
}

bool cpu_has_shani() {
    unsigned a, b, c, d;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    const bool sha = (b >> 29) & 1;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
    const bool sse41 = (c >> 19) & 1, ssse3 = (c >> 9) & 1;
    return sha && sse41 && ssse3;
}

const bool kShaNi = cpu_has_shani();

}  // namespace

Sha256::Sha256() {
    static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    std::memcpy(h_, iv, sizeof(h_));
}

void Sha256::compress(const uint8_t* p, size_t nblocks) {
    if (kShaNi) blocks_shani(h_, p, nblocks);
    else blocks_portable(h_, p, nblocks);
}

void Sha256::update(const void* data, size_t n) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    total_ += n;
    if (fill_ > 0) {
        const size_t take = std::min(n, size_t(64) - fill_);
        std::memcpy(buf_ + fill_, p, take);
        fill_ += take;
        p += take;
        n -= take;
        if (fill_ == 64) {
            compress(buf_, 1);
            fill_ = 0;
        }
    }
    if (n >= 64) {
        compress(p, n / 64);
        p += (n / 64) * 64;
        n %= 64;
    }
    if (n > 0) {
        std::memcpy(buf_, p, n);
        fill_ = n;
    }
}

void Sha256::final(uint8_t out[32]) {
    const uint64_t bits = total_ * 8;
    uint8_t pad[72] = {0x80};
    const size_t padlen = (fill_ < 56) ? (56 - fill_) : (120 - fill_);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = uint8_t(bits >> (56 - 8 * i));
    update(pad, padlen);
    update(len, 8);
    for (int i = 0; i < 8; ++i) {
        out[4 * i] = uint8_t(h_[i] >> 24);
        out[4 * i + 1] = uint8_t(h_[i] >> 16);
        out[4 * i + 2] = uint8_t(h_[i] >> 8);
        out[4 * i + 3] = uint8_t(h_[i]);
    }
}

bool sha_ni_available() { return kShaNi; }

// Canonical bytes (detcore.cpp:73-84), little-endian: [T][tok...][T][(V, logits_bits...) x T].
// The host is little-endian, so token and logit arrays are hashed in place.
void hash_canonical(const uint32_t* tokens, uint32_t T, const float* logits, uint32_t V, uint8_t out[32]) {
    Sha256 s;
    s.update(&T, 4);
    if (T > 0) s.update(tokens, 4 * size_t(T));
    s.update(&T, 4);
    for (uint32_t t = 0; t < T; ++t) {
        s.update(&V, 4);
        s.update(logits + size_t(t) * V, 4 * size_t(V));
    }
    s.final(out);
}

// ---- receipt v2: per-step Merkle roots over 4 KiB leaves, da.cpp tree rules ----
void merkle_leaf(const void* blob, size_t n, uint8_t out[32]) {   // H(0x00 || blob), da.cpp:27-34
    const uint8_t tag = 0x00;
    Sha256 s;
    s.update(&tag, 1);
    if (n) s.update(blob, n);
    s.final(out);
}
void merkle_node(const uint8_t l[32], const uint8_t r[32], uint8_t out[32]) {   // H(0x01 || l || r)
    const uint8_t tag = 0x01;
    Sha256 s;
    s.update(&tag, 1);
    s.update(l, 32);
    s.update(r, 32);
    s.final(out);
}
void step_root(const float* logits, uint32_t V, uint8_t out[32]) {
    const size_t bytes = 4 * size_t(V);
    std::vector<std::array<uint8_t, 32>> level((bytes + kV2LeafBytes - 1) / kV2LeafBytes);
    const uint8_t* b = reinterpret_cast<const uint8_t*>(logits);
    for (size_t j = 0; j < level.size(); ++j)
        merkle_leaf(b + j * kV2LeafBytes, std::min<size_t>(kV2LeafBytes, bytes - j * kV2LeafBytes), level[j].data());
    if (level.empty()) {   // da.cpp:45-46 sentinel (V = 0 never occurs)
        merkle_leaf(nullptr, 0, out);
        return;
    }
    while (level.size() > 1) {   // odd level: last node paired with itself (da.cpp:48-61)
        std::vector<std::array<uint8_t, 32>> next((level.size() + 1) / 2);
        for (size_t i = 0; i < next.size(); ++i)
            merkle_node(level[2 * i].data(), level[2 * i + 1 < level.size() ? 2 * i + 1 : 2 * i].data(), next[i].data());
        level.swap(next);
    }
    std::memcpy(out, level[0].data(), 32);
}
// SHA-256 of "RCPTv2\0\0" || [T][tokens][T][(V, root) x T], little-endian like the v1 layout.
void hash_canonical_v2_roots(const uint32_t* tokens, uint32_t T, const uint8_t* roots, uint32_t V, uint8_t out[32]) {
    static const char tag[8] = {'R', 'C', 'P', 'T', 'v', '2', 0, 0};
    Sha256 s;
    s.update(tag, 8);
    s.update(&T, 4);
    if (T > 0) s.update(tokens, 4 * size_t(T));
    s.update(&T, 4);
    for (uint32_t t = 0; t < T; ++t) {
        s.update(&V, 4);
        s.update(roots + 32 * size_t(t), 32);
    }
    s.final(out);
}

}  // namespace detgpu

using namespace detgpu;

namespace {
void put_be32(std::string& o, uint32_t v) {
    o.push_back(char(v >> 24));
    o.push_back(char(v >> 16));
    o.push_back(char(v >> 8));
    o.push_back(char(v));
}
uint32_t load_be32(const uint8_t* p) {
    return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}
}  // namespace

extern "C" {

void detgpu_sha256(const uint8_t* data, size_t n, uint8_t out[32]) {
    Sha256 s;
    s.update(data, n);
    s.final(out);
}

size_t detgpu_canonical_size(uint32_t T, uint32_t V) { return 8 + 4 * size_t(T) + size_t(T) * (4 + 4 * size_t(V)); }

void detgpu_encode_canonical(const uint32_t* tokens, uint32_t T, const float* logits, uint32_t V, uint8_t* out) {
    uint8_t* p = out;
    std::memcpy(p, &T, 4);
    p += 4;
    if (T > 0) std::memcpy(p, tokens, 4 * size_t(T));
    p += 4 * size_t(T);
    std::memcpy(p, &T, 4);
    p += 4;
    for (uint32_t t = 0; t < T; ++t) {
        std::memcpy(p, &V, 4);
        p += 4;
        std::memcpy(p, logits + size_t(t) * V, 4 * size_t(V));
        p += 4 * size_t(V);
    }
}

void detgpu_hash_canonical(const uint32_t* tokens, uint32_t T, const float* logits, uint32_t V, uint8_t out[32]) {
    hash_canonical(tokens, T, logits, V, out);
}

void detgpu_step_root(const float* logits, uint32_t V, uint8_t out[32]) { step_root(logits, V, out); }

void detgpu_hash_canonical_v2(const uint32_t* tokens, uint32_t T, const float* logits, uint32_t V, uint8_t out[32]) {
    std::vector<uint8_t> roots(32 * size_t(T));
    for (uint32_t t = 0; t < T; ++t) step_root(logits + size_t(t) * V, V, roots.data() + 32 * size_t(t));
    hash_canonical_v2_roots(tokens, T, roots.data(), V, out);
}

// codec.cpp:93-104 and encode_policy codec.cpp:67-74
size_t detgpu_encode_exec_tuple(const char* model_id, const uint8_t container_digest[32], const char* arch,
                                const char* driver_tag, const detgpu_policy* policy, uint64_t seed,
                                const uint32_t* prompt, uint32_t prompt_len, uint8_t* out) {
    std::string w;
    auto str = [&](const char* s) {
        const size_t n = std::strlen(s);
        put_be32(w, uint32_t(n));
        w.append(s, n);
    };
    str(model_id);
    w.append(reinterpret_cast<const char*>(container_digest), 32);
    str(arch);
    str(driver_tag);
    w.push_back(char(policy->kind));
    w.push_back(char(policy->has_k ? 1 : 0));
    put_be32(w, policy->has_k ? policy->k : 0);
    w.push_back(char(policy->has_p ? 1 : 0));
    const float pv = policy->has_p ? policy->p : 0.0f;
    uint32_t pb;
    std::memcpy(&pb, &pv, 4);
    put_be32(w, pb);
    put_be32(w, policy->max_tokens);
    put_be32(w, uint32_t(seed >> 32));
    put_be32(w, uint32_t(seed));
    put_be32(w, prompt_len);
    for (uint32_t i = 0; i < prompt_len; ++i) put_be32(w, prompt[i]);
    if (out != nullptr) std::memcpy(out, w.data(), w.size());
    return w.size();
}

int detgpu_decode_exec_tuple(const uint8_t* b, size_t n, char* model_id, size_t model_id_cap,
                             uint8_t container_digest[32], char* arch, size_t arch_cap, char* driver_tag,
                             size_t driver_cap, detgpu_policy* policy, uint64_t* seed, uint32_t* prompt_out,
                             uint32_t prompt_cap, uint32_t* prompt_len) {
    size_t pos = 0;
    auto need = [&](size_t k) { return pos + k <= n; };
    auto u8 = [&](uint8_t* v) {
        if (!need(1)) return false;
        *v = b[pos++];
        return true;
    };
    auto u32 = [&](uint32_t* v) {
        if (!need(4)) return false;
        *v = load_be32(b + pos);
        pos += 4;
        return true;
    };
    auto str = [&](char* dst, size_t cap) {
        uint32_t len;
        if (!u32(&len) || !need(len) || size_t(len) + 1 > cap) return false;
        std::memcpy(dst, b + pos, len);
        dst[len] = 0;
        if (std::memchr(dst, 0, len) != nullptr) return false;   // embedded NUL cannot round-trip
        pos += len;
        return true;
    };
    if (!str(model_id, model_id_cap)) return DETGPU_EINVAL;
    if (!need(32)) return DETGPU_EINVAL;
    std::memcpy(container_digest, b + pos, 32);
    pos += 32;
    if (!str(arch, arch_cap) || !str(driver_tag, driver_cap)) return DETGPU_EINVAL;
    uint8_t kind, has_k, has_p;
    uint32_t k, pbits, max_tokens, hi, lo, count;
    if (!u8(&kind) || !u8(&has_k) || !u32(&k) || !u8(&has_p) || !u32(&pbits) || !u32(&max_tokens)) return DETGPU_EINVAL;
    // strict: flags are 0/1 and absent fields carry a zero payload, so decode(encode(x)) is the
    // only preimage (fixes the malleability of codec.cpp:76-91)
    if (kind > 2 || has_k > 1 || has_p > 1 || (!has_k && k != 0) || (!has_p && pbits != 0)) return DETGPU_EINVAL;
    if (!u32(&hi) || !u32(&lo) || !u32(&count)) return DETGPU_EINVAL;
    if (count > prompt_cap || !need(size_t(count) * 4)) return DETGPU_EINVAL;
    for (uint32_t i = 0; i < count; ++i) u32(&prompt_out[i]);
    if (pos != n) return DETGPU_EINVAL;
    policy->kind = kind;
    policy->has_k = has_k;
    policy->has_p = has_p;
    policy->reserved = 0;
    policy->k = k;
    std::memcpy(&policy->p, &pbits, 4);
    policy->max_tokens = max_tokens;
    *seed = (uint64_t(hi) << 32) | lo;
    *prompt_len = count;
    return DETGPU_OK;
}

}  // extern "C"
