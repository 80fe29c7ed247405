// Receipt v2 digest on the GPU: per generated step, the
// Merkle root of the step's f32 logits split into 4 KiB leaves, with the reference's DA tree rules
//   leaf  H(0x00 || blob)           (reference proj/src/da.cpp:27-34)
//   node  H(0x01 || left || right)  (da.cpp:36-43)
//   odd level: the last hash is paired with a copy of itself (da.cpp:48-61)
// so the host hashes only tokens and one 32-byte root per step instead of 131 MB of logits
// (receipt.cpp hash_canonical_v2). One CTA per (request slot, step): each thread hashes leaves
// (65 SHA-256 compressions per 4 KiB leaf), then the CTA folds the level in shared memory.
#include <cstdint>

#include "digest.cuh"

namespace detgpu {

namespace {

__constant__ uint32_t kK256[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void sha_init(uint32_t h[8]) {
    h[0] = 0x6a09e667u; h[1] = 0xbb67ae85u; h[2] = 0x3c6ef372u; h[3] = 0xa54ff53au;
    h[4] = 0x510e527fu; h[5] = 0x9b05688cu; h[6] = 0x1f83d9abu; h[7] = 0x5be0cd19u;
}

// One 64-byte block given as 16 big-endian message words.
__device__ __forceinline__ void sha_block(uint32_t h[8], uint32_t w[16]) {
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
#pragma unroll
    for (int t = 0; t < 64; ++t) {
        uint32_t wt;
        if (t < 16) {
            wt = w[t];
        } else {
            const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
            const uint32_t s0 = rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10);
            wt = w[t & 15] = w[t & 15] + s0 + w[(t - 7) & 15] + s1;
        }
        const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = hh + S1 + ch + kK256[t] + wt;
        const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + S0 + mj;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// H(0x00 || data[0..len)), len a multiple of 4 (f32 logits), data in little-endian memory order.
// Message word w holds data bytes 4w-1 .. 4w+2 (the tag byte shifts everything by one).
__device__ void leaf_hash(const uint32_t* __restrict__ d, int len, uint32_t out[8]) {
    const int nw = len / 4, lm = len + 1, nblk = (lm + 8) / 64 + 1;
    uint32_t h[8];
    sha_init(h);
    uint32_t prev = 0;   // data word w-1 (the tag byte 0x00 sits in its top byte for w = 0)
    for (int b = 0; b < nblk; ++b) {
        uint32_t w[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            const int wi = b * 16 + t;
            uint32_t v;
            if (wi < nw) {
                const uint32_t cur = __ldg(d + wi);
                v = __byte_perm(prev, cur, 0x3456);
                prev = cur;
            } else if (wi == nw) {
                v = __byte_perm(prev, 0x80u, 0x3456);   // last data byte, then the 0x80 pad byte
            } else {
                v = 0;
            }
            w[t] = v;
        }
        if (b == nblk - 1) w[15] = static_cast<uint32_t>(lm) * 8u;   // bit length (< 2^32)
        sha_block(h, w);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = h[i];
}

// H(0x01 || l || r) with l, r as big-endian digest words: a 65-byte message, two blocks.
__device__ void node_hash(const uint32_t l[8], const uint32_t r[8], uint32_t out[8]) {
    uint32_t h[8];
    sha_init(h);
    uint32_t w[16];
    w[0] = 0x01000000u | (l[0] >> 8);
#pragma unroll
    for (int t = 1; t < 8; ++t) w[t] = (l[t - 1] << 24) | (l[t] >> 8);
    w[8] = (l[7] << 24) | (r[0] >> 8);
#pragma unroll
    for (int t = 9; t < 16; ++t) w[t] = (r[t - 9] << 24) | (r[t - 8] >> 8);
    sha_block(h, w);
    w[0] = (r[7] << 24) | 0x00800000u;
#pragma unroll
    for (int t = 1; t < 15; ++t) w[t] = 0;
    w[15] = 65u * 8u;
    sha_block(h, w);
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = h[i];
}

constexpr int kThreads = 128;
constexpr int kMaxLeaves = 512;   // V <= 512 * 1024 floats

__global__ void __launch_bounds__(kThreads) receipt_roots_kernel(const float* __restrict__ trace, int64_t slot_stride,
                                                                 const int* __restrict__ steps, int V,
                                                                 uint8_t* __restrict__ roots, int tcap) {
    __shared__ uint32_t lv[kMaxLeaves][8];
    const int t = blockIdx.x, slot = blockIdx.y;
    if (t >= steps[slot]) return;
    const int bytes = 4 * V;
    const int L = (bytes + kLeafBytes - 1) / kLeafBytes;
    const uint32_t* base = reinterpret_cast<const uint32_t*>(trace + slot * slot_stride + static_cast<int64_t>(t) * V);
    for (int j = threadIdx.x; j < L; j += kThreads) {
        const int len = min(kLeafBytes, bytes - j * kLeafBytes);
        uint32_t hv[8];
        leaf_hash(base + j * (kLeafBytes / 4), len, hv);
#pragma unroll
        for (int i = 0; i < 8; ++i) lv[j][i] = hv[i];
    }
    __syncthreads();
    for (int n = L; n > 1; n = (n + 1) / 2) {   // odd level: the last node pairs with itself
        const int m = (n + 1) / 2;                  // <= kMaxLeaves / 2 = 2 * kThreads
        uint32_t h0[8], h1[8];
        const int k0 = threadIdx.x, k1 = threadIdx.x + kThreads;
        if (k0 < m) node_hash(lv[2 * k0], lv[2 * k0 + 1 < n ? 2 * k0 + 1 : 2 * k0], h0);
        if (k1 < m) node_hash(lv[2 * k1], lv[2 * k1 + 1 < n ? 2 * k1 + 1 : 2 * k1], h1);
        __syncthreads();   // every read of this level done before it is overwritten
        if (k0 < m)
#pragma unroll
            for (int i = 0; i < 8; ++i) lv[k0][i] = h0[i];
        if (k1 < m)
#pragma unroll
            for (int i = 0; i < 8; ++i) lv[k1][i] = h1[i];
        __syncthreads();
    }
    if (threadIdx.x < 8) {
        const uint32_t v = lv[0][threadIdx.x];
        uint8_t* o = roots + (static_cast<int64_t>(slot) * tcap + t) * 32 + threadIdx.x * 4;
        o[0] = static_cast<uint8_t>(v >> 24);
        o[1] = static_cast<uint8_t>(v >> 16);
        o[2] = static_cast<uint8_t>(v >> 8);
        o[3] = static_cast<uint8_t>(v);
    }
}

}  // namespace

cudaError_t launch_receipt_roots(const float* trace, int64_t slot_stride, const int* steps_dev, int n_slots, int tmax,
                                 int V, uint8_t* roots_dev, int tcap, cudaStream_t stream) {
    if (V <= 0 || (4LL * V + kLeafBytes - 1) / kLeafBytes > kMaxLeaves || n_slots <= 0 || tmax <= 0)
        return tmax <= 0 || n_slots <= 0 ? cudaSuccess : cudaErrorInvalidValue;
    receipt_roots_kernel<<<dim3(tmax, n_slots), kThreads, 0, stream>>>(trace, slot_stride, steps_dev, V, roots_dev,
                                                                      tcap);
    return cudaGetLastError();
}

}  // namespace detgpu
