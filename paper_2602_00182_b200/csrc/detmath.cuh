// Deterministic arithmetic shared by every kernel of the engine.
//
// The numeric contract is the reference's: IEEE f32 round-to-nearest, no implicit
// contraction (the library is compiled with --fmad=false, mirroring -ffp-contract=off in
// reference proj/CMakeLists.txt:10-12), fused multiply-add only where written as __fmaf_rn, and
// sums in the reference's canonical tree order (detcore.cpp:135-150).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace detgpu {

// ------------------------------------------------------------------ exp
// det_expf: the exp the reference's det_softmax calls (std::exp on f32, detcore.cpp:193), as the
// x86-64 glibc 2.39 FMA variant evaluates it: x*32/ln2 = k + r, 2^(k/32) from a 32-entry table,
// cubic in r, all in binary64 with fused multiply-adds. Verified bit-exact against libm's expf for
// every float in [-104, 88.72] (oracle/check_expf.c); the oracle restates the same algorithm.
__device__ __constant__ static const unsigned long long kExp2Tab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};

__device__ __forceinline__ float det_expf(float x) {
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {                       // |x| >= 88 or non-finite
        if (ux == 0xff800000u) return 0.0f;      // -inf
        if (abstop >= 0x7f8) return x + x;       // +inf, NaN
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);  // overflow
        if (x < -0x1.9fe368p6f) return 0.0f;                       // underflow
    }
    const double InvLn2N = 0x1.71547652b82fep+0 * 32.0;
    const double Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
    const double C1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const double xd = static_cast<double>(x);
    double kd = __fma_rn(InvLn2N, xd, Shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, Shift);
    const double r = __fma_rn(InvLn2N, xd, -kd);
    unsigned long long t = kExp2Tab[ki % 32];
    t += ki << 47;
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double z = __fma_rn(C0, r, C1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(C2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

// The same function for warp-uniform call sites, with the 32-entry table held one entry per lane
// and fetched by shuffle (a divergent __constant__ lookup serialises up to 32 ways). Every lane of
// the warp must call it; the result is bit-identical to det_expf.
struct ExpTab {
    uint32_t lo, hi;
};
// The same 32 entries in global memory: a warp fetches them with one coalesced 256-byte load (a
// __constant__ read with 32 different addresses is serialised); call it early, off the critical path.
__device__ const unsigned long long kExp2TabG[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull,
};
__device__ __forceinline__ ExpTab exp_tab_lane() {
    const unsigned long long t = __ldg(&kExp2TabG[threadIdx.x & 31]);
    return ExpTab{static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32)};
}
__device__ __forceinline__ float det_expf_shfl(float x, ExpTab tab) {
    const double InvLn2N = 0x1.71547652b82fep+0 * 32.0;
    const double Shift = 0x1.8p+52;
    const double C0 = 0x1.c6af84b912394p-5 / 32.0 / 32.0 / 32.0;
    const double C1 = 0x1.ebfce50fac4f3p-3 / 32.0 / 32.0;
    const double C2 = 0x1.62e42ff0c52d6p-1 / 32.0;
    const double xd = static_cast<double>(x);
    double kd = __fma_rn(InvLn2N, xd, Shift);
    const unsigned long long ki = static_cast<unsigned long long>(__double_as_longlong(kd));
    kd = __dsub_rn(kd, Shift);
    const double r = __fma_rn(InvLn2N, xd, -kd);
    const int idx = static_cast<int>(ki & 31);
    const uint32_t lo = __shfl_sync(0xffffffffu, tab.lo, idx);
    const uint32_t hi = __shfl_sync(0xffffffffu, tab.hi, idx);
    unsigned long long t = (static_cast<unsigned long long>(hi) << 32) | lo;
    t += ki << 47;
    const double s = __longlong_as_double(static_cast<long long>(t));
    const double z = __fma_rn(C0, r, C1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(C2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    float res = __double2float_rn(y);
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ff;
    if (abstop >= 0x42b) {   // same special cases as det_expf, applied after the uniform shuffles
        if (ux == 0xff800000u) res = 0.0f;
        else if (abstop >= 0x7f8) res = x + x;
        else if (x > 0x1.62e42ep6f) res = __int_as_float(0x7f800000);
        else if (x < -0x1.9fe368p6f) res = 0.0f;
    }
    return res;
}

// packed f32x2 arithmetic (FMUL2 / FFMA2): each lane of the pair is an IEEE round-to-nearest f32
// operation, bit-identical to the scalar __fmul_rn / __fmaf_rn
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// fma(a, b, c) per lane. Used only where a*b is exact in f32 (a product of two bf16 values has at
// most 16 significant bits), so it equals add(round(a*b), c) bit for bit.
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// Per lane exactly __fmaf_rn(a, b, c) (a single rounding of the exact a*b+c): any operands.
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    return (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ float lo32(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi32(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

// Canonical 8-product block of a q.k dot product (local_tree_sum<8> of the exact products):
// ((p0+p1)+(p2+p3)) + ((p4+p5)+(p6+p7)), p_i = q_i * k_i with k_i the 8 bf16 values of `kv` and q
// stored as f32 quads in the order q0 q2 q1 q3 | q4 q6 q5 q7 (qa, qb). Products of two bf16
// values are exact in f32, so the packed fma equals the sum of the rounded products.
__device__ __forceinline__ float qk_block8(uint4 kv, ulonglong2 qa, ulonglong2 qb) {
    const uint64_t k02 = (static_cast<uint64_t>(kv.y << 16) << 32) | (kv.x << 16);
    const uint64_t k13 = (static_cast<uint64_t>(kv.y & 0xffff0000u) << 32) | (kv.x & 0xffff0000u);
    const uint64_t k46 = (static_cast<uint64_t>(kv.w << 16) << 32) | (kv.z << 16);
    const uint64_t k57 = (static_cast<uint64_t>(kv.w & 0xffff0000u) << 32) | (kv.z & 0xffff0000u);
    const uint64_t s0 = fma2(qa.x, k02, mul2(qa.y, k13));   // {p0+p1, p2+p3}
    const uint64_t s1 = fma2(qb.x, k46, mul2(qb.y, k57));   // {p4+p5, p6+p7}
    return __fadd_rn(__fadd_rn(lo32(s0), hi32(s0)), __fadd_rn(lo32(s1), hi32(s1)));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// The same canonical 8-product block with the second level packed too: q stored per 8-block as
// q0 q4 q1 q5 | q2 q6 q3 q7 (qa, qb), so the level-1 pairs land as (p0+p1, p4+p5) and
// (p2+p3, p6+p7) and one packed add forms (p0..3, p4..7). Same tree, same bits as qk_block8.
__device__ __forceinline__ float qk_block8_x2(uint4 kv, ulonglong2 qa, ulonglong2 qb) {
    const uint64_t k04 = (static_cast<uint64_t>(kv.z << 16) << 32) | (kv.x << 16);
    const uint64_t k15 = (static_cast<uint64_t>(kv.z & 0xffff0000u) << 32) | (kv.x & 0xffff0000u);
    const uint64_t k26 = (static_cast<uint64_t>(kv.w << 16) << 32) | (kv.y << 16);
    const uint64_t k37 = (static_cast<uint64_t>(kv.w & 0xffff0000u) << 32) | (kv.y & 0xffff0000u);
    const uint64_t sa = fma2(qa.x, k04, mul2(qa.y, k15));   // {p0+p1, p4+p5}
    const uint64_t sb = fma2(qb.x, k26, mul2(qb.y, k37));   // {p2+p3, p6+p7}
    const uint64_t t = add2(sa, sb);                         // {p0+..+p3, p4+..+p7}
    return __fadd_rn(lo32(t), hi32(t));
}
// index of q element i in the permuted quad layout qk_block8 reads (swap 1 <-> 2 in each quad)
__host__ __device__ constexpr int qperm(int i) { return (i & ~3) | ((i & 3) == 1 ? 2 : (i & 3) == 2 ? 1 : (i & 3)); }

// ------------------------------------------------------------------ bf16
__device__ __forceinline__ __nv_bfloat16 f2bf(float v) { return __float2bfloat16_rn(v); }
__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

// ------------------------------------------------------------------ canonical tree
// The reference tree (detcore.cpp:135-150: adjacent pairs level by level, odd tail promoted
// unchanged) equals the perfect binary tree over the input padded with -0.0f to a power of two,
// because x + (-0.0f) == x bit-exactly for every x. All GPU reductions below are perfect trees
// over power-of-two extents with that padding.
constexpr float kNegZero = -0.0f;

// Butterfly across the 32 lanes: level L pairs lanes differing in bit L, i.e. adjacent blocks,
// lowest bit first. f32 addition is commutative, so every lane ends with the identical tree sum.
__device__ __forceinline__ float warp_tree_sum(float v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

// In-register perfect tree over N (power of two) consecutive values.
template <int N>
__device__ __forceinline__ float local_tree_sum(float (&v)[N]) {
#pragma unroll
    for (int w = 1; w < N; w <<= 1) {
#pragma unroll
        for (int i = 0; i < N; i += 2 * w) v[i] = __fadd_rn(v[i], v[i + w]);
    }
    return v[0];
}

// Block-level tree: each warp has already produced the tree sum of its contiguous block; combine
// the NW (power of two) warp sums as a perfect tree. `scratch` holds >= NW floats.
template <int NW>
__device__ __forceinline__ float block_tree_combine(float warp_sum, float* scratch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) scratch[warp] = warp_sum;
    __syncthreads();
    float r;
    if (NW == 1) {
        r = scratch[0];
    } else {
        float v = lane < NW ? scratch[lane] : kNegZero;
        // lanes >= NW hold -0 padding; a 32-wide butterfly over [s_0..s_{NW-1}, -0, ...] reduces the
        // first NW lanes as a perfect tree and adds -0 sums afterwards, which leaves them unchanged.
        v = warp_tree_sum(v);
        r = v;
    }
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ PRNG (reference prng.hpp)
__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
// xoshiro256++ step (prng.hpp:46-56).
__device__ __forceinline__ uint64_t xoshiro_next(uint64_t* s) {
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
// splitmix64 output number n (n >= 1) of a generator seeded with `seed` (prng.hpp:18-23): counter
// based, so weight element i of a tensor is one evaluation at n = i + 1.
__host__ __device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t n) {
    uint64_t z = seed + n * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace detgpu
