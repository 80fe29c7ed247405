// Non-GEMM kernels: RMSNorm (+embedding gather), paged decode attention with a fixed KV-chunk
// order, vocabulary softmax + decode (greedy / top-k / nucleus), counter-based weight generation.
// Every reduction is a perfect binary tree over a -0.0f-padded power-of-two extent, which equals
// the reference's canonical tree (detcore.cpp:135-150); every multiply-add is explicit.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "detmath.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace detgpu {

namespace {

__device__ __forceinline__ int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

// Perfect tree over [0, n) padded with -0 to P2 = max(128, pow2 >= n): 128-element tiles reduced by
// (ld(i, valid) must return -0.0f for !valid)
// one warp each (4 consecutive per lane, then the lane butterfly), tile sums reduced level by level
// in shared memory. Requires blockDim.x == 1024 and n <= 131072.
template <class Load>
__device__ float block_tree_sum_1024(int n, Load ld, float* s_tiles) {
    const int P2 = max(128, next_pow2(n));
    const int ntiles = P2 / 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = warp; t < ntiles; t += 32) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = t * 128 + lane * 4 + j;
            v[j] = ld(i, i < n);   // called by every lane (warp-uniform), returns -0 when !valid
        }
        float s = local_tree_sum<4>(v);
        s = warp_tree_sum(s);
        if (lane == 0) s_tiles[t] = s;
    }
    __syncthreads();
    for (int w = 1; w < ntiles; w <<= 1) {
        for (int i = threadIdx.x * 2 * w; i < ntiles; i += blockDim.x * 2 * w)
            s_tiles[i] = __fadd_rn(s_tiles[i], s_tiles[i + w]);
        __syncthreads();
    }
    const float r = s_tiles[0];
    __syncthreads();
    return r;
}

// The same tree when producing a leaf needs a global load followed by a store (the softmax exp
// pass): fetch(i, ok) only loads, map(i, ok, raw) computes / stores and returns the leaf. The next
// tile's loads are issued before this tile's stores, so loads are not serialised behind stores
// the compiler cannot prove disjoint.
template <class Fetch, class Map>
__device__ float block_tree_sum_1024_fm(int n, Fetch fetch, Map map, float* s_tiles) {
    const int P2 = max(128, next_pow2(n));
    const int ntiles = P2 / 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float nxt[4];
    if (warp < ntiles) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = warp * 128 + lane * 4 + j;
            nxt[j] = fetch(i, i < n);
        }
    }
    for (int t = warp; t < ntiles; t += 32) {
        float raw[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) raw[j] = nxt[j];
        if (t + 32 < ntiles) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = (t + 32) * 128 + lane * 4 + j;
                nxt[j] = fetch(i, i < n);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int i = t * 128 + lane * 4 + j;
            v[j] = map(i, i < n, raw[j]);   // called by every lane (warp-uniform), -0 when !valid
        }
        float s = local_tree_sum<4>(v);
        s = warp_tree_sum(s);
        if (lane == 0) s_tiles[t] = s;
    }
    __syncthreads();
    for (int w = 1; w < ntiles; w <<= 1) {
        for (int i = threadIdx.x * 2 * w; i < ntiles; i += blockDim.x * 2 * w)
            s_tiles[i] = __fadd_rn(s_tiles[i], s_tiles[i + w]);
        __syncthreads();
    }
    const float r = s_tiles[0];
    __syncthreads();
    return r;
}

// ------------------------------------------------------------------ RMSNorm
// E contiguous bf16 <-> f32 per thread, 16-byte vectors when E % 8 == 0 (a warp then touches whole
// sectors instead of one 2-byte element per sector per instruction)
template <int E>
__device__ __forceinline__ void load_bf16_row(const __nv_bfloat16* __restrict__ src, float (&v)[E]) {
    if constexpr (E % 8 == 0) {
#pragma unroll
        for (int j = 0; j < E; j += 8) {
            const uint4 w = *reinterpret_cast<const uint4*>(src + j);
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[j + 2 * k] = __uint_as_float(ws[k] << 16);
                v[j + 2 * k + 1] = __uint_as_float(ws[k] & 0xffff0000u);
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = bf2f(src[j]);
    }
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    return static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(a))) |
           (static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(b))) << 16);
}

// y_i = bf16((x_i * rstd) * gamma_i), rstd = 1 / sqrt(tree(x*x)/d + eps)
template <int E>
__global__ void __launch_bounds__(256) rmsnorm_kernel(const float* __restrict__ x_in, float* __restrict__ x_out,
                                                      const __nv_bfloat16* __restrict__ embed,
                                                      const int* __restrict__ col_token,
                                                      const __nv_bfloat16* __restrict__ gamma,
                                                      __nv_bfloat16* __restrict__ out, const int* __restrict__ col_index,
                                                      const int* __restrict__ out_index, int d, float eps,
                                                      float* __restrict__ ss_out) {
    __shared__ float scratch[32];
    pdl_wait();
    pdl_trigger();
    const int col = blockIdx.x;
    const int base = threadIdx.x * E;
    float v[E];
    if (embed != nullptr) {
        const int tok = col_token[col];
        load_bf16_row<E>(embed + static_cast<int64_t>(tok) * d + base, v);
        float* dst = x_out + static_cast<int64_t>(col) * d + base;
        if constexpr (E % 4 == 0) {
#pragma unroll
            for (int j = 0; j < E; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < E; ++j) dst[j] = v[j];
        }
        if (ss_out != nullptr) {
            // per-128-element partial sums of squares of the new residual row (fused-norm decode):
            // warp w reduces tiles w, w+8, ... with 4 contiguous elements per lane + the butterfly
            __syncthreads();
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            const float* xr = x_out + static_cast<int64_t>(col) * d;
            for (int t = warp; t < d / 128; t += 8) {
                const float4 f = *reinterpret_cast<const float4*>(xr + t * 128 + lane * 4);
                float q[4] = {__fmul_rn(f.x, f.x), __fmul_rn(f.y, f.y), __fmul_rn(f.z, f.z), __fmul_rn(f.w, f.w)};
                const float tsum = warp_tree_sum(local_tree_sum<4>(q));
                if (lane == 0) ss_out[static_cast<int64_t>(col) * (d / 128) + t] = tsum;
            }
        }
    } else {
        const int row = col_index != nullptr ? col_index[col] : col;
        const float* src = x_in + static_cast<int64_t>(row) * d + base;
        if constexpr (E % 4 == 0) {
#pragma unroll
            for (int j = 0; j < E; j += 4) {
                const float4 f = *reinterpret_cast<const float4*>(src + j);
                v[j] = f.x;
                v[j + 1] = f.y;
                v[j + 2] = f.z;
                v[j + 3] = f.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = src[j];
        }
    }
    float sq[E];
#pragma unroll
    for (int j = 0; j < E; ++j) sq[j] = __fmul_rn(v[j], v[j]);
    float s = local_tree_sum<E>(sq);
    s = warp_tree_sum(s);
    s = block_tree_combine<8>(s, scratch);
    const float ms = __fdiv_rn(s, static_cast<float>(d));
    const float rstd = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, eps)));
    const int orow = out_index != nullptr ? out_index[col] : col;
    __nv_bfloat16* o = out + static_cast<int64_t>(orow) * d + base;
    float g[E];
    load_bf16_row<E>(gamma + base, g);
    if constexpr (E % 8 == 0) {
#pragma unroll
        for (int j = 0; j < E; j += 8) {
            uint4 w;
            w.x = pack_bf16x2(__fmul_rn(__fmul_rn(v[j], rstd), g[j]), __fmul_rn(__fmul_rn(v[j + 1], rstd), g[j + 1]));
            w.y = pack_bf16x2(__fmul_rn(__fmul_rn(v[j + 2], rstd), g[j + 2]), __fmul_rn(__fmul_rn(v[j + 3], rstd), g[j + 3]));
            w.z = pack_bf16x2(__fmul_rn(__fmul_rn(v[j + 4], rstd), g[j + 4]), __fmul_rn(__fmul_rn(v[j + 5], rstd), g[j + 5]));
            w.w = pack_bf16x2(__fmul_rn(__fmul_rn(v[j + 6], rstd), g[j + 6]), __fmul_rn(__fmul_rn(v[j + 7], rstd), g[j + 7]));
            *reinterpret_cast<uint4*>(o + j) = w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < E; ++j) o[j] = f2bf(__fmul_rn(__fmul_rn(v[j], rstd), g[j]));
    }
}

// ------------------------------------------------------------------ misc test kernels
// Both exp variants; a disagreement between them is reported as the NaN payload 0x7fc00bad.
__global__ void expf_kernel(const float* x, float* y, int64_t n) {
    const ExpTab tab = exp_tab_lane();
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        const float xv = i < n ? x[i] : 0.0f;
        const float a = det_expf_shfl(xv, tab);   // warp-uniform loop: every lane calls
        if (i < n) {
            const float b = det_expf(xv);
            y[i] = __float_as_uint(a) == __float_as_uint(b) ? a : __uint_as_float(0x7fc00badu);
        }
    }
}

__global__ void __launch_bounds__(1024) tree_sum_kernel(const float* x, float* out, int n) {
    __shared__ float tiles[1024];
    const float* row = x + static_cast<int64_t>(blockIdx.x) * n;
    const float s = block_tree_sum_1024(n, [&](int i, bool ok) { return ok ? row[i] : kNegZero; }, tiles);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ------------------------------------------------------------------ weights
// Logical element (r, c) of a tensor seeded with `seed`: z = splitmix64 output r*cols+c+1;
// u = (z >> 40) * 2^-23 - 1 in [-1, 1) (prng.hpp:68-70 next_symmetric_f32); value u * 2^scale_exp
// (exact) or, for norm gains, fma(u, 1/8, 1); stored as bf16 (RNE) at physical row r*row_mul+row_add.
__global__ void init_kernel(__nv_bfloat16* dst, uint64_t seed, int64_t rows, int64_t cols, float scale,
                            int is_gamma, int row_mul, int row_add, int tiled) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t z = splitmix64_at(seed, static_cast<uint64_t>(i) + 1);
        const float u = __fsub_rn(__fmul_rn(static_cast<float>(z >> 40), 0x1.0p-23f), 1.0f);
        const float v = is_gamma ? __fmaf_rn(u, 0.125f, 1.0f) : __fmul_rn(u, scale);
        const int64_t r = i / cols, c = i % cols;
        const int64_t pr = r * row_mul + row_add;
        const int64_t o = tiled ? (((pr >> 7) * (cols >> 6) + (c >> 6)) * 128 + (pr & 127)) * 64 + (c & 63)
                                : pr * cols + c;
        dst[o] = f2bf(v);
    }
}


// ------------------------------------------------------------------ softmax + decode
// reference: det_softmax (detcore.cpp:187-198), decode_with_draw / decode_step (detcore.cpp:202-262)
__device__ __forceinline__ uint64_t prob_key(float p, int idx) {
    return (static_cast<uint64_t>(__float_as_uint(p)) << 32) | static_cast<uint32_t>(0xFFFFFFFFu - idx);
}
__device__ __forceinline__ float key_prob(uint64_t k) { return __uint_as_float(static_cast<uint32_t>(k >> 32)); }
__device__ __forceinline__ int key_idx(uint64_t k) { return static_cast<int>(0xFFFFFFFFu - static_cast<uint32_t>(k)); }

struct SampleSmem {
    float tiles[1024];
    uint64_t sort[1024];
    unsigned int hist[256];
    float red_f[32];
    int red_i[32];
    unsigned int count;
    int flag;
    float fval;
    uint64_t kval;
};

// The row's tail (detcore.cpp:202-262): p_i = e_i / S, argmax, top-k / nucleus selection, one
// token, bookkeeping. P holds e_i on entry. Called by one 1024-thread CTA per row.
// p_i = e_i / S over [i_begin, i_end) in place, and the CTA's argmax with the smallest-index
// tie-break (detcore.cpp:202-208); the result is valid in thread 0 (and warp 0).
__device__ __forceinline__ void sample_divide_argmax(SampleSmem& sm, float* P, float S, int i_begin, int i_end,
                                                     int tid, int warp, int lane, float& bp, int& bi) {
    bp = -1.0f;
    bi = 0x7fffffff;
    for (int i0 = i_begin + tid; i0 < i_end; i0 += 8 * 1024) {   // 8 loads in flight before the stores
        float e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) e[u] = i0 + u * 1024 < i_end ? P[i0 + u * 1024] : 0.0f;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * 1024;   // increasing per thread: the first maximum is kept
            if (i < i_end) {
                const float p = __fdiv_rn(e[u], S);
                P[i] = p;
                if (p > bp) {
                    bp = p;
                    bi = i;
                }
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float op = __shfl_xor_sync(0xffffffffu, bp, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (op > bp || (op == bp && oi < bi)) {
            bp = op;
            bi = oi;
        }
    }
    __syncthreads();
    if (lane == 0) {
        sm.red_f[warp] = bp;
        sm.red_i[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
        bp = sm.red_f[lane];
        bi = sm.red_i[lane];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float op = __shfl_xor_sync(0xffffffffu, bp, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (op > bp || (op == bp && oi < bi)) {
                bp = op;
                bi = oi;
            }
        }
    }
}

// The row's tail (detcore.cpp:202-262) once P holds the probabilities and thread 0 the argmax:
// top-k / nucleus selection, one token, bookkeeping. One 1024-thread CTA per row.
__device__ __forceinline__ void sample_tail(const SampleParams& sp, SampleSmem& sm, int r, int slot, int step,
                                            const DevPolicy& pol, int V, float* P, uint64_t* sorted, int argmax,
                                            float rdraw, int tid, int warp, int lane) {
    (void)warp;
    (void)lane;
    int token = argmax;   // valid in thread 0
    int32_t err = DETGPU_OK;

    if (pol.kind != DETGPU_GREEDY) {
        __syncthreads();
        // Candidates in (probability desc, index asc) order, produced 1024 at a time: radix-select
        // the 1024-th largest key below `upper`, gather, bitonic sort. Thread 0 runs the reference's
        // sequential cumulative rules over the sorted prefix.
        uint64_t upper = ~0ull;
        int consumed = 0;
        int kept = 0;          // length of the kept prefix once decided
        bool decided = false;
        const int target_k = pol.kind == DETGPU_TOP_K ? static_cast<int>(pol.k < static_cast<uint32_t>(V) ? pol.k : static_cast<uint32_t>(V)) : V;
        float cum = 0.0f;      // nucleus running sum (thread 0)
        while (!decided) {
            const int remaining = V - consumed;
            const int take = min(1024, remaining);
            uint64_t kappa = 0;
            if (remaining > 1024) {
                uint64_t prefix = 0, mask = 0;
                unsigned int want = 1024;
                for (int shift = 56; shift >= 0; shift -= 8) {
                    if (tid < 256) sm.hist[tid] = 0;
                    __syncthreads();
                    for (int i = tid; i < V; i += 1024) {
                        const uint64_t k = prob_key(P[i], i);
                        if (k < upper && (k & mask) == prefix) atomicAdd(&sm.hist[(k >> shift) & 255], 1u);
                    }
                    __syncthreads();
                    if (tid == 0) {
                        unsigned int acc = 0;
                        int b = 255;
                        for (; b > 0; --b) {
                            if (acc + sm.hist[b] >= want) break;
                            acc += sm.hist[b];
                        }
                        sm.kval = static_cast<uint64_t>(b);
                        sm.count = want - acc;
                        sm.flag = sm.hist[b] == want - acc;   // the whole bin is taken: lower bits free
                    }
                    __syncthreads();
                    prefix |= sm.kval << shift;
                    mask |= 255ull << shift;
                    want = sm.count;
                    const bool whole_bin = sm.flag != 0;
                    __syncthreads();
                    if (whole_bin) break;   // every key with this prefix is >= kappa = prefix
                }
                kappa = prefix;
            }
            // gather keys in [kappa, upper)
            if (tid == 0) sm.count = 0;
            sm.sort[tid] = 0;
            __syncthreads();
            for (int i = tid; i < V; i += 1024) {
                const uint64_t k = prob_key(P[i], i);
                if (k < upper && k >= kappa) sm.sort[atomicAdd(&sm.count, 1u)] = k;
            }
            __syncthreads();
            // bitonic sort, descending
            for (int kk = 2; kk <= 1024; kk <<= 1) {
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const int ixj = tid ^ j;
                    if (ixj > tid) {
                        const uint64_t x = sm.sort[tid], y = sm.sort[ixj];
                        const bool desc = (tid & kk) == 0;
                        if (desc ? (x < y) : (x > y)) {
                            sm.sort[tid] = y;
                            sm.sort[ixj] = x;
                        }
                    }
                    __syncthreads();
                }
            }
            if (tid < take) sorted[consumed + tid] = sm.sort[tid];   // all threads: one store each
            if (tid == 0) {
                int dec = 0;
                for (int j = 0; j < take; ++j) {
                    const uint64_t k = sm.sort[j];
                    if (dec) break;
                    if (pol.kind == DETGPU_TOP_K) {
                        if (consumed + j + 1 >= target_k) {
                            kept = target_k;
                            dec = 1;
                        }
                    } else {
                        cum = __fadd_rn(cum, key_prob(k));
                        if (cum >= pol.p) {
                            kept = consumed + j + 1;
                            dec = 1;
                        }
                    }
                }
                if (!dec && consumed + take >= V) {
                    kept = V;
                    dec = 1;
                }
                sm.flag = dec;
                sm.count = kept;
                sm.kval = sm.sort[take - 1];
            }
            __syncthreads();
            decided = sm.flag != 0;
            kept = static_cast<int>(sm.count);
            upper = sm.kval;
            consumed += take;
            __syncthreads();
        }
        // renormalise with the canonical tree over the kept prefix, in sorted order. A prefix
        // decided in the first round (consumed == 1024 or V) is still in shared memory.
        const bool in_smem = consumed <= 1024;
        auto kept_key = [&](int i) { return in_smem ? sm.sort[i] : sorted[i]; };
        const float mass = block_tree_sum_1024(kept, [&](int i, bool ok) { return ok ? key_prob(kept_key(i)) : kNegZero; },
                                               sm.tiles);
        if (in_smem && mass > 0.0f) {   // the quotients p_i / mass in parallel (same divisions)
            __syncthreads();            // sm.tiles is free again
            if (tid < kept) sm.tiles[tid] = __fdiv_rn(key_prob(sm.sort[tid]), mass);
            __syncthreads();
        }
        if (tid == 0) {
            if (!(mass > 0.0f)) {
                err = DETGPU_EINVAL;
                token = 0;
            } else {
                float c2 = 0.0f;
                token = key_idx(kept_key(kept - 1));   // rounding left cum slightly below r
                for (int i = 0; i < kept; ++i) {
                    c2 = __fadd_rn(c2, in_smem ? sm.tiles[i] : __fdiv_rn(key_prob(sorted[i]), mass));
                    if (c2 >= rdraw) {
                        token = key_idx(kept_key(i));
                        break;
                    }
                }
            }
        }
    }

    if (tid == 0) {
        const int sr = sp.state_by_slot ? slot : r;   // where the decode state of this row lives
        sp.token_out[sr] = static_cast<uint32_t>(token);
        if (err != DETGPU_OK) sp.status[slot] = err;
        if (sp.tokens_hist != nullptr) sp.tokens_hist[static_cast<int64_t>(slot) * sp.tcap + step] = token;
        if (sp.col_step_mut != nullptr) {
            if (err != DETGPU_OK || step + 1 >= pol.max_tokens) {
                sp.col_step_mut[sr] = -1;
                sp.col_pos[sr] = -1;
            } else {
                sp.col_step_mut[sr] = step + 1;
                sp.col_pos[sr] = sp.col_pos[sr] + 1;
            }
        }
    }
}

__device__ __forceinline__ float sample_draw(const SampleParams& sp, int slot) {   // one xoshiro step per token
    uint64_t* st = sp.prng + static_cast<int64_t>(slot) * 4;
    uint64_t s[4] = {st[0], st[1], st[2], st[3]};
    const uint64_t u = xoshiro_next(s);
    st[0] = s[0];
    st[1] = s[1];
    st[2] = s[2];
    st[3] = s[3];
    return __fmul_rn(static_cast<float>(u >> 40), 0x1.0p-24f);
}

__device__ __forceinline__ void sample_fail_nonfinite(const SampleParams& sp, int r, int slot) {
    sp.status[slot] = DETGPU_ENONFINITE;
    const int sr = sp.state_by_slot ? slot : r;
    sp.token_out[sr] = 0;
    if (sp.col_step_mut != nullptr) {
        sp.col_step_mut[sr] = -1;
        sp.col_pos[sr] = -1;
    }
}

__global__ void __launch_bounds__(1024) sample_kernel(const SampleParams sp) {
    __shared__ SampleSmem sm;
    const ExpTab tab = exp_tab_lane();   // before the dependency wait: off the critical path
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int slot = r, step = 0;
    if (sp.col_step != nullptr) {
        step = sp.col_step[r];
        if (step < 0) return;
        slot = sp.col_slot[r];
    }
    const DevPolicy pol = sp.policy[slot];
    const int V = sp.vocab;
    const float* L = sp.col_step != nullptr
                         ? sp.logits + static_cast<int64_t>(slot) * sp.slot_stride + static_cast<int64_t>(step) * V
                         : sp.logits + static_cast<int64_t>(r) * sp.logit_row_stride;
    float* P = sp.probs + static_cast<int64_t>(r) * V;
    uint64_t* sorted = sp.scratch + static_cast<int64_t>(r) * V;

    // pass 1: max (left scan order is irrelevant for max) + finiteness (detcore.cpp:127-133)
    float m = -FLT_MAX;
    int bad = 0;
    for (int i = tid; i < V; i += 1024) {
        const float v = L[i];
        if (!isfinite(v)) bad = 1;
        m = fmaxf(m, v);
    }
    m = warp_max(m);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        sm.red_f[warp] = m;
        sm.red_i[warp] = bad;
    }
    if (tid == 0) sm.flag = 0;
    __syncthreads();
    if (warp == 0) {
        float mm = sm.red_f[lane];
        int bb = sm.red_i[lane];
        mm = warp_max(mm);
        bb = __any_sync(0xffffffffu, bb);
        if (lane == 0) {
            sm.fval = mm;
            sm.flag = bb;
        }
    }
    __syncthreads();
    const float maxv = sm.fval;
    // one generator step per token, drawn before the policy branch (detcore.cpp:256-262)
    const float rdraw = tid == 0 ? sample_draw(sp, slot) : 0.0f;
    if (sm.flag) {
        if (tid == 0) sample_fail_nonfinite(sp, r, slot);
        return;
    }

    // pass 2: e_i = exp(l_i - max); S = canonical tree of e
    const float S = block_tree_sum_1024_fm(
        V, [&](int i, bool ok) { return ok ? L[i] : 0.0f; },
        [&](int i, bool ok, float l) {
            const float e = det_expf_shfl(ok ? __fsub_rn(l, maxv) : 0.0f, tab);
            if (!ok) return kNegZero;
            P[i] = e;
            return e;
        },
        sm.tiles);
    float bp;
    int bi;
    sample_divide_argmax(sm, P, S, 0, V, tid, warp, lane, bp, bi);
    sample_tail(sp, sm, r, slot, step, pol, V, P, sorted, bi, rdraw, tid, warp, lane);
}

// Small batches: the row is split over nblk CTAs of kSampleBlock logits (aligned subtrees of the
// canonical tree over next_pow2(V)). sample_max_kernel leaves each block's max and finiteness;
// sample_multi_kernel computes e_i and the block's subtree sum, the last block of the row (a
// ticket) folds the subtree sums with the same tree into S; sample_div_kernel divides and takes
// block argmaxes, its last block reduces them and runs sample_tail. Bits equal the single-CTA
// kernel's; the exp and divide passes run on nblk SMs instead of one.
constexpr int kSampleBlock = 4096;

__global__ void __launch_bounds__(256) sample_max_kernel(const SampleParams sp) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x, r = blockIdx.y;
    int slot = r, step = 0;
    if (sp.col_step != nullptr) {
        step = sp.col_step[r];
        if (step < 0) return;
        slot = sp.col_slot[r];
    }
    const int V = sp.vocab;
    const float* L = sp.col_step != nullptr
                         ? sp.logits + static_cast<int64_t>(slot) * sp.slot_stride + static_cast<int64_t>(step) * V
                         : sp.logits + static_cast<int64_t>(r) * sp.logit_row_stride;
    float m = -FLT_MAX;
    int bad = 0;
    const int i1 = min(V, (b + 1) * kSampleBlock);
    for (int i = b * kSampleBlock + threadIdx.x; i < i1; i += 256) {
        const float v = L[i];
        if (!isfinite(v)) bad = 1;
        m = fmaxf(m, v);
    }
    __shared__ float rm[8];
    __shared__ int rb[8];
    m = warp_max(m);
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        rm[threadIdx.x >> 5] = m;
        rb[threadIdx.x >> 5] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) {
            m = fmaxf(m, rm[w]);
            bad |= rb[w];
        }
        float* ws = sp.blk_ws + (static_cast<int64_t>(r) * kSampleMaxBlocks + b) * 4;
        ws[0] = m;
        ws[1] = bad ? 1.0f : 0.0f;
    }
}

__global__ void __launch_bounds__(1024) sample_multi_kernel(const SampleParams sp) {
    __shared__ SampleSmem sm;
    __shared__ int s_last;
    const ExpTab tab = exp_tab_lane();   // before the dependency wait: off the critical path
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x, r = blockIdx.y, nblk = gridDim.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int slot = r, step = 0;
    if (sp.col_step != nullptr) {
        step = sp.col_step[r];
        if (step < 0) return;
        slot = sp.col_slot[r];
    }
    const DevPolicy pol = sp.policy[slot];
    const int V = sp.vocab;
    const float* L = sp.col_step != nullptr
                         ? sp.logits + static_cast<int64_t>(slot) * sp.slot_stride + static_cast<int64_t>(step) * V
                         : sp.logits + static_cast<int64_t>(r) * sp.logit_row_stride;
    float* P = sp.probs + static_cast<int64_t>(r) * V;
    float* ws = sp.blk_ws + static_cast<int64_t>(r) * kSampleMaxBlocks * 4;
    if (warp == 0) {   // lane j reads block j: one round trip (max is order-free)
        float mj = lane < nblk ? __ldcg(ws + 4 * lane) : -FLT_MAX;
        const int bj = __any_sync(0xffffffffu, lane < nblk && __ldcg(ws + 4 * lane + 1) != 0.0f);
        mj = warp_max(mj);
        if (lane == 0) {
            sm.fval = mj;
            sm.flag = bj;
        }
    }
    __syncthreads();
    const float m = sm.fval;
    const int bad = sm.flag;
    __syncthreads();
    if (bad) {   // block 0 reports, with the row's one generator step
        if (b == 0 && tid == 0) {
            sample_draw(sp, slot);
            sample_fail_nonfinite(sp, r, slot);
        }
        return;
    }

    const int i0 = b * kSampleBlock;
    const int nloc = max(0, min(kSampleBlock, V - i0));
    const float part = block_tree_sum_1024_fm(
        nloc, [&](int i, bool ok) { return ok ? L[i0 + i] : 0.0f; },
        [&](int i, bool ok, float l) {
            const float e = det_expf_shfl(ok ? __fsub_rn(l, m) : 0.0f, tab);
            if (!ok) return kNegZero;
            P[i0 + i] = e;
            return e;
        },
        sm.tiles);
    if (tid == 0) {
        ws[4 * b + 2] = part;
        __threadfence();
        const int prev = atomicAdd(sp.tickets + r, 1);
        s_last = prev == nblk - 1;
        if (s_last) sp.tickets[r] = 0;   // re-armed for the next launch
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // S: the subtree sums folded by the same perfect tree (absent subtrees are -0)
    const int nbp = max(128, next_pow2(V)) / min(max(128, next_pow2(V)), kSampleBlock);
    if (tid < 32) {
        float v = tid < nblk ? __ldcg(ws + 4 * tid + 2) : kNegZero;
        for (int off = 1; off < nbp; off <<= 1) {
            const float o = __shfl_xor_sync(0xffffffffu, v, off);
            v = __fadd_rn(v, o);
        }
        if (tid == 0) sm.fval = v;
    }
    if (tid == 0) ws[3] = sm.fval;   // S for sample_div_kernel
}

// p_i = e_i / S over the block, block argmax; the last block of the row reduces the block
// candidates (smallest index on ties, as the sequential scan) and runs sample_tail.
__global__ void __launch_bounds__(1024) sample_div_kernel(const SampleParams sp) {
    __shared__ SampleSmem sm;
    __shared__ int s_last;
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x, r = blockIdx.y, nblk = gridDim.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int slot = r, step = 0;
    if (sp.col_step != nullptr) {
        step = sp.col_step[r];
        if (step < 0) return;
        slot = sp.col_slot[r];
    }
    float* ws = sp.blk_ws + static_cast<int64_t>(r) * kSampleMaxBlocks * 4;
    if (warp == 0) {   // non-finite row: reported by sample_multi_kernel
        const int bj = __any_sync(0xffffffffu, lane < nblk && __ldcg(ws + 4 * lane + 1) != 0.0f);
        if (lane == 0) sm.flag = bj;
    }
    __syncthreads();
    if (sm.flag) return;
    const DevPolicy pol = sp.policy[slot];
    const int V = sp.vocab;
    float* P = sp.probs + static_cast<int64_t>(r) * V;
    const float S = __ldcg(ws + 3);
    float bp;
    int bi;
    sample_divide_argmax(sm, P, S, b * kSampleBlock, min(V, (b + 1) * kSampleBlock), tid, warp, lane, bp, bi);
    if (tid == 0) {
        ws[4 * b + 0] = bp;   // the block max slot is free again
        reinterpret_cast<int*>(ws)[4 * b + 2] = bi;
        __threadfence();
        const int prev = atomicAdd(sp.tickets + r, 1);
        s_last = prev == nblk - 1;
        if (s_last) sp.tickets[r] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp == 0) {
        bp = lane < nblk ? __ldcg(ws + 4 * lane) : -1.0f;
        bi = lane < nblk ? __ldcg(reinterpret_cast<const int*>(ws) + 4 * lane + 2) : 0x7fffffff;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float op = __shfl_xor_sync(0xffffffffu, bp, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (op > bp || (op == bp && oi < bi)) {
                bp = op;
                bi = oi;
            }
        }
    }
    __syncthreads();
    uint64_t* sorted = sp.scratch + static_cast<int64_t>(r) * V;
    const float rdraw = tid == 0 ? sample_draw(sp, slot) : 0.0f;
    sample_tail(sp, sm, r, slot, step, pol, V, P, sorted, bi, rdraw, tid, warp, lane);
}

cudaLaunchConfig_t make_cfg(dim3 grid, dim3 block, size_t smem, cudaStream_t stream, cudaLaunchAttribute* attr,
                            bool pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

}  // namespace

cudaError_t launch_rmsnorm(const float* x_in, float* x_out, const __nv_bfloat16* embed, const int* col_token,
                           const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* col_index, int ncols, int d,
                           float eps, cudaStream_t stream, bool pdl) {
    return launch_rmsnorm_ex(x_in, x_out, embed, col_token, gamma, out, col_index, nullptr, ncols, d, eps, stream, pdl);
}

cudaError_t launch_embed(const __nv_bfloat16* embed, const int* col_token, float* x_out, float* ss_out,
                         const __nv_bfloat16* gamma, __nv_bfloat16* h_out, int ncols, int d, float eps,
                         cudaStream_t stream, bool pdl) {
    return launch_rmsnorm_ex(nullptr, x_out, embed, col_token, gamma, h_out, nullptr, nullptr, ncols, d, eps, stream, pdl,
                             ss_out);
}

cudaError_t launch_rmsnorm_ex(const float* x_in, float* x_out, const __nv_bfloat16* embed, const int* col_token,
                              const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* in_index, const int* out_index,
                              int ncols, int d, float eps, cudaStream_t stream, bool pdl, float* ss_out) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = make_cfg(dim3(ncols), dim3(256), 0, stream, attr, pdl);
    const int* ii = in_index;
    const int* oi = out_index;
    switch (d) {
        case 256:
            return cudaLaunchKernelEx(&cfg, rmsnorm_kernel<1>, x_in, x_out, embed, col_token, gamma, out, ii, oi, d, eps, ss_out);
        case 512:
            return cudaLaunchKernelEx(&cfg, rmsnorm_kernel<2>, x_in, x_out, embed, col_token, gamma, out, ii, oi, d, eps, ss_out);
        case 1024:
            return cudaLaunchKernelEx(&cfg, rmsnorm_kernel<4>, x_in, x_out, embed, col_token, gamma, out, ii, oi, d, eps, ss_out);
        case 2048:
            return cudaLaunchKernelEx(&cfg, rmsnorm_kernel<8>, x_in, x_out, embed, col_token, gamma, out, ii, oi, d, eps, ss_out);
        case 4096:
            return cudaLaunchKernelEx(&cfg, rmsnorm_kernel<16>, x_in, x_out, embed, col_token, gamma, out, ii, oi, d, eps, ss_out);
        default:
            return cudaErrorInvalidValue;
    }
}

cudaError_t launch_rmsnorm_gather(const float* x, const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* in_index,
                                  const int* out_index, int n, int d, float eps, cudaStream_t stream, bool pdl) {
    return launch_rmsnorm_ex(x, nullptr, nullptr, nullptr, gamma, out, in_index, out_index, n, d, eps, stream, pdl);
}

cudaError_t launch_expf(const float* x, float* y, int64_t n, cudaStream_t stream) {
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 16));
    expf_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(x, y, n);
    return cudaGetLastError();
}

cudaError_t launch_tree_sum(const float* x, float* out, int rows, int n, cudaStream_t stream) {
    if (n > 131072 || rows <= 0) return cudaErrorInvalidValue;
    tree_sum_kernel<<<rows, 1024, 0, stream>>>(x, out, n);
    return cudaGetLastError();
}

cudaError_t launch_init_tensor(__nv_bfloat16* dst, uint64_t seed, int64_t rows, int64_t cols, int scale_exp,
                               int is_gamma, int row_mul, int row_add, cudaStream_t stream, bool tiled) {
    const float scale = ldexpf(1.0f, scale_exp);
    const int64_t n = rows * cols;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
    init_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(dst, seed, rows, cols, scale, is_gamma, row_mul, row_add,
                                                             tiled ? 1 : 0);
    return cudaGetLastError();
}

size_t sample_scratch_bytes(int rows, int vocab) { return sizeof(uint64_t) * static_cast<size_t>(rows) * vocab; }

cudaError_t launch_sample(const SampleParams& sp, cudaStream_t stream, bool pdl) {
    if (sp.vocab > 131072 || sp.vocab <= 0) return cudaErrorInvalidValue;
    const int nblk = (sp.vocab + kSampleBlock - 1) / kSampleBlock;
    if (sp.blk_ws != nullptr && sp.tickets != nullptr && nblk > 1 && sp.rows <= kSampleMultiMaxRows) {
        cudaLaunchAttribute a1[1], a2[1];
        cudaLaunchConfig_t c1 = make_cfg(dim3(nblk, sp.rows), dim3(256), 0, stream, a1, pdl);
        cudaError_t e = cudaLaunchKernelEx(&c1, sample_max_kernel, sp);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t c2 = make_cfg(dim3(nblk, sp.rows), dim3(1024), 0, stream, a2, pdl);
        e = cudaLaunchKernelEx(&c2, sample_multi_kernel, sp);
        if (e != cudaSuccess) return e;
        cudaLaunchAttribute a3[1];
        cudaLaunchConfig_t c3 = make_cfg(dim3(nblk, sp.rows), dim3(1024), 0, stream, a3, pdl);
        return cudaLaunchKernelEx(&c3, sample_div_kernel, sp);
    }
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = make_cfg(dim3(sp.rows), dim3(1024), 0, stream, attr, pdl);
    return cudaLaunchKernelEx(&cfg, sample_kernel, sp);
}

}  // namespace detgpu
