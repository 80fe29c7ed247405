// tcgen05 / TMEM / TMA GEMM with fused epilogues. See gemm.cuh for the contract.
//
// Warp roles (256 threads, one CTA per SM):
//   warp 0      TMA producer (one lane): weight tile 128x64 + up to 4 activation tiles 64x64 / stage
//   warp 1      MMA issuer (one lane): 4 x (K=16) tcgen05.mma per sub-tile per stage into TMEM
//   warp 2      TMEM allocator (256 columns = 4 sub-tiles x 64 f32 columns)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> fused epilogue -> global
// Reference counterpart: det_matvec (reference proj/src/detcore.cpp:165-185), one output element
// per weight row; here the reduction order over K is fixed by the k-block loop below and never
// split across CTAs.
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "gemm.cuh"
#include "detmath.cuh"
#include "ptx.cuh"

namespace detgpu {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int SUB_N = 64;
constexpr int A_BYTES = BM * BK * 2;        // 16 KB
constexpr int B_BYTES = SUB_N * BK * 2;     // 8 KB
constexpr int kMaxBc = 35;                  // k-blocks of a fused B buffer
constexpr int kRecvBytes = 4096;            // push combine: (S-1) peers x owned columns x 128 rows x f32

template <int NSUB>
struct Cfg {
    // <= 128 columns: ~100 KB of shared memory so that two CTAs fit per SM (the next GEMM's CTAs,
    // launched early by programmatic dependent launch, stream their weights while this one drains);
    // 256-column tiles keep a deep ring at one CTA per SM.
    static constexpr int STAGE_BYTES = A_BYTES + NSUB * B_BYTES;
    static constexpr int BUDGET = NSUB <= 2 ? 96 * 1024 : 192 * 1024;
    static constexpr int STAGES = BUDGET / STAGE_BYTES;
    // one-column-group decode: 10 KB more: 6 KB so the fused B buffer (the B ring + this) holds 35
    // k-blocks, then the 4 KB receive buffer of the pushed K-segment partials (kRecvBytes)
    static constexpr int BC_EXTRA = NSUB == 1 ? 10 * 1024 : 0;
    static constexpr int RECV_OFF = STAGES * NSUB * B_BYTES + 6 * 1024;   // from sB
    static constexpr int SMEM = STAGES * STAGE_BYTES + BC_EXTRA + 1024 /*align*/ + 640 /*barriers*/;
    static constexpr int MIN_CTAS = NSUB <= 2 ? 2 : 1;
    static constexpr uint32_t TMEM = NSUB * SUB_N;   // f32 accumulator columns (power of two)
};

__device__ __forceinline__ float epilogue_store(const GemmParams& p, int row, int col, float v) {
    switch (p.mode) {
        case kEpiStoreF32: {
            int64_t off;
            if (p.col_step != nullptr) {
                const int st = p.col_step[col];
                if (st < 0) return v;
                off = static_cast<int64_t>(p.col_slot[col]) * p.slot_stride + static_cast<int64_t>(st) * p.n_out;
            } else {
                off = static_cast<int64_t>(col) * p.ld_out;
            }
            p.out[off + row] = v;
            return v;
        }
        case kEpiAddF32: {
            float* dst = p.out + static_cast<int64_t>(col) * p.ld_out + row;
            const float r = __fadd_rn(*dst, v);
            *dst = r;
            return r;
        }
        default:
            return v;
    }
}

// RoPE on interleaved pairs (2i, 2i+1) of each head (the original Llama complex-pair convention):
//   x0' = x0*c - x1*s ; x1' = x0*s + x1*c   (each product rounded, no contraction)
__device__ __forceinline__ void epilogue_qkv(const GemmParams& p, int row, int col, float v, float partner) {
    const int pos = p.col_pos[col];
    if (pos < 0) return;
    const int qrows = p.hq * p.hd, krows = p.hkv * p.hd;
    const int d = row % p.hd;
    if (row < qrows + krows) {
        const int i = d >> 1;
        const float c = p.rope_cos[static_cast<int64_t>(pos) * (p.hd / 2) + i];
        const float s = p.rope_sin[static_cast<int64_t>(pos) * (p.hd / 2) + i];
        if ((d & 1) == 0) v = __fsub_rn(__fmul_rn(v, c), __fmul_rn(partner, s));
        else v = __fadd_rn(__fmul_rn(partner, s), __fmul_rn(v, c));
    }
    const __nv_bfloat16 b = f2bf(v);
    if (row < qrows) {
        p.q_out[static_cast<int64_t>(col) * qrows + row] = b;
        return;
    }
    const bool is_k = row < qrows + krows;
    const int kvh = (row - (is_k ? qrows : qrows + krows)) / p.hd;
    const int slot = p.col_req[col];
    const int page_id = p.block_table[static_cast<int64_t>(slot) * p.max_pages + pos / p.page];
    const int64_t off = ((static_cast<int64_t>(page_id) * p.hkv + kvh) * p.page + pos % p.page) * p.hd + d;
    (is_k ? p.kcache : p.vcache)[off] = b;
}

// The same epilogue with the row's and the column's parts computed once (many columns): a thread's
// row is fixed, and each column's position and KV-cache destination come from shared memory.
struct QkvRow {
    int d;           // dimension within the head
    bool rope;       // q or k row
    int dst;         // 0 q_out, 1 kcache, 2 vcache
    int64_t off;     // q: row; k/v: kvh * page * hd + d
};
__device__ __forceinline__ QkvRow qkv_row(const GemmParams& p, int row) {
    const int qrows = p.hq * p.hd, krows = p.hkv * p.hd;
    QkvRow r;
    r.d = row % p.hd;
    r.rope = row < qrows + krows;
    r.dst = row < qrows ? 0 : r.rope ? 1 : 2;
    const int kvh = r.dst == 0 ? 0 : (row - (r.dst == 1 ? qrows : qrows + krows)) / p.hd;
    r.off = r.dst == 0 ? row : static_cast<int64_t>(kvh) * p.page * p.hd + r.d;
    return r;
}
// kvbase = ((page_id * hkv) * page + pos % page) * hd for the column's position
__device__ __forceinline__ void epilogue_qkv_col(const GemmParams& p, const QkvRow& r, int col, int pos,
                                                 int64_t kvbase, float v, float partner) {
    if (pos < 0) return;
    if (r.rope) {
        const int64_t i = static_cast<int64_t>(pos) * (p.hd / 2) + (r.d >> 1);
        const float c = p.rope_cos[i], s = p.rope_sin[i];
        if ((r.d & 1) == 0) v = __fsub_rn(__fmul_rn(v, c), __fmul_rn(partner, s));
        else v = __fadd_rn(__fmul_rn(partner, s), __fmul_rn(v, c));
    }
    const __nv_bfloat16 b = f2bf(v);
    if (r.dst == 0) p.q_out[static_cast<int64_t>(col) * (p.hq * p.hd) + r.off] = b;
    else (r.dst == 1 ? p.kcache : p.vcache)[kvbase + r.off] = b;
}

// silu(g) * u with g = gate row 2j, u = up row 2j+1; silu(g) = g / (1 + exp(-g)).
__device__ __forceinline__ void epilogue_swiglu(const GemmParams& p, int row, int col, float v, float partner,
                                                float e /* det_expf(-v) */) {
    if ((row & 1) != 0) return;
    const float sg = __fdiv_rn(v, __fadd_rn(1.0f, e));
    p.act[static_cast<int64_t>(col) * (p.n_out / 2) + (row >> 1)] = f2bf(__fmul_rn(sg, partner));
}

// SwiGLU of two adjacent columns at once: the even lane (gate row) finishes column c, the odd lane
// (up row) column c + 1, so every lane evaluates one exp / division instead of both lanes of a pair
// evaluating one. Same scalar arithmetic per output as epilogue_swiglu.
__device__ __forceinline__ void epilogue_swiglu_pair(const GemmParams& p, int row, int col, float v0, float v1,
                                                     ExpTab tab) {
    const bool odd = (row & 1) != 0;
    const float recv = __shfl_xor_sync(0xffffffffu, odd ? v0 : v1, 1);
    const float g = odd ? recv : v0, u = odd ? v1 : recv;
    const float e = det_expf_shfl(-g, tab);
    const float sg = __fdiv_rn(g, __fadd_rn(1.0f, e));
    p.act[static_cast<int64_t>(col + (odd ? 1 : 0)) * (p.n_out / 2) + (row >> 1)] = f2bf(__fmul_rn(sg, u));
}

__device__ __forceinline__ float epilogue_any(const GemmParams& p, int row, int col, float v, ExpTab tab) {
    if (p.mode == kEpiQkvRope || p.mode == kEpiSwiglu) {
        const float partner = __shfl_xor_sync(0xffffffffu, v, 1);   // callers keep `col` warp-uniform
        if (p.mode == kEpiQkvRope) epilogue_qkv(p, row, col, v, partner);
        else epilogue_swiglu(p, row, col, v, partner, det_expf_shfl(-v, tab));   // all lanes
        return v;
    }
    return epilogue_store(p, row, col, v);
}

// Decode: while the accumulator builds, the epilogue warps load what the epilogue of (row, col)
// will read (the residual for AddF32; RoPE factors and the destination for QKV; the trace slot for
// the lm_head), so the epilogue after the last MMA has no dependent global round trip.
struct EpiPre {
    float a, b;     // AddF32: residual x; QKV: cos, sin
    int64_t off;    // QKV / StoreF32: destination element offset (< 0: nothing to store)
    int where;      // QKV: 0 q_out, 1 kcache, 2 vcache
};

__device__ __forceinline__ EpiPre epilogue_preload(const GemmParams& p, int row, int col) {
    EpiPre e{0.0f, 0.0f, -1, 0};
    if (p.mode == kEpiAddF32) {
        e.a = p.out[static_cast<int64_t>(col) * p.ld_out + row];
    } else if (p.mode == kEpiQkvRope) {
        const int pos = p.col_pos[col];
        if (pos < 0) return e;
        const int qrows = p.hq * p.hd, krows = p.hkv * p.hd;
        const int d = row % p.hd;
        if (row < qrows + krows) {
            const int64_t i = static_cast<int64_t>(pos) * (p.hd / 2) + (d >> 1);
            e.a = p.rope_cos[i];
            e.b = p.rope_sin[i];
        }
        if (row < qrows) {
            e.off = static_cast<int64_t>(col) * qrows + row;
        } else {
            const bool is_k = row < qrows + krows;
            const int kvh = (row - (is_k ? qrows : qrows + krows)) / p.hd;
            const int page_id = p.block_table[static_cast<int64_t>(p.col_req[col]) * p.max_pages + pos / p.page];
            e.off = ((static_cast<int64_t>(page_id) * p.hkv + kvh) * p.page + pos % p.page) * p.hd + d;
            e.where = is_k ? 1 : 2;
        }
    } else if (p.mode == kEpiStoreF32) {
        if (p.col_step != nullptr) {
            const int st = p.col_step[col];
            e.off = st < 0 ? -1 : static_cast<int64_t>(p.col_slot[col]) * p.slot_stride + static_cast<int64_t>(st) * p.n_out + row;
        } else {
            e.off = static_cast<int64_t>(col) * p.ld_out + row;
        }
    }
    return e;
}

// epilogue_any with the preloaded operands (same arithmetic, bit for bit)
__device__ __forceinline__ float epilogue_pre(const GemmParams& p, int row, int col, float v, const EpiPre& e,
                                              ExpTab tab) {
    if (p.mode == kEpiAddF32) {
        const float r = __fadd_rn(e.a, v);
        p.out[static_cast<int64_t>(col) * p.ld_out + row] = r;
        return r;
    }
    if (p.mode == kEpiQkvRope) {
        const float partner = __shfl_xor_sync(0xffffffffu, v, 1);
        if (e.off < 0) return v;
        const int qrows = p.hq * p.hd, krows = p.hkv * p.hd;
        if (row < qrows + krows) {
            if ((row & 1) == 0) v = __fsub_rn(__fmul_rn(v, e.a), __fmul_rn(partner, e.b));
            else v = __fadd_rn(__fmul_rn(partner, e.b), __fmul_rn(v, e.a));
        }
        (e.where == 0 ? p.q_out : e.where == 1 ? p.kcache : p.vcache)[e.off] = f2bf(v);
        return v;
    }
    if (p.mode == kEpiStoreF32) {
        if (e.off >= 0) p.out[e.off] = v;
        return v;
    }
    return epilogue_any(p, row, col, v, tab);
}

__device__ __forceinline__ void epi_bar();

// Sum of squares of the updated residual over this tile's 128 rows for one column (perfect tree:
// lane butterfly over 32 consecutive rows, then the 4 warps), stored as the tile's partial of the
// next RMSNorm. All 128 epilogue threads call it with the same column.
__device__ __forceinline__ void tile_sumsq(const GemmParams& p, int tile, int col, float xnew, int ew, int lane,
                                           float* s_red) {
    float q = warp_tree_sum(__fmul_rn(xnew, xnew));
    if (lane == 0) s_red[ew] = q;
    epi_bar();
    if (ew == 0 && lane == 0)
        p.ss_out[static_cast<int64_t>(col) * p.ss_tiles + tile] =
            __fadd_rn(__fadd_rn(s_red[0], s_red[1]), __fadd_rn(s_red[2], s_red[3]));
    epi_bar();
}

// Perfect-tree sum of squares of a row of d = 32*E floats (lane owns E contiguous): float4 chunks
// merged with a binary counter, then the lane butterfly == the canonical tree over d.
template <int E>
__device__ __forceinline__ float warp_sumsq(const float* __restrict__ row, int lane) {
    constexpr int NC = E / 4;
    constexpr int DEPTH = (NC >= 32 ? 5 : NC >= 16 ? 4 : NC >= 8 ? 3 : NC >= 4 ? 2 : NC >= 2 ? 1 : 0) + 1;
    float stack[DEPTH];
    const float4* src = reinterpret_cast<const float4*>(row + lane * E);
#pragma unroll
    for (int g = 0; g < NC; ++g) {
        const float4 v = src[g];
        float q[4] = {__fmul_rn(v.x, v.x), __fmul_rn(v.y, v.y), __fmul_rn(v.z, v.z), __fmul_rn(v.w, v.w)};
        float carry = local_tree_sum<4>(q);
        int lvl = 0;
#pragma unroll
        for (int b = g; b & 1; b >>= 1, ++lvl) carry = __fadd_rn(stack[lvl], carry);
        stack[lvl] = carry;
    }
    return warp_tree_sum(stack[DEPTH - 1]);
}

__device__ __forceinline__ float norm_sumsq(const float* row, int d, int lane) {
    switch (d) {
        case 256: return warp_sumsq<8>(row, lane);
        case 512: return warp_sumsq<16>(row, lane);
        case 1024: return warp_sumsq<32>(row, lane);
        case 2048: return warp_sumsq<64>(row, lane);
        default: return warp_sumsq<128>(row, lane);   // 4096
    }
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Fused B operand (decode, <= 8 columns). The epilogue warps, idle until the accumulator is
// ready, build the B tiles of the CTA's whole K-segment once, straight into a compact shared
// buffer: k-block i occupies 1 KB at bc + i*1024 holding rows 0..7 in the 128B-swizzled K-major
// layout (16-byte chunk j of row r stored at chunk j ^ r). The MMA's 64-row descriptor at
// bc + i*1024 also covers rows 8..63, which are the following k-blocks' bytes: those are the
// padding columns of the N=64 instruction and are never stored (columns are independent).
// Values (bits identical to the unfused kernels):
//   norm: bf16((x * rstd) * gamma), rstd from the producer's per-tile sums of squares
//   attn: bf16(O / L) of the chunk partials combined in chunk order (attention.cu)
__device__ __forceinline__ void put_b(uint8_t* bc, int i, int c, int kq, float v0, float v1, float v2, float v3) {
    uint2 packed;
    packed.x = static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(v0))) |
               (static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(v1))) << 16);
    packed.y = static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(v2))) |
               (static_cast<uint32_t>(__bfloat16_as_ushort(f2bf(v3))) << 16);
    const int chunk = (kq >> 3) ^ (c & 7);
    *reinterpret_cast<uint2*>(bc + i * 1024 + c * 128 + chunk * 16 + (kq & 7) * 2) = packed;
}

// every producer thread: make its k-block writes visible to the tensor core, then arrive
__device__ __forceinline__ void release_b(uint64_t* bready, int i) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&bready[i]);
}

// Arrive on k-blocks [released, done) of the fused B buffer (every producer thread, same sequence).
__device__ __forceinline__ void release_b_range(uint64_t* bready, int& released, int done) {
    if (done <= released) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = released; i < done; ++i) mbar_arrive(&bready[i]);
    released = done;
}

// Items are (k-block, column, 4 consecutive k) in k-block-major order, 128 per round, so k-blocks
// are released to the MMA as soon as their last item is stored. x and gamma of the next round are
// in flight while the current one is converted; the sums of squares load with the first round.
__device__ void norm_b_setup(const GemmParams& p, uint8_t* bc, uint64_t* bready, int kb0, int nkb, int col0,
                             int ncols, int ew, int lane) {
    __shared__ float s_rstd[8];
    constexpr int R = 4;   // items per thread per round
    const int d = p.norm_d, ntiles = d / 128;
    const int t = ew * 32 + lane;
    const int per_kb = ncols * 16, total = nkb * per_kb;
    float part[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {   // the producer of x left one partial per 128-row tile
        const int cc = ew + 4 * j;
        part[j] = cc < ncols && lane < ntiles ? __ldcg(p.norm_ss + static_cast<int64_t>(col0 + cc) * ntiles + lane)
                                              : kNegZero;
    }
    float4 xn[R];
    uint2 gn[R];
    auto load = [&](int q0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = q0 + r * 128 + t;
            if (q < total) {
                const int i = q / per_kb, rem = q % per_kb, c = rem >> 4, kq = (rem & 15) * 4;
                const int k = (kb0 + i) * BK + kq;
                xn[r] = __ldcg(reinterpret_cast<const float4*>(p.norm_x + static_cast<int64_t>(col0 + c) * d + k));
                gn[r] = __ldg(reinterpret_cast<const uint2*>(p.norm_gamma + k));
            }
        }
    };
    load(0);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int cc = ew + 4 * j;
        const float ss = warp_tree_sum(part[j]);   // == the tree over d
        if (cc < ncols && lane == 0) {
            const float ms = __fdiv_rn(ss, static_cast<float>(d));
            s_rstd[cc] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(ms, p.norm_eps)));
        }
    }
    epi_bar();
    int released = 0;
    for (int q0 = 0; q0 < total; q0 += R * 128) {
        float4 xc[R];
        uint2 gc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            xc[r] = xn[r];
            gc[r] = gn[r];
        }
        if (q0 + R * 128 < total) load(q0 + R * 128);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = q0 + r * 128 + t;
            if (q < total) {
                const int i = q / per_kb, rem = q % per_kb, c = rem >> 4, kq = (rem & 15) * 4;
                const float rstd = s_rstd[c];
                put_b(bc, i, c, kq, __fmul_rn(__fmul_rn(xc[r].x, rstd), __uint_as_float(gc[r].x << 16)),
                      __fmul_rn(__fmul_rn(xc[r].y, rstd), __uint_as_float(gc[r].x & 0xffff0000u)),
                      __fmul_rn(__fmul_rn(xc[r].z, rstd), __uint_as_float(gc[r].y << 16)),
                      __fmul_rn(__fmul_rn(xc[r].w, rstd), __uint_as_float(gc[r].y & 0xffff0000u)));
            }
        }
        release_b_range(bready, released, q0 + R * 128 >= total ? nkb : (q0 + R * 128) / per_kb);
    }
}

// Grid (S, n_out/128, column groups), cluster (S,1,1): the S CTAs of a cluster own the same 128
// weight rows and columns and the fixed K-segments [s*nkb/S, (s+1)*nkb/S) of the reduction. Each
// runs its segment as one tcgen05 accumulation chain in TMEM; the S partial tiles are exchanged
// through distributed shared memory and combined per element with the reference tree over the S
// partials in segment order (detcore.cpp:135-150). S depends only on the GEMM shape.
// Cluster combine of the S_ K-segment partial tiles (> 8 columns) and the epilogue: CTA `seg`
// finalises column quads seg, seg + S_, ...; warp group wg takes every other round of QB_ quads.
// Per element the reference tree over the S_ partials in segment order (local_tree_sum<8>, -0
// padded: the padding adds are exact and compile away for a constant S_).
// The S_ partials of one column quad (v[s], segment order) -> the reference tree per element ->
// the fused epilogue of the quad's live columns.
template <int S_>
__device__ __forceinline__ void finish_quad(const GemmParams& p, const float4 (&v)[S_], int q, int nq, int ncols,
                                            int m0, int rl, int col0, const QkvRow& qr, const int* s_cpos,
                                            const int64_t* s_ckv, ExpTab tab) {
    float sum[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float t[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
            t[s] = s >= S_ ? kNegZero : e == 0 ? v[s].x : e == 1 ? v[s].y : e == 2 ? v[s].z : v[s].w;
        sum[e] = local_tree_sum<8>(t);
    }
    if (p.mode == kEpiAddF32) {   // residual add: the quad's four loads first
        float res[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            res[e] = q < nq && q * 4 + e < ncols ? p.out[static_cast<int64_t>(col0 + q * 4 + e) * p.ld_out + m0 + rl] : 0.0f;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (q < nq && q * 4 + e < ncols)
                p.out[static_cast<int64_t>(col0 + q * 4 + e) * p.ld_out + m0 + rl] = __fadd_rn(res[e], sum[e]);
        return;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int cl = q * 4 + e;
        if (q >= nq || cl >= ncols) continue;   // warp-uniform
        if (p.mode == kEpiStoreF32) {
            if (s_ckv[cl] >= 0) p.out[s_ckv[cl] + m0 + rl] = sum[e];
            continue;
        }
        if (p.mode == kEpiQkvRope) {
            const float partner = __shfl_xor_sync(0xffffffffu, sum[e], 1);
            epilogue_qkv_col(p, qr, col0 + cl, s_cpos[cl], s_ckv[cl], sum[e], partner);
            continue;
        }
        if (p.mode == kEpiSwiglu && (e & 1) == 0 && cl + 1 < ncols) {
            epilogue_swiglu_pair(p, m0 + rl, col0 + cl, sum[e], sum[e + 1], tab);
            ++e;   // both columns done
            continue;
        }
        epilogue_any(p, m0 + rl, col0 + cl, sum[e], tab);   // ss_out: <= 8 cols
    }
}

// Many-column combine (cluster form): CTA `seg` finalises column quads seg, seg + S_, ... reading
// every segment's partial tile over DSMEM; warp group wg takes every other round of QB_ quads.
// Per element the reference tree over the S_ partials in segment order (local_tree_sum<8>, -0
// padded: the padding adds are exact and compile away for a constant S_).
template <int S_, int QB_>
__device__ __forceinline__ void combine_quads(const GemmParams& p, uint32_t pbase, int seg, int wg, int nq, int ncols,
                                              int m0, int rl, int col0, const QkvRow& qr, const int* s_cpos,
                                              const int64_t* s_ckv, ExpTab tab, int rstride = 1, int roff = 0) {
    for (int q0 = seg + wg * QB_ * S_; q0 < nq; q0 += 2 * QB_ * S_) {
        float4 v[QB_][S_];
#pragma unroll
        for (int u = 0; u < QB_; ++u) {
            const int q = q0 + u * S_;
#pragma unroll
            for (int s = 0; s < S_; ++s)
                v[u][s] = q < nq ? ld_dsmem_f32x4(mapa_shared(pbase + 16u * static_cast<uint32_t>(q * BM + rl),
                                                              static_cast<uint32_t>(s * rstride + roff)))
                                 : make_float4(kNegZero, kNegZero, kNegZero, kNegZero);
        }
#pragma unroll
        for (int u = 0; u < QB_; ++u)
            finish_quad<S_>(p, v[u], q0 + u * S_, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab);
    }
}
// Persistent form: the partials were pushed into this CTA's receive buffer R
// [source segment][owned quad j][row] (quad q = seg + j * S_), so every read is local.
template <int S_>
__device__ __forceinline__ void combine_local(const GemmParams& p, const float4* R, int qmax, int seg, int nq, int ncols,
                                              int m0, int rl, int col0, const QkvRow& qr, const int* s_cpos,
                                              const int64_t* s_ckv, ExpTab tab) {
    for (int j = 0, q = seg; q < nq; ++j, q += S_) {
        float4 v[S_];
#pragma unroll
        for (int s = 0; s < S_; ++s) v[s] = R[(s * qmax + j) * BM + rl];
        finish_quad<S_>(p, v, q, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab);
    }
}

template <int NSUB>
__global__ void __launch_bounds__(256, Cfg<NSUB>::MIN_CTAS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmParams p) {
    using C = Cfg<NSUB>;
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (128B-swizzled tiles); offset arithmetic on the shared array keeps every
    // access to it an LDS/STS (a pointer rebuilt from an integer would be generic)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * NSUB * B_BYTES + C::BC_EXTRA);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* bready = tfull + 1;        // [kMaxBc] fused B: k-block i ready (128 producer arrivals)
    uint64_t* recv_bar = bready + kMaxBc;   // push combine: peers' partials landed
    uint32_t* tslot = reinterpret_cast<uint32_t*>(recv_bar + 1);

    __shared__ float s_red[4];
    __shared__ int s_cpos[NSUB * SUB_N];        // QKV, many columns: each column's position ...
    __shared__ int64_t s_ckv[NSUB * SUB_N];     // ... and KV-cache row base (epilogue_qkv_col); f32
                                                // store: the column's output base (-1: inactive)
    __shared__ uint64_t s_tm[kTraceMarks];   // timeline marks (p.trace only)
    const bool tracing = p.trace != nullptr;
    if (tracing && threadIdx.x < kTraceMarks) s_tm[threadIdx.x] = threadIdx.x == 0 ? globaltimer_ns() : 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.ksplit;
    const int seg = blockIdx.x;                 // == %cluster_ctarank
    // grid (S, column groups, tiles): the column groups of one weight tile run back to back, so
    // the tile's weights are read from HBM once and from L2 by the other groups
    const int tile = blockIdx.z, cgrp = blockIdx.y, ntiles = gridDim.z;
    const int m0 = tile * BM;
    const int col0 = cgrp * (NSUB * SUB_N);
    const int ncols = min(NSUB * SUB_N, p.ncols - col0);
    const int nb = (ncols + SUB_N - 1) / SUB_N;
    const int nkb_all = p.k / BK;
    const int kb0 = seg * nkb_all / S, kb1 = (seg + 1) * nkb_all / S;
    const int nkb = kb1 - kb0;
    // Fused RMSNorm (decode, <= 8 columns): the B operand is produced in shared memory by the
    // epilogue warps from the f32 residual stream instead of being loaded by TMA from a separately
    // normalised bf16 copy; bits are identical to rmsnorm_kernel + TMA.
    const bool fused = p.norm_x != nullptr;
    uint8_t* bc = sB;   // fused B buffer: 1 KB per k-block (see norm_b_setup)
    // Decode (<= 8 columns): column cl is finalised by CTA cl % S; every other segment pushes its
    // partial of that column straight into the owner's receive buffer (st.async + mbarrier), so the
    // owner never waits on a remote read and nobody waits for the owner.
    const int recv_cols = (ncols + S - 1) / S;   // owned columns per CTA, at most
    const bool push = NSUB == 1 && S > 1 && ncols <= 8 && (S - 1) * recv_cols * BM * 4 <= kRecvBytes;
    float* recv = reinterpret_cast<float*>(sB + C::RECV_OFF);   // [peer slot][owned column][row]
    const int owned = seg < ncols ? (ncols - 1 - seg) / S + 1 : 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        for (int i = 0; i < kMaxBc; ++i) mbar_init(&bready[i], 128);
        mbar_init(recv_bar, 1);
        if (push && owned > 0) mbar_arrive_expect_tx(recv_bar, static_cast<uint32_t>((S - 1) * owned * BM * 4));
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tslot, C::TMEM);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (push) cluster_arrive();   // receive barriers initialised (waited on before the first push)
    const uint32_t tbase = *tslot;

    // Weight tile (128 rows x 64 k) through a 3D tensor map: pre-tiled weights are one contiguous
    // 16 KB block per (tile, k-block) -> coordinate (0, 0, tile*nkb + kb); a plain row-major matrix
    // is viewed as [rows][K/64][64] -> coordinate (0, kb, m0). Same smem image either way.
    auto load_w = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int kb) {
        if (p.w_tiled) tma_load_3d(dst, m, bar, 0, 0, tile * nkb_all + kb, kEvictFirst);
        else tma_load_3d(dst, m, bar, 0, kb, m0, kEvictFirst);
    };
    const uint32_t stage_tx = fused ? A_BYTES : A_BYTES + nb * B_BYTES;
    const int pre = min(STAGES, nkb);
    if (warp == 0 && lane == 0) {
        // Weight tiles do not depend on the previous kernel: stream them before the PDL wait.
        for (int i = 0; i < pre; ++i) {
            mbar_arrive_expect_tx(&full[i], stage_tx);
            load_w(sA + i * A_BYTES, &tmW, &full[i], kb0 + i);
        }
    }
    if (warp == 3 && lane == 0) {
        l2_prefetch_slice(p.l2pf, p.l2pf_bytes, blockIdx.x + S * (tile + ntiles * cgrp), S * gridDim.y * gridDim.z);
        // the segment is contiguous in the tiled layout: k-blocks [pre, pre + self_pf_kb) in one request
        const int npf = min(nkb - pre, p.self_pf_kb);
        if (p.w_tiled && p.w_raw != nullptr && npf > 0)
            l2_prefetch_bulk(static_cast<const uint8_t*>(p.w_raw) +
                                 (static_cast<int64_t>(tile) * nkb_all + kb0 + pre) * A_BYTES,
                             static_cast<uint32_t>(npf) * A_BYTES);
    }
    if (fused && warp >= 4)   // RMSNorm gamma of this K-segment (a weight): warm L2 before the wait
        for (int i = threadIdx.x - 128; i < nkb; i += 128) prefetch_l2(p.norm_gamma + (kb0 + i) * BK);
    // Every kernel waits for its predecessor before triggering its dependents, so when a kernel
    // starts, all kernels before its predecessor have completed (attention relies on this).
    pdl_wait();
    pdl_trigger();
    if (tracing && threadIdx.x == 0) s_tm[1] = globaltimer_ns();
    if (warp == 0) {
        if (lane == 0) {
            if (!fused)
                for (int i = 0; i < pre; ++i)
                    for (int j = 0; j < nb; ++j)
                        tma_load_2d(sB + (i * NSUB + j) * B_BYTES, &tmX, &full[i], (kb0 + i) * BK, col0 + j * SUB_N,
                                    kEvictLast);
            int s = pre % STAGES, ph = (pre / STAGES) & 1;   // ring slot and phase, advanced incrementally
            for (int i = pre; i < nkb; ++i) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], stage_tx);
                load_w(sA + s * A_BYTES, &tmW, &full[s], kb0 + i);
                if (!fused)
                    for (int j = 0; j < nb; ++j)
                        tma_load_2d(sB + (s * NSUB + j) * B_BYTES, &tmX, &full[s], (kb0 + i) * BK,
                                    col0 + j * SUB_N, kEvictLast);
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, SUB_N);
            const bool wide = p.mma_wide && !fused && nb > 1;
            const uint32_t idesc_wide = umma_idesc_bf16(BM, nb * SUB_N);
            int s = 0, ph = 0;
            for (int i = 0; i < nkb; ++i) {
                if (fused) mbar_wait(&bready[i], 0);
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = fused ? smem_u32(bc + i * 1024) : smem_u32(sB + s * NSUB * B_BYTES);
                if (wide) {
                    // all live sub-tiles as one N = nb*64 instruction (A read once from smem)
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc_mma_bf16(tbase, umma_desc_k128(a_base + k * 32), umma_desc_k128(b_base + k * 32), idesc_wide,
                                    (i | k) != 0 ? 1u : 0u);
                } else {
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t adesc = umma_desc_k128(a_base + k * 32);
                        for (int j = 0; j < nb; ++j) {
                            const uint64_t bdesc = umma_desc_k128(b_base + j * B_BYTES + k * 32);
                            tc_mma_bf16(tbase + j * SUB_N, adesc, bdesc, idesc, (i | k) != 0 ? 1u : 0u);
                        }
                    }
                }
                tc_commit(&empty[s]);   // frees the smem stage once these MMAs retire
                if (++s == STAGES) {
                    s = 0;
                    ph ^= 1;
                }
            }
            tc_commit(tfull);           // accumulator complete
        }
    } else if (warp >= 4) {
        const int ew = warp - 4;       // == warp % 4: TMEM lanes 32*ew .. 32*ew+31
        const int rl = ew * 32 + lane;
        const ExpTab tab = exp_tab_lane();
        if (fused) norm_b_setup(p, bc, bready, kb0, nkb, col0, ncols, ew, lane);
        if (tracing && threadIdx.x == 128) s_tm[2] = globaltimer_ns();   // B operand built (fused)
        if (p.mode == kEpiStoreF32 && ncols > 8 && S > 1 && !push)   // each column's output base (or -1)
            for (int c = rl; c < ncols; c += 128) {
                int64_t off = static_cast<int64_t>(col0 + c) * p.ld_out;
                if (p.col_step != nullptr) {
                    const int st = p.col_step[col0 + c];
                    off = st < 0 ? -1
                                 : static_cast<int64_t>(p.col_slot[col0 + c]) * p.slot_stride +
                                       static_cast<int64_t>(st) * p.n_out;
                }
                s_ckv[c] = off;
            }
        if (p.mode == kEpiQkvRope && ncols > 8 && S > 1 && !push)   // read after the cluster barrier
            for (int c = rl; c < ncols; c += 128) {
                const int pos = p.col_pos[col0 + c];
                s_cpos[c] = pos;
                s_ckv[c] = pos < 0 ? 0
                                   : ((static_cast<int64_t>(p.block_table[static_cast<int64_t>(p.col_req[col0 + c]) *
                                                                               p.max_pages + pos / p.page]) * p.hkv) *
                                          p.page + pos % p.page) * p.hd;
            }
        EpiPre pre{0.0f, 0.0f, -1, 0};   // the first owned column's epilogue operands (decode)
        if (push && seg < ncols) pre = epilogue_preload(p, m0 + rl, col0 + seg);
        mbar_wait(tfull, 0);
        tc_fence_after();
        if (tracing && threadIdx.x == 128) s_tm[3] = globaltimer_ns();   // accumulator complete
        float* P = reinterpret_cast<float*>(smem);   // partial tile [col][128] (stages are idle now)
        if (push) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + (static_cast<uint32_t>(ew * 32) << 16), r);
            tc_wait_ld();
            cluster_wait();
            const uint32_t rbase = smem_u32(recv);
#pragma unroll
            for (int cl = 0; cl < 8; ++cl) {
                const int o = cl % S;
                if (cl < ncols && o != seg) {
                    const int slot = seg < o ? seg : seg - 1;
                    const uint32_t off = 4u * static_cast<uint32_t>((slot * recv_cols + cl / S) * BM + rl);
                    st_async_f32(mapa_shared(rbase + off, o), __uint_as_float(r[cl]), mapa_shared(smem_u32(recv_bar), o));
                }
            }
            if (tracing && threadIdx.x == 128) s_tm[4] = globaltimer_ns();   // partials pushed
            if (owned > 0) {
                mbar_wait(recv_bar, 0);
                if (tracing && threadIdx.x == 128) s_tm[5] = globaltimer_ns();   // peers' partials landed
#pragma unroll
                for (int cl = 0; cl < 8; ++cl) {
                    if (cl < ncols && cl % S == seg) {
                        float v[8];
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2) {
                            const int slot = s2 < seg ? s2 : s2 - 1;
                            v[s2] = s2 >= S ? kNegZero
                                  : s2 == seg ? __uint_as_float(r[cl])
                                              : recv[(slot * recv_cols + cl / S) * BM + rl];
                        }
                        const float sum = local_tree_sum<8>(v);
                        const float xn = cl == seg ? epilogue_pre(p, m0 + rl, col0 + cl, sum, pre, tab)
                                                   : epilogue_any(p, m0 + rl, col0 + cl, sum, tab);
                        if (p.ss_out != nullptr) tile_sumsq(p, tile, col0 + cl, xn, ew, lane, s_red);
                    }
                }
                if (tracing && threadIdx.x == 128) s_tm[7] = globaltimer_ns();   // epilogue done
            }
        }
        for (int j = 0; j < nb && !push; ++j) {
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tbase + (static_cast<uint32_t>(ew * 32) << 16) + j * SUB_N + h * 32, r);
                tc_wait_ld();
                const int cl0 = j * SUB_N + h * 32;
                if (S == 1) {
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (cl0 + c < ncols) {
                            const float xn = epilogue_any(p, m0 + rl, col0 + cl0 + c, __uint_as_float(r[c]), tab);
                            if (p.ss_out != nullptr) tile_sumsq(p, tile, col0 + cl0 + c, xn, ew, lane, s_red);
                        }
                } else {
                    float4* P4 = reinterpret_cast<float4*>(P);   // [column quad][row] x 4 columns
#pragma unroll
                    for (int c = 0; c < 32; c += 4)
                        P4[((cl0 + c) >> 2) * BM + rl] = make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                                                                     __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
                }
            }
        }
    }
    if (tracing && threadIdx.x == 128 && !push) s_tm[4] = globaltimer_ns();   // partial tile / epilogue written
    if (push && warp < 4) cluster_wait();   // pairs the arrive above (long complete by now)
    if (S > 1 && !push) {
        cluster_sync_all();   // partial tiles of all segments visible cluster-wide
        if (tracing && threadIdx.x == 128) s_tm[5] = globaltimer_ns();   // cluster exchange ready
        {
            // all eight warps: the partials come from shared memory, not TMEM, so any warp can take
            // any rows; warp group wg = warp / 4 takes every other round of column quads
            const int rl = (warp & 3) * 32 + lane, wg = warp >> 2;
            const ExpTab tab = exp_tab_lane();
            const uint32_t pbase = smem_u32(smem);
            // CTA `seg` finalises column quads seg, seg+S, ...; QB quads per round trip so that all
            // their DSMEM loads are in flight together.
            constexpr int QB = NSUB <= 2 ? 1 : 2;
            const int nq = ncols <= 8 ? 0 : (ncols + 3) >> 2;
            const QkvRow qr = qkv_row(p, m0 + rl);
            for (int cl = seg; warp >= 4 && ncols <= 8 && cl < ncols; cl += S) {   // one column per CTA
                float v[8];
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    v[s] = s < S ? ld_dsmem_f32(mapa_shared(
                                       pbase + 16u * static_cast<uint32_t>((cl >> 2) * BM + rl) + 4u * (cl & 3), s))
                                 : kNegZero;
                const float sum = local_tree_sum<8>(v);
                if (tracing && threadIdx.x == 128 && s_tm[6] == 0) s_tm[6] = globaltimer_ns();   // DSMEM loads
                const float xn = epilogue_any(p, m0 + rl, col0 + cl, sum, tab);
                if (p.ss_out != nullptr) tile_sumsq(p, tile, col0 + cl, xn, warp - 4, lane, s_red);
            }
            switch (S) {
                case 2: combine_quads<2, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 3: combine_quads<3, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 4: combine_quads<4, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 5: combine_quads<5, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 6: combine_quads<6, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 7: combine_quads<7, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                default: combine_quads<8, QB>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
            }
        }
        if (tracing && threadIdx.x == 128) s_tm[7] = globaltimer_ns();   // combine + epilogue done
        cluster_sync_all();   // peers keep their shared memory until every reader is done
        if (tracing && threadIdx.x == 128) s_tm[8] = globaltimer_ns();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, C::TMEM);
    }
    if (tracing && threadIdx.x == 0)
        trace_record(p.trace, (p.trace_tag << 24) | (blockIdx.x + S * (tile + ntiles * cgrp)), s_tm);
}

// ---------------------------------------------------------------------------------------------
// Many columns (> 64), persistent: a cluster of S CTAs (one per K-segment, one CTA per SM) walks
// the (weight tile, 128-column group) units round robin, so the grid is one wave whatever the
// shape. TMEM holds two 128-column accumulators: the MMA of unit i+1 runs while the epilogue
// warps move unit i's partial to shared memory, combine the S partials of their columns over DSMEM
// (the segment tree, combine_quads) and run the fused epilogue. Per unit and column the arithmetic
// is exactly gemm_tc_kernel's (same K-segments, same chains, same tree), so bits are identical
// (tests/test_gpu_gemm.py::test_persistent_gemm_bit_identical).
//
// Cross-CTA hand-offs are mbarriers, not cluster barriers (the producer and MMA warps never stop).
// The combine is a push: each CTA sends every column quad of its partial straight into the owner
// CTA's receive buffer (st.async, completing bytes on the owner's `recv` barrier), so the owner
// reads all S partials of its quads from local shared memory (no DSMEM round trip):
//   recv     : the S partials of this CTA's quads of the unit have landed
//   rfree    : every CTA finished combining the unit (S remote arrivals) -> receive buffers reusable
//   tfull[b] / tempty[b] : TMEM accumulator b complete / drained (MMA <-> epilogue)
constexpr int kPN = 128;                                   // columns per unit (two 64-wide sub-tiles)
constexpr int kPStages = 4;
constexpr int kPStageBytes = A_BYTES + 2 * B_BYTES;        // 32 KB
constexpr int kPRecvBytes = 36 * BM * 16;                  // max over S of S * ceil(32 / S) quads x 128 rows x 16 B
constexpr int kPSmem = kPStages * kPStageBytes + kPRecvBytes + 1024 /*align*/ + 256 /*barriers*/;

__global__ void __launch_bounds__(256, 1)
    gemm_persist_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPStages * A_BYTES;
    float4* R = reinterpret_cast<float4*>(sB + kPStages * 2 * B_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(R) + kPRecvBytes);
    uint64_t* empty = full + kPStages;
    uint64_t* tfull = empty + kPStages;    // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint64_t* recv = tempty + 2;
    uint64_t* rfree = recv + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(rfree + 1);
    __shared__ int s_cpos[kPN];
    __shared__ int64_t s_ckv[kPN];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.ksplit;
    const int seg = static_cast<int>(cluster_ctarank());
    const int cid = blockIdx.x / S, ncl = gridDim.x / S;
    const int ntiles = p.n_out / BM, ncg = (p.ncols + kPN - 1) / kPN;
    const int nunits = ntiles * ncg;
    const int nkb_all = p.k / BK;
    const int kb0 = seg * nkb_all / S, kb1 = (seg + 1) * nkb_all / S, nkb = kb1 - kb0;
    const int qmax = (kPN / 4 + S - 1) / S;   // owned quads per CTA, at most
    const uint64_t t_start = globaltimer_ns();

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int i = 0; i < kPStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 1);
        }
        mbar_init(recv, 1);
        mbar_init(rfree, S);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tslot, 2 * kPN);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync_all();   // every CTA's barriers initialised before any remote arrive / push
    const uint32_t tbase = *tslot;

    auto unit_geom = [&](int u, int& tile, int& col0, int& ncols) {
        tile = u / ncg;   // consecutive units: the column groups of one tile (weights read once from HBM)
        col0 = (u % ncg) * kPN;
        ncols = min(kPN, p.ncols - col0);
    };
    auto load_w = [&](void* dst, uint64_t* bar, int tile, int kb) {
        if (p.w_tiled) tma_load_3d(dst, &tmW, bar, 0, 0, tile * nkb_all + kb, kEvictFirst);
        else tma_load_3d(dst, &tmW, bar, 0, kb, tile * BM, kEvictFirst);
    };

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int s = 0, ph = 0;
            bool first = true;
            for (int u = cid; u < nunits; u += ncl) {
                int tile, col0, ncols;
                unit_geom(u, tile, col0, ncols);
                const int nb = (ncols + SUB_N - 1) / SUB_N;
                const uint32_t tx = A_BYTES + nb * B_BYTES;
                int i0 = 0;
                if (first) {   // weights do not depend on the previous kernel: stream them before the PDL wait
                    const int pre = min(kPStages, nkb);
                    for (int i = 0; i < pre; ++i) {
                        mbar_arrive_expect_tx(&full[i], tx);
                        load_w(sA + i * A_BYTES, &full[i], tile, kb0 + i);
                    }
                    pdl_wait();
                    pdl_trigger();
                    for (int i = 0; i < pre; ++i)
                        for (int j = 0; j < nb; ++j)
                            tma_load_2d(sB + (i * 2 + j) * B_BYTES, &tmX, &full[i], (kb0 + i) * BK, col0 + j * SUB_N,
                                        kEvictLast);
                    s = pre % kPStages;
                    ph = (pre / kPStages) & 1;
                    i0 = pre;
                    first = false;
                }
                for (int i = i0; i < nkb; ++i) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], tx);
                    load_w(sA + s * A_BYTES, &full[s], tile, kb0 + i);
                    for (int j = 0; j < nb; ++j)
                        tma_load_2d(sB + (s * 2 + j) * B_BYTES, &tmX, &full[s], (kb0 + i) * BK, col0 + j * SUB_N,
                                    kEvictLast);
                    if (++s == kPStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            if (first) {   // no unit for this cluster
                pdl_wait();
                pdl_trigger();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int s = 0, ph = 0, it = 0;
            for (int u = cid; u < nunits; u += ncl, ++it) {
                int tile, col0, ncols;
                unit_geom(u, tile, col0, ncols);
                const int nb = (ncols + SUB_N - 1) / SUB_N;
                const uint32_t idesc = umma_idesc_bf16(BM, nb * SUB_N);
                const int b = it & 1, use = it >> 1;
                if (use > 0) mbar_wait(&tempty[b], (use - 1) & 1);   // the epilogue drained this buffer
                tc_fence_after();
                const uint32_t d = tbase + b * kPN;
                for (int i = 0; i < nkb; ++i) {
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                    const uint32_t b_base = smem_u32(sB + s * 2 * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)   // one N = nb*64 instruction (bit-identical to per sub-tile)
                        tc_mma_bf16(d, umma_desc_k128(a_base + k * 32), umma_desc_k128(b_base + k * 32), idesc,
                                    (i | k) != 0 ? 1u : 0u);
                    tc_commit(&empty[s]);
                    if (++s == kPStages) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                tc_commit(&tfull[b]);
            }
        }
    } else if (warp == 3 && lane == 0) {
        l2_prefetch_slice(p.l2pf, p.l2pf_bytes, blockIdx.x, gridDim.x);
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue: TMEM -> push -> combine
        const int ew = warp - 4, rl = ew * 32 + lane;
        const ExpTab tab = exp_tab_lane();
        const uint32_t rbase = smem_u32(R), recv_addr = smem_u32(recv);
        int it = 0;
        for (int u = cid; u < nunits; u += ncl, ++it) {
            int tile, col0, ncols;
            unit_geom(u, tile, col0, ncols);
            const int nb = (ncols + SUB_N - 1) / SUB_N;
            const int nq = (ncols + 3) >> 2;
            const int m0 = tile * BM;
            const int b = it & 1, use = it >> 1;
            // this unit's per-column epilogue operands (read only by this CTA's epilogue warps)
            if (p.mode == kEpiStoreF32)
                for (int c = rl; c < ncols; c += 128) {
                    int64_t off = static_cast<int64_t>(col0 + c) * p.ld_out;
                    if (p.col_step != nullptr) {
                        const int st = p.col_step[col0 + c];
                        off = st < 0 ? -1
                                     : static_cast<int64_t>(p.col_slot[col0 + c]) * p.slot_stride +
                                           static_cast<int64_t>(st) * p.n_out;
                    }
                    s_ckv[c] = off;
                }
            if (p.mode == kEpiQkvRope)
                for (int c = rl; c < ncols; c += 128) {
                    const int pos = p.col_pos[col0 + c];
                    s_cpos[c] = pos;
                    s_ckv[c] = pos < 0 ? 0
                                       : ((static_cast<int64_t>(p.block_table[static_cast<int64_t>(p.col_req[col0 + c]) *
                                                                                   p.max_pages + pos / p.page]) * p.hkv) *
                                              p.page + pos % p.page) * p.hd;
                }
            const QkvRow qr = p.mode == kEpiQkvRope ? qkv_row(p, m0 + rl) : QkvRow{};
            mbar_wait(&tfull[b], use & 1);
            tc_fence_after();
            if (it > 0) mbar_wait_cluster(rfree, (it - 1) & 1);   // every receive buffer of the cluster is free
            if (threadIdx.x == 128) {   // our quads' S partials: arrival + expected bytes
                const int own = seg < nq ? (nq - 1 - seg) / S + 1 : 0;
                mbar_arrive_expect_tx(recv, static_cast<uint32_t>(S * own * BM * 16));
            }
            for (int j = 0; j < nb; ++j) {
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tbase + (static_cast<uint32_t>(ew * 32) << 16) + b * kPN + j * SUB_N + h * 32, r);
                    tc_wait_ld();
                    const int q0 = (j * SUB_N + h * 32) >> 2;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int q = q0 + c;
                        if (q >= nq) break;   // warp-uniform
                        const uint32_t o = static_cast<uint32_t>(q % S);
                        const uint32_t off = 16u * static_cast<uint32_t>((seg * qmax + q / S) * BM + rl);
                        st_async_v4(mapa_shared(rbase + off, o), r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3],
                                    mapa_shared(recv_addr, o));
                    }
                }
            }
            tc_fence_before();
            epi_bar();
            if (threadIdx.x == 128) mbar_arrive(&tempty[b]);   // the accumulator may be reused (unit it + 2)
            mbar_wait_cluster(recv, it & 1);                   // all S partials of our quads landed
            switch (S) {
                case 2: combine_local<2>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 3: combine_local<3>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 4: combine_local<4>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 5: combine_local<5>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 6: combine_local<6>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                case 7: combine_local<7>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
                default: combine_local<8>(p, R, qmax, seg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab); break;
            }
            epi_bar();   // every epilogue thread's reads of R are complete
            if (threadIdx.x == 128)
                for (int r = 0; r < S; ++r) mbar_arrive_remote(mapa_shared(smem_u32(rfree), static_cast<uint32_t>(r)));
        }
    }
    // nobody leaves while a peer may still push into it (every push lands before its owner's last recv wait)
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, 2 * kPN);
    }
    if (p.trace != nullptr && threadIdx.x == 0) {
        uint64_t marks[kTraceMarks] = {};
        marks[0] = t_start;
        trace_record(p.trace, (p.trace_tag << 24) | blockIdx.x, marks);
    }
}

cudaError_t launch_persist(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p, cudaStream_t stream,
                           bool pdl) {
    static std::atomic<uint64_t> attr_devs{0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(gemm_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem);
        if (e != cudaSuccess) return e;
        attrs_done(attr_devs, dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = kPSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = p.ksplit;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    // as many clusters as are co-resident (clusters live inside one GPC: S = 5 or 8 leaves SMs idle),
    // never more than there are units
    static int max_clusters[9][64] = {};
    int& mc = max_clusters[p.ksplit][dev & 63];
    if (mc == 0) {
        cfg.gridDim = dim3(p.ksplit * 148, 1, 1);
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, gemm_persist_kernel, &cfg) != cudaSuccess || n <= 0) return cudaErrorInvalidConfiguration;
        mc = n;
        if (std::getenv("DETGPU_DEBUG_PERSIST")) std::fprintf(stderr, "gemm_persist: S=%d -> %d clusters\n", p.ksplit, n);
    }
    const int nunits = (p.n_out / BM) * ((p.ncols + kPN - 1) / kPN);
    cfg.gridDim = dim3(p.ksplit * (mc < nunits ? mc : nunits), 1, 1);
    return cudaLaunchKernelEx(&cfg, gemm_persist_kernel, tmW, tmX, p);
}

// ---------------------------------------------------------------------------------------------
// Many columns (> 64): CTA pairs (cta_group::2). A pair computes a 256-row x 128-column tile of one
// K-segment chain: each CTA loads its 128 weight rows and 64 of the 128 activation columns per
// k-block (24 KB instead of 32 KB for the same 128 x 128 x 64 MACs per SM, four stages in flight
// instead of three), the even CTA issues one M = 256, N = 128 tcgen05.mma per K step, and each
// CTA's TMEM holds its 128 rows x 128 columns. The S K-segments are S pairs of one cluster (rank
// 2s + v) and are combined exactly as in gemm_tc_kernel (combine_quads over ranks 2s' + v), so
// every output element has the same K order, chains and tree: the bits equal the one-CTA form
// (tests/test_gpu_gemm.py).
constexpr int kPairStages = 4;
constexpr int kPairSmem = kPairStages * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers*/;

__global__ void __launch_bounds__(256, 2)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPairStages * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kPairStages * B_BYTES);
    uint64_t* empty = full + kPairStages;
    uint64_t* tfull = empty + kPairStages;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
    __shared__ int s_cpos[2 * SUB_N];
    __shared__ int64_t s_ckv[2 * SUB_N];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.ksplit;
    const int rank = static_cast<int>(blockIdx.x), v = rank & 1, seg = rank >> 1;
    const uint32_t leader = static_cast<uint32_t>(rank & ~1);
    const int m0 = static_cast<int>(blockIdx.z) * 2 * BM + v * BM, tile = m0 / BM;
    const int col0 = static_cast<int>(blockIdx.y) * 2 * SUB_N;
    const int ncols = min(2 * SUB_N, p.ncols - col0);
    const int bcol = col0 + v * SUB_N;   // this CTA's half of the pair's B columns
    const int nkb_all = p.k / BK;
    const int kb0 = seg * nkb_all / S, nkb = (seg + 1) * nkb_all / S - kb0;
    constexpr uint32_t kStageTx = 2 * (A_BYTES + B_BYTES);   // both CTAs' bytes land on the leader's barrier

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc_pair(tslot, 2 * SUB_N);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    cluster_sync_all();   // every pair member's barriers exist before any remote arrive / complete_tx
    const uint32_t tbase = *tslot;

    auto load_w = [&](int s, int kb) {
        const uint32_t bar = mapa_shared(smem_u32(&full[s]), leader);
        if (p.w_tiled) tma_load_3d_pair(sA + s * A_BYTES, &tmW, bar, 0, 0, tile * nkb_all + kb, kEvictFirst);
        else tma_load_3d_pair(sA + s * A_BYTES, &tmW, bar, 0, kb, m0, kEvictFirst);
    };
    auto load_x = [&](int s, int kb) {
        tma_load_2d_pair(sB + s * B_BYTES, &tmX, mapa_shared(smem_u32(&full[s]), leader), kb * BK, bcol, kEvictLast);
    };
    const int pre = min(kPairStages, nkb);
    if (threadIdx.x == 0)   // weight tiles do not depend on the previous kernel
        for (int i = 0; i < pre; ++i) {
            if (v == 0) mbar_arrive_expect_tx(&full[i], kStageTx);
            load_w(i, kb0 + i);
        }
    pdl_wait();
    pdl_trigger();
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < pre; ++i) load_x(i, kb0 + i);
            int s = pre % kPairStages, ph = (pre / kPairStages) & 1;
            for (int i = pre; i < nkb; ++i) {
                mbar_wait(&empty[s], ph ^ 1);
                if (v == 0) mbar_arrive_expect_tx(&full[s], kStageTx);
                load_w(s, kb0 + i);
                load_x(s, kb0 + i);
                if (++s == kPairStages) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && v == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, 2 * SUB_N);
            const uint16_t mask = static_cast<uint16_t>(3u << leader);
            int s = 0, ph = 0;
            for (int i = 0; i < nkb; ++i) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA + s * A_BYTES), b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    tc_mma_bf16_pair(tbase, umma_desc_k128(a_base + k * 32), umma_desc_k128(b_base + k * 32), idesc,
                                     (i | k) != 0 ? 1u : 0u);
                tc_commit_pair_mc(&empty[s], mask);   // frees this stage in both pair members
                if (++s == kPairStages) {
                    s = 0;
                    ph ^= 1;
                }
            }
            tc_commit_pair_mc(tfull, mask);
        }
    } else if (warp >= 4) {
        const int ew = warp - 4, rl = ew * 32 + lane;
        // per-column epilogue operands (read after the cluster barrier below)
        if (p.mode == kEpiStoreF32)
            for (int c = rl; c < ncols; c += 128) {
                int64_t off = static_cast<int64_t>(col0 + c) * p.ld_out;
                if (p.col_step != nullptr) {
                    const int st = p.col_step[col0 + c];
                    off = st < 0 ? -1
                                 : static_cast<int64_t>(p.col_slot[col0 + c]) * p.slot_stride +
                                       static_cast<int64_t>(st) * p.n_out;
                }
                s_ckv[c] = off;
            }
        if (p.mode == kEpiQkvRope)
            for (int c = rl; c < ncols; c += 128) {
                const int pos = p.col_pos[col0 + c];
                s_cpos[c] = pos;
                s_ckv[c] = pos < 0 ? 0
                                   : ((static_cast<int64_t>(p.block_table[static_cast<int64_t>(p.col_req[col0 + c]) *
                                                                               p.max_pages + pos / p.page]) * p.hkv) *
                                          p.page + pos % p.page) * p.hd;
            }
        mbar_wait(tfull, 0);
        tc_fence_after();
        float4* P4 = reinterpret_cast<float4*>(smem);   // partial tile [column quad][row] (stages idle)
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tbase + (static_cast<uint32_t>(ew * 32) << 16) + h * 32, r);
            tc_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; c += 4)
                P4[((h * 32 + c) >> 2) * BM + rl] = make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                                                                __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
        }
    }
    cluster_sync_all();   // every segment's partial tile visible cluster-wide
    {
        const int rl = (warp & 3) * 32 + lane, wg = warp >> 2;
        const ExpTab tab = exp_tab_lane();
        const uint32_t pbase = smem_u32(smem);
        const int nq = (ncols + 3) >> 2;
        const QkvRow qr = qkv_row(p, m0 + rl);
        switch (S) {
            case 1: combine_quads<1, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 2: combine_quads<2, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 3: combine_quads<3, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 4: combine_quads<4, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 5: combine_quads<5, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 6: combine_quads<6, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            case 7: combine_quads<7, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
            default: combine_quads<8, 1>(p, pbase, seg, wg, nq, ncols, m0, rl, col0, qr, s_cpos, s_ckv, tab, 2, v); break;
        }
    }
    cluster_sync_all();   // peers keep their shared memory until every reader is done
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_pair(tbase, 2 * SUB_N);
    }
}

cudaError_t launch_pair(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p, cudaStream_t stream,
                        bool pdl) {
    static std::atomic<uint64_t> attr_devs{0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPairSmem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attrs_done(attr_devs, dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * p.ksplit, (p.ncols + 2 * SUB_N - 1) / (2 * SUB_N), p.n_out / (2 * BM));
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = kPairSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2 * p.ksplit;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, gemm_pair_kernel, tmW, tmX, p);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeFn>(nullptr);
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

template <int NSUB>
cudaError_t launch_nsub(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p, cudaStream_t stream,
                        bool pdl) {
    using C = Cfg<NSUB>;
    static std::atomic<uint64_t> attr_devs{0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attrs_done(attr_devs, dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.ksplit, (p.ncols + NSUB * SUB_N - 1) / (NSUB * SUB_N), p.n_out / BM);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = p.ksplit;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<NSUB>, tmW, tmX, p);
}

}  // namespace

bool make_tmap_weights(CUtensorMap* m, const void* ptr, uint64_t n_out, uint64_t k, bool tiled) {
    EncodeFn enc = get_encode();
    if (enc == nullptr) return false;
    cuuint64_t dims[3];
    cuuint64_t strides[2];
    cuuint32_t box[3];
    if (tiled) {   // [tiles*nkb][128 rows][64 k], each (tile, kb) block contiguous
        dims[0] = 64; dims[1] = 128; dims[2] = (n_out / 128) * (k / 64);
        strides[0] = 128; strides[1] = 128 * 128;
        box[0] = 64; box[1] = 128; box[2] = 1;
    } else {       // row-major [n_out][k] viewed as [n_out][k/64][64]
        dims[0] = 64; dims[1] = k / 64; dims[2] = n_out;
        strides[0] = 128; strides[1] = k * 2;
        box[0] = 64; box[1] = 1; box[2] = 128;
    }
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint32_t box_rows) {
    EncodeFn enc = get_encode();
    if (enc == nullptr) return false;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The sub-tile count only sizes the smem pipeline (deeper for small batches); the MMA shape, the
// K order and each column's TMEM accumulation sequence are identical for every choice.
// S = min(K/64, max(2, min(8, 256 / tiles))): enough CTAs (with two resident per SM) to keep every
// SM streaming weights; chosen from measured B200 scans (tools/gemm_split_scan.py).
int gemm_ksplit(int n_out, int k) {
    const int tiles = n_out / BM, nkb = k / BK;
    int s = 256 / (tiles > 0 ? tiles : 1);
    s = s > 8 ? 8 : s;
    s = s < 2 ? 2 : s;
    return s > nkb ? nkb : s;
}

cudaError_t gemm_launch(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p_in, cudaStream_t stream,
                        bool pdl) {
    if (p_in.n_out % BM != 0 || p_in.k % BK != 0 || p_in.k <= 0 || p_in.ncols <= 0) return cudaErrorInvalidValue;
    GemmParams p = p_in;
    if (p.ksplit <= 0) p.ksplit = gemm_ksplit(p.n_out, p.k);
    if (p.ksplit > 8 || p.ksplit > p.k / BK) return cudaErrorInvalidValue;
    const int seg_kb = (p.k / BK + p.ksplit - 1) / p.ksplit;
    if (p.norm_x != nullptr && (p.ncols > 8 || seg_kb > 35)) return cudaErrorInvalidValue;
    if (p.norm_x != nullptr && (p.ncols > 8 || p.norm_ss == nullptr || p.k != p.norm_d || (p.norm_d & (p.norm_d - 1)) != 0 ||
                                p.norm_d < 256 || p.norm_d > 4096))
        return cudaErrorInvalidValue;
    if (p.ss_out != nullptr && (p.mode != kEpiAddF32 || p.n_out != p.ss_tiles * BM || p.ncols > 8))
        return cudaErrorInvalidValue;
    if (p.ncols <= 64) return launch_nsub<1>(tmW, tmX, p, stream, pdl);
    // persistent clusters: faster for S = 2 (gate/up, lm_head: long K-segments keep the main loop
    // busy while the push combine runs); at S = 5 / 8 the per-unit combine is longer than the main
    // loop of 8-13 k-blocks and the one-unit clusters (two CTAs per SM) win (tools/gemm_persist_bench.py)
    if (p.persist > 0 && p.ksplit > 1 && (p.ksplit <= 2 || p.persist > 1) && p.norm_x == nullptr && p.ss_out == nullptr)
        return launch_persist(tmW, tmX, p, stream, pdl);
    // > 128 columns: 128-column tiles at two CTAs per SM (one CTA's epilogue overlaps the other's
    // main loop) beat 256-column tiles at one CTA per SM by 25 % on the 512-token prefill
    if (p.pair > 0 && p.n_out % (2 * BM) == 0 && 2 * p.ksplit <= 16 && p.norm_x == nullptr && p.ss_out == nullptr)
        return launch_pair(tmW, tmX, p, stream, pdl);
    if (p.max_nsub != 4) return launch_nsub<2>(tmW, tmX, p, stream, pdl);
    return launch_nsub<4>(tmW, tmX, p, stream, pdl);
}

}  // namespace detgpu
