// Streamed decode attention for many columns (DESIGN.md §3.5 arithmetic, §4 layout).
//
// The per-chunk arithmetic is attention.cu's (attn_chunk_kernel): scores are the canonical tree
// over d of exact q*k products times 1/sqrt(hd); chunk max m, e = exp(s - m), l = tree(e), o_d =
// fma chain over positions in order; chunks combined in chunk order (a_c = exp(m_c - max m),
// out = bf16(fma-chain(o a) / fma-chain(l a))). Only the schedule differs:
//
// * one persistent CTA per SM walks a contiguous range of the step's (column, kv head, chunk)
//   stream, so every SM reads the same number of 64-position chunks whatever the batch mix;
// * a producer warp streams each chunk's K and V (one contiguous 16 KB block per (page, head)) with
//   TMA into a ring of shared-memory stages (K 128B-swizzled so the thread-per-position score reads
//   are conflict-free), plus the column's q (1D bulk copy), completing on the stage's mbarrier;
// * four consumer groups of 64 threads take the ring's chunks round robin: chunk j -> group j % 4.
//   Each chunk's partial (m, l, o) goes to the workspace; the group that completes a (column, kv
//   head) combines it. Completion is counted per CTA in shared memory; only an item split between
//   two CTAs' ranges (at most two per CTA) also goes through a global ticket.
//
// A chunk's bits do not depend on which CTA, group or stage computes it, and the combine order is
// fixed, so the output is identical to attn_chunk_kernel's (tests/test_gpu_engine.py).
#include <cfloat>

#include "common.h"
#include "detmath.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace detgpu {

namespace {

constexpr int kCH = kAttnChunk;            // 64 positions per chunk
constexpr int kGroups = 4;                 // consumer groups
constexpr int kGT = 64;                    // threads per consumer group (two warps)
constexpr int kThreads = kGroups * kGT + 32;   // + producer warp
constexpr int kProducerWarp = kGroups * kGT / 32;
constexpr int kMaxCols = 256;              // columns staged in shared memory
constexpr int kLocalSlots = 256;           // per-CTA chunk counters of (column, kv head) items
constexpr int kMaxCombine = 128;           // chunks per (column, kv head) the combine scratch holds

template <int HD, int G>
struct Cfg {
    static constexpr int KB = kCH * HD * 2;                       // K (or V) bytes of one chunk
    static constexpr int QB = G * HD * 2;                         // the column's q for this kv head
    static constexpr int STAGE = (2 * KB + QB + 1023) / 1024 * 1024;
    static constexpr int S = HD == 128 ? 6 : 8;                   // ring stages
    static constexpr int WORK = G * (HD + 2 * kCH) * 4;           // q f32, scores, e (per group)
    static constexpr int COMB = 2 * G * kMaxCombine * 4;          // combine: a_c and l_c (aliases WORK)
    static constexpr int SCR = (WORK > COMB ? WORK : COMB) + 2 * G * 4 * 2;   // + m, l
    static constexpr int DYN = 1024 + S * STAGE + kGroups * SCR;  // + alignment slack
    static constexpr int DPT = HD / kGT;                          // PV dimensions per thread
};

__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kGT) : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem_dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t hint) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(smem_dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(hint)
        : "memory");
}

// byte offset of dimension d (even when 2 dims are read together) of row p in a 128B-swizzled
// [64 rows][HD] block loaded as HD/64 boxes of [64 rows][64 dims]
__device__ __forceinline__ uint32_t swz(int p, int d) {
    const int half = d >> 6, dd = d & 63;
    return static_cast<uint32_t>(half * (kCH * 128) + p * 128 + ((((dd >> 3) ^ (p & 7))) << 4) + (dd & 7) * 2);
}

struct ChunkInfo {
    int col, kvh, c, n, nch;
    int key;     // the item's first chunk in this CTA's range, relative to the range start
    int cnt;     // the item's chunks in this CTA's range
    int whole;   // every chunk of the item is in this CTA's range
};

template <int HD, int G>
__global__ void __launch_bounds__(kThreads, 1)
    attn_stream_kernel(const AttnParams a, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, float scale) {
    using C = Cfg<HD, G>;
    constexpr int S = C::S;
    constexpr int NV = HD / 8;
    constexpr int DEPTH = (NV >= 16 ? 4 : NV >= 8 ? 3 : NV >= 4 ? 2 : 1) + 1;
    constexpr int DPT = C::DPT;
    static_assert(HD == 64 || HD == 128, "head dim");
    static_assert(G >= 1 && G <= 4, "group size");
    extern __shared__ uint8_t st_dsm[];
    // 1024-byte aligned ring (128B-swizzled TMA boxes); offset arithmetic on the shared array keeps
    // every access an LDS (a pointer rebuilt from an integer would be generic)
    uint8_t* ring = st_dsm + ((1024u - (smem_u32(st_dsm) & 1023u)) & 1023u);
    uint8_t* scr_all = ring + S * C::STAGE;
    __shared__ uint64_t full[S], empty[S];
    __shared__ int4 sinfo[S];
    __shared__ int s_pos[kMaxCols], s_pref[kMaxCols + 1];
    __shared__ int s_last[kGroups];
    __shared__ int s_cnt[kLocalSlots];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ncols = a.ncols;
    for (int i = tid; i < ncols; i += kThreads) s_pos[i] = a.col_pos[i];
    for (int i = tid; i < kLocalSlots; i += kThreads) s_cnt[i] = 0;
    if (tid < S) {
        mbar_init(&full[tid], 1);
        mbar_init(&empty[tid], kGT);
    }
    if (tid == 0) fence_mbar_init();
    __syncthreads();
    if (warp == 0) {   // s_pref[col] = sum over earlier columns of hkv * chunks
        const int per = (ncols + 31) / 32;
        const int c0 = lane * per, c1 = min(ncols, c0 + per);
        int sum = 0;
        for (int col = c0; col < c1; ++col) sum += s_pos[col] >= 0 ? (s_pos[col] / kCH + 1) * a.hkv : 0;
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        int run = incl - sum;
        for (int col = c0; col < c1; ++col) {
            s_pref[col] = run;
            run += s_pos[col] >= 0 ? (s_pos[col] / kCH + 1) * a.hkv : 0;
        }
        if (lane == 31) s_pref[ncols] = incl;
    }
    __syncthreads();
    const int T = s_pref[ncols];
    const int nb = gridDim.x, b = blockIdx.x;
    const int t0 = static_cast<int>(static_cast<int64_t>(b) * T / nb);
    const int nloc = static_cast<int>(static_cast<int64_t>(b + 1) * T / nb) - t0;

    if (warp == kProducerWarp) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            l2_prefetch_slice(a.l2pf, a.l2pf_bytes, b, nb);
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
        }
        auto locate = [&](int j) {
            const int t = t0 + j;
            int lo = 0, hi = ncols;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (s_pref[mid] <= t) lo = mid;
                else hi = mid;
            }
            ChunkInfo ci;
            ci.col = lo;
            const int r = t - s_pref[lo];
            ci.nch = s_pos[lo] / kCH + 1;
            ci.kvh = r / ci.nch;
            ci.c = r % ci.nch;
            ci.n = min(kCH, s_pos[lo] + 1 - ci.c * kCH);
            const int i0 = s_pref[lo] + ci.kvh * ci.nch, i1 = i0 + ci.nch;
            const int l0 = max(i0, t0), l1 = min(i1, t0 + nloc);
            ci.key = l0 - t0;
            ci.cnt = l1 - l0;
            ci.whole = i0 >= t0 && i1 <= t0 + nloc;
            return ci;
        };
        auto page_of = [&](const ChunkInfo& ci) {
            const int slot = __ldg(a.col_req + ci.col);
            return __ldg(a.block_table + static_cast<int64_t>(slot) * a.max_pages + ci.c);
        };
        auto issue_kv = [&](int s, const ChunkInfo& ci, int pid) {
            uint8_t* st = ring + s * C::STAGE;
            const int row = static_cast<int>(a.kv_row0 + (static_cast<int64_t>(pid) * a.hkv + ci.kvh) * kCH);
#pragma unroll
            for (int h = 0; h < HD / 64; ++h) {
                tma_load_2d(st + h * (kCH * 128), &tmK, &full[s], h * 64, row, kEvictFirst);
                tma_load_2d(st + C::KB + h * (kCH * 128), &tmV, &full[s], h * 64, row, kEvictFirst);
            }
        };
        auto issue_q = [&](int s, const ChunkInfo& ci) {
            const __nv_bfloat16* src = a.q + static_cast<int64_t>(ci.col) * a.hq * HD + static_cast<int64_t>(ci.kvh) * G * HD;
            bulk_load(ring + s * C::STAGE + 2 * C::KB, src, C::QB, &full[s], kEvictLast);
        };
        auto publish = [&](int s, const ChunkInfo& ci) {
            sinfo[s] = make_int4(ci.col, ci.kvh | (ci.c << 16), ci.n | (ci.nch << 16),
                                 ci.cnt | (ci.whole << 8) | (ci.key << 9));
            mbar_arrive_expect_tx(&full[s], 2 * C::KB + C::QB);
        };
        // first fill: history chunks stream before the dependency wait (the QKV GEMM, our
        // predecessor, writes q and the newest K/V row, which lives in each column's last chunk)
        const int nfirst = min(S, nloc);
        ChunkInfo ci0{};
        int pid0 = 0;
        if (lane < nfirst) {
            ci0 = locate(lane);
            pid0 = page_of(ci0);
            publish(lane, ci0);
            if (ci0.c < ci0.nch - 1) issue_kv(lane, ci0, pid0);
        }
        pdl_wait();
        pdl_trigger();
        if (lane < nfirst) {
            if (ci0.c == ci0.nch - 1) issue_kv(lane, ci0, pid0);
            issue_q(lane, ci0);
        }
        for (int jb = S; jb < nloc; jb += 32) {
            ChunkInfo ci{};
            int pid = 0;
            if (jb + lane < nloc) {
                ci = locate(jb + lane);
                pid = page_of(ci);
            }
            const int cnt = min(32, nloc - jb);
            for (int i = 0; i < cnt; ++i) {
                if (lane == i) {
                    const int j = jb + i, s = j % S;
                    mbar_wait(&empty[s], ((j / S) - 1) & 1, j);
                    publish(s, ci);
                    issue_kv(s, ci, pid);
                    issue_q(s, ci);
                }
                __syncwarp();
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    const int gi = warp >> 1, gt = tid & (kGT - 1), wg = warp & 1;
    float* gQ = reinterpret_cast<float*>(scr_all + gi * C::SCR);   // [G][HD], {0,2,1,3}-permuted quads
    float* gS = gQ + G * HD;                                        // [G][64] scores
    float* gE = gS + G * kCH;                                       // [64][G] exp(s - m)
    float* gM = reinterpret_cast<float*>(scr_all + gi * C::SCR + (C::SCR - 2 * G * 4 * 2));
    float* gL = gM + G;
    float* cA = gQ;                                                 // combine: [G][kMaxCombine] a_c
    float* cLs = gQ + G * kMaxCombine;                              //          [G][kMaxCombine] l_c
    const ExpTab tab = exp_tab_lane();
    const int64_t cstride = static_cast<int64_t>(G) * (HD + 4);

    for (int j = gi; j < nloc; j += kGroups) {
        const int s = j % S;
        // Stage s is consumed by different groups on successive uses (S is not a multiple of the
        // group count), so this group has not itself waited for the stage's previous use j - S:
        // while that phase is still in flight, a parity wait for chunk j passes at once (the
        // phase-parity ABA). First wait until chunk j - S has been released (empty[s] phase k - 1;
        // exact: phase k - 2 is complete, since the producer published chunk j - S, and phase k is
        // this group's own release of chunk j), after which full[s] is in phase k or k + 1 and the
        // parity wait for chunk j is exact.
        const int k = j / S;
        if (k > 0) mbar_wait(&empty[s], (k - 1) & 1, gt == 0 ? j : -1);
        mbar_wait(&full[s], k & 1, gt == 0 ? j : -1);
        const int4 inf = sinfo[s];
        const int col = inf.x, kvh = inf.y & 0xffff, c = inf.y >> 16, n = inf.z & 0xffff, nch = inf.z >> 16;
        const int lcnt = inf.w & 0xff, whole = (inf.w >> 8) & 1, key = inf.w >> 9;
        const uint8_t* st = ring + s * C::STAGE;
        const uint16_t* sq = reinterpret_cast<const uint16_t*>(st + 2 * C::KB);
        for (int i = gt * 8; i < G * HD; i += kGT * 8) {   // q -> f32; within each quad the order 0,2,1,3
            const uint4 w = *reinterpret_cast<const uint4*>(sq + i);
            *reinterpret_cast<float4*>(gQ + i) = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.y << 16),
                                                             __uint_as_float(w.x & 0xffff0000u),
                                                             __uint_as_float(w.y & 0xffff0000u));
            *reinterpret_cast<float4*>(gQ + i + 4) = make_float4(__uint_as_float(w.z << 16), __uint_as_float(w.w << 16),
                                                                 __uint_as_float(w.z & 0xffff0000u),
                                                                 __uint_as_float(w.w & 0xffff0000u));
        }
        group_bar(gi);
        // scores: thread = position, all G heads over the same unpacked K row
        if (gt < n) {
            const int p = gt;
            const uint32_t kbase = static_cast<uint32_t>(p * 128);
            float stk[G][DEPTH];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint4 kv = *reinterpret_cast<const uint4*>(st + kbase + (((v & 7) ^ (p & 7)) << 4) + (v >> 3) * (kCH * 128));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float carry = qk_block8(kv, *reinterpret_cast<const ulonglong2*>(gQ + g * HD + v * 8),
                                            *reinterpret_cast<const ulonglong2*>(gQ + g * HD + v * 8 + 4));
                    int lvl = 0;
#pragma unroll
                    for (int bb = v; bb & 1; bb >>= 1, ++lvl) carry = __fadd_rn(stk[g][lvl], carry);
                    stk[g][lvl] = carry;
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) gS[g * kCH + p] = __fmul_rn(stk[g][DEPTH - 1], scale);
        }
        group_bar(gi);
        // chunk softmax (chunk_softmax's arithmetic): warp wg owns heads wg, wg + 2, ...
        for (int g = wg; g < G; g += 2) {
            constexpr int PPL = kCH / 32;
            float sv[PPL], e[PPL];
            float m = -FLT_MAX;
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                const int p = lane * PPL + q;
                sv[q] = p < n ? gS[g * kCH + p] : 0.0f;
                if (p < n) m = fmaxf(m, sv[q]);
            }
            m = warp_max(m);
#pragma unroll
            for (int q = 0; q < PPL; ++q) {
                const int p = lane * PPL + q;
                const float ev = det_expf_shfl(p < n ? __fsub_rn(sv[q], m) : 0.0f, tab);
                e[q] = p < n ? ev : kNegZero;
                gE[p * G + g] = e[q];
            }
            float l = local_tree_sum<PPL>(e);
            l = warp_tree_sum(l);
            if (lane == 0) {
                gM[g] = m;
                gL[g] = l;
            }
        }
        group_bar(gi);
        // PV: thread = DPT dimensions x G heads; fma chains over positions in order. With two
        // dimensions per thread the pair of chains of one head is one packed FFMA2 per position
        // (each lane an independent fma.rn: the same bits as two scalar __fmaf_rn chains).
        float acc[G][DPT];
        {
            const int d0 = gt * DPT;
            const uint8_t* sV = st + C::KB;
            uint32_t voff[8];   // swizzled offset of (row r, d0) for r = p mod 8; rows 8 apart are 1 KB apart
#pragma unroll
            for (int r = 0; r < 8; ++r) voff[r] = swz(r, d0);
            auto load_e = [&](int p, float (&ev)[G]) {
                if constexpr (G == 4) {
                    const float4 e4 = *reinterpret_cast<const float4*>(gE + p * 4);
                    ev[0] = e4.x;
                    ev[1] = e4.y;
                    ev[2] = e4.z;
                    ev[3] = e4.w;
                } else {
#pragma unroll
                    for (int g = 0; g < G; ++g) ev[g] = gE[p * G + g];
                }
            };
            if constexpr (DPT == 2) {
                uint64_t acc2[G];
#pragma unroll
                for (int g = 0; g < G; ++g) acc2[g] = 0;
                auto pv_step = [&](int p, uint32_t off) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(sV + off);
                    const uint64_t vv = pack2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
                    float ev[G];
                    load_e(p, ev);
#pragma unroll
                    for (int g = 0; g < G; ++g) acc2[g] = ffma2(pack2(ev[g], ev[g]), vv, acc2[g]);
                };
                int p = 0;
                for (; p + 8 <= n; p += 8) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) pv_step(p + r, voff[r] + p * 128);
                }
                for (; p < n; ++p) pv_step(p, swz(p, d0));
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    acc[g][0] = lo32(acc2[g]);
                    acc[g][1] = hi32(acc2[g]);
                }
            } else {
#pragma unroll
                for (int g = 0; g < G; ++g)
#pragma unroll
                    for (int k = 0; k < DPT; ++k) acc[g][k] = 0.0f;
                auto pv_step = [&](int p, uint32_t off) {
                    const float v0 = __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(sV + off)) << 16);
                    float ev[G];
                    load_e(p, ev);
#pragma unroll
                    for (int g = 0; g < G; ++g) acc[g][0] = __fmaf_rn(ev[g], v0, acc[g][0]);
                };
                int p = 0;
                for (; p + 8 <= n; p += 8) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) pv_step(p + r, voff[r] + p * 128);
                }
                for (; p < n; ++p) pv_step(p, swz(p, d0));
            }
        }
        mbar_arrive(&empty[s]);   // this thread's reads of the stage are done
        __nv_bfloat16* outp = a.out + static_cast<int64_t>(col) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD;
        if (nch == 1) {   // the combine weight is exp(0) == 1 exactly (as attn_chunk_kernel)
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float L = __fmaf_rn(gL[g], 1.0f, 0.0f);
#pragma unroll
                for (int k = 0; k < DPT; ++k)
                    outp[g * HD + gt * DPT + k] = f2bf(__fdiv_rn(__fmaf_rn(acc[g][k], 1.0f, 0.0f), L));
            }
            continue;
        }
        float* wsb = a.ws + (static_cast<int64_t>(col) * a.hkv + kvh) * a.max_chunks * cstride;
        {
            float* w = wsb + c * cstride;
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int k = 0; k < DPT; ++k) w[g * (HD + 4) + 4 + gt * DPT + k] = acc[g][k];
            if (gt < G) {
                w[gt * (HD + 4)] = gM[gt];
                w[gt * (HD + 4) + 1] = gL[gt];
            }
        }
        // Completion of the item: this CTA's chunks count in shared memory (release/acquire at CTA
        // scope: the barrier orders the group's partial stores before thread 0's fence); the CTA
        // completing its share of an item that spans CTAs adds it to the item's global ticket.
        group_bar(gi);
        if (gt == 0) {
            int last = 0;
            int* tk = a.tickets + static_cast<int64_t>(col) * a.hkv + kvh;
            if (key < kLocalSlots) {
                __threadfence_block();
                const int done = atomicAdd(&s_cnt[key], 1) + 1;
                if (done == lcnt) {
                    __threadfence_block();
                    if (whole) {
                        last = 1;
                    } else {
                        __threadfence();
                        last = atomicAdd(tk, lcnt) + lcnt == nch;
                        if (last) *tk = 0;   // re-armed for the next launch
                    }
                }
            } else {
                __threadfence();
                last = atomicAdd(tk, 1) == nch - 1;
                if (last) *tk = 0;
            }
            if (last) __threadfence();
            s_last[gi] = last;
        }
        group_bar(gi);
        if (!s_last[gi]) continue;   // group-uniform
        // ---- combine the column's nch chunk partials in chunk order (combine_ws_chain's arithmetic)
        for (int i = gt; i < G * nch; i += kGT) {
            const int g = i / nch, cc = i % nch;
            const float* w = wsb + cc * cstride + g * (HD + 4);
            cA[g * kMaxCombine + cc] = __ldcg(w);
            cLs[g * kMaxCombine + cc] = __ldcg(w + 1);
        }
        group_bar(gi);
        for (int g = wg; g < G; g += 2) {
            float M = -FLT_MAX;
            for (int cc = lane; cc < nch; cc += 32) M = fmaxf(M, cA[g * kMaxCombine + cc]);
            M = warp_max(M);
            for (int c0 = 0; c0 < nch; c0 += 32) {
                const int cc = c0 + lane;
                const float al = det_expf_shfl(cc < nch ? __fsub_rn(cA[g * kMaxCombine + cc], M) : 0.0f, tab);
                if (cc < nch) cA[g * kMaxCombine + cc] = al;
            }
        }
        group_bar(gi);
        {
            float L[G], O[G][DPT];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                L[g] = 0.0f;
#pragma unroll
                for (int k = 0; k < DPT; ++k) O[g][k] = 0.0f;
            }
            const float* wo = wsb + 4 + gt * DPT;
            constexpr int U = 4;
            for (int c0 = 0; c0 < nch; c0 += U) {
                float ov[U][G][DPT];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        if (c0 + u < nch) {
                            if constexpr (DPT == 2) {
                                const float2 t = __ldcg(reinterpret_cast<const float2*>(wo + (c0 + u) * cstride + g * (HD + 4)));
                                ov[u][g][0] = t.x;
                                ov[u][g][1] = t.y;
                            } else {
                                ov[u][g][0] = __ldcg(wo + (c0 + u) * cstride + g * (HD + 4));
                            }
                        }
                    }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (c0 + u >= nch) break;
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float al = cA[g * kMaxCombine + c0 + u];
                        L[g] = __fmaf_rn(cLs[g * kMaxCombine + c0 + u], al, L[g]);
#pragma unroll
                        for (int k = 0; k < DPT; ++k) O[g][k] = __fmaf_rn(ov[u][g][k], al, O[g][k]);
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int k = 0; k < DPT; ++k) outp[g * HD + gt * DPT + k] = f2bf(__fdiv_rn(O[g][k], L[g]));
        }
        group_bar(gi);   // the combine scratch aliases the next chunk's q / scores
    }
}

template <int HD, int G>
cudaError_t launch_stream_hg(const AttnParams& a, cudaStream_t stream, bool pdl) {
    using C = Cfg<HD, G>;
    static std::atomic<uint64_t> attr_devs{0};
    static int n_sm[64] = {0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(attn_stream_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::DYN);
        if (e != cudaSuccess) return e;
        int sms = 0;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if (dev < 64) n_sm[dev] = sms;
        attrs_done(attr_devs, dev);
    }
    int sms = dev < 64 ? n_sm[dev] : 0;
    if (sms <= 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::DYN;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(HD)));
    return cudaLaunchKernelEx(&cfg, attn_stream_kernel<HD, G>, a, *a.tm_k, *a.tm_v, scale);
}

}  // namespace

bool attention_stream_supported(const AttnParams& a) {
    if (a.tm_k == nullptr || a.tm_v == nullptr || !a.decode) return false;
    if (a.page != kAttnChunk || a.ncols > kMaxCols || a.max_chunks > kMaxCombine) return false;
    if (a.hkv <= 0 || a.hq % a.hkv != 0) return false;
    const int G = a.hq / a.hkv;
    return (a.hd == 128 && (G == 1 || G == 2 || G == 4)) || (a.hd == 64 && (G == 1 || G == 2 || G == 4));
}

cudaError_t launch_attention_stream(const AttnParams& a, cudaStream_t stream, bool pdl) {
    if (!attention_stream_supported(a)) return cudaErrorInvalidValue;
    const int G = a.hq / a.hkv;
    if (a.hd == 128) {
        switch (G) {
            case 1: return launch_stream_hg<128, 1>(a, stream, pdl);
            case 2: return launch_stream_hg<128, 2>(a, stream, pdl);
            default: return launch_stream_hg<128, 4>(a, stream, pdl);
        }
    }
    switch (G) {
        case 1: return launch_stream_hg<64, 1>(a, stream, pdl);
        case 2: return launch_stream_hg<64, 2>(a, stream, pdl);
        default: return launch_stream_hg<64, 4>(a, stream, pdl);
    }
}

}  // namespace detgpu
