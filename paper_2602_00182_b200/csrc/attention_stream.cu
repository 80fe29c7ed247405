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
// * four chunk groups take the ring's chunks round robin (chunk j -> group j % 4); a chunk group is
//   HS consumer groups of 64 threads, each owning G/HS of the kv head's query heads (scores,
//   softmax, PV chains). A consumer group hands its chunk partial (o, m, l) to the combiner warps
//   through its shared-memory scratch and moves on to its next chunk;
// * the combiner warps take the partials in chunk order: they store them to the workspace (or, for
//   a one-chunk item, finish the output), and when a (column, kv head) item is complete (its last
//   chunk in this CTA's range; an item split between two CTAs' ranges also counts a global
//   ticket) they combine it. The workspace stores, the completion count and the combine are thus
//   off the consumers' critical path.
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
constexpr int kGroups = 4;                 // chunk groups (chunk j -> group j % kGroups)
constexpr int kGT = 64;                    // threads per consumer group (two warps)
constexpr int kPT = 64;                    // copier threads (two warps)
constexpr int kCT = 128;                   // combiner threads (four warps)
constexpr int kMaxCols = 256;              // columns staged in shared memory
constexpr int kMaxCombine = 128;           // chunks per (column, kv head): contexts up to 8192
constexpr int kCopyBar = 14;               // named barrier of the copier warps
constexpr int kCombBar = 15;               // named barrier of the combiner warps
// Head split: each chunk group is HS consumer groups of 64 threads, each owning G/HS of the kv
// head's query heads for the whole chunk. The per-(head, position) and per-(head, dim)
// arithmetic is unchanged, so the split never changes a bit.
template <int G>
struct Split {
#ifndef DETGPU_ATTN_HS
#define DETGPU_ATTN_HS 1   // 2: measured slower (each half re-reads K and V: shared-memory traffic)
#endif
    static constexpr int HS = G % DETGPU_ATTN_HS == 0 ? DETGPU_ATTN_HS : 1;
    static constexpr int GH = G / HS;                        // query heads per consumer group
    static constexpr int NCG = kGroups * HS;                 // consumer groups
    static constexpr int PRODUCER_WARP = NCG * kGT / 32;
    static constexpr int COPY_WARP0 = PRODUCER_WARP + 1;
    static constexpr int COMB_WARP0 = COPY_WARP0 + kPT / 32;
    static constexpr int THREADS = NCG * kGT + 32 + kPT + kCT;   // + producer, copier, combiner warps
};

template <int HD, int G>
struct Cfg {
    using SP = Split<G>;
    static constexpr int GH = SP::GH;
    static constexpr int KB = kCH * HD * 2;                       // K (or V) bytes of one chunk
    static constexpr int QB = G * HD * 2;                         // the column's q for this kv head
    static constexpr int STAGE = (2 * KB + QB + 1023) / 1024 * 1024;
    static constexpr int S = HD == 128 ? 6 : 8;                   // ring stages
    // consumer group scratch: q f32 [GH][HD], scores [GH][64], e [64][GH], m [GH], l [GH]
    static constexpr int SCR = (GH * (HD + 2 * kCH) * 4 + 2 * GH * 4 + 15) / 16 * 16;
    static constexpr int CBUF = 2 * G * kMaxCombine * 4;          // one item's (m or a_c, l) per chunk
    static constexpr int DYN = 1024 + S * STAGE + SP::NCG * SCR + 2 * CBUF;   // + alignment slack
    static constexpr int DPT = HD / kGT;                          // PV dimensions per consumer thread
    static constexpr int PDT = G * HD / kPT;                      // copied dimensions per copier thread
    static constexpr int CDT = G * HD / kCT > 0 ? G * HD / kCT : 1;   // combine dimensions per thread
    static constexpr int CTA_ACTIVE = G * HD / CDT;               // combiner threads with output
    // hand-off in the stage's K area once both halves are past their scores: o [G][HD], m [G], l [G]
    static constexpr int HO_ML = G * HD * 4;
    static_assert(HO_ML + 2 * G * 4 <= KB, "hand-off fits the K area");
};

__device__ __forceinline__ void group_bar(int g) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(kGT) : "memory");
}
__device__ __forceinline__ void comb_bar() {
    asm volatile("bar.sync %0, %1;" ::"r"(kCombBar), "r"(kCT) : "memory");
}
__device__ __forceinline__ void copy_bar() {
    asm volatile("bar.sync %0, %1;" ::"r"(kCopyBar), "r"(kPT) : "memory");
}
// both consumer groups of chunk group gi (head split): barrier 1 + NCG + gi
__device__ __forceinline__ void chunk_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(2 * kGT) : "memory");
}
// combine queue entry: one per (column, kv head) item this CTA touches, in chunk order
struct CombItem {
    int col, kvh, nch;
    int mode;   // 0: nothing to combine here, 1: combine with (m, l) staged, 2: reload (m, l), 3: end
};

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
__global__ void __launch_bounds__(Split<G>::THREADS, 1)
    attn_stream_kernel(const AttnParams a, const __grid_constant__ CUtensorMap tmK,
                       const __grid_constant__ CUtensorMap tmV, float scale) {
    using C = Cfg<HD, G>;
    using SP = Split<G>;
    constexpr int HS = SP::HS, GH = SP::GH, NCG = SP::NCG, kThreads = SP::THREADS;
    constexpr int S = C::S;
    constexpr int NV = HD / 8;
    constexpr int DEPTH = (NV >= 16 ? 4 : NV >= 8 ? 3 : NV >= 4 ? 2 : 1) + 1;
    constexpr int DPT = C::DPT;
    static_assert(HD == 64 || HD == 128, "head dim");
    static_assert(G >= 1 && G <= 4, "group size");
    static_assert(1 + NCG + kGroups <= kCopyBar, "named barriers");
    extern __shared__ uint8_t st_dsm[];
    // 1024-byte aligned ring (128B-swizzled TMA boxes); offset arithmetic on the shared array keeps
    // every access an LDS (a pointer rebuilt from an integer would be generic)
    uint8_t* ring = st_dsm + ((1024u - (smem_u32(st_dsm) & 1023u)) & 1023u);
    uint8_t* scr_all = ring + S * C::STAGE;
    // two combine buffers [2][G][kMaxCombine]: m (then a_c) and l of each chunk of an item
    float* cbuf = reinterpret_cast<float*>(scr_all + NCG * C::SCR);
    __shared__ uint64_t full[S], empty[S];
    __shared__ uint64_t pready[S];              // consumers -> copier: the stage holds the hand-off
    __shared__ uint64_t qfull[2], qempty[2];    // copier -> combiner queue
    __shared__ CombItem qdesc[2];
    __shared__ int4 sinfo[S];
    __shared__ int s_pos[kMaxCols], s_pref[kMaxCols + 1];
    __shared__ int s_last;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ncols = a.ncols;
    for (int i = tid; i < ncols; i += kThreads) s_pos[i] = a.col_pos[i];
    if (tid < S) {
        mbar_init(&full[tid], 1);
        mbar_init(&empty[tid], kPT);
        mbar_init(&pready[tid], kGT * HS);
    }
    if (tid < 2) {
        mbar_init(&qfull[tid], 1);
        mbar_init(&qempty[tid], kCT);
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
    const ExpTab tab = exp_tab_lane();
    const int64_t cstride = static_cast<int64_t>(G) * (HD + 4);   // workspace [col][kvh][chunk][head][4 + HD]

    if (warp == SP::PRODUCER_WARP) {
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
        // (prefill: the predecessor writes every chunk's K/V of the prompt, so everything waits)
        const bool early = a.decode != 0;
        if (lane < nfirst) {
            ci0 = locate(lane);
            pid0 = page_of(ci0);
            publish(lane, ci0);
            if (early && ci0.c < ci0.nch - 1) issue_kv(lane, ci0, pid0);
        }
        pdl_wait();
        pdl_trigger();
        if (lane < nfirst) {
            if (!early || ci0.c == ci0.nch - 1) issue_kv(lane, ci0, pid0);
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

    if (warp >= SP::COPY_WARP0 && warp < SP::COMB_WARP0) {
        // ------------------------------------------------------------ copier
        // Takes the hand-offs in chunk order: stores each partial to the workspace (or finishes a
        // one-chunk item), stages an item's (m, l) for its combine, releases the stage, and queues
        // every item it completes here for the combiner.
        const int pt = tid - SP::COPY_WARP0 * 32;
        constexpr int PDT = C::PDT;
        const int ph = pt * PDT / HD, pd0 = pt * PDT % HD;   // this thread's head and first dimension
        int qs = -1;   // queue sequence of the current item
        auto push = [&](const CombItem& it) {
            // queue slot qs & 1 was freed by the combiner when it finished item qs - 2
            if (pt == 0) {
                qdesc[qs & 1] = it;
                mbar_arrive(&qfull[qs & 1]);
            }
        };
        for (int j = 0; j < nloc; ++j) {
            const int s = j % S;
            mbar_wait(&pready[s], (j / S) & 1, pt == 0 ? j : -1);
            const int4 inf = sinfo[s];
            const int col = inf.x, kvh = inf.y & 0xffff, c = inf.y >> 16, nch = inf.z >> 16;
            const int lcnt = inf.w & 0xff, whole = (inf.w >> 8) & 1, key = inf.w >> 9;
            const float* ho = reinterpret_cast<const float*>(ring + s * C::STAGE);   // o [G][HD], m [G], l [G]
            if (j == key) {   // the item's first chunk in this range: a new queue entry
                ++qs;
                if (qs >= 2) mbar_wait(&qempty[qs & 1], ((qs >> 1) - 1) & 1, pt == 0 ? j : -1);
            }
            float* cb = cbuf + (qs & 1) * 2 * G * kMaxCombine;
            if (nch == 1) {   // the combine weight is exp(0) == 1 exactly (as attn_chunk_kernel)
                __nv_bfloat16* outp = a.out + static_cast<int64_t>(col) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD;
                const float L = __fmaf_rn(ho[C::HO_ML / 4 + G + ph], 1.0f, 0.0f);
#pragma unroll
                for (int k = 0; k < PDT; ++k)
                    outp[ph * HD + pd0 + k] = f2bf(__fdiv_rn(__fmaf_rn(ho[ph * HD + pd0 + k], 1.0f, 0.0f), L));
            } else {
                float* w = a.ws + ((static_cast<int64_t>(col) * a.hkv + kvh) * a.max_chunks + c) * cstride;
                if constexpr (PDT % 4 == 0) {
#pragma unroll
                    for (int k = 0; k < PDT; k += 4)
                        *reinterpret_cast<float4*>(w + ph * (HD + 4) + 4 + pd0 + k) =
                            *reinterpret_cast<const float4*>(ho + ph * HD + pd0 + k);
                } else {
#pragma unroll
                    for (int k = 0; k < PDT; ++k) w[ph * (HD + 4) + 4 + pd0 + k] = ho[ph * HD + pd0 + k];
                }
                if (pt < G) {
                    const float m = ho[C::HO_ML / 4 + pt], l = ho[C::HO_ML / 4 + G + pt];
                    w[pt * (HD + 4)] = m;
                    w[pt * (HD + 4) + 1] = l;
                    cb[pt * kMaxCombine + c] = m;
                    cb[(G + pt) * kMaxCombine + c] = l;
                }
            }
            mbar_arrive(&empty[s]);   // stage released (its hand-off is copied)
            if (j != key + lcnt - 1) continue;   // not the item's last chunk in this range
            CombItem it{col, kvh, nch, 0};
            if (nch > 1) {
                if (whole) {
                    it.mode = 1;
                } else {   // an item spanning CTAs: the CTA completing its global ticket combines
                    copy_bar();   // every copier thread's partial stores precede thread 0's release
                    if (pt == 0) {
                        __threadfence();
                        int* tk = a.tickets + static_cast<int64_t>(col) * a.hkv + kvh;
                        const int last = atomicAdd(tk, lcnt) + lcnt == nch;
                        if (last) {
                            *tk = 0;   // re-armed for the next launch
                            __threadfence();
                        }
                        s_last = last;
                    }
                    copy_bar();
                    it.mode = s_last ? 2 : 0;
                }
            }
            // the copier threads' workspace stores are ordered before the combiner's reads: every
            // copier thread fences (CTA scope) and the queue entry is published after the barrier
            __threadfence_block();
            copy_bar();
            push(it);
        }
        ++qs;
        if (qs >= 2) mbar_wait(&qempty[qs & 1], ((qs >> 1) - 1) & 1, pt == 0 ? nloc : -1);
        push(CombItem{0, 0, 0, 3});
        return;
    }

    if (warp >= SP::COMB_WARP0) {
        // ------------------------------------------------------------ combiner
        const int ct = tid - SP::COMB_WARP0 * 32, cw = ct >> 5;
        constexpr int CDT = C::CDT;
        const int ch = ct * CDT / HD, cd0 = ct * CDT % HD;   // this thread's head and first dimension
        const bool cact = ct < C::CTA_ACTIVE;
        for (int qs = 0;; ++qs) {
            mbar_wait(&qfull[qs & 1], (qs >> 1) & 1, ct == 0 ? qs : -1);
            const CombItem it = qdesc[qs & 1];
            if (it.mode == 3) break;
            float* cA = cbuf + (qs & 1) * 2 * G * kMaxCombine;   // [G][kMaxCombine] m, then a_c
            float* cLs = cA + G * kMaxCombine;                   // [G][kMaxCombine] l
            const int nch = it.nch;
            float* wsb = a.ws + (static_cast<int64_t>(it.col) * a.hkv + it.kvh) * a.max_chunks * cstride;
            if (it.mode != 0) {
                if (it.mode == 2) {   // chunks of another CTA's range: (m, l) from the workspace
                    for (int i = ct; i < G * nch; i += kCT) {
                        const int g = i / nch, cc = i % nch;
                        const float* w = wsb + cc * cstride + g * (HD + 4);
                        cA[g * kMaxCombine + cc] = __ldcg(w);
                        cLs[g * kMaxCombine + cc] = __ldcg(w + 1);
                    }
                }
                comb_bar();
                // ---- combine the item's nch chunk partials in chunk order (combine_ws_chain's arithmetic)
                for (int g = cw; g < G; g += kCT / 32) {
                    float M = -FLT_MAX;
                    for (int cc = lane; cc < nch; cc += 32) M = fmaxf(M, cA[g * kMaxCombine + cc]);
                    M = warp_max(M);
                    for (int c0 = 0; c0 < nch; c0 += 32) {
                        const int cc = c0 + lane;
                        const float al = det_expf_shfl(cc < nch ? __fsub_rn(cA[g * kMaxCombine + cc], M) : 0.0f, tab);
                        if (cc < nch) cA[g * kMaxCombine + cc] = al;
                    }
                }
                comb_bar();
                if (cact) {
                    __nv_bfloat16* outp =
                        a.out + static_cast<int64_t>(it.col) * a.hq * HD + static_cast<int64_t>(it.kvh) * G * HD;
                    float L = 0.0f, O[CDT];
#pragma unroll
                    for (int k = 0; k < CDT; ++k) O[k] = 0.0f;
                    const float* wo = wsb + ch * (HD + 4) + 4 + cd0;
                    constexpr int U = 8;   // partials in flight per round trip
                    for (int c0 = 0; c0 < nch; c0 += U) {
                        float ov[U][CDT];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (c0 + u < nch) {
                                if constexpr (CDT == 4) {
                                    const float4 t4 = __ldcg(reinterpret_cast<const float4*>(wo + (c0 + u) * cstride));
                                    ov[u][0] = t4.x;
                                    ov[u][1] = t4.y;
                                    ov[u][2] = t4.z;
                                    ov[u][3] = t4.w;
                                } else if constexpr (CDT == 2) {
                                    const float2 t2 = __ldcg(reinterpret_cast<const float2*>(wo + (c0 + u) * cstride));
                                    ov[u][0] = t2.x;
                                    ov[u][1] = t2.y;
                                } else {
#pragma unroll
                                    for (int k = 0; k < CDT; ++k) ov[u][k] = __ldcg(wo + (c0 + u) * cstride + k);
                                }
                            }
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (c0 + u >= nch) break;
                            const float al = cA[ch * kMaxCombine + c0 + u];
                            L = __fmaf_rn(cLs[ch * kMaxCombine + c0 + u], al, L);
#pragma unroll
                            for (int k = 0; k < CDT; ++k) O[k] = __fmaf_rn(ov[u][k], al, O[k]);
                        }
                    }
#pragma unroll
                    for (int k = 0; k < CDT; ++k) outp[ch * HD + cd0 + k] = f2bf(__fdiv_rn(O[k], L));
                }
            }
            mbar_arrive(&qempty[qs & 1]);   // the queue slot and its combine buffer are free
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // consumer group cg (64 threads) = half hh of chunk group gi; it owns query heads
    // g0 .. g0 + GH - 1 of every chunk the chunk group takes
    const int cg = warp >> 1, gi = cg / HS, hh = cg % HS, gt = tid & (kGT - 1), wg = warp & 1;
    const int g0 = hh * GH;
    float* gQ = reinterpret_cast<float*>(scr_all + cg * C::SCR);   // [GH][HD], 8-blocks as q0 q4 q1 q5 q2 q6 q3 q7 (qk_block8_x2)
    float* gS = gQ + GH * HD;                                       // [GH][64] scores
    float* gE = gS + GH * kCH;                                      // [64][GH] exp(s - m)
    float* gM = gE + kCH * GH;                                      // [GH] chunk max
    float* gL = gM + GH;                                            // [GH] l

    for (int j = gi; j < nloc; j += kGroups) {
        const int s = j % S;
        // Stage s is consumed by different chunk groups on successive uses (S is not a multiple of
        // the group count), so this group has not itself waited for the stage's previous use j - S:
        // while that phase is still in flight, a parity wait for chunk j passes at once (the
        // phase-parity ABA). First wait until chunk j - S has been released (empty[s] phase k - 1;
        // exact: phase k - 2 is complete, since the producer published chunk j - S, and phase k is
        // this group's own release of chunk j), after which full[s] is in phase k or k + 1 and the
        // parity wait for chunk j is exact.
        const int k = j / S;
        if (k > 0) mbar_wait(&empty[s], (k - 1) & 1, gt == 0 ? j : -1);
        mbar_wait(&full[s], k & 1, gt == 0 ? j : -1);
        const int4 inf = sinfo[s];
        const int n = inf.z & 0xffff;
        const uint8_t* st = ring + s * C::STAGE;
        const uint16_t* sq = reinterpret_cast<const uint16_t*>(st + 2 * C::KB) + g0 * HD;
        for (int i = gt * 8; i < GH * HD; i += kGT * 8) {   // q -> f32, each 8-block as q0 q4 q1 q5 q2 q6 q3 q7
            const uint4 w = *reinterpret_cast<const uint4*>(sq + i);
            *reinterpret_cast<float4*>(gQ + i) = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.z << 16),
                                                             __uint_as_float(w.x & 0xffff0000u),
                                                             __uint_as_float(w.z & 0xffff0000u));
            *reinterpret_cast<float4*>(gQ + i + 4) = make_float4(__uint_as_float(w.y << 16), __uint_as_float(w.w << 16),
                                                                 __uint_as_float(w.y & 0xffff0000u),
                                                                 __uint_as_float(w.w & 0xffff0000u));
        }
        group_bar(cg);
        // scores: thread = position, the group's GH heads over the same unpacked K row
        if (gt < n) {
            const int p = gt;
            const uint32_t kbase = static_cast<uint32_t>(p * 128);
            float stk[GH][DEPTH];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint4 kv = *reinterpret_cast<const uint4*>(st + kbase + (((v & 7) ^ (p & 7)) << 4) + (v >> 3) * (kCH * 128));
#pragma unroll
                for (int g = 0; g < GH; ++g) {
                    float carry = qk_block8_x2(kv, *reinterpret_cast<const ulonglong2*>(gQ + g * HD + v * 8),
                                               *reinterpret_cast<const ulonglong2*>(gQ + g * HD + v * 8 + 4));
                    int lvl = 0;
#pragma unroll
                    for (int bb = v; bb & 1; bb >>= 1, ++lvl) carry = __fadd_rn(stk[g][lvl], carry);
                    stk[g][lvl] = carry;
                }
            }
#pragma unroll
            for (int g = 0; g < GH; ++g) gS[g * kCH + p] = __fmul_rn(stk[g][DEPTH - 1], scale);
        }
        // both halves are done with K before either writes its hand-off over it
        if constexpr (HS > 1) chunk_bar(1 + NCG + gi);
        else group_bar(cg);
        // chunk softmax (chunk_softmax's arithmetic): warp wg owns heads wg, wg + 2, ...
        for (int g = wg; g < GH; g += 2) {
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
                gE[p * GH + g] = e[q];
            }
            float l = local_tree_sum<PPL>(e);
            l = warp_tree_sum(l);
            if (lane == 0) {
                gM[g] = m;
                gL[g] = l;
            }
        }
        group_bar(cg);
        // PV: thread = DPT dimensions x GH heads; fma chains over positions in order. With two
        // dimensions per thread the pair of chains of one head is one packed FFMA2 per position
        // (each lane an independent fma.rn: the same bits as two scalar __fmaf_rn chains).
        float acc[GH][DPT];
        {
            const int d0 = gt * DPT;
            const uint8_t* sV = st + C::KB;
            uint32_t voff[8];   // swizzled offset of (row r, d0) for r = p mod 8; rows 8 apart are 1 KB apart
#pragma unroll
            for (int r = 0; r < 8; ++r) voff[r] = swz(r, d0);
            auto load_e = [&](int p, float (&ev)[GH]) {
                if constexpr (GH == 2) {
                    const float2 e2 = *reinterpret_cast<const float2*>(gE + p * 2);
                    ev[0] = e2.x;
                    ev[1] = e2.y;
                } else {
#pragma unroll
                    for (int g = 0; g < GH; ++g) ev[g] = gE[p * GH + g];
                }
            };
            if constexpr (DPT == 2) {
                uint64_t acc2[GH];
#pragma unroll
                for (int g = 0; g < GH; ++g) acc2[g] = 0;
                auto pv_step = [&](int p, uint32_t off) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(sV + off);
                    const uint64_t vv = pack2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
                    float ev[GH];
                    load_e(p, ev);
#pragma unroll
                    for (int g = 0; g < GH; ++g) acc2[g] = ffma2(pack2(ev[g], ev[g]), vv, acc2[g]);
                };
                int p = 0;
                for (; p + 8 <= n; p += 8) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) pv_step(p + r, voff[r] + p * 128);
                }
                for (; p < n; ++p) pv_step(p, swz(p, d0));
#pragma unroll
                for (int g = 0; g < GH; ++g) {
                    acc[g][0] = lo32(acc2[g]);
                    acc[g][1] = hi32(acc2[g]);
                }
            } else {
#pragma unroll
                for (int g = 0; g < GH; ++g)
#pragma unroll
                    for (int k = 0; k < DPT; ++k) acc[g][k] = 0.0f;
                auto pv_step = [&](int p, uint32_t off) {
                    const float v0 = __uint_as_float(static_cast<uint32_t>(*reinterpret_cast<const uint16_t*>(sV + off)) << 16);
                    float ev[GH];
                    load_e(p, ev);
#pragma unroll
                    for (int g = 0; g < GH; ++g) acc[g][0] = __fmaf_rn(ev[g], v0, acc[g][0]);
                };
                int p = 0;
                for (; p + 8 <= n; p += 8) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) pv_step(p + r, voff[r] + p * 128);
                }
                for (; p < n; ++p) pv_step(p, swz(p, d0));
            }
        }
        // hand-off in the stage's K area: o [G][HD] (this group's heads), m [G], l [G]; the arrive
        // releases these stores to the copier (CTA scope), which releases the stage
        float* ho = reinterpret_cast<float*>(ring + s * C::STAGE);
#pragma unroll
        for (int g = 0; g < GH; ++g) {
            if constexpr (DPT == 2)
                *reinterpret_cast<float2*>(ho + (g0 + g) * HD + gt * 2) = make_float2(acc[g][0], acc[g][1]);
            else
#pragma unroll
                for (int k = 0; k < DPT; ++k) ho[(g0 + g) * HD + gt * DPT + k] = acc[g][k];
        }
        if (gt < GH) {
            ho[C::HO_ML / 4 + g0 + gt] = gM[gt];
            ho[C::HO_ML / 4 + G + g0 + gt] = gL[gt];
        }
        mbar_arrive(&pready[s]);
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
    cfg.blockDim = dim3(Split<G>::THREADS);
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
    if (a.tm_k == nullptr || a.tm_v == nullptr || (!a.decode && !a.stream_prefill)) return false;
    if (a.page != kAttnChunk || (a.decode && a.ncols > kMaxCols) || a.max_chunks > kMaxCombine) return false;
    if (a.hkv <= 0 || a.hq % a.hkv != 0) return false;
    const int G = a.hq / a.hkv;
    return (a.hd == 128 && (G == 1 || G == 2 || G == 4)) || (a.hd == 64 && (G == 1 || G == 2 || G == 4));
}

cudaError_t launch_attention_stream(const AttnParams& a_in, cudaStream_t stream, bool pdl) {
    if (!attention_stream_supported(a_in)) return cudaErrorInvalidValue;
    if (a_in.ncols > kMaxCols) {   // prefill chunks: consecutive launches of <= kMaxCols columns each
        const int G = a_in.hq / a_in.hkv;
        const int64_t cstride = static_cast<int64_t>(G) * (a_in.hd + 4);
        for (int c0 = 0; c0 < a_in.ncols; c0 += kMaxCols) {
            AttnParams a = a_in;
            a.ncols = a_in.ncols - c0 < kMaxCols ? a_in.ncols - c0 : kMaxCols;
            a.col_pos += c0;
            a.col_req += c0;
            a.q += static_cast<int64_t>(c0) * a.hq * a.hd;
            a.out += static_cast<int64_t>(c0) * a.hq * a.hd;
            a.ws += static_cast<int64_t>(c0) * a.hkv * a.max_chunks * cstride;
            a.tickets += static_cast<int64_t>(c0) * a.hkv;
            if (c0 > 0) a.l2pf_bytes = 0;
            const cudaError_t e = launch_attention_stream(a, stream, pdl);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
    const AttnParams& a = a_in;
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
