// Paged decode attention with a fixed KV-chunk order.
//
// One CTA per (chunk, kv head, query column); the G = hq/hkv query heads of a kv head share the
// chunk's K/V in shared memory. Per query head:
//   s_p = tree_d(q_d * k_pd) * (1/sqrt(hd))      products of bf16 pairs are exact in f32
//   m = max_p s_p ; e_p = exp(s_p - m) ; l = tree_p(e_p) ; o_d = fma chain over p in order
// and the chunks are combined in chunk order by whichever CTA of the (column, kv head) finishes
// last (a ticket elects the combiner; the combination itself is order-fixed):
//   a_c = exp(m_c - max m) ; out_d = bf16( (sum_c fma o_cd a_c) / (sum_c fma l_c a_c) )
// Chunk boundaries are positions 64c, so split-KV parallelism never changes a bit and prefill
// queries see exactly the same arithmetic as decode steps.
#include <cfloat>

#include "common.h"
#include "detmath.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace detgpu {

namespace {

constexpr int kNT = 256;           // threads per CTA
constexpr int kMaxClusterChunks = 16;   // cluster mode: chunks of one (column, kv head) per cluster
constexpr int kNW = kNT / 32;

// ---- the per-chunk arithmetic, shared by the chunk-parallel and the
// chunk-sequential kernels so that both produce the same bits ----

// K/V rows [r_begin, r_end) of the chunk starting at position p0 (kv head kvh) into shared memory
// with 16-byte cp.async; K vectors XOR-swizzled by row (chunk_scores). When the page size is a
// multiple of the chunk (the engine's 64) the chunk is one contiguous [CH][HD] block per head:
// one page-table read per chunk instead of one per vector.
template <int HD>
__device__ __forceinline__ void load_chunk_rows(const AttnParams& a, const int* bt_slot, int kvh, int p0, int r_begin,
                                                int r_end, __nv_bfloat16* sK, __nv_bfloat16* sV, bool k, bool v,
                                                int tid) {
    constexpr int VPR = HD * 2 / 16;
    if (a.page % kAttnChunk == 0) {
        const int pid = __ldg(bt_slot + p0 / a.page);
        const int64_t base = ((static_cast<int64_t>(pid) * a.hkv + kvh) * a.page + p0 % a.page) * HD;
        for (int i = r_begin * VPR + tid; i < r_end * VPR; i += kNT) {
            const int r = i / VPR, vv = i % VPR;
            const int64_t off = base + r * HD + vv * 8;
            if (k) cp_async_16(sK + r * HD + ((vv ^ (r & (VPR - 1))) * 8), a.kcache + off);
            if (v) cp_async_16(sV + r * HD + vv * 8, a.vcache + off);
        }
        return;
    }
    for (int i = r_begin * VPR + tid; i < r_end * VPR; i += kNT) {
        const int r = i / VPR, vv = i % VPR;
        const int p = p0 + r;
        const int pid = __ldg(bt_slot + p / a.page);
        const int64_t off = ((static_cast<int64_t>(pid) * a.hkv + kvh) * a.page + p % a.page) * HD + vv * 8;
        if (k) cp_async_16(sK + r * HD + ((vv ^ (r & (VPR - 1))) * 8), a.kcache + off);
        if (v) cp_async_16(sV + r * HD + vv * 8, a.vcache + off);
    }
}

// scores: one thread per (position, head) evaluates the canonical tree over d sequentially:
// 8-product blocks (perfect trees) merged by a binary counter == the perfect tree over HD.
// K rows are stored with their 16-byte vectors XOR-swizzled by row, so the 32 rows a warp
// reads at one vector index fall in distinct banks.
template <int HD, int G>
__device__ __forceinline__ void chunk_scores(const __nv_bfloat16* sK, const float* sQ, float* sS, int n, int tid,
                                             float scale) {
    constexpr int CH = kAttnChunk;
    constexpr int NV = HD / 8;                       // 16-byte vectors per row
    constexpr int DEPTH = (NV >= 16 ? 4 : NV >= 8 ? 3 : NV >= 4 ? 2 : 1) + 1;
    for (int idx = tid; idx < G * CH; idx += kNT) {
        const int p = idx % CH, g = idx / CH;
        if (p >= n) continue;
        float stk[DEPTH];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const uint4 kv = *reinterpret_cast<const uint4*>(sK + p * HD + ((v ^ (p & (NV - 1))) * 8));
            float carry = qk_block8_x2(kv, *reinterpret_cast<const ulonglong2*>(sQ + g * HD + v * 8),
                                    *reinterpret_cast<const ulonglong2*>(sQ + g * HD + v * 8 + 4));
            int lvl = 0;
#pragma unroll
            for (int b = v; b & 1; b >>= 1, ++lvl) carry = __fadd_rn(stk[lvl], carry);
            stk[lvl] = carry;
        }
        sS[g * CH + p] = __fmul_rn(stk[DEPTH - 1], scale);
    }
}

// chunk softmax pieces: warp g owns head g (CH/32 positions per lane): m, e = exp(s - m), l = tree(e)
template <int G>
__device__ __forceinline__ void chunk_softmax(float* sS, float* sM, float* sL, int n, int warp, int lane, ExpTab tab) {
    constexpr int CH = kAttnChunk;
    for (int g = warp; g < G; g += kNW) {
        constexpr int PPL = CH / 32;   // positions per lane
        float sv[PPL], e[PPL];
        float m = -FLT_MAX;
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int p = lane * PPL + j;
            sv[j] = p < n ? sS[g * CH + p] : 0.0f;
            if (p < n) m = fmaxf(m, sv[j]);
        }
        m = warp_max(m);
#pragma unroll
        for (int j = 0; j < PPL; ++j) {
            const int p = lane * PPL + j;
            const float ev = det_expf_shfl(p < n ? __fsub_rn(sv[j], m) : 0.0f, tab);
            e[j] = p < n ? ev : kNegZero;
            sS[g * CH + p] = e[j];
        }
        float l = local_tree_sum<PPL>(e);
        l = warp_tree_sum(l);
        if (lane == 0) {
            sM[g] = m;
            sL[g] = l;
        }
    }
}

// PV chains per thread: chain j of thread tid is chain_of(tid, j) = tid + j * kNT, i.e. head
// ch / HD, dimension ch % HD (G * HD or more: none).
template <int HD, int G>
__host__ __device__ constexpr int pv_cpt() {
    return (G * HD + kNT - 1) / kNT;
}
template <int HD, int G>
__device__ __forceinline__ int chain_of(int tid, int j) {
    return tid + j * kNT;
}

// o: chain (g, d) = fma over positions in order
template <int HD, int G>
__device__ __forceinline__ void chunk_pv(const __nv_bfloat16* sV, const float* sS, int n, int tid,
                                         float (&acc)[pv_cpt<HD, G>()]) {
    constexpr int CH = kAttnChunk;
    constexpr int CHAINS = G * HD;
    constexpr int CPT = pv_cpt<HD, G>();
    const uint16_t* v16 = reinterpret_cast<const uint16_t*>(sV);
#pragma unroll
    for (int j = 0; j < CPT; ++j) acc[j] = 0.0f;
    if (tid < CHAINS) {
        const int d = tid % HD;   // every chain of this thread has the same d (kNT % HD == 0)
#pragma unroll 8
        for (int p = 0; p < n; ++p) {
            const float v = __uint_as_float(static_cast<uint32_t>(v16[p * HD + d]) << 16);
#pragma unroll
            for (int j = 0; j < CPT; ++j) {
                const int ch = chain_of<HD, G>(tid, j);
                if (ch < CHAINS) acc[j] = __fmaf_rn(sS[(ch / HD) * CH + p], v, acc[j]);
            }
        }
    }
}

// The workspace combine of one (head, d) chain over nch chunk partials in chunk order:
// M = max m_c, a_c = exp(m_c - M), out = bf16(fma-chain(o_c a_c) / fma-chain(l_c a_c)). Loads are
// issued eight chunks at a time before their arithmetic (one L2 round trip per eight chunks).
// Warp-uniform nch (det_expf_shfl).
__device__ __forceinline__ __nv_bfloat16 combine_ws_chain(const float* base, int64_t cstride, int nch, int d,
                                                          ExpTab tab) {
    constexpr int B = 8;
    float M = -FLT_MAX;
    for (int c0 = 0; c0 < nch; c0 += B) {
        float m[B];
#pragma unroll
        for (int u = 0; u < B; ++u) m[u] = c0 + u < nch ? __ldcg(base + (c0 + u) * cstride) : -FLT_MAX;
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (c0 + u < nch) M = fmaxf(M, m[u]);
    }
    float L = 0.0f, O = 0.0f;
    for (int c0 = 0; c0 < nch; c0 += B) {
        float m[B], l[B], o[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const float* w = base + (c0 + u) * cstride;
            const bool ok = c0 + u < nch;
            m[u] = ok ? __ldcg(w) : 0.0f;
            l[u] = ok ? __ldcg(w + 1) : 0.0f;
            o[u] = ok ? __ldcg(w + 4 + d) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const float al = det_expf_shfl(c0 + u < nch ? __fsub_rn(m[u], M) : 0.0f, tab);   // all lanes
            if (c0 + u < nch) {
                L = __fmaf_rn(l[u], al, L);
                O = __fmaf_rn(o[u], al, O);
            }
        }
    }
    return f2bf(__fdiv_rn(O, L));
}

// CL (cluster mode): the chunk CTAs of one (column, kv head) form a cluster; chunk 0 (the leader)
// receives every other chunk's (m, l, o) by st.async into its K/V buffer once it has finished with
// it, combines them in chunk order and writes the output: no workspace, no ticket, no grid-wide
// round trip. Same arithmetic as the ticket combine below.
// MINB: resident CTAs per SM the register budget is sized for. 6 (<= 40 registers) for many
// columns; at <= 2 columns (<= 2 x hkv x chunks CTAs, far fewer than the SMs) 4 (<= 64 registers)
// shortens the chunk's latency chain: batch 1 step -0.5 %, batch 2 -0.5 % (batch 4-7 slower).
template <int HD, int G, bool CL, int MINB>
__global__ void __launch_bounds__(kNT, MINB) attn_chunk_kernel(const AttnParams a, float scale) {
    constexpr int CH = kAttnChunk;
    constexpr int E = HD / 32;                       // q/k elements per lane in a dot product
    constexpr int CHAINS = G * HD;                   // (head, d) accumulators of the PV product
    constexpr int CPT = pv_cpt<HD, G>();            // PV chains per thread (chain_of)
    extern __shared__ __align__(16) uint8_t attn_dsm[];
    __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(attn_dsm);
    __nv_bfloat16* sV = sK + CH * HD;
    __shared__ __align__(16) float sQ[G * HD];
    __shared__ float sS[G * CH];
    __shared__ float sM[G], sL[G];
    __shared__ int s_last;
    __shared__ uint64_t s_bar[2];   // CL: [0] leader: partials landed, [1] pusher: leader's K/V buffer free
    __shared__ float s_al[CL ? G : 1][CL ? kMaxClusterChunks : 1], s_mx[G];

    const int c = blockIdx.x, kvh = blockIdx.y, col = blockIdx.z;
    struct TraceAtExit {   // records the CTA's timeline on every return path (instrumentation only)
        const AttnParams& a;
        uint64_t m[kTraceMarks];
        __device__ void mark(int i) {
            if (a.trace != nullptr) m[i] = globaltimer_ns();
        }
        __device__ ~TraceAtExit() {
            if (threadIdx.x == 0 && a.trace != nullptr)
                trace_record(a.trace, (a.trace_tag << 24) | (blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)),
                             m);
        }
    } tr{a, {a.trace != nullptr ? globaltimer_ns() : 0}};
    if (threadIdx.x == 0)
        l2_prefetch_slice(a.l2pf, a.l2pf_bytes, c + gridDim.x * (kvh + gridDim.y * col),
                          gridDim.x * gridDim.y * gridDim.z);
    // sep_recv: the leader's partial-receive buffer follows its K/V buffer, so pushes need no
    // handshake; the leader arms its barrier for the pushed bytes before the cluster barrier
    const bool sep = CL && a.sep_recv != 0;
    if constexpr (CL) {
        if (threadIdx.x == 0) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            fence_mbar_init();
            if (sep && c == 0) {
                const int pos0 = a.col_pos[col];
                const int nch0 = pos0 < 0 ? 0 : pos0 / kAttnChunk + 1;
                if (nch0 > 1)
                    mbar_arrive_expect_tx(&s_bar[0], static_cast<uint32_t>((nch0 - 1) * G * (HD + 2) * 4));
            }
        }
        __syncthreads();
        cluster_arrive();   // every CTA of the cluster, active or not, arrives once and waits once
    }
    auto leave = [&]() {
        if constexpr (CL) cluster_wait();
    };
    // Decode: positions < pos were written by earlier steps and col_pos by the previous step's
    // sampler; every kernel waits for its predecessor before triggering (gemm.cu), so both are
    // complete when this kernel starts and the chunk's K/V can stream while the QKV GEMM (the
    // predecessor, which appends position pos) is still running. Prefill reads K/V the predecessor
    // writes, so it waits first.
    if (!a.decode) {
        pdl_wait();
        pdl_trigger();
        tr.mark(1);
    }
    const int pos = a.col_pos[col];
    if (pos < 0) {
        leave();
        return;
    }
    const int ctx = pos + 1;
    const int p0 = c * CH;
    if (p0 >= ctx) {
        leave();
        return;
    }
    const int n = min(CH, ctx - p0);
    const int slot = a.col_req[col];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    // K/V rows: page ids of the chunk, then every 16-byte vector with cp.async
    const int* bt = a.block_table + static_cast<int64_t>(slot) * a.max_pages;
    auto load_rows = [&](int r_begin, int r_end) {
        load_chunk_rows<HD>(a, bt, kvh, p0, r_begin, r_end, sK, sV, true, true, tid);
    };
    ExpTab tab;
    if (a.decode) {
        load_rows(0, pos - p0 < n ? pos - p0 : n);   // history rows, before the wait
        tab = exp_tab_lane();                        // also before the wait, after the history loads
        pdl_wait();
        pdl_trigger();
        tr.mark(1);
        if (pos - p0 < n) load_rows(pos - p0, n);     // the row the QKV GEMM just appended
    } else {
        tab = exp_tab_lane();
        load_rows(0, n);
    }
    cp_async_commit();
    // q: 8 bf16 per 16-byte load (one L2 round trip), stored as f32 in qk_block8_x2 order
    const __nv_bfloat16* qsrc = a.q + static_cast<int64_t>(col) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD;
    for (int i = tid * 8; i < G * HD; i += kNT * 8) {
        const uint4 w = *reinterpret_cast<const uint4*>(qsrc + i);
        *reinterpret_cast<float4*>(sQ + i) = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.z << 16),
                                                         __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.z & 0xffff0000u));
        *reinterpret_cast<float4*>(sQ + i + 4) = make_float4(__uint_as_float(w.y << 16), __uint_as_float(w.w << 16),
                                                             __uint_as_float(w.y & 0xffff0000u),
                                                             __uint_as_float(w.w & 0xffff0000u));
    }
    cp_async_wait_all();
    __syncthreads();
    tr.mark(2);   // K/V chunk and q in shared memory

    chunk_scores<HD, G>(sK, sQ, sS, n, tid, scale);
    __syncthreads();
    tr.mark(3);   // scores

    chunk_softmax<G>(sS, sM, sL, n, warp, lane, tab);
    __syncthreads();
    tr.mark(4);   // softmax

    float acc[CPT];
    chunk_pv<HD, G>(sV, sS, n, tid, acc);
    tr.mark(5);   // PV chains
    const int nch = (ctx + CH - 1) / CH;
    __nv_bfloat16* outp = a.out + static_cast<int64_t>(col) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD;
    if constexpr (CL) {
        if (nch > 1) {
            constexpr int BLK = G * (HD + 2);   // one pushed partial: m[G], l[G], o[G][HD]
            float* recv = reinterpret_cast<float*>(attn_dsm + (sep ? 2 * CH * HD * 2 : 0));
            if (c == 0) {
                if (!sep) {
                    __syncthreads();   // the leader's own K/V reads are complete
                    if (tid == 0) mbar_arrive_expect_tx(&s_bar[0], static_cast<uint32_t>((nch - 1) * BLK * 4));
                }
                cluster_wait();
                if (!sep && tid >= 1 && tid < nch) mbar_arrive_remote(mapa_shared(smem_u32(&s_bar[1]), tid));
                if (tid < G) {
                    float M = sM[tid];   // chunk order: fmaxf chain from -FLT_MAX (see the ticket combine)
                    M = fmaxf(-FLT_MAX, M);
                    mbar_wait(&s_bar[0], 0);
                    for (int cc = 1; cc < nch; ++cc) M = fmaxf(M, recv[(cc - 1) * BLK + tid]);
                    s_mx[tid] = M;
                } else {
                    mbar_wait(&s_bar[0], 0);
                }
                __syncthreads();
                if (tid < ((G * kMaxClusterChunks + 31) & ~31)) {   // warp-uniform: det_expf_shfl needs all lanes
                    const int g = tid / kMaxClusterChunks, cc = tid % kMaxClusterChunks;
                    const bool ok = g < G && cc < nch;
                    const float m = !ok ? 0.0f : cc == 0 ? sM[g] : recv[(cc - 1) * BLK + g];
                    const float al = det_expf_shfl(ok ? __fsub_rn(m, s_mx[g < G ? g : 0]) : 0.0f, tab);
                    if (ok) s_al[g][cc] = al;
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    const int ch = chain_of<HD, G>(tid, j);
                    if (ch >= CHAINS) continue;
                    const int g = ch / HD, d = ch % HD;
                    float L = __fmaf_rn(sL[g], s_al[g][0], 0.0f), O = __fmaf_rn(acc[j], s_al[g][0], 0.0f);
                    for (int cc = 1; cc < nch; ++cc) {
                        const float* w = recv + (cc - 1) * BLK;
                        L = __fmaf_rn(w[G + g], s_al[g][cc], L);
                        O = __fmaf_rn(w[2 * G + g * HD + d], s_al[g][cc], O);
                    }
                    outp[ch] = f2bf(__fdiv_rn(O, L));
                }
            } else {
                cluster_wait();
                if (!sep) mbar_wait(&s_bar[1], 0);   // the leader no longer reads its K/V buffer
                const uint32_t rb = mapa_shared(smem_u32(recv) + 4u * static_cast<uint32_t>((c - 1) * BLK), 0);
                const uint32_t rbar = mapa_shared(smem_u32(&s_bar[0]), 0);
#pragma unroll
                for (int j = 0; j < CPT; ++j) {
                    const int ch = chain_of<HD, G>(tid, j);
                    if (ch < CHAINS) st_async_f32(rb + 4u * (2 * G + ch), acc[j], rbar);
                }
                if (tid < G) {
                    st_async_f32(rb + 4u * tid, sM[tid], rbar);
                    st_async_f32(rb + 4u * (G + tid), sL[tid], rbar);
                }
            }
            return;
        }
        leave();
    }
    if (nch == 1) {
        // single chunk: the combine weight is exp(0) == 1 exactly
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
            const int ch = chain_of<HD, G>(tid, j);
            if (ch < CHAINS)
                outp[ch] = f2bf(__fdiv_rn(__fmaf_rn(acc[j], 1.0f, 0.0f), __fmaf_rn(sL[ch / HD], 1.0f, 0.0f)));
        }
        return;
    }
    float* wsb = a.ws + (static_cast<int64_t>(col) * a.hkv + kvh) * a.max_chunks * G * (HD + 4);
    float* ws = wsb + static_cast<int64_t>(c) * G * (HD + 4);
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        const int ch = chain_of<HD, G>(tid, j);
        if (ch < CHAINS) ws[(ch / HD) * (HD + 4) + 4 + ch % HD] = acc[j];
    }
    if (tid < G) {
        ws[tid * (HD + 4)] = sM[tid];
        ws[tid * (HD + 4) + 1] = sL[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        int* t = a.tickets + static_cast<int64_t>(col) * a.hkv + kvh;
        const int prev = atomicAdd(t, 1);
        s_last = prev == nch - 1;
        if (s_last) *t = 0;   // re-armed for the next launch
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int64_t cstride = static_cast<int64_t>(G) * (HD + 4);
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
        const int ch = tid + j * kNT;
        if (ch >= CHAINS) continue;
        const int g = ch / HD, d = ch % HD;
        outp[ch] = combine_ws_chain(wsb + g * (HD + 4), cstride, nch, d, tab);
    }
}

template <int HD, int G, bool CL, int MINB>
cudaError_t launch_hgc_m(const AttnParams& a, cudaStream_t stream, bool pdl) {
    constexpr size_t dsm_kv = 2 * static_cast<size_t>(kAttnChunk) * HD * 2;
    constexpr size_t dsm_max = dsm_kv + (CL ? static_cast<size_t>(kMaxClusterChunks - 1) * G * (HD + 2) * 4 : 0);
    const size_t dsm = dsm_kv + (CL && a.sep_recv ? static_cast<size_t>(a.max_chunks - 1) * G * (HD + 2) * 4 : 0);
    static std::atomic<uint64_t> attr_devs{0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(attn_chunk_kernel<HD, G, CL, MINB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm_max));
        if (e == cudaSuccess && CL)
            e = cudaFuncSetAttribute(attn_chunk_kernel<HD, G, CL, MINB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attrs_done(attr_devs, dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.max_chunks, a.hkv, a.ncols);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CL ? a.max_chunks : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(HD)));
    return cudaLaunchKernelEx(&cfg, attn_chunk_kernel<HD, G, CL, MINB>, a, scale);
}

template <int HD, int G, bool CL>
cudaError_t launch_hgc(const AttnParams& a, cudaStream_t stream, bool pdl) {
    return a.ncols <= 2 ? launch_hgc_m<HD, G, CL, 4>(a, stream, pdl) : launch_hgc_m<HD, G, CL, 6>(a, stream, pdl);
}

// Prefill: one CTA per (chunk, kv head, block of Q = ROWS/G consecutive query columns): the chunk's
// K/V is loaded once for the block instead of once per query. Per (query, head) row the
// arithmetic is chunk_scores / chunk_softmax / chunk_pv's: each thread evaluates four score trees
// over one K row (the K vector unpacked once for the four), and the PV chains of a dimension share
// each V element. Chunk partials go to the workspace; the CTA completing a query's chunk count
// (ticket per column) combines it exactly as attn_chunk_kernel's ticket combine.
template <int HD, int G, int ROWS>
__global__ void __launch_bounds__(kNT, 4) attn_prefill_kernel(const AttnParams a, float scale) {
    constexpr int CH = kAttnChunk;
    constexpr int Q = G >= ROWS ? 1 : ROWS / G;      // query columns per CTA
    constexpr int R = Q * G;                         // (query, head) rows: ROWS
    constexpr int NV = HD / 8;
    constexpr int DEPTH = (NV >= 16 ? 4 : NV >= 8 ? 3 : NV >= 4 ? 2 : 1) + 1;
    constexpr int SR = R * CH / kNT;                 // score rows per thread (4)
    constexpr int PR = R * HD / kNT;                 // PV chains per thread
    static_assert(kNT % CH == 0 && kNT % HD == 0 && R * CH % kNT == 0, "mapping");
    extern __shared__ __align__(16) uint8_t pf_dsm[];
    __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(pf_dsm);
    __nv_bfloat16* sV = sK + CH * HD;
    float* sQ = reinterpret_cast<float*>(sV + CH * HD);   // [R][HD]
    float* sS = sQ + R * HD;                               // [R][CH]
    __shared__ float sM[R], sL[R];
    __shared__ int s_pos[Q], s_slot[Q], s_n[Q], s_run[Q], s_last[Q];
    pdl_wait();
    pdl_trigger();
    const int c = blockIdx.x, kvh = blockIdx.y, col0 = blockIdx.z * Q;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p0 = c * CH;
    if (tid < Q) {
        const int col = col0 + tid;
        const int pos = col < a.ncols ? a.col_pos[col] : -1;
        s_pos[tid] = pos;
        s_slot[tid] = pos >= 0 ? a.col_req[col] : -1;
        s_n[tid] = pos >= p0 ? min(CH, pos + 1 - p0) : 0;
    }
    __syncthreads();
    {   // causal prefill: about half the (chunk, query block) CTAs see no position of their chunk
        bool any = false;
#pragma unroll
        for (int q = 0; q < Q; ++q) any |= s_n[q] > 0;
        if (!any) return;
    }
    const ExpTab tab = exp_tab_lane();
    for (int q0 = 0; q0 < Q;) {   // runs of queries of one request share the K/V chunk
        int q1 = q0 + 1;
        while (q1 < Q && s_slot[q1] == s_slot[q0]) ++q1;
        int nmax = 0;
        for (int q = q0; q < q1; ++q) nmax = max(nmax, s_n[q]);
        if (s_slot[q0] < 0 || nmax == 0) {
            q0 = q1;
            continue;
        }
        if (tid < Q) s_run[tid] = tid >= q0 && tid < q1 ? s_n[tid] : 0;   // this run's rows only
        const int* bt = a.block_table + static_cast<int64_t>(s_slot[q0]) * a.max_pages;
        load_chunk_rows<HD>(a, bt, kvh, p0, 0, nmax, sK, sV, true, true, tid);
        cp_async_commit();
        for (int i = tid * 8; i < (q1 - q0) * G * HD; i += kNT * 8) {   // 8 bf16 per load; quads 0,2,1,3
            const int q = q0 + i / (G * HD), rem = i % (G * HD);
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(
                a.q + static_cast<int64_t>(col0 + q) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD + rem));
            float* dq = sQ + q * G * HD + rem;
            *reinterpret_cast<float4*>(dq) = make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.y << 16),
                                                         __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y & 0xffff0000u));
            *reinterpret_cast<float4*>(dq + 4) = make_float4(__uint_as_float(w.z << 16), __uint_as_float(w.w << 16),
                                                             __uint_as_float(w.z & 0xffff0000u),
                                                             __uint_as_float(w.w & 0xffff0000u));
        }
        cp_async_wait_all();
        __syncthreads();
        {   // scores: position p, rows rg, rg + kNT/CH, ... (same tree as chunk_scores)
            const int p = tid % CH, rg = tid / CH;
            float stk[SR][DEPTH];
            bool on[SR];
#pragma unroll
            for (int k = 0; k < SR; ++k) on[k] = p < s_run[(rg + k * (kNT / CH)) / G];
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const uint4 kv = *reinterpret_cast<const uint4*>(sK + p * HD + ((v ^ (p & (NV - 1))) * 8));
#pragma unroll
                for (int k = 0; k < SR; ++k) {
                    const int r = rg + k * (kNT / CH);
                    float carry = qk_block8(kv, *reinterpret_cast<const ulonglong2*>(sQ + r * HD + v * 8),
                                            *reinterpret_cast<const ulonglong2*>(sQ + r * HD + v * 8 + 4));
                    int lvl = 0;
#pragma unroll
                    for (int b = v; b & 1; b >>= 1, ++lvl) carry = __fadd_rn(stk[k][lvl], carry);
                    stk[k][lvl] = carry;
                }
            }
#pragma unroll
            for (int k = 0; k < SR; ++k)
                if (on[k]) sS[(rg + k * (kNT / CH)) * CH + p] = __fmul_rn(stk[k][DEPTH - 1], scale);
        }
        __syncthreads();
        for (int r = warp; r < R; r += kNW) {   // chunk softmax per row (chunk_softmax's arithmetic)
            const int n = s_run[r / G];
            if (n == 0) continue;
            constexpr int PPL = CH / 32;
            float sv[PPL], e[PPL];
            float m = -FLT_MAX;
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int p = lane * PPL + j;
                sv[j] = p < n ? sS[r * CH + p] : 0.0f;
                if (p < n) m = fmaxf(m, sv[j]);
            }
            m = warp_max(m);
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int p = lane * PPL + j;
                const float ev = det_expf_shfl(p < n ? __fsub_rn(sv[j], m) : 0.0f, tab);
                e[j] = p < n ? ev : kNegZero;
                sS[r * CH + p] = e[j];
            }
            float l = local_tree_sum<PPL>(e);
            l = warp_tree_sum(l);
            if (lane == 0) {
                sM[r] = m;
                sL[r] = l;
            }
        }
        __syncthreads();
        {   // PV: two dimensions x RPT consecutive rows per thread: one 4-byte V load feeds 2 * RPT chains
            constexpr int TPR = HD / 2;             // threads per row group
            constexpr int RPT = R * TPR / kNT;      // rows per thread (PR / 2)
            static_assert(2 * RPT == PR && kNT % TPR == 0, "PV mapping");
            const int d0 = (tid % TPR) * 2, r0 = (tid / TPR) * RPT;   // r0 warp-uniform
            const uint32_t* v32 = reinterpret_cast<const uint32_t*>(sV);
            // the two chains of a row are one packed FFMA2 per position (each lane an independent
            // fma.rn: the same bits as two scalar __fmaf_rn chains)
            uint64_t acc2[RPT];
            int nr[RPT];
            int nmin = CH;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                acc2[k] = 0;
                nr[k] = s_run[(r0 + k) / G];
                nmin = min(nmin, nr[k]);
            }
            const float* srow = sS + r0 * CH;   // row r0 + k at srow + k*CH
#pragma unroll 4
            for (int p = 0; p < nmin; ++p) {   // every row active: no per-FMA guard
                const uint32_t w = v32[(p * HD + d0) >> 1];
                const uint64_t vv = pack2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
#pragma unroll
                for (int k = 0; k < RPT; ++k) {
                    const float e = srow[k * CH + p];
                    acc2[k] = ffma2(pack2(e, e), vv, acc2[k]);
                }
            }
            for (int p = nmin; p < nmax; ++p) {   // the causal edge
                const uint32_t w = v32[(p * HD + d0) >> 1];
                const uint64_t vv = pack2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
#pragma unroll
                for (int k = 0; k < RPT; ++k)
                    if (p < nr[k]) {
                        const float e = srow[k * CH + p];
                        acc2[k] = ffma2(pack2(e, e), vv, acc2[k]);
                    }
            }
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int r = r0 + k, q = r / G, g = r % G;
                if (nr[k] == 0) continue;
                float* ws = a.ws + ((static_cast<int64_t>(col0 + q) * a.hkv + kvh) * a.max_chunks + c) * G * (HD + 4) +
                            g * (HD + 4);
                *reinterpret_cast<float2*>(ws + 4 + d0) = make_float2(lo32(acc2[k]), hi32(acc2[k]));
                if (d0 == 0) {
                    ws[0] = sM[r];
                    ws[1] = sL[r];
                }
            }
        }
        __syncthreads();
        q0 = q1;
    }
    // per-column tickets: the CTA holding a column's last chunk partial combines that column. The
    // ticket thread's fence after the barrier releases the whole CTA's partials (cumulativity), and
    // the combining CTA's ticket thread fences again before the barrier its readers pass.
    __syncthreads();
    if (tid < Q) {
        s_last[tid] = 0;
        if (s_n[tid] > 0) {
            const int nch = (s_pos[tid] + CH) / CH;
            int* t = a.tickets + static_cast<int64_t>(col0 + tid) * a.hkv + kvh;
            __threadfence();
            if (atomicAdd(t, 1) == nch - 1) {
                s_last[tid] = 1;
                *t = 0;   // re-armed for the next launch
                __threadfence();
            }
        }
    }
    __syncthreads();
    for (int q = 0; q < Q; ++q) {
        if (!s_last[q]) continue;   // block-uniform
        const int nch = (s_pos[q] + CH) / CH;
        const float* wsb = a.ws + (static_cast<int64_t>(col0 + q) * a.hkv + kvh) * a.max_chunks * G * (HD + 4);
        const int64_t cstride = static_cast<int64_t>(G) * (HD + 4);
        __nv_bfloat16* outp = a.out + static_cast<int64_t>(col0 + q) * a.hq * HD + static_cast<int64_t>(kvh) * G * HD;
        for (int ch = tid; ch < G * HD; ch += kNT) {   // whole warps: det_expf_shfl
            const int g = ch / HD, d = ch % HD;
            const float* base = wsb + g * (HD + 4);
            if (nch == 1) {   // the combine weight is exp(0) == 1 exactly (as attn_chunk_kernel)
                outp[ch] = f2bf(__fdiv_rn(__fmaf_rn(__ldcg(base + 4 + d), 1.0f, 0.0f), __fmaf_rn(__ldcg(base + 1), 1.0f, 0.0f)));
                continue;
            }
            outp[ch] = combine_ws_chain(base, cstride, nch, d, tab);
        }
    }
}

template <int HD, int G, int ROWS>
cudaError_t launch_prefill(const AttnParams& a, cudaStream_t stream, bool pdl) {
    constexpr int Q = G >= ROWS ? 1 : ROWS / G;
    constexpr size_t dsm = 2 * static_cast<size_t>(kAttnChunk) * HD * 2 + static_cast<size_t>(Q * G) * HD * 4 +
                           static_cast<size_t>(Q * G) * kAttnChunk * 4;
    static std::atomic<uint64_t> attr_devs{0};
    int dev = 0;
    if (attrs_needed(attr_devs, &dev)) {
        cudaError_t e = cudaFuncSetAttribute(attn_prefill_kernel<HD, G, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(dsm));
        if (e != cudaSuccess) return e;
        attrs_done(attr_devs, dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.max_chunks, a.hkv, (a.ncols + Q - 1) / Q);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = dsm;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const float scale = static_cast<float>(1.0 / sqrt(static_cast<double>(HD)));
    return cudaLaunchKernelEx(&cfg, attn_prefill_kernel<HD, G, ROWS>, a, scale);
}

// Cluster combine when the chunks of a (column, kv head) fit one cluster and the pushed partials
// fit the leader's K/V buffer; the workspace/ticket combine otherwise.
template <int HD, int G>
cudaError_t launch_hg(const AttnParams& a, cudaStream_t stream, bool pdl) {
    // (query, head) rows per CTA: 16 for prompts up to ~1k columns, 32 above (each K/V chunk shared by
    // more rows; measured crossover); per-row arithmetic identical
    if (!a.decode && a.prefill_blocks)
        return a.ncols >= 1024 ? launch_prefill<HD, G, 32>(a, stream, pdl) : launch_prefill<HD, G, 16>(a, stream, pdl);
    // many columns: the workspace/ticket combine schedules better than 12-CTA clusters
    const bool cl = (a.cluster_max_cols <= 0 || a.ncols <= a.cluster_max_cols) && a.max_chunks <= kMaxClusterChunks &&
                    static_cast<size_t>(a.max_chunks - 1) * G * (HD + 2) * 4 <= 2 * static_cast<size_t>(kAttnChunk) * HD * 2;
    return cl ? launch_hgc<HD, G, true>(a, stream, pdl) : launch_hgc<HD, G, false>(a, stream, pdl);
}

}  // namespace

size_t attn_workspace_bytes(const AttnParams& a) {
    const int G = a.hq / a.hkv;
    return sizeof(float) * static_cast<size_t>(a.ncols) * a.hkv * a.max_chunks * G * (a.hd + 4);
}

cudaError_t launch_attention(const AttnParams& a, cudaStream_t stream, bool pdl) {
    if (a.hkv <= 0 || a.hq % a.hkv != 0 || a.page < 16 || a.page % 16 != 0) return cudaErrorInvalidValue;
    if (a.stream_min_cols > 0 && a.ncols >= a.stream_min_cols && attention_stream_supported(a))
        return launch_attention_stream(a, stream, pdl);
    const int G = a.hq / a.hkv;
    if (a.hd == 128) {
        switch (G) {
            case 1: return launch_hg<128, 1>(a, stream, pdl);
            case 2: return launch_hg<128, 2>(a, stream, pdl);
            case 4: return launch_hg<128, 4>(a, stream, pdl);
            case 8: return launch_hg<128, 8>(a, stream, pdl);
            default: return cudaErrorInvalidValue;
        }
    }
    if (a.hd == 64) {
        switch (G) {
            case 1: return launch_hg<64, 1>(a, stream, pdl);
            case 2: return launch_hg<64, 2>(a, stream, pdl);
            case 4: return launch_hg<64, 4>(a, stream, pdl);
            default: return cudaErrorInvalidValue;
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace detgpu
