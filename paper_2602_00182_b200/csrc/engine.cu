// The deterministic inference engine: weights, paged KV cache, prefill + decode loop (CUDA graph
// per batch size), host receipt hashing, and the engine part of the C-ABI (include/detgpu.h).
//
// Reference path replaced: detcore::infer / infer_batch (reference proj/src/detcore.cpp:319-410)
// and out_hash = SHA-256(canonical_bytes) (proj/src/receipts.cpp:120). One engine = one GPU
// replica; requests of a generate() call are decoded in groups of batch_size with per-request
// state (prng, position, trace step) living in device memory.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <future>
#include <deque>
#include <thread>
#include <vector>

#include "common.h"
#include "detgpu.h"
#include "digest.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "model.h"
#include "receipt.h"
#include "toy.cuh"

namespace detgpu {

namespace {

constexpr int kPage = 64;          // KV positions per page
constexpr int kPrefillCols = 2048; // max activation columns per forward pass

// Every engine buffer is followed by a canary region (kCanaryBytes of 0xA5). compute-sanitizer is
// not available on the GPU pool, so detgpu_debug_check_canaries() is the out-of-bounds-write
// check the tests run after their workloads (tests/test_gpu_engine.py, tools/sanitize_run.py).
constexpr size_t kCanaryBytes = 4096;
struct CanaryReg {
    std::mutex mu;
    std::map<void*, std::pair<size_t, int>> live;   // base -> (payload bytes, device)
};
CanaryReg& canaries() {
    static CanaryReg r;
    return r;
}
template <class T>
cudaError_t dalloc(T** p, size_t count) {
    const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), bytes + kCanaryBytes);
    if (e != cudaSuccess) return e;
    e = cudaMemset(reinterpret_cast<uint8_t*>(*p) + bytes, 0xA5, kCanaryBytes);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(canaries().mu);
    canaries().live[*p] = {bytes, dev};
    return cudaSuccess;
}
void dfree(void* p) {
    if (p == nullptr) return;
    {
        std::lock_guard<std::mutex> lk(canaries().mu);
        canaries().live.erase(p);
    }
    cudaFree(p);
}

struct Layer {
    __nv_bfloat16 *attn_norm = nullptr, *wqkv = nullptr, *wo = nullptr, *ffn_norm = nullptr, *wgu = nullptr,
                  *wdown = nullptr;
    CUtensorMap tm_qkv, tm_o, tm_gu, tm_down;
};

}  // namespace

struct Engine {
    int device = 0;
    std::string model_id, arch;
    ModelConfig cfg{};
    bool toy = false;
    uint32_t max_batch = 0, max_context = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    std::vector<void*> allocs;

    // weights
    __nv_bfloat16 *embed = nullptr, *lm_head = nullptr, *final_norm = nullptr;
    CUtensorMap tm_lm;
    CUtensorMap tm_kpool, tm_vpool;   // whole K / V pools as [rows][hd] (streamed decode attention)
    std::vector<Layer> layers;
    uint64_t n_params = 0;
    // activations
    int col_cap = 0;
    float* x = nullptr;
    __nv_bfloat16 *h = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr, *h_last = nullptr;
    // KV cache (paged, static page ownership per slot)
    __nv_bfloat16 *kpool = nullptr, *vpool = nullptr;
    int pages_per_slot = 0, total_pages = 0, max_chunks = 0;
    int* block_table = nullptr;
    float* attn_ws = nullptr;
    float* norm_ss = nullptr;   // [cols][d/128] per-tile sums of squares (fused-norm decode)
    int* attn_tickets = nullptr;
    float *rope_cos = nullptr, *rope_sin = nullptr;
    // prefill plan
    int *p_tok = nullptr, *p_pos = nullptr, *p_req = nullptr, *p_last_in = nullptr, *p_last_out = nullptr;
    // per-slot decode state
    int *d_tok = nullptr, *d_pos = nullptr, *d_req = nullptr, *d_step = nullptr, *d_status = nullptr;
    uint64_t* d_prng = nullptr;
    DevPolicy* d_pol = nullptr;
    float* probs = nullptr;
    uint64_t* sort_scratch = nullptr;
    float* sample_ws = nullptr;     // multi-CTA sampler: per-row block max / subtree sums
    int* sample_tickets = nullptr;
    // outputs (grown on demand)
    float* trace = nullptr;
    size_t trace_cap = 0;
    uint32_t* tok_hist = nullptr;
    uint8_t* d_roots = nullptr;   // receipt v2: [slot][tcap][32] per-step Merkle roots
    int* d_steps = nullptr;       // receipt v2: steps per slot
    size_t roots_cap = 0;
    size_t tok_cap = 0;
    int64_t slot_stride = 0;
    int tcap = 0;
    // pinned staging for D2H
    float* pinned[2] = {nullptr, nullptr};
    size_t pinned_floats = 0;
    // pinned host buffers for traces hashed off the decode loop (collect_slot), reused once their
    // hashing task is done
    struct HashBuf {
        float* p = nullptr;
        size_t cap = 0;
        std::shared_future<void> busy;
    };
    std::deque<HashBuf> hash_bufs;   // deque: growing it never moves a buffer in use
    size_t hash_next = 0;            // round-robin victim when every buffer is busy
    // decode graphs keyed by (ncols, slot_stride)
    std::map<std::pair<int, int64_t>, cudaGraphExec_t> graphs;
    std::map<std::pair<int, int64_t>, uint64_t> graph_used;   // LRU stamps (get_graph)
    uint64_t graph_clock = 0;
    // pinned host staging for the serving loop's small H2D copies (admission state, prefill
    // plans): ring of buffers, each reused only after the event recorded behind its copies
    struct Stage {
        void* p = nullptr;
        size_t cap = 0;
        cudaEvent_t ev = nullptr;
        bool pending = false;
    };
    Stage stage[4];
    int stage_next = 0;
    uint64_t launches_per_step = 0;
    bool use_pdl = true;
    // toy model
    ToyWeights toyw{};

    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<std::pair<cudaEvent_t, int>>* prof = nullptr;
    unsigned skip_mask = 0;   // timing experiments only (detgpu_profile_graph): kernel classes left out
    // Decode: which kernels warm the NEXT kernel's weights into L2 at their start (bit 0: attention ->
    // o, 1: o -> gate/up, 2: gate/up -> down, 3: down -> next QKV, 4: QKV -> o), at most l2pf_cap
    // bytes each. Scheduling only: results are unaffected. DETGPU_L2PF / DETGPU_L2PF_MB override.
    // Default: the o-projection warms the first 16 MB of gate/up (tools/l2pf_scan.py).
    unsigned l2pf_mask = 2;
    // per-GEMM overrides of self_pf_kb (-1: self_pf_kb), order qkv, o, gate/up, down, lm_head. The
    // down GEMM launches during the gate/up tail, where its prefetch competes with gate/up's own
    // stream; for o and down 0 measured best (tools/l2pf_scan.py, batch 1: -1.5 % and -0.4 %)
    int self_pf_kb_cls[5] = {-1, 0, -1, 0, -1};
    int self_pf_kb = 4;   // GemmParams::self_pf_kb (tools/l2pf_scan.py: 4 beat 8 by ~1 % at batch 1 and 8)
    int gemm_pair = 0;    // GemmParams::pair: CTA-pair (cta_group::2) GEMMs above 64 columns
    // GemmParams::persist: persistent double-buffered GEMMs above 64 columns. Bit-identical and
    // faster standalone for S = 2, but slower inside the PDL pipeline (one CTA per SM: the next
    // kernel cannot start streaming during the tail; tools/persist_ab.py), so off by default.
    int gemm_persist = 0;
    int max_nsub = 0;     // GemmParams::max_nsub
    bool prefill_blocks = true;   // AttnParams::prefill_blocks
    int fuse_max_cols = 8;           // decode RMSNorm fused into the consuming GEMMs up to this many columns (<= 8)
    int attn_stream_min_cols = 8;    // AttnParams::stream_min_cols (0: off); 8: batch 8 3.95 -> 3.86 ms, 5-7 slower (tools/l2pf_scan.py)
    bool mixed_steps = true;         // continuous batching: admitted prompts' last prefill chunk + one decode step in one forward
    int attn_stream_prefill = 1;     // AttnParams::stream_prefill: 512-token prefill 18.45 -> 17.21 ms, 2,000 tokens 107.3 -> 98.7 ms
    int attn_sep_recv_max_cols = 2;   // AttnParams::sep_recv up to this many columns (0: never)
    int attn_cluster_max_cols = 8;   // AttnParams::cluster_max_cols (crossover measured with tools/l2pf_scan.py)
    TraceRec* trace_buf = nullptr;   // per-CTA timeline (detgpu_set_option "trace"), instrumentation only
    int64_t l2pf_cap = 16ll << 20;

    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        cudaError_t e = dalloc(p, count);
        if (e == cudaSuccess) allocs.push_back(*p);
        return e;
    }
    ~Engine() {
        cudaSetDevice(device);
        for (auto& g : graphs) cudaGraphExecDestroy(g.second);
        for (void* p : allocs) dfree(p);
        if (trace) dfree(trace);
        if (trace_buf) cudaFree(trace_buf);
        for (auto& hb : hash_bufs) {
            if (hb.busy.valid()) hb.busy.wait();
            if (hb.p) cudaFreeHost(hb.p);
        }
        if (tok_hist) dfree(tok_hist);
        if (d_roots) dfree(d_roots);
        if (d_steps) dfree(d_steps);
        for (float* p : pinned)
            if (p) cudaFreeHost(p);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& st : stage) {
            if (st.ev) cudaEventSynchronize(st.ev), cudaEventDestroy(st.ev);
            if (st.p) cudaFreeHost(st.p);
        }
        toy_free(toyw);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace {

int fail(Engine* e, int code, const std::string& msg) {
    if (e) e->err = msg;
    set_global_error(msg);
    return code;
}

constexpr size_t kMaxGraphs = 24;
constexpr uint32_t kBosToken = 0;   // what an empty b200 prompt means (detgpu_generate)

// Next pinned staging buffer of at least `bytes` (waits only if its previous copies are still
// queued); stage_release() records the event behind the copies issued from it.
cudaError_t stage_acquire(Engine* E, size_t bytes, void** out, int* idx) {
    const int i = E->stage_next++ % 4;
    Engine::Stage& st = E->stage[i];
    cudaError_t e = cudaSuccess;
    if (st.ev == nullptr && (e = cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    if (st.pending && (e = cudaEventSynchronize(st.ev)) != cudaSuccess) return e;
    st.pending = false;
    if (st.cap < bytes) {
        if (st.p) cudaFreeHost(st.p);
        st.p = nullptr;
        st.cap = 0;
        if ((e = cudaHostAlloc(&st.p, bytes, cudaHostAllocDefault)) != cudaSuccess) return e;
        st.cap = bytes;
    }
    *out = st.p;
    *idx = i;
    return cudaSuccess;
}
cudaError_t stage_release(Engine* E, int idx) {
    E->stage[idx].pending = true;
    return cudaEventRecord(E->stage[idx].ev, E->stream);
}

#define ENG_CUDA(expr)                                                                                 \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess) return fail(E, DETGPU_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

int init_weights(Engine* E) {
    const ModelConfig& c = E->cfg;
    const int d = c.d, qd = c.hq * c.hd, kd = c.hkv * c.hd, F = c.F, V = c.V;
    const int sd = -half_log2_round(d), sq = -half_log2_round(qd), sf = -half_log2_round(F);
    const uint64_t base = fnv1a64(E->model_id.c_str());
    auto seed = [&](int tid) { return mix_seed(base, static_cast<uint64_t>(tid)); };
    cudaStream_t s = E->stream;
    ENG_CUDA(E->alloc(&E->embed, size_t(V) * d));
    ENG_CUDA(E->alloc(&E->lm_head, size_t(V) * d));
    ENG_CUDA(E->alloc(&E->final_norm, d));
    ENG_CUDA(launch_init_tensor(E->embed, seed(0), V, d, 0, 0, 1, 0, s));
    ENG_CUDA(launch_init_tensor(E->lm_head, seed(1), V, d, 4 + sd, 0, 1, 0, s, true));
    ENG_CUDA(launch_init_tensor(E->final_norm, seed(2), 1, d, 0, 1, 1, 0, s));
    if (!make_tmap_weights(&E->tm_lm, E->lm_head, V, d, true)) return fail(E, DETGPU_ECUDA, "tensor map (lm_head)");
    E->n_params = 2ull * V * d + d;
    E->layers.resize(c.L);
    for (int l = 0; l < c.L; ++l) {
        Layer& Ly = E->layers[l];
        ENG_CUDA(E->alloc(&Ly.attn_norm, d));
        ENG_CUDA(E->alloc(&Ly.ffn_norm, d));
        ENG_CUDA(E->alloc(&Ly.wqkv, size_t(qd + 2 * kd) * d));
        ENG_CUDA(E->alloc(&Ly.wo, size_t(d) * qd));
        ENG_CUDA(E->alloc(&Ly.wgu, size_t(2 * F) * d));
        ENG_CUDA(E->alloc(&Ly.wdown, size_t(d) * F));
        ENG_CUDA(launch_init_tensor(Ly.attn_norm, seed(layer_tensor_id(l, kAttnNorm)), 1, d, 0, 1, 1, 0, s));
        ENG_CUDA(launch_init_tensor(Ly.ffn_norm, seed(layer_tensor_id(l, kFfnNorm)), 1, d, 0, 1, 1, 0, s));
        // fused QKV rows: [wq ; wk ; wv]
        ENG_CUDA(launch_init_tensor(Ly.wqkv, seed(layer_tensor_id(l, kWq)), qd, d, sd, 0, 1, 0, s, true));
        ENG_CUDA(launch_init_tensor(Ly.wqkv, seed(layer_tensor_id(l, kWk)), kd, d, sd, 0, 1, qd, s, true));
        ENG_CUDA(launch_init_tensor(Ly.wqkv, seed(layer_tensor_id(l, kWv)), kd, d, sd, 0, 1, qd + kd, s, true));
        ENG_CUDA(launch_init_tensor(Ly.wo, seed(layer_tensor_id(l, kWo)), d, qd, sq, 0, 1, 0, s, true));
        // gate/up interleaved by row: physical 2j = gate j, 2j+1 = up j (SwiGLU epilogue pairs)
        ENG_CUDA(launch_init_tensor(Ly.wgu, seed(layer_tensor_id(l, kWgate)), F, d, sd, 0, 2, 0, s, true));
        ENG_CUDA(launch_init_tensor(Ly.wgu, seed(layer_tensor_id(l, kWup)), F, d, sd, 0, 2, 1, s, true));
        ENG_CUDA(launch_init_tensor(Ly.wdown, seed(layer_tensor_id(l, kWdown)), d, F, sf, 0, 1, 0, s, true));
        if (!make_tmap_weights(&Ly.tm_qkv, Ly.wqkv, qd + 2 * kd, d, true) || !make_tmap_weights(&Ly.tm_o, Ly.wo, d, qd, true) ||
            !make_tmap_weights(&Ly.tm_gu, Ly.wgu, 2 * F, d, true) || !make_tmap_weights(&Ly.tm_down, Ly.wdown, d, F, true))
            return fail(E, DETGPU_ECUDA, "tensor map (layer)");
        E->n_params += 2ull * d + size_t(qd + 2 * kd) * d + size_t(d) * qd + 3ull * F * d;
    }
    return DETGPU_OK;
}

int init_buffers(Engine* E) {
    const ModelConfig& c = E->cfg;
    const int d = c.d, qd = c.hq * c.hd, kd = c.hkv * c.hd;
    const int B = static_cast<int>(E->max_batch);
    E->col_cap = std::max(B, kPrefillCols);
    const int C = E->col_cap;
    ENG_CUDA(E->alloc(&E->x, size_t(C) * d));
    ENG_CUDA(E->alloc(&E->h, size_t(C) * d));
    ENG_CUDA(E->alloc(&E->q, size_t(C) * qd));
    ENG_CUDA(E->alloc(&E->attn, size_t(C) * qd));
    ENG_CUDA(E->alloc(&E->act, size_t(C) * c.F));
    ENG_CUDA(E->alloc(&E->h_last, size_t(B) * d));
    ENG_CUDA(cudaMemsetAsync(E->h, 0, sizeof(__nv_bfloat16) * size_t(C) * d, E->stream));
    ENG_CUDA(cudaMemsetAsync(E->attn, 0, sizeof(__nv_bfloat16) * size_t(C) * qd, E->stream));
    ENG_CUDA(cudaMemsetAsync(E->act, 0, sizeof(__nv_bfloat16) * size_t(C) * c.F, E->stream));
    ENG_CUDA(cudaMemsetAsync(E->h_last, 0, sizeof(__nv_bfloat16) * size_t(B) * d, E->stream));
    // KV pool: static page ownership, slot b owns pages [b*pps, (b+1)*pps)
    E->pages_per_slot = (static_cast<int>(E->max_context) + kPage - 1) / kPage;
    E->total_pages = E->pages_per_slot * B;
    E->max_chunks = (E->pages_per_slot * kPage + kAttnChunk - 1) / kAttnChunk;
    const size_t per_layer = size_t(E->total_pages) * kPage * kd;
    ENG_CUDA(E->alloc(&E->kpool, per_layer * c.L));
    ENG_CUDA(E->alloc(&E->vpool, per_layer * c.L));
    if (!make_tmap_bf16(&E->tm_kpool, E->kpool, c.hd, per_layer * c.L / c.hd, 64) ||
        !make_tmap_bf16(&E->tm_vpool, E->vpool, c.hd, per_layer * c.L / c.hd, 64))
        return fail(E, DETGPU_ECUDA, "tensor map (kv pool)");
    std::vector<int> bt(size_t(B) * E->pages_per_slot);
    for (size_t i = 0; i < bt.size(); ++i) bt[i] = static_cast<int>(i);
    ENG_CUDA(E->alloc(&E->block_table, bt.size()));
    ENG_CUDA(cudaMemcpy(E->block_table, bt.data(), sizeof(int) * bt.size(), cudaMemcpyHostToDevice));
    {
        AttnParams a{};
        a.ncols = C;
        a.hq = c.hq;
        a.hkv = c.hkv;
        a.hd = c.hd;
        a.max_chunks = E->max_chunks;
        ENG_CUDA(E->alloc(&E->attn_ws, attn_workspace_bytes(a) / sizeof(float)));
        ENG_CUDA(E->alloc(&E->attn_tickets, size_t(C) * c.hkv));
        ENG_CUDA(E->alloc(&E->norm_ss, size_t(C) * (d / 128)));

        ENG_CUDA(cudaMemset(E->attn_tickets, 0, sizeof(int) * size_t(C) * c.hkv));
    }
    // RoPE tables, host binary64 -> f32; identical expression in the oracle.
    const int npos = static_cast<int>(E->max_context), h2 = c.hd / 2;
    std::vector<float> cs(size_t(npos) * h2), sn(size_t(npos) * h2);
    for (int p = 0; p < npos; ++p)
        for (int i = 0; i < h2; ++i) {
            const double inv = std::pow(c.theta, -2.0 * i / c.hd);
            const double ang = double(p) * inv;
            cs[size_t(p) * h2 + i] = static_cast<float>(std::cos(ang));
            sn[size_t(p) * h2 + i] = static_cast<float>(std::sin(ang));
        }
    ENG_CUDA(E->alloc(&E->rope_cos, cs.size()));
    ENG_CUDA(E->alloc(&E->rope_sin, sn.size()));
    ENG_CUDA(cudaMemcpy(E->rope_cos, cs.data(), sizeof(float) * cs.size(), cudaMemcpyHostToDevice));
    ENG_CUDA(cudaMemcpy(E->rope_sin, sn.data(), sizeof(float) * sn.size(), cudaMemcpyHostToDevice));
    ENG_CUDA(E->alloc(&E->p_tok, C));
    ENG_CUDA(E->alloc(&E->p_pos, C));
    ENG_CUDA(E->alloc(&E->p_req, C));
    ENG_CUDA(E->alloc(&E->p_last_in, B));
    ENG_CUDA(E->alloc(&E->p_last_out, B));
    ENG_CUDA(E->alloc(&E->d_tok, B));
    ENG_CUDA(E->alloc(&E->d_pos, B));
    ENG_CUDA(E->alloc(&E->d_req, B));
    ENG_CUDA(E->alloc(&E->d_step, B));
    ENG_CUDA(E->alloc(&E->d_status, B));
    ENG_CUDA(E->alloc(&E->d_prng, size_t(B) * 4));
    ENG_CUDA(E->alloc(&E->d_pol, B));
    ENG_CUDA(E->alloc(&E->probs, size_t(B) * c.V));
    ENG_CUDA(E->alloc(&E->sort_scratch, size_t(B) * c.V));
    ENG_CUDA(E->alloc(&E->sample_ws, size_t(4) * kSampleMaxBlocks * B));
    ENG_CUDA(E->alloc(&E->sample_tickets, size_t(B)));
    ENG_CUDA(cudaMemset(E->sample_tickets, 0, sizeof(int) * B));
    std::vector<int> ident(B);
    for (int i = 0; i < B; ++i) ident[i] = i;
    ENG_CUDA(cudaMemcpy(E->d_req, ident.data(), sizeof(int) * B, cudaMemcpyHostToDevice));
    return DETGPU_OK;
}

// ------------------------------------------------------------------ forward pass
// Optional per-launch event trail (detgpu_profile_decode_step): kernel classes below.
enum ProfClass { kProfNorm = 0, kProfQkv, kProfAttn, kProfO, kProfGateUp, kProfDown, kProfLmHead, kProfSample, kProfN };
void mark(Engine* E, int cls) {
    if (E->prof == nullptr) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, E->stream);
    E->prof->push_back({ev, cls});
}
GemmParams gemm_base(const Engine* E, const void* w, int n_out, int k, int ncols) {
    GemmParams p{};
    p.w_raw = w;
    p.self_pf_kb = E->self_pf_kb;
    p.max_nsub = E->max_nsub;
    p.pair = E->gemm_pair;
    p.persist = E->gemm_persist;
    p.w_tiled = 1;   // engine weights are stored pre-tiled
    p.mma_wide = 1;  // one N = 64*sub-tiles MMA per K step: column bits identical (tools/wide_mma_check.py)

    p.n_out = n_out;
    p.k = k;
    p.ncols = ncols;
    p.trace = E->trace_buf;
    return p;
}

// All layers for `ncols` columns. Input: tokens/pos/req per column. Output: x (residual) and, when
// `final_all`, h = final_norm(x) for all columns; else h_last[out_idx[i]] = final_norm(x[in_idx[i]])
// for n_last gathered columns.
cudaError_t forward(Engine* E, int ncols, const int* tok, const int* pos, const int* req, bool final_all,
                    int n_last, uint64_t* nlaunch) {
    const ModelConfig& c = E->cfg;
    const int d = c.d, qd = c.hq * c.hd, kd = c.hkv * c.hd;
    cudaStream_t s = E->stream;
    const bool pdl = E->use_pdl;
    const size_t per_layer = size_t(E->total_pages) * kPage * kd;
    cudaError_t e;
    uint64_t n = 0;
    // activation tensor maps over exactly `ncols` rows: the MMA's padding rows are TMA zero-fill
    CUtensorMap tm_h, tm_attn, tm_act;
    if (!make_tmap_bf16(&tm_h, E->h, d, ncols, 64) || !make_tmap_bf16(&tm_attn, E->attn, qd, ncols, 64) ||
        !make_tmap_bf16(&tm_act, E->act, c.F, ncols, 64))
        return cudaErrorInvalidValue;
    // Decode with <= 8 columns: RMSNorm is fused into the consuming GEMMs (QKV, gate/up, lm_head),
    // which build their B operand from the f32 residual stream; bits are identical.
    const bool fuse = final_all && ncols <= E->fuse_max_cols;
    e = launch_embed(E->embed, tok, E->x, fuse ? E->norm_ss : nullptr, E->layers[0].attn_norm, E->h, ncols, d, c.eps, s,
                     pdl);
    if (e != cudaSuccess) return e;
    mark(E, kProfNorm);
    ++n;
    for (int l = 0; l < c.L; ++l) {
        const Layer& Ly = E->layers[l];
        GemmParams g = gemm_base(E, Ly.wqkv, qd + 2 * kd, d, ncols);
        if (E->self_pf_kb_cls[0] >= 0) g.self_pf_kb = E->self_pf_kb_cls[0];
        g.mode = kEpiQkvRope;
        g.trace_tag = kProfQkv;
        g.q_out = E->q;
        g.hq = c.hq;
        g.hkv = c.hkv;
        g.hd = c.hd;
        g.col_pos = pos;
        g.col_req = req;
        g.rope_cos = E->rope_cos;
        g.rope_sin = E->rope_sin;
        g.kcache = E->kpool + per_layer * l;
        g.vcache = E->vpool + per_layer * l;
        g.block_table = E->block_table;
        g.max_pages = E->pages_per_slot;
        g.page = kPage;
        if (fuse) {
            g.norm_x = E->x;
            g.norm_ss = E->norm_ss;
            g.norm_gamma = Ly.attn_norm;
            g.norm_d = d;
            g.norm_eps = c.eps;
        }
        const int64_t wb_qkv = int64_t(qd + 2 * kd) * d * 2, wb_o = int64_t(d) * qd * 2,
                      wb_gu = int64_t(2 * c.F) * d * 2, wb_down = int64_t(d) * c.F * 2;
        const unsigned pf = fuse ? E->l2pf_mask : 0u;
        auto pf_bytes = [&](int64_t b) { return b < E->l2pf_cap ? b : E->l2pf_cap; };
        if (pf & 16u) {
            g.l2pf = Ly.wo;
            g.l2pf_bytes = pf_bytes(wb_o);
        }
        if (!(E->skip_mask & (1u << kProfQkv)) && (e = gemm_launch(Ly.tm_qkv, tm_h, g, s, pdl)) != cudaSuccess) return e;
        mark(E, kProfQkv);
        AttnParams a{};
        a.q = E->q;
        a.kcache = E->kpool + per_layer * l;
        a.vcache = E->vpool + per_layer * l;
        a.block_table = E->block_table;
        a.col_pos = pos;
        a.col_req = req;
        a.out = E->attn;
        a.ws = E->attn_ws;
        a.tickets = E->attn_tickets;
        a.ncols = ncols;
        a.hq = c.hq;
        a.hkv = c.hkv;
        a.hd = c.hd;
        a.page = kPage;
        a.max_pages = E->pages_per_slot;
        a.max_chunks = E->max_chunks;
        a.decode = final_all ? 1 : 0;   // decode steps (final_all) vs prefill chunks
        a.prefill_blocks = E->prefill_blocks ? 1 : 0;
        a.cluster_max_cols = E->attn_cluster_max_cols;
        a.sep_recv = ncols <= E->attn_sep_recv_max_cols ? 1 : 0;
        a.tm_k = &E->tm_kpool;
        a.tm_v = &E->tm_vpool;
        a.kv_row0 = static_cast<int64_t>(per_layer / c.hd) * l;
        a.stream_min_cols = E->attn_stream_min_cols;
        a.stream_prefill = E->attn_stream_prefill;
        a.trace = E->trace_buf;
        a.trace_tag = kProfAttn;
        if (pf & 1u) {
            a.l2pf = Ly.wo;
            a.l2pf_bytes = pf_bytes(wb_o);
        }
        if (!(E->skip_mask & (1u << kProfAttn)) && (e = launch_attention(a, s, pdl)) != cudaSuccess) return e;
        mark(E, kProfAttn);
        GemmParams go = gemm_base(E, Ly.wo, d, qd, ncols);
        if (E->self_pf_kb_cls[1] >= 0) go.self_pf_kb = E->self_pf_kb_cls[1];
        go.mode = kEpiAddF32;
        go.trace_tag = kProfO;
        go.out = E->x;
        go.ld_out = d;
        if (fuse) {
            go.ss_out = E->norm_ss;
            go.ss_tiles = d / 128;
        }
        if (pf & 2u) {
            go.l2pf = Ly.wgu;
            go.l2pf_bytes = pf_bytes(wb_gu);
        }
        if (!(E->skip_mask & (1u << kProfO)) && (e = gemm_launch(Ly.tm_o, tm_attn, go, s, pdl)) != cudaSuccess) return e;
        mark(E, kProfO);
        if (!fuse && !(E->skip_mask & (1u << kProfNorm))) {
            if ((e = launch_rmsnorm(E->x, nullptr, nullptr, nullptr, Ly.ffn_norm, E->h, nullptr, ncols, d, c.eps, s,
                                    pdl)) != cudaSuccess)
                return e;
            mark(E, kProfNorm);
            ++n;
        }
        GemmParams gu = gemm_base(E, Ly.wgu, 2 * c.F, d, ncols);
        if (E->self_pf_kb_cls[2] >= 0) gu.self_pf_kb = E->self_pf_kb_cls[2];
        gu.mode = kEpiSwiglu;
        gu.trace_tag = kProfGateUp;
        gu.act = E->act;
        if (fuse) {
            gu.norm_x = E->x;
            gu.norm_ss = E->norm_ss;
            gu.norm_gamma = Ly.ffn_norm;
            gu.norm_d = d;
            gu.norm_eps = c.eps;
        }
        if (pf & 4u) {
            gu.l2pf = Ly.wdown;
            gu.l2pf_bytes = pf_bytes(wb_down);
        }
        if (!(E->skip_mask & (1u << kProfGateUp)) && (e = gemm_launch(Ly.tm_gu, tm_h, gu, s, pdl)) != cudaSuccess) return e;
        mark(E, kProfGateUp);
        GemmParams gd = gemm_base(E, Ly.wdown, d, c.F, ncols);
        gd.mode = kEpiAddF32;
        if (E->self_pf_kb_cls[3] >= 0) gd.self_pf_kb = E->self_pf_kb_cls[3];
        gd.trace_tag = kProfDown;
        gd.out = E->x;
        gd.ld_out = d;
        if (fuse) {
            gd.ss_out = E->norm_ss;
            gd.ss_tiles = d / 128;
        }
        if ((pf & 8u) && l + 1 < c.L) {
            gd.l2pf = E->layers[l + 1].wqkv;
            gd.l2pf_bytes = pf_bytes(wb_qkv);
        }
        if (!(E->skip_mask & (1u << kProfDown)) && (e = gemm_launch(Ly.tm_down, tm_act, gd, s, pdl)) != cudaSuccess) return e;
        mark(E, kProfDown);
        n += 6;
        if (fuse) {
            // norms fused into the next QKV GEMM / lm_head
        } else if (l + 1 < c.L && (E->skip_mask & (1u << kProfNorm))) {
            // timing experiments only: RMSNorm left out
        } else if (l + 1 < c.L) {
            e = launch_rmsnorm(E->x, nullptr, nullptr, nullptr, E->layers[l + 1].attn_norm, E->h, nullptr, ncols, d,
                               c.eps, s, pdl);
            ++n;
        } else if (final_all) {
            e = launch_rmsnorm(E->x, nullptr, nullptr, nullptr, E->final_norm, E->h, nullptr, ncols, d, c.eps, s, pdl);
            ++n;
        } else if (n_last > 0) {
            e = launch_rmsnorm_gather(E->x, E->final_norm, E->h_last, E->p_last_in, E->p_last_out, n_last, d, c.eps, s,
                                      pdl);
            ++n;
        }
        if (e != cudaSuccess) return e;
        if (!fuse) mark(E, kProfNorm);
    }
    if (nlaunch) *nlaunch += n;
    return cudaSuccess;
}

// lm_head over `ncols` columns of X (tmX) into the trace at (slot, d_step[col]), then the sampler.
// col_step / col_slot: the trace step and slot of each column (default: the decode state, one
// column per slot); by_slot: the sampler updates the decode state of the column's slot (compact
// columns of newly admitted requests in continuous batching).
cudaError_t head_and_sample(Engine* E, const __nv_bfloat16* X, int ncols, uint64_t* nlaunch, bool fuse_norm = false,
                            const int* col_step = nullptr, const int* col_slot = nullptr, bool by_slot = false) {
    if (col_step == nullptr) col_step = E->d_step;
    if (col_slot == nullptr) col_slot = E->d_req;
    const ModelConfig& c = E->cfg;
    CUtensorMap tmX;
    if (!make_tmap_bf16(&tmX, X, c.d, ncols, 64)) return cudaErrorInvalidValue;
    GemmParams g = gemm_base(E, E->lm_head, c.V, c.d, ncols);
    if (E->self_pf_kb_cls[4] >= 0) g.self_pf_kb = E->self_pf_kb_cls[4];
    g.mode = kEpiStoreF32;
    g.trace_tag = kProfLmHead;
    if (fuse_norm) {   // final RMSNorm fused into the lm_head's B operand (decode, <= 8 columns)
        g.norm_x = E->x;
        g.norm_ss = E->norm_ss;
        g.norm_gamma = E->final_norm;
        g.norm_d = c.d;
        g.norm_eps = c.eps;
    }
    g.out = E->trace;
    g.col_step = col_step;
    g.col_slot = col_slot;
    g.slot_stride = E->slot_stride;
    cudaError_t e = gemm_launch(E->tm_lm, tmX, g, E->stream, E->use_pdl);
    if (e != cudaSuccess) return e;
    mark(E, kProfLmHead);
    SampleParams sp{};
    sp.logits = E->trace;
    sp.col_step = col_step;
    sp.col_slot = col_slot;
    sp.state_by_slot = by_slot ? 1 : 0;
    sp.slot_stride = E->slot_stride;
    sp.rows = ncols;
    sp.vocab = c.V;
    sp.policy = E->d_pol;
    sp.prng = E->d_prng;
    sp.probs = E->probs;
    sp.scratch = E->sort_scratch;
    sp.blk_ws = E->sample_ws;
    sp.tickets = E->sample_tickets;
    sp.token_out = reinterpret_cast<uint32_t*>(E->d_tok);
    sp.status = E->d_status;
    sp.tokens_hist = E->tok_hist;
    sp.tcap = E->tcap;
    sp.col_pos = E->d_pos;
    sp.col_step_mut = E->d_step;
    e = launch_sample(sp, E->stream, E->use_pdl);
    mark(E, kProfSample);
    if (nlaunch) *nlaunch += 2 + ((c.V + 4095) / 4096 > 1 && ncols <= kSampleMultiMaxRows ? 2 : 0);   // lm_head, sampler
    return e;
}

int ensure_outputs(Engine* E, int nslots, int tmax) {
    // the slot stride is bucketed (powers of two up to 64 steps, then multiples of 64) so a server
    // seeing many distinct max_tokens captures a bounded set of decode graphs (layout only: the
    // logits of step t of a slot are at slot * stride + t * V whatever the stride)
    tmax = tmax <= 64 ? (tmax <= 1 ? 1 : 1 << (32 - __builtin_clz(unsigned(tmax - 1)))) : (tmax + 63) / 64 * 64;
    const size_t need_trace = size_t(nslots) * tmax * E->cfg.V;
    if (need_trace > E->trace_cap) {
        if (E->trace) dfree(E->trace);
        E->trace = nullptr;
        ENG_CUDA(dalloc(&E->trace, need_trace));
        E->trace_cap = need_trace;
        for (auto& gph : E->graphs) cudaGraphExecDestroy(gph.second);
        E->graphs.clear();
        E->graph_used.clear();
    }
    const size_t need_tok = size_t(nslots) * tmax;
    if (need_tok > E->tok_cap) {
        if (E->tok_hist) dfree(E->tok_hist);
        E->tok_hist = nullptr;
        ENG_CUDA(dalloc(&E->tok_hist, need_tok));
        E->tok_cap = need_tok;
        for (auto& gph : E->graphs) cudaGraphExecDestroy(gph.second);
        E->graphs.clear();
        E->graph_used.clear();
    }
    if (E->tcap != tmax || E->slot_stride != int64_t(tmax) * E->cfg.V) {
        E->tcap = tmax;
        E->slot_stride = int64_t(tmax) * E->cfg.V;
    }
    return DETGPU_OK;
}

int get_graph(Engine* E, int ncols, cudaGraphExec_t* out) {
    auto key = std::make_pair(ncols, E->slot_stride);
    E->graph_used[key] = ++E->graph_clock;
    auto it = E->graphs.find(key);
    if (it != E->graphs.end()) {
        *out = it->second;
        return DETGPU_OK;
    }
    if (E->graphs.size() >= kMaxGraphs) {   // bounded cache: drop the least recently used graph
        auto victim = E->graphs.end();
        for (auto g = E->graphs.begin(); g != E->graphs.end(); ++g)
            if (victim == E->graphs.end() || E->graph_used[g->first] < E->graph_used[victim->first]) victim = g;
        ENG_CUDA(cudaStreamSynchronize(E->stream));   // never destroy a graph that may still run
        cudaGraphExecDestroy(victim->second);
        E->graph_used.erase(victim->first);
        E->graphs.erase(victim);
    }
    cudaGraph_t g;
    ENG_CUDA(cudaStreamBeginCapture(E->stream, cudaStreamCaptureModeThreadLocal));
    uint64_t n = 0;
    cudaError_t e = forward(E, ncols, E->d_tok, E->d_pos, E->d_req, true, 0, &n);
    if (e == cudaSuccess) e = head_and_sample(E, E->h, ncols, &n, ncols <= E->fuse_max_cols);
    cudaError_t e2 = cudaStreamEndCapture(E->stream, &g);
    ENG_CUDA(e);
    ENG_CUDA(e2);
    cudaGraphExec_t ex;
    ENG_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    E->graphs[key] = ex;
    E->launches_per_step = n;
    *out = ex;
    return DETGPU_OK;
}

std::string validate_policy(const detgpu_policy& p) {
    // DecodePolicy::validate (detcore.cpp:52-69)
    switch (p.kind) {
        case DETGPU_GREEDY:
            if (p.has_k || p.has_p) return "greedy policy must not carry k or p";
            return "";
        case DETGPU_TOP_K:
            if (!p.has_k) return "top_k policy requires k";
            if (p.k == 0) return "top_k k must be positive";
            if (p.has_p) return "top_k policy must not carry p";
            return "";
        case DETGPU_NUCLEUS:
            if (!p.has_p) return "nucleus policy requires p";
            if (!(p.p > 0.0f) || p.p > 1.0f) return "nucleus p must be in (0,1]";
            if (p.has_k) return "nucleus policy must not carry k";
            return "";
        default:
            return "unknown decode kind";
    }
}

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double ms() const {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
};

// One group of n <= max_batch requests through prefill + decode; results left in trace/tok_hist.
int run_group(Engine* E, uint32_t n, const uint32_t* const* prompts, const uint32_t* lens, const detgpu_policy* pols,
              const uint64_t* seeds, detgpu_stats* st) {
    const ModelConfig& c = E->cfg;
    cudaStream_t s = E->stream;
    int tmax = 0;
    for (uint32_t i = 0; i < n; ++i) tmax = std::max<int>(tmax, static_cast<int>(pols[i].max_tokens));
    if (tmax == 0) return DETGPU_OK;
    if (int rc = ensure_outputs(E, static_cast<int>(n), tmax)) return rc;
    // per-slot state
    std::vector<int> step(n), pos(n), zero(n, 0);
    std::vector<uint64_t> prng(size_t(n) * 4);
    std::vector<DevPolicy> dp(n);
    for (uint32_t i = 0; i < n; ++i) {
        const bool active = pols[i].max_tokens > 0;
        step[i] = active ? 0 : -1;
        pos[i] = active ? static_cast<int>(lens[i]) - 1 : -1;
        prng_seeded(seeds[i], &prng[size_t(i) * 4]);
        dp[i] = to_dev_policy(pols[i]);
    }
    ENG_CUDA(cudaMemcpyAsync(E->d_step, step.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_pos, pos.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_status, zero.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_tok, zero.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_prng, prng.data(), sizeof(uint64_t) * prng.size(), cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_pol, dp.data(), sizeof(DevPolicy) * n, cudaMemcpyHostToDevice, s));
    if (st) st->h2d_bytes += n * (4 * sizeof(int) + 32 + sizeof(DevPolicy));
    ENG_CUDA(cudaEventRecord(E->ev[0], s));
    // prefill: all prompt tokens (of active requests) as columns, chunked; chunking is invisible in
    // the bits because every column is independent (batch invariance)
    std::vector<int> ctok, cpos, creq, lin, lout;
    uint64_t nl = 0;
    auto flush = [&]() -> int {
        if (ctok.empty()) return DETGPU_OK;
        const int nc = static_cast<int>(ctok.size());
        ENG_CUDA(cudaMemcpyAsync(E->p_tok, ctok.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, s));
        ENG_CUDA(cudaMemcpyAsync(E->p_pos, cpos.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, s));
        ENG_CUDA(cudaMemcpyAsync(E->p_req, creq.data(), sizeof(int) * nc, cudaMemcpyHostToDevice, s));
        const int nlast = static_cast<int>(lin.size());
        if (nlast > 0) {
            ENG_CUDA(cudaMemcpyAsync(E->p_last_in, lin.data(), sizeof(int) * nlast, cudaMemcpyHostToDevice, s));
            ENG_CUDA(cudaMemcpyAsync(E->p_last_out, lout.data(), sizeof(int) * nlast, cudaMemcpyHostToDevice, s));
        }
        if (st) st->h2d_bytes += sizeof(int) * (3ull * nc + 2ull * nlast);
        ENG_CUDA(forward(E, nc, E->p_tok, E->p_pos, E->p_req, false, nlast, &nl));
        // the host vectors are reused next chunk: wait for the async copies to be consumed
        ENG_CUDA(cudaStreamSynchronize(s));
        ctok.clear();
        cpos.clear();
        creq.clear();
        lin.clear();
        lout.clear();
        return DETGPU_OK;
    };
    for (uint32_t i = 0; i < n; ++i) {
        if (pols[i].max_tokens == 0) continue;
        for (uint32_t t = 0; t < lens[i]; ++t) {
            if (static_cast<int>(ctok.size()) == E->col_cap)
                if (int rc = flush()) return rc;
            if (t + 1 == lens[i]) {
                lin.push_back(static_cast<int>(ctok.size()));
                lout.push_back(static_cast<int>(i));
            }
            ctok.push_back(static_cast<int>(prompts[i][t]));
            cpos.push_back(static_cast<int>(t));
            creq.push_back(static_cast<int>(i));
        }
    }
    if (int rc = flush()) return rc;
    ENG_CUDA(head_and_sample(E, E->h_last, static_cast<int>(n), &nl));
    ENG_CUDA(cudaEventRecord(E->ev[1], s));
    // decode loop: one graph replay per step
    cudaGraphExec_t gx = nullptr;
    if (tmax > 1)
        if (int rc = get_graph(E, static_cast<int>(n), &gx)) return rc;
    for (int t = 1; t < tmax; ++t) ENG_CUDA(cudaGraphLaunch(gx, s));
    ENG_CUDA(cudaEventRecord(E->ev[2], s));
    ENG_CUDA(cudaEventSynchronize(E->ev[2]));
    if (st) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, E->ev[0], E->ev[1]);
        cudaEventElapsedTime(&b, E->ev[1], E->ev[2]);
        st->prefill_ms += a;
        st->decode_ms += b;
        st->decode_steps += static_cast<uint64_t>(tmax - 1);
        st->kernel_launches += nl + static_cast<uint64_t>(tmax - 1) * E->launches_per_step;
    }
    return DETGPU_OK;
}

// Outputs of one finished slot: status, tokens, logits (D2H through two pinned staging buffers,
// hashing piece k while k+1 lands) and out_hash (v1: SHA-256 of the canonical bytes; v2: the
// per-step Merkle roots computed on the GPU).
int collect_slot(Engine* E, int slot, uint32_t T, uint32_t* tokens_out, float* logits_out, uint8_t* out_hash, bool v2,
                 detgpu_stats* st, std::vector<std::future<void>>* hashers = nullptr) {
    const int V = E->cfg.V;
    cudaStream_t s = E->stream;
    int status = 0;
    ENG_CUDA(cudaMemcpy(&status, E->d_status + slot, sizeof(int), cudaMemcpyDeviceToHost));
    if (status == DETGPU_ENONFINITE) return fail(E, DETGPU_EINVAL, "det_softmax: non-finite value");
    if (status != 0) return fail(E, DETGPU_EINVAL, "decode: zero probability mass after truncation");
    Timer tcopy;
    std::vector<uint32_t> toks(std::max<uint32_t>(T, 1));
    if (T > 0)
        ENG_CUDA(cudaMemcpy(toks.data(), E->tok_hist + size_t(slot) * E->tcap, sizeof(uint32_t) * T,
                            cudaMemcpyDeviceToHost));
    if (st) st->d2h_bytes += sizeof(uint32_t) * size_t(T);
    if (tokens_out && T) std::memcpy(tokens_out, toks.data(), sizeof(uint32_t) * T);
    double copy_ms = tcopy.ms(), hash_ms = 0;
    if (v2 && out_hash != nullptr) {
        Timer th;
        std::vector<uint8_t> roots(32 * size_t(std::max<uint32_t>(T, 1)));
        if (T > 0) {
            const size_t need = 32 * size_t(T);
            if (need > E->roots_cap) {
                if (E->d_roots) dfree(E->d_roots);
                E->d_roots = nullptr;
                ENG_CUDA(dalloc(&E->d_roots, std::max(need, size_t(E->max_batch) * E->tcap * 32)));
                E->roots_cap = std::max(need, size_t(E->max_batch) * E->tcap * 32);
            }
            if (E->d_steps == nullptr) ENG_CUDA(dalloc(&E->d_steps, size_t(E->max_batch)));
            const int steps = static_cast<int>(T);
            ENG_CUDA(cudaMemcpyAsync(E->d_steps, &steps, sizeof(int), cudaMemcpyHostToDevice, s));
            ENG_CUDA(launch_receipt_roots(E->trace + size_t(slot) * E->slot_stride, E->slot_stride, E->d_steps, 1, steps,
                                          V, E->d_roots, E->tcap, s));
            ENG_CUDA(cudaMemcpyAsync(roots.data(), E->d_roots, need, cudaMemcpyDeviceToHost, s));
            ENG_CUDA(cudaStreamSynchronize(s));
            if (st) st->d2h_bytes += need;
        }
        hash_canonical_v2_roots(toks.data(), T, roots.data(), static_cast<uint32_t>(V), out_hash);
        hash_ms += th.ms();
    }
    const bool want_hash = out_hash != nullptr && !v2;
    if (want_hash && hashers != nullptr && T > 0) {
        // continuous batching: copy the slot's trace out and hash it on a worker thread, so that
        // the v1 SHA-256 (sequential, ~71 ms per 8B request) does not stall the decode loop
        const size_t n = size_t(T) * V;
        Timer tw;
        float* dst = logits_out;
        Engine::HashBuf* hb = nullptr;
        if (dst == nullptr) {
            // a pinned buffer whose previous hash is done; the pool grows to one buffer per spare
            // host thread (3..16), so many requests finishing together hash in parallel; when all
            // are busy, wait for the oldest
            static const size_t kMaxBufs = std::max<size_t>(3, std::min<size_t>(16, std::thread::hardware_concurrency() > 2
                                                                                         ? std::thread::hardware_concurrency() - 2
                                                                                         : 3));
            for (auto& b : E->hash_bufs)
                if (!b.busy.valid() || b.busy.wait_for(std::chrono::seconds(0)) == std::future_status::ready) {
                    hb = &b;
                    break;
                }
            if (hb == nullptr && E->hash_bufs.size() < kMaxBufs) {
                E->hash_bufs.emplace_back();
                hb = &E->hash_bufs.back();
            }
            if (hb == nullptr) {
                hb = &E->hash_bufs[E->hash_next++ % E->hash_bufs.size()];
                hb->busy.wait();
            }
            if (hb->cap < n) {
                if (hb->p) cudaFreeHost(hb->p);
                hb->p = nullptr;
                hb->cap = 0;
                ENG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&hb->p), sizeof(float) * n, cudaHostAllocDefault));
                hb->cap = n;
            }
            dst = hb->p;
        }
        ENG_CUDA(cudaMemcpy(dst, E->trace + size_t(slot) * E->slot_stride, sizeof(float) * n, cudaMemcpyDeviceToHost));
        copy_ms += tw.ms();
        if (st) st->d2h_bytes += 4 * n;
        auto tk = std::make_shared<std::vector<uint32_t>>(toks.begin(), toks.begin() + T);
        std::future<void> f = std::async(std::launch::async, [tk, dst, T, V, out_hash]() {
            hash_canonical(tk->data(), T, dst, static_cast<uint32_t>(V), out_hash);
        });
        if (hb != nullptr) {
            hb->busy = f.share();
            hashers->push_back(std::async(std::launch::deferred, [sf = hb->busy]() { sf.wait(); }));
        } else {
            hashers->push_back(std::move(f));
        }
        if (st) st->d2h_ms += static_cast<float>(copy_ms);
        return DETGPU_OK;
    }
    if (logits_out != nullptr || want_hash) {
        const size_t piece = E->pinned_floats;
        Sha256 sha;
        if (want_hash) {
            sha.update(&T, 4);
            if (T) sha.update(toks.data(), 4 * size_t(T));
            sha.update(&T, 4);
        }
        const size_t total = size_t(T) * V;
        const float* src = E->trace + size_t(slot) * E->slot_stride;
        size_t done = 0;
        int buf = 0;
        size_t inflight = std::min(piece, total);
        if (total > 0) ENG_CUDA(cudaMemcpyAsync(E->pinned[0], src, sizeof(float) * inflight, cudaMemcpyDeviceToHost, s));
        while (done < total) {
            Timer tw;
            ENG_CUDA(cudaStreamSynchronize(s));
            copy_ms += tw.ms();
            const size_t cur = inflight;
            const size_t next_off = done + cur;
            size_t next = 0;
            if (next_off < total) {
                next = std::min(piece, total - next_off);
                ENG_CUDA(cudaMemcpyAsync(E->pinned[buf ^ 1], src + next_off, sizeof(float) * next,
                                         cudaMemcpyDeviceToHost, s));
            }
            Timer th;
            const float* hp = E->pinned[buf];
            if (logits_out) std::memcpy(logits_out + done, hp, sizeof(float) * cur);
            if (want_hash) {
                // step boundaries inside this piece: each step is prefixed by its u32 vocab size
                size_t off = 0;
                while (off < cur) {
                    const size_t g = done + off;
                    if (g % V == 0) sha.update(&V, 4);
                    const size_t run = std::min(cur - off, size_t(V) - g % V);
                    sha.update(hp + off, 4 * run);
                    off += run;
                }
            }
            hash_ms += th.ms();
            done += cur;
            inflight = next;
            buf ^= 1;
        }
        if (st) st->d2h_bytes += 4 * total;
        if (want_hash) sha.final(out_hash);
    }
    if (st) {
        st->d2h_ms += static_cast<float>(copy_ms);
        st->hash_ms += static_cast<float>(hash_ms);
    }
    return DETGPU_OK;
}

int collect_group(Engine* E, uint32_t n, const detgpu_policy* pols, uint32_t* const* tokens_out,
                  float* const* logits_out, uint8_t* out_hash, bool v2, detgpu_stats* st) {
    // several requests: hash them on worker threads (one request: the streamed, copy-overlapped hash)
    std::vector<std::future<void>> hashers;
    int rc = DETGPU_OK;
    for (uint32_t i = 0; i < n && rc == DETGPU_OK; ++i) {
        if (pols[i].max_tokens == 0) continue;   // handled by the caller (empty canonical output)
        rc = collect_slot(E, static_cast<int>(i), pols[i].max_tokens, tokens_out ? tokens_out[i] : nullptr,
                          logits_out ? logits_out[i] : nullptr, out_hash ? out_hash + 32 * size_t(i) : nullptr, v2, st,
                          n > 1 ? &hashers : nullptr);
    }
    for (auto& f : hashers) f.wait();
    return rc;
}

// Continuous batching: `slots` decode slots stay busy; a request is admitted into a
// slot as soon as one frees, its prompt prefilled between decode steps and its first token sampled
// from compact columns that update the slot's decode state. Every column is computed
// independently of the others, so a request's bytes do not depend on what it shares
// a step with: outputs equal the static-group path's bit for bit (tests/test_gpu_engine.py). The
// host knows each slot's finishing step (one token per step), so decode steps run back to back in
// graph replays with no per-step synchronisation.
int run_continuous(Engine* E, uint32_t n_req, const uint32_t* const* prompts, const uint32_t* lens,
                   const detgpu_policy* pols, const uint64_t* seeds, uint32_t slots, uint32_t* const* tokens_out,
                   float* const* logits_out, uint8_t* out_hash, bool v2, detgpu_stats* st) {
    cudaStream_t s = E->stream;
    int tmax = 1;
    for (uint32_t i = 0; i < n_req; ++i) tmax = std::max<int>(tmax, static_cast<int>(pols[i].max_tokens));
    if (int rc = ensure_outputs(E, static_cast<int>(slots), tmax)) return rc;
    std::vector<int> init(slots, -1), zero(slots, 0);
    ENG_CUDA(cudaMemcpyAsync(E->d_step, init.data(), sizeof(int) * slots, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_pos, init.data(), sizeof(int) * slots, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_status, zero.data(), sizeof(int) * slots, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaMemcpyAsync(E->d_tok, zero.data(), sizeof(int) * slots, cudaMemcpyHostToDevice, s));
    ENG_CUDA(cudaStreamSynchronize(s));
    cudaGraphExec_t gx = nullptr;
    if (tmax > 1)
        if (int rc = get_graph(E, static_cast<int>(slots), &gx)) return rc;
    std::vector<int> slot_req(slots, -1), slot_left(slots, 0);
    uint32_t next = 0;
    uint64_t nl = 0, decode_steps = 0, graph_steps = 0;
    Timer tall;
    double prefill_ms = 0;
    std::vector<int> ctok, cpos, creq, lin, lout, adm;
    std::vector<std::future<void>> hashers;   // v1 receipts hashed off the decode loop
    struct Join {
        std::vector<std::future<void>>& h;
        ~Join() {
            for (auto& f : h)
                if (f.valid()) f.wait();
        }
    } join{hashers};
    for (;;) {
        // 1. collect the slots that finished (the stream is idle here: synchronised at the end of
        //    the previous round), freeing them for admission in this round
        for (uint32_t sl = 0; sl < slots; ++sl) {
            if (slot_req[sl] < 0 || slot_left[sl] != 0) continue;
            const int r = slot_req[sl];
            if (int rc = collect_slot(E, static_cast<int>(sl), pols[r].max_tokens, tokens_out ? tokens_out[r] : nullptr,
                                      logits_out ? logits_out[r] : nullptr, out_hash ? out_hash + 32 * size_t(r) : nullptr,
                                      v2, st, &hashers))
                return rc;
            slot_req[sl] = -1;
        }
        // 2. admit pending requests into free slots (max_tokens == 0 needs no GPU work). Nothing
        //    below waits for the GPU: the small H2D copies come from pinned staging buffers.
        adm.clear();
        for (uint32_t sl = 0; sl < slots && next < n_req; ++sl) {
            if (slot_req[sl] >= 0) continue;
            while (next < n_req && pols[next].max_tokens == 0) {
                if (out_hash) {
                    if (v2) hash_canonical_v2_roots(nullptr, 0, nullptr, E->cfg.V, out_hash + 32 * size_t(next));
                    else hash_canonical(nullptr, 0, nullptr, E->cfg.V, out_hash + 32 * size_t(next));
                }
                ++next;
            }
            if (next >= n_req) break;
            slot_req[sl] = static_cast<int>(next++);
            adm.push_back(static_cast<int>(sl));
        }
        if (!adm.empty()) {
            Timer tp;
            // Slots still decoding ride along: the last prefill chunk of the admitted prompts and one
            // decode step of every decoding slot run as ONE forward pass (columns [0, slots) = the
            // slots' decode columns, then the prompt columns), so the weights are streamed once for
            // both. Columns are independent (batch invariance), so the bytes are unchanged.
            std::vector<char> admitted(slots, 0);
            for (int sl : adm) admitted[sl] = 1;
            int ndec = 0;
            for (uint32_t sl = 0; sl < slots; ++sl)
                if (slot_req[sl] >= 0 && !admitted[sl] && slot_left[sl] > 0) ++ndec;
            const bool mix = ndec > 0 && E->mixed_steps && static_cast<int>(slots) + 64 <= E->col_cap;
            const int base = mix ? static_cast<int>(slots) : 0;
            const int cap = E->col_cap - base;
            auto flush = [&](bool last) -> int {
                if (ctok.empty() && !(last && mix)) return DETGPU_OK;
                const bool with_dec = last && mix;
                const int nc = static_cast<int>(ctok.size());
                if (with_dec)   // decoding slots: column sl -> h_last row sl
                    for (uint32_t sl = 0; sl < slots; ++sl)
                        if (slot_req[sl] >= 0 && !admitted[sl]) {
                            lin.push_back(-1 - static_cast<int>(sl));   // marker: decode column sl
                            lout.push_back(static_cast<int>(sl));
                        }
                const int nlast = static_cast<int>(lin.size());
                const int off = with_dec ? base : 0;
                void* bp = nullptr;
                int bi = 0;
                ENG_CUDA(stage_acquire(E, sizeof(int) * (3 * size_t(nc) + 2 * size_t(nlast)), &bp, &bi));
                int* bb = static_cast<int*>(bp);
                std::copy(ctok.begin(), ctok.end(), bb);
                std::copy(cpos.begin(), cpos.end(), bb + nc);
                std::copy(creq.begin(), creq.end(), bb + 2 * nc);
                for (int i = 0; i < nlast; ++i)   // prompt lasts: chunk index -> column off + index
                    bb[3 * nc + i] = lin[i] < 0 ? -1 - lin[i] : off + lin[i];
                std::copy(lout.begin(), lout.end(), bb + 3 * nc + nlast);
                if (with_dec) {   // the slots' decode state as the first `slots` columns
                    ENG_CUDA(cudaMemcpyAsync(E->p_tok, E->d_tok, sizeof(int) * slots, cudaMemcpyDeviceToDevice, s));
                    ENG_CUDA(cudaMemcpyAsync(E->p_pos, E->d_pos, sizeof(int) * slots, cudaMemcpyDeviceToDevice, s));
                    ENG_CUDA(cudaMemcpyAsync(E->p_req, E->d_req, sizeof(int) * slots, cudaMemcpyDeviceToDevice, s));
                }
                if (nc > 0) {
                    ENG_CUDA(cudaMemcpyAsync(E->p_tok + off, bb, sizeof(int) * nc, cudaMemcpyHostToDevice, s));
                    ENG_CUDA(cudaMemcpyAsync(E->p_pos + off, bb + nc, sizeof(int) * nc, cudaMemcpyHostToDevice, s));
                    ENG_CUDA(cudaMemcpyAsync(E->p_req + off, bb + 2 * nc, sizeof(int) * nc, cudaMemcpyHostToDevice, s));
                }
                if (nlast > 0) {
                    ENG_CUDA(cudaMemcpyAsync(E->p_last_in, bb + 3 * nc, sizeof(int) * nlast, cudaMemcpyHostToDevice, s));
                    ENG_CUDA(cudaMemcpyAsync(E->p_last_out, bb + 3 * nc + nlast, sizeof(int) * nlast, cudaMemcpyHostToDevice, s));
                }
                ENG_CUDA(stage_release(E, bi));
                if (st) st->h2d_bytes += sizeof(int) * (3ull * nc + 2ull * nlast) + sizeof(uint32_t) * nc;
                ENG_CUDA(forward(E, off + nc, E->p_tok, E->p_pos, E->p_req, false, nlast, &nl));
                ctok.clear();
                cpos.clear();
                creq.clear();
                lin.clear();
                lout.clear();
                return DETGPU_OK;
            };
            for (size_t j = 0; j < adm.size(); ++j) {   // prompts as prefill columns; h_last[slot] = last position
                const int r = slot_req[adm[j]];
                for (uint32_t t = 0; t < lens[r]; ++t) {
                    if (static_cast<int>(ctok.size()) == cap)
                        if (int rc = flush(false)) return rc;
                    if (t + 1 == lens[r]) {
                        lin.push_back(static_cast<int>(ctok.size()));
                        lout.push_back(adm[j]);
                    }
                    ctok.push_back(static_cast<int>(prompts[r][t]));
                    cpos.push_back(static_cast<int>(t));
                    creq.push_back(adm[j]);
                }
            }
            if (int rc = flush(true)) return rc;
            // the admitted slots' decode state (after the forward: their columns were not decode
            // columns in it), then one sampler pass over the slots: the first token of each admitted
            // request (trace step 0) and, when mixed, the next token of every decoding slot
            struct AdmState {   // the slot's decode state before its first token is sampled
                uint64_t prng[4];
                DevPolicy dp;
                int pos, status, step;
            };
            void* sp = nullptr;
            int si = 0;
            ENG_CUDA(stage_acquire(E, sizeof(AdmState) * adm.size(), &sp, &si));
            AdmState* as = static_cast<AdmState*>(sp);
            for (size_t j = 0; j < adm.size(); ++j) {
                const int sl = adm[j], r = slot_req[sl];
                prng_seeded(seeds[r], as[j].prng);
                as[j].dp = to_dev_policy(pols[r]);
                as[j].pos = static_cast<int>(lens[r]) - 1;
                as[j].status = 0;
                as[j].step = 0;
                ENG_CUDA(cudaMemcpyAsync(E->d_prng + 4 * size_t(sl), as[j].prng, sizeof(as[j].prng), cudaMemcpyHostToDevice, s));
                ENG_CUDA(cudaMemcpyAsync(E->d_pol + sl, &as[j].dp, sizeof(DevPolicy), cudaMemcpyHostToDevice, s));
                ENG_CUDA(cudaMemcpyAsync(E->d_pos + sl, &as[j].pos, sizeof(int), cudaMemcpyHostToDevice, s));
                ENG_CUDA(cudaMemcpyAsync(E->d_status + sl, &as[j].status, sizeof(int), cudaMemcpyHostToDevice, s));
                ENG_CUDA(cudaMemcpyAsync(E->d_step + sl, &as[j].step, sizeof(int), cudaMemcpyHostToDevice, s));
                if (st) st->h2d_bytes += sizeof(as[j].prng) + sizeof(DevPolicy) + 3 * sizeof(int);
            }
            ENG_CUDA(stage_release(E, si));
            ENG_CUDA(head_and_sample(E, E->h_last, static_cast<int>(slots), &nl, false, E->d_step, E->d_req, false));
            for (int sl : adm) slot_left[sl] = static_cast<int>(pols[slot_req[sl]].max_tokens) - 1;
            if (mix) {
                for (uint32_t sl = 0; sl < slots; ++sl)
                    if (slot_req[sl] >= 0 && !admitted[sl]) slot_left[sl] -= 1;
                decode_steps += 1;
            }
            prefill_ms += tp.ms();
        }
        // 3. decode steps until the next slot finishes (0 steps if an admitted request needs just
        //    its first token), then wait once for the stream so that slot can be collected
        int k = INT32_MAX;
        for (uint32_t sl = 0; sl < slots; ++sl)
            if (slot_req[sl] >= 0) k = std::min(k, slot_left[sl]);
        if (k == INT32_MAX) {   // no active slot
            if (next >= n_req) break;
            continue;
        }
        for (int t = 0; t < k; ++t) ENG_CUDA(cudaGraphLaunch(gx, s));
        decode_steps += static_cast<uint64_t>(k);
        graph_steps += static_cast<uint64_t>(k);
        for (uint32_t sl = 0; sl < slots; ++sl)
            if (slot_req[sl] >= 0) slot_left[sl] -= k;
        ENG_CUDA(cudaStreamSynchronize(s));
    }
    if (st) {
        st->prefill_ms += static_cast<float>(prefill_ms);
        st->decode_ms += static_cast<float>(tall.ms() - prefill_ms);
        st->decode_steps += decode_steps;
        st->kernel_launches += nl + graph_steps * E->launches_per_step;
    }
    return DETGPU_OK;
}

}  // namespace

}  // namespace detgpu

using namespace detgpu;

struct detgpu_engine {
    std::unique_ptr<Engine> e;
};

extern "C" {

int detgpu_arch_supported(const char* arch) {
    return arch && (std::strcmp(arch, "archA") == 0 || std::strcmp(arch, "archB") == 0 || std::strcmp(arch, "b200") == 0);
}

int detgpu_create(int device, const char* model_id, const char* arch, uint32_t max_batch, uint32_t max_context,
                  detgpu_engine** out) {
    if (out == nullptr || model_id == nullptr || arch == nullptr) return fail(nullptr, DETGPU_EINVAL, "null argument");
    *out = nullptr;
    if (!detgpu_arch_supported(arch))
        return fail(nullptr, DETGPU_EINVAL, std::string("infer: unknown arch profile '") + arch + "'");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(nullptr, DETGPU_ENODEV, "no such CUDA device");
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, device);
    if (prop.major != 10) return fail(nullptr, DETGPU_ENODEV, "detgpu needs an sm_100 (B200) device");
    auto E = std::make_unique<Engine>();
    E->device = device;
    E->model_id = model_id;
    E->arch = arch;
    E->max_batch = std::max<uint32_t>(1, std::min<uint32_t>(max_batch, 256));
    E->max_context = std::max<uint32_t>(1, max_context);
    if (const char* v = std::getenv("DETGPU_L2PF")) E->l2pf_mask = static_cast<unsigned>(std::strtoul(v, nullptr, 0));
    if (const char* v = std::getenv("DETGPU_L2PF_MB")) E->l2pf_cap = std::strtoll(v, nullptr, 0) << 20;
    cudaSetDevice(device);
    Engine* Ep = E.get();
    {
        Engine* E = Ep;   // for ENG_CUDA
        ENG_CUDA(cudaStreamCreateWithFlags(&E->stream, cudaStreamNonBlocking));
        for (auto& ev : E->ev) ENG_CUDA(cudaEventCreate(&ev));
        if (std::strcmp(arch, "b200") != 0) {
            E->toy = true;
            if (int rc = toy_init(E->toyw, model_id, std::strcmp(arch, "archA") == 0 ? 0 : 1, E->stream))
                return fail(E, rc, "toy model init failed");
        } else {
            const ModelConfig* c = find_model_config(model_id);
            if (c == nullptr)
                return fail(nullptr, DETGPU_EINVAL,
                            std::string("unknown model config for '") + model_id + "' (expected llama-tiny[:tag], llama-mid[:tag] or llama3-8b[:tag])");
            E->cfg = *c;
            if (int rc = init_weights(E)) return rc;
            if (int rc = init_buffers(E)) return rc;
            E->pinned_floats = size_t(1) << 24;   // 64 MiB per staging buffer
            for (auto& p : E->pinned) ENG_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(float) * E->pinned_floats));
        }
        ENG_CUDA(cudaStreamSynchronize(E->stream));
    }
    *out = new detgpu_engine{std::move(E)};
    return DETGPU_OK;
}

void detgpu_destroy(detgpu_engine* h) { delete h; }

const char* detgpu_last_error(const detgpu_engine* h) { return h ? h->e->err.c_str() : detgpu_global_error(); }

int detgpu_get_model_info(const detgpu_engine* h, detgpu_model_info* o) {
    if (!h || !o) return DETGPU_EINVAL;
    const Engine* E = h->e.get();
    std::memset(o, 0, sizeof(*o));
    if (E->toy) {
        o->toy = 1;
        o->vocab = kToyVocab;
        o->d_model = kToyDim;
        o->n_layers = 2;
        o->n_params = 2 * kToyVocab * kToyDim + 2 * kToyDim * kToyDim;
        o->weight_bytes = 4 * o->n_params;
        return DETGPU_OK;
    }
    o->n_layers = E->cfg.L;
    o->d_model = E->cfg.d;
    o->n_heads = E->cfg.hq;
    o->n_kv_heads = E->cfg.hkv;
    o->head_dim = E->cfg.hd;
    o->ffn = E->cfg.F;
    o->vocab = E->cfg.V;
    o->rope_theta = static_cast<float>(E->cfg.theta);
    o->rms_eps = E->cfg.eps;
    o->n_params = E->n_params;
    o->weight_bytes = 2 * E->n_params;
    return DETGPU_OK;
}

int detgpu_generate(detgpu_engine* h, uint32_t n_req, const uint32_t* const* prompts, const uint32_t* prompt_lens,
                    const detgpu_policy* policies, const uint64_t* seeds, uint32_t batch_size,
                    uint32_t* const* tokens_out, float* const* logits_out, uint8_t* out_hash, uint32_t flags,
                    detgpu_stats* stats) {
    if (h == nullptr) return fail(nullptr, DETGPU_EINVAL, "null engine");
    Engine* E = h->e.get();
    cudaSetDevice(E->device);
    if (stats) std::memset(stats, 0, sizeof(*stats));
    if (batch_size == 0) return fail(E, DETGPU_EINVAL, "infer_batch: batch_size must be positive");
    if (n_req == 0) return DETGPU_OK;
    if (!prompts || !prompt_lens || !policies || !seeds) return fail(E, DETGPU_EINVAL, "null argument");
    const uint32_t vocab = E->toy ? kToyVocab : static_cast<uint32_t>(E->cfg.V);
    // start_run validation (detcore.cpp:332-343), all requests before any work
    for (uint32_t i = 0; i < n_req; ++i) {
        const std::string perr = validate_policy(policies[i]);
        if (!perr.empty()) return fail(E, DETGPU_EINVAL, "infer: " + perr);
        for (uint32_t t = 0; t < prompt_lens[i]; ++t)
            if (prompts[i][t] >= vocab) return fail(E, DETGPU_EINVAL, "infer: prompt token out of vocabulary");
        if (!E->toy && uint64_t(std::max(prompt_lens[i], 1u)) + policies[i].max_tokens > E->max_context)
            return fail(E, DETGPU_EINVAL, "infer: prompt + max_tokens exceeds the engine's max_context");
    }
    // Empty prompts: the reference accepts them (detcore.cpp:340-352: the ToyModel decodes from its
    // zero state). A transformer needs a position to predict from, so for the b200 models an empty
    // prompt is the one-token prompt [kBosToken] (the oracle applies the same rule).
    static const uint32_t kBos[1] = {kBosToken};
    std::vector<const uint32_t*> pr_eff(prompts, prompts + n_req);
    std::vector<uint32_t> len_eff(prompt_lens, prompt_lens + n_req);
    if (!E->toy)
        for (uint32_t i = 0; i < n_req; ++i)
            if (len_eff[i] == 0) {
                pr_eff[i] = kBos;
                len_eff[i] = 1;
            }
    prompts = pr_eff.data();
    prompt_lens = len_eff.data();
    if (E->toy)
        return toy_generate(E->toyw, n_req, prompts, prompt_lens, policies, seeds, batch_size, tokens_out, logits_out,
                            out_hash, flags, stats, E->stream, &E->err);
    const uint32_t group = std::min(batch_size, E->max_batch);
    if ((flags & DETGPU_F_CONTINUOUS) && !(flags & DETGPU_F_DEVICE_ONLY)) {
        if (int rc = run_continuous(E, n_req, prompts, prompt_lens, policies, seeds, group, tokens_out, logits_out,
                                    out_hash, (flags & DETGPU_F_RECEIPT_V2) != 0, stats))
            return rc;
        if (stats)
            for (uint32_t i = 0; i < n_req; ++i) stats->tokens += policies[i].max_tokens;
        return DETGPU_OK;
    }
    Timer total;
    for (uint32_t base = 0; base < n_req; base += group) {
        const uint32_t n = std::min(group, n_req - base);
        if (stats) stats->h2d_bytes += 0;
        if (int rc = run_group(E, n, prompts + base, prompt_lens + base, policies + base, seeds + base, stats)) return rc;
        if (stats)
            for (uint32_t i = 0; i < n; ++i) stats->tokens += policies[base + i].max_tokens;
        if (!(flags & DETGPU_F_DEVICE_ONLY)) {
            uint32_t* const* to = tokens_out ? tokens_out + base : nullptr;
            float* const* lo = logits_out ? logits_out + base : nullptr;
            if (int rc = collect_group(E, n, policies + base, to, lo, out_hash ? out_hash + 32 * size_t(base) : nullptr,
                                       (flags & DETGPU_F_RECEIPT_V2) != 0, stats))
                return rc;
        } else {
            std::vector<int> status(n);
            ENG_CUDA(cudaMemcpy(status.data(), E->d_status, sizeof(int) * n, cudaMemcpyDeviceToHost));
            for (uint32_t i = 0; i < n; ++i)
                if (status[i] != 0) return fail(E, DETGPU_EINVAL, "decode: non-finite value or zero probability mass");
        }
    }
    // max_tokens == 0 requests: tokens empty, canonical bytes = [0][0]
    if (out_hash && !(flags & DETGPU_F_DEVICE_ONLY))
        for (uint32_t i = 0; i < n_req; ++i)
            if (policies[i].max_tokens == 0) {
                if (flags & DETGPU_F_RECEIPT_V2) hash_canonical_v2_roots(nullptr, 0, nullptr, vocab, out_hash + 32 * size_t(i));
                else hash_canonical(nullptr, 0, nullptr, vocab, out_hash + 32 * size_t(i));
            }
    (void)total;
    return DETGPU_OK;
}

}  // extern "C"

extern "C" {

void* detgpu_stream(const detgpu_engine* h) { return h ? static_cast<void*>(h->e->stream) : nullptr; }

int detgpu_debug_check_canaries(uint64_t* n_checked, uint64_t* n_bad) {
    std::vector<std::pair<void*, std::pair<size_t, int>>> bufs;
    {
        std::lock_guard<std::mutex> lk(canaries().mu);
        bufs.assign(canaries().live.begin(), canaries().live.end());
    }
    std::vector<uint8_t> host(kCanaryBytes);
    uint64_t bad = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& b : bufs) {
        cudaSetDevice(b.second.second);
        if (cudaMemcpy(host.data(), static_cast<uint8_t*>(b.first) + b.second.first, kCanaryBytes,
                       cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(nullptr, DETGPU_ECUDA, "check_canaries: cudaMemcpy failed");
        for (uint8_t v : host)
            if (v != 0xA5) {
                ++bad;
                break;
            }
    }
    cudaSetDevice(cur);
    if (n_checked) *n_checked = bufs.size();
    if (n_bad) *n_bad = bad;
    return DETGPU_OK;
}

// One decode forward + lm_head + sample for `ncols` slots at context `ctx`, launched without graph
// or PDL, with a CUDA event after every launch on the engine stream. ms_by_class[k] is the mean
// time per step spent in kernel class k (0 norm, 1 qkv gemm, 2 attention, 3 o gemm, 4 gate/up gemm,
// 5 down gemm, 6 lm_head gemm, 7 sample); launches_by_class[k] the launches per step.
int detgpu_profile_decode_step(detgpu_engine* h, uint32_t ncols, uint32_t ctx, uint32_t reps, float* ms_by_class,
                               uint32_t* launches_by_class) {
    if (h == nullptr || h->e->toy) return fail(nullptr, DETGPU_EINVAL, "profile: transformer engine required");
    Engine* E = h->e.get();
    cudaSetDevice(E->device);
    if (ncols == 0 || ncols > E->max_batch || ctx == 0 || ctx > E->max_context || reps == 0)
        return fail(E, DETGPU_EINVAL, "profile: bad ncols/ctx/reps");
    if (int rc = ensure_outputs(E, static_cast<int>(ncols), 2)) return rc;
    std::vector<int> step(ncols, 0), pos(ncols, static_cast<int>(ctx) - 1), tok(ncols, 1), zero(ncols, 0);
    std::vector<uint64_t> prng(size_t(ncols) * 4);
    std::vector<DevPolicy> dp(ncols);
    for (uint32_t i = 0; i < ncols; ++i) {
        prng_seeded(i, &prng[size_t(i) * 4]);
        dp[i] = DevPolicy{DETGPU_GREEDY, 0, 0.0f, 2};
    }
    ENG_CUDA(cudaMemcpy(E->d_prng, prng.data(), sizeof(uint64_t) * prng.size(), cudaMemcpyHostToDevice));
    ENG_CUDA(cudaMemcpy(E->d_pol, dp.data(), sizeof(DevPolicy) * ncols, cudaMemcpyHostToDevice));
    std::vector<std::pair<cudaEvent_t, int>> trail;
    const bool pdl = E->use_pdl;
    E->use_pdl = false;
    std::vector<double> acc(kProfN, 0.0);
    std::vector<uint32_t> cnt(kProfN, 0);
    cudaError_t err = cudaSuccess;
    for (uint32_t r = 0; r < reps && err == cudaSuccess; ++r) {
        cudaMemcpyAsync(E->d_step, step.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, E->stream);
        cudaMemcpyAsync(E->d_pos, pos.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, E->stream);
        cudaMemcpyAsync(E->d_tok, tok.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, E->stream);
        cudaMemcpyAsync(E->d_status, zero.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice, E->stream);
        trail.clear();
        E->prof = &trail;
        mark(E, -1);
        err = forward(E, static_cast<int>(ncols), E->d_tok, E->d_pos, E->d_req, true, 0, nullptr);
        if (err == cudaSuccess) err = head_and_sample(E, E->h, static_cast<int>(ncols), nullptr, static_cast<int>(ncols) <= E->fuse_max_cols);
        E->prof = nullptr;
        if (err == cudaSuccess) err = cudaStreamSynchronize(E->stream);
        for (size_t i = 1; i < trail.size() && err == cudaSuccess; ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, trail[i - 1].first, trail[i].first);
            acc[trail[i].second] += ms;
            if (r == 0) cnt[trail[i].second] += 1;
        }
        for (auto& t : trail) cudaEventDestroy(t.first);
    }
    E->use_pdl = pdl;
    ENG_CUDA(err);
    for (int k = 0; k < kProfN; ++k) {
        if (ms_by_class) ms_by_class[k] = static_cast<float>(acc[k] / reps);
        if (launches_by_class) launches_by_class[k] = cnt[k];
    }
    return DETGPU_OK;
}

}  // extern "C"

extern "C" {

// Timing experiment: capture a decode-step graph for ncols slots at context ctx with the kernel
// classes in skip_mask left out (bit k = class k of detgpu_profile_decode_step), replay it `reps`
// times and return the mean ms per step. Numerically meaningless when skip_mask != 0; never used
// by generate().
int detgpu_set_option(detgpu_engine* h, const char* name, int64_t value) {
    if (h == nullptr || name == nullptr) return fail(nullptr, DETGPU_EINVAL, "set_option: null argument");
    Engine* E = h->e.get();
    if (std::strcmp(name, "l2pf_mask") == 0) E->l2pf_mask = static_cast<unsigned>(value);
    else if (std::strcmp(name, "l2pf_cap_mb") == 0) E->l2pf_cap = value << 20;
    else if (std::strcmp(name, "pdl") == 0) E->use_pdl = value != 0;
    else if (std::strcmp(name, "self_pf_kb") == 0) E->self_pf_kb = static_cast<int>(value);
    else if (std::strncmp(name, "self_pf_kb_", 11) == 0) {
        static const char* kCls[5] = {"qkv", "o", "gate_up", "down", "lm_head"};
        int i = 0;
        while (i < 5 && std::strcmp(name + 11, kCls[i]) != 0) ++i;
        if (i == 5) return fail(E, DETGPU_EINVAL, std::string("set_option: unknown option '") + name + "'");
        E->self_pf_kb_cls[i] = static_cast<int>(value);
    }
    else if (std::strcmp(name, "max_nsub") == 0) E->max_nsub = static_cast<int>(value);
    else if (std::strcmp(name, "gemm_pair") == 0) E->gemm_pair = static_cast<int>(value);
    else if (std::strcmp(name, "gemm_persist") == 0) E->gemm_persist = static_cast<int>(value);
    else if (std::strcmp(name, "prefill_blocks") == 0) E->prefill_blocks = value != 0;
    else if (std::strcmp(name, "attn_cluster_max_cols") == 0) E->attn_cluster_max_cols = static_cast<int>(value);
    else if (std::strcmp(name, "attn_sep_recv_max_cols") == 0) E->attn_sep_recv_max_cols = static_cast<int>(value);
    else if (std::strcmp(name, "attn_stream_min_cols") == 0) E->attn_stream_min_cols = static_cast<int>(value);
    else if (std::strcmp(name, "attn_stream_prefill") == 0) E->attn_stream_prefill = static_cast<int>(value);
    else if (std::strcmp(name, "mixed_steps") == 0) E->mixed_steps = value != 0;
    else if (std::strcmp(name, "fuse_max_cols") == 0) E->fuse_max_cols = static_cast<int>(value < 0 ? 0 : value > 8 ? 8 : value);
    else if (std::strcmp(name, "trace") == 0) {
        cudaSetDevice(E->device);
        if (E->trace_buf != nullptr) cudaFree(E->trace_buf);
        E->trace_buf = nullptr;
        if (value > 0) {
            const uint32_t cap = static_cast<uint32_t>(value < (1 << 24) ? value : (1 << 24));
            ENG_CUDA(cudaMalloc(&E->trace_buf, sizeof(TraceRec) * (cap + 1)));
            const uint32_t hdr[2] = {0u, cap};
            ENG_CUDA(cudaMemcpy(E->trace_buf, hdr, sizeof(hdr), cudaMemcpyHostToDevice));
        }
    }
    else return fail(E, DETGPU_EINVAL, std::string("set_option: unknown option '") + name + "'");
    cudaSetDevice(E->device);
    for (auto& kv : E->graphs) cudaGraphExecDestroy(kv.second);
    E->graphs.clear();
    E->graph_used.clear();
    return DETGPU_OK;
}

int detgpu_trace_read(detgpu_engine* h, void* out, uint32_t max_records, uint32_t* n_records) {
    if (h == nullptr || n_records == nullptr) return fail(nullptr, DETGPU_EINVAL, "trace_read: null argument");
    Engine* E = h->e.get();
    *n_records = 0;
    if (E->trace_buf == nullptr) return fail(E, DETGPU_EINVAL, "trace_read: tracing is off");
    cudaSetDevice(E->device);
    ENG_CUDA(cudaStreamSynchronize(E->stream));
    uint32_t hdr[2];
    ENG_CUDA(cudaMemcpy(hdr, E->trace_buf, sizeof(hdr), cudaMemcpyDeviceToHost));
    const uint32_t n = std::min(std::min(hdr[0], hdr[1]), max_records);
    if (out != nullptr && n > 0)
        ENG_CUDA(cudaMemcpy(out, E->trace_buf + 1, sizeof(TraceRec) * n, cudaMemcpyDeviceToHost));
    *n_records = n;
    hdr[0] = 0;
    ENG_CUDA(cudaMemcpy(E->trace_buf, hdr, sizeof(uint32_t), cudaMemcpyHostToDevice));
    return DETGPU_OK;
}

int detgpu_profile_graph(detgpu_engine* h, uint32_t ncols, uint32_t ctx, uint32_t skip_mask, uint32_t reps,
                         float* ms_per_step) {
    if (h == nullptr || h->e->toy) return fail(nullptr, DETGPU_EINVAL, "profile: transformer engine required");
    Engine* E = h->e.get();
    cudaSetDevice(E->device);
    if (ncols == 0 || ncols > E->max_batch || ctx == 0 || ctx > E->max_context || reps == 0)
        return fail(E, DETGPU_EINVAL, "profile: bad ncols/ctx/reps");
    if (int rc = ensure_outputs(E, static_cast<int>(ncols), 2)) return rc;
    std::vector<int> step(ncols, -1), pos(ncols, static_cast<int>(ctx) - 1), tok(ncols, 1), zero(ncols, 0);
    std::vector<DevPolicy> dp(ncols, DevPolicy{DETGPU_GREEDY, 0, 0.0f, 1 << 30});
    ENG_CUDA(cudaMemcpy(E->d_pol, dp.data(), sizeof(DevPolicy) * ncols, cudaMemcpyHostToDevice));
    ENG_CUDA(cudaMemcpy(E->d_tok, tok.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice));
    ENG_CUDA(cudaMemcpy(E->d_status, zero.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice));
    // positions stay fixed across replays: the sampler is skipped via step = -1 unless asked for
    ENG_CUDA(cudaMemcpy(E->d_pos, pos.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice));
    ENG_CUDA(cudaMemcpy(E->d_step, step.data(), sizeof(int) * ncols, cudaMemcpyHostToDevice));
    E->skip_mask = skip_mask;
    cudaGraph_t g;
    ENG_CUDA(cudaStreamBeginCapture(E->stream, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = forward(E, static_cast<int>(ncols), E->d_tok, E->d_pos, E->d_req, true, 0, nullptr);
    if (e == cudaSuccess) e = head_and_sample(E, E->h, static_cast<int>(ncols), nullptr, static_cast<int>(ncols) <= E->fuse_max_cols);
    cudaError_t e2 = cudaStreamEndCapture(E->stream, &g);
    E->skip_mask = 0;
    ENG_CUDA(e);
    ENG_CUDA(e2);
    cudaGraphExec_t ex;
    ENG_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    for (int i = 0; i < 3; ++i) ENG_CUDA(cudaGraphLaunch(ex, E->stream));
    ENG_CUDA(cudaEventRecord(E->ev[0], E->stream));
    for (uint32_t i = 0; i < reps; ++i) ENG_CUDA(cudaGraphLaunch(ex, E->stream));
    ENG_CUDA(cudaEventRecord(E->ev[1], E->stream));
    ENG_CUDA(cudaEventSynchronize(E->ev[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, E->ev[0], E->ev[1]);
    cudaGraphExecDestroy(ex);
    if (ms_per_step) *ms_per_step = ms / reps;
    return DETGPU_OK;
}

}  // extern "C"
