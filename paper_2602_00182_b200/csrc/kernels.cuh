// Non-GEMM kernels of the deterministic decode path (declarations).
#pragma once
#include "trace.h"
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "detgpu.h"

namespace detgpu {

// Attention KV chunk: positions [c*kAttnChunk, (c+1)*kAttnChunk) form one online-softmax chunk,
// combined in chunk order. Part of the numeric definition; never batch-dependent.
constexpr int kAttnChunk = 64;

// ---- RMSNorm (optionally with the embedding gather fused in) ----
// x_in [rows][d] f32 (row = col_index ? col_index[col] : col); when embed != nullptr the input row
// is embed[col_token[col]] (bf16) and is also written to x_out[col][d] as f32.
cudaError_t launch_rmsnorm(const float* x_in, float* x_out, const __nv_bfloat16* embed, const int* col_token,
                           const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* col_index, int ncols, int d,
                           float eps, cudaStream_t stream, bool pdl);

cudaError_t launch_rmsnorm_ex(const float* x_in, float* x_out, const __nv_bfloat16* embed, const int* col_token,
                              const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* in_index, const int* out_index,
                              int ncols, int d, float eps, cudaStream_t stream, bool pdl, float* ss_out = nullptr);
// Embedding gather x = embed[tok] (+ normalised h); with ss_out also the per-128-element partial
// sums of squares of x that a fused-norm GEMM consumes.
cudaError_t launch_embed(const __nv_bfloat16* embed, const int* col_token, float* x_out, float* ss_out,
                         const __nv_bfloat16* gamma, __nv_bfloat16* h_out, int ncols, int d, float eps,
                         cudaStream_t stream, bool pdl);
// out[out_index[i]] = rmsnorm(x[in_index[i]]) for i < n
cudaError_t launch_rmsnorm_gather(const float* x, const __nv_bfloat16* gamma, __nv_bfloat16* out, const int* in_index,
                                  const int* out_index, int n, int d, float eps, cudaStream_t stream, bool pdl);
cudaError_t launch_expf(const float* x, float* y, int64_t n, cudaStream_t stream);
cudaError_t launch_tree_sum(const float* x, float* out, int rows, int n, cudaStream_t stream);
// tiled: store GEMM-tiled [phys_rows/128][cols/64][128][64] instead of row-major
cudaError_t launch_init_tensor(__nv_bfloat16* dst, uint64_t seed, int64_t rows, int64_t cols, int scale_exp,
                               int is_gamma, int row_mul, int row_add, cudaStream_t stream, bool tiled = false);

// ---- attention ----
struct AttnParams {
    const __nv_bfloat16* q;        // [ncols][hq*hd]
    const __nv_bfloat16* kcache;   // [pages][hkv][page][hd]
    const __nv_bfloat16* vcache;
    const int* block_table;        // [slots][max_pages]
    const int* col_pos;            // query position (<0 inactive); attends to [0, pos]
    const int* col_req;            // slot of each column
    __nv_bfloat16* out;            // [ncols][hq*hd]
    float* ws;                     // partials
    int* tickets;                  // [ncols][hkv], zero-initialised; reset by the combining CTA
    int ncols, hq, hkv, hd, page, max_pages, max_chunks;
    int decode;                    // 1: every column's positions < pos were written by earlier launches
    int prefill_blocks;            // prefill: query blocks share each K/V chunk (attn_prefill_kernel)
    int cluster_max_cols;          // decode: cluster combine up to this many columns (0: always)
    int sep_recv;                  // cluster combine: separate receive buffer (no push handshake)
    const void* l2pf;              // optional: bytes warmed into L2 at kernel start (the o weights)
    int64_t l2pf_bytes;
    TraceRec* trace;        // optional per-CTA timeline (timing instrumentation)
    uint32_t trace_tag;
    // streamed decode attention (attention_stream.cu): 2D tensor maps over the whole K / V pools
    // ([rows][hd], 64x64 boxes, 128B swizzle), this layer's first row, and the column count from
    // which it replaces attn_chunk_kernel (0: never)
    const CUtensorMap* tm_k;
    const CUtensorMap* tm_v;
    int64_t kv_row0;
    int stream_min_cols;
    int stream_prefill;            // prefill chunks through the streamed kernel too (every K/V load after the wait)
};
size_t attn_workspace_bytes(const AttnParams& a);
cudaError_t launch_attention(const AttnParams& a, cudaStream_t stream, bool pdl);
bool attention_stream_supported(const AttnParams& a);
cudaError_t launch_attention_stream(const AttnParams& a, cudaStream_t stream, bool pdl);

// ---- softmax + decode ----
struct DevPolicy {
    int kind;        // DETGPU_GREEDY / TOP_K / NUCLEUS
    uint32_t k;
    float p;
    int max_tokens;
};
inline DevPolicy to_dev_policy(const detgpu_policy& p) {
    DevPolicy d;
    d.kind = p.kind;
    d.k = p.has_k ? p.k : 0;
    d.p = p.has_p ? p.p : 0.0f;
    d.max_tokens = static_cast<int>(p.max_tokens);
    return d;
}

struct SampleParams {
    const float* logits;        // row r at logits + row_off(r)
    int64_t logit_row_stride;   // used when col_step == nullptr
    const int* col_step;        // engine: trace step of each row (<0 inactive)
    const int* col_slot;
    int64_t slot_stride;
    int rows, vocab;
    const DevPolicy* policy;    // per row (engine: per slot via col_slot)
    uint64_t* prng;             // [slot][4]
    float* probs;               // [rows][vocab] scratch / output
    uint64_t* scratch;          // sample_scratch_bytes
    uint32_t* token_out;        // [rows] (engine: next input token)
    int32_t* status;            // [rows] (or per slot)
    // engine bookkeeping (nullable): tokens_hist[slot*tcap + step] = token; pos/step advance
    uint32_t* tokens_hist;
    int tcap;
    int* col_pos;
    int* col_step_mut;
    int state_by_slot;          // token_out / col_pos / col_step_mut indexed by slot (else by row)
    // small batches (rows <= kSampleMultiMaxRows, nullable): the row is split over several CTAs
    float* blk_ws;              // [rows][kSampleMaxBlocks][4] block max / non-finite / subtree sum
    int* tickets;               // [rows], zero-initialised; reset by the last block
};
constexpr int kSampleMaxBlocks = 32;   // vocab <= 32 * 4096
constexpr int kSampleMultiMaxRows = 16;
size_t sample_scratch_bytes(int rows, int vocab);
cudaError_t launch_sample(const SampleParams& sp, cudaStream_t stream, bool pdl);

}  // namespace detgpu
