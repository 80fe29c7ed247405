// Batch-invariant bf16 GEMM on tcgen05 (declarations shared by gemm.cu and the engine).
//
//   Y[col, n] = sum_k X[col, k] * W[n, k]      W: [n_out, K] bf16 (weights), X: [ncols, K] bf16
//
// Swap-AB: weight rows are the MMA M dimension (128 per CTA), activation columns (tokens) are the
// MMA N dimension in fixed 64-wide sub-tiles. The instruction shape (M=128, N=64, K=16), the K
// order (k-block 0..K/64-1, four K=16 steps each, accumulated in TMEM) and the tile of every column
// are the same for every batch size: a column's bits depend only on its own activations and the
// weights (tested by tests/test_gpu_gemm.py::test_batch_invariance).
#pragma once
#include "trace.h"
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace detgpu {

enum GemmMode : int {
    kEpiStoreF32 = 0,   // out[off(col) + row] = acc            (logits, generic)
    kEpiAddF32 = 1,     // out[col*ld + row] += acc              (residual stream)
    kEpiQkvRope = 2,    // RoPE(q,k) -> q bf16, k/v appended to the paged KV cache
    kEpiSwiglu = 3,     // interleaved gate/up rows -> silu(g)*u bf16
};

struct GemmParams {
    int n_out;   // rows of W (multiple of 128)
    int k;       // reduction extent (multiple of 64)
    int ncols;   // number of activation columns
    int mode;
    int ksplit;  // 0: gemm_ksplit(n_out, k) (the engine's numeric definition); >0: explicit (test hooks)
    int w_tiled; // weights pre-tiled [n_out/128][K/64][128][64] (engine) or plain row-major
    int mma_wide;// 1: one N = nb*64 MMA per K=16 step instead of nb N=64 ones (same column bits)
    // kEpiStoreF32 / kEpiAddF32
    float* out;
    int64_t ld_out;            // per-column stride of `out` (elements)
    const int* col_step;       // optional: logits trace step per column (<0 = inactive)
    const int* col_slot;       // optional: request slot per column (with col_step)
    int64_t slot_stride;       // elements per slot in the trace (with col_step)
    // kEpiQkvRope
    __nv_bfloat16* q_out;      // [ncols][hq*hd]
    int hq, hkv, hd;
    const int* col_pos;        // position of each column
    const int* col_req;        // request slot of each column (block table row)
    const float* rope_cos;     // [max_pos][hd/2]
    const float* rope_sin;
    __nv_bfloat16* kcache;     // this layer's K pool [pages][hkv][page][hd]
    __nv_bfloat16* vcache;
    const int* block_table;    // [slots][max_pages]
    int max_pages;
    int page;                  // positions per page
    // kEpiSwiglu
    __nv_bfloat16* act;        // [ncols][n_out/2]
    // fused RMSNorm of the B operand (<= 8 columns, K == norm_d): X = bf16(rmsnorm(norm_x) * gamma)
    const float* norm_x;       // [ncols][norm_d] f32 residual stream, or nullptr (X via tmX)
    const float* norm_ss;      // [ncols][norm_d/128] per-tile sums of squares of norm_x
    const __nv_bfloat16* norm_gamma;
    int norm_d;
    float norm_eps;
    // kEpiAddF32 in fused decode: emit the next RMSNorm's per-tile sums of squares of the result
    float* ss_out;             // [ncols][ss_tiles] or nullptr
    int ss_tiles;              // n_out / 128
    const void* w_raw;         // tiled weights (w_tiled): base pointer for the L2 self-prefetch below
    int max_nsub;              // > 128 columns: widest tile in 64-column sub-tiles (4, or 0: 2)
    int pair;                  // > 64 columns: CTA-pair tiles (gemm_pair_kernel, cta_group::2) when 1
    int persist;               // > 64 columns: persistent clusters, double-buffered TMEM (gemm_persist_kernel)
    int self_pf_kb;            // before the PDL wait, warm up to this many of the CTA's own weight
                               // k-blocks beyond the shared-memory ring into L2 (0: off)
    const void* l2pf;          // optional: bytes warmed into L2 at kernel start (the next kernel's weights)
    int64_t l2pf_bytes;
    TraceRec* trace;    // optional per-CTA timeline (timing instrumentation)
    uint32_t trace_tag;
};

// 3D tensor map of a weight matrix [n_out][k] (row-major view or pre-tiled, see gemm.cu load_w).
bool make_tmap_weights(CUtensorMap* m, const void* ptr, uint64_t n_out, uint64_t k, bool tiled);
// Tensor map for a row-major [rows, inner] bf16 matrix, box = 64 (inner) x box_rows, 128B swizzle.
bool make_tmap_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint32_t box_rows);

// Number of fixed K-segments for a GEMM shape (part of the numeric definition):
// S = min(K/64, max(2, min(8, 256 / (n_out/128)))). Never depends on the batch.
int gemm_ksplit(int n_out, int k);

// Launch (PDL-enabled) on `stream`. tmW: make_tmap_weights; tmX: box 64 rows over exactly ncols
// rows, so the MMA's padding rows are TMA zero-fill and cost no memory traffic.
cudaError_t gemm_launch(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p,
                        cudaStream_t stream, bool pdl);

}  // namespace detgpu
