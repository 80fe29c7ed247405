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

template <int NSUB>
struct Cfg {
    // <= 128 columns: ~100 KB of shared memory so that two CTAs fit per SM (the next GEMM's CTAs,
    // launched early by programmatic dependent launch, stream their weights while this one drains);
    // 256-column tiles keep a deep ring at one CTA per SM.
    static constexpr int STAGE_BYTES = A_BYTES + NSUB * B_BYTES;
    static constexpr int BUDGET = NSUB <= 2 ? 96 * 1024 : 192 * 1024;
    static constexpr int STAGES = BUDGET / STAGE_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int MIN_CTAS = NSUB <= 2 ? 2 : 1;
    static constexpr uint32_t TMEM = NSUB * SUB_N;   // f32 accumulator columns (power of two)
};

__device__ __forceinline__ void epilogue_store(const GemmParams& p, int row, int col, float v) {
    switch (p.mode) {
        case kEpiStoreF32: {
            int64_t off;
            if (p.col_step != nullptr) {
                const int st = p.col_step[col];
                if (st < 0) return;
                off = static_cast<int64_t>(p.col_slot[col]) * p.slot_stride + static_cast<int64_t>(st) * p.n_out;
            } else {
                off = static_cast<int64_t>(col) * p.ld_out;
            }
            p.out[off + row] = v;
            return;
        }
        case kEpiAddF32: {
            float* dst = p.out + static_cast<int64_t>(col) * p.ld_out + row;
            *dst = __fadd_rn(*dst, v);
            return;
        }
        default:
            return;
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

// silu(g) * u with g = gate row 2j, u = up row 2j+1; silu(g) = g / (1 + exp(-g)).
__device__ __forceinline__ void epilogue_swiglu(const GemmParams& p, int row, int col, float v, float partner) {
    if ((row & 1) != 0) return;
    const float e = det_expf(-v);
    const float sg = __fdiv_rn(v, __fadd_rn(1.0f, e));
    p.act[static_cast<int64_t>(col) * (p.n_out / 2) + (row >> 1)] = f2bf(__fmul_rn(sg, partner));
}

__device__ __forceinline__ void epilogue_any(const GemmParams& p, int row, int col, float v) {
    if (p.mode == kEpiQkvRope || p.mode == kEpiSwiglu) {
        const float partner = __shfl_xor_sync(0xffffffffu, v, 1);   // callers keep `col` warp-uniform
        if (p.mode == kEpiQkvRope) epilogue_qkv(p, row, col, v, partner);
        else epilogue_swiglu(p, row, col, v, partner);
    } else {
        epilogue_store(p, row, col, v);
    }
}

// Grid (S, n_out/128, column groups), cluster (S,1,1): the S CTAs of a cluster own the same 128
// weight rows and columns and the fixed K-segments [s*nkb/S, (s+1)*nkb/S) of the reduction. Each
// runs its segment as one tcgen05 accumulation chain in TMEM; the S partial tiles are exchanged
// through distributed shared memory and combined per element with the reference tree over the S
// partials in segment order (detcore.cpp:135-150). S depends only on the GEMM shape.
template <int NSUB>
__global__ void __launch_bounds__(256, Cfg<NSUB>::MIN_CTAS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmParams p) {
    using C = Cfg<NSUB>;
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * NSUB * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.ksplit;
    const int seg = blockIdx.x;                 // == %cluster_ctarank
    const int m0 = blockIdx.y * BM;
    const int col0 = blockIdx.z * (NSUB * SUB_N);
    const int ncols = min(NSUB * SUB_N, p.ncols - col0);
    const int nb = (ncols + SUB_N - 1) / SUB_N;
    const int nkb_all = p.k / BK;
    const int kb0 = seg * nkb_all / S, kb1 = (seg + 1) * nkb_all / S;
    const int nkb = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tslot, C::TMEM);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    // Weight tile (128 rows x 64 k) through a 3D tensor map: pre-tiled weights are one contiguous
    // 16 KB block per (tile, k-block) -> coordinate (0, 0, tile*nkb + kb); a plain row-major matrix
    // is viewed as [rows][K/64][64] -> coordinate (0, kb, m0). Same smem image either way.
    auto load_w = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int kb) {
        if (p.w_tiled) tma_load_3d(dst, m, bar, 0, 0, blockIdx.y * nkb_all + kb, kEvictFirst);
        else tma_load_3d(dst, m, bar, 0, kb, m0, kEvictFirst);
    };
    const uint32_t stage_tx = A_BYTES + nb * B_BYTES;
    const int pre = min(STAGES, nkb);
    if (warp == 0 && lane == 0) {
        // Weight tiles do not depend on the previous kernel: stream them before the PDL wait.
        for (int i = 0; i < pre; ++i) {
            mbar_arrive_expect_tx(&full[i], stage_tx);
            load_w(sA + i * A_BYTES, &tmW, &full[i], kb0 + i);
        }
    }
    // Every kernel waits for its predecessor before triggering its dependents, so when a kernel
    // starts, all kernels before its predecessor have completed (attention relies on this).
    pdl_wait();
    pdl_trigger();
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < pre; ++i)
                for (int j = 0; j < nb; ++j)
                    tma_load_2d(sB + (i * NSUB + j) * B_BYTES, &tmX, &full[i], (kb0 + i) * BK, col0 + j * SUB_N,
                                kEvictLast);
            for (int i = pre; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], stage_tx);
                load_w(sA + s * A_BYTES, &tmW, &full[s], kb0 + i);
                for (int j = 0; j < nb; ++j)
                    tma_load_2d(sB + (s * NSUB + j) * B_BYTES, &tmX, &full[s], (kb0 + i) * BK, col0 + j * SUB_N,
                                kEvictLast);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, SUB_N);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                mbar_wait(&full[s], (i / STAGES) & 1);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = smem_u32(sB + s * NSUB * B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint64_t adesc = umma_desc_k128(a_base + k * 32);
                    for (int j = 0; j < nb; ++j) {
                        const uint64_t bdesc = umma_desc_k128(b_base + j * B_BYTES + k * 32);
                        tc_mma_bf16(tbase + j * SUB_N, adesc, bdesc, idesc, (i | k) != 0 ? 1u : 0u);
                    }
                }
                tc_commit(&empty[s]);   // frees the smem stage once these MMAs retire
            }
            tc_commit(tfull);           // accumulator complete
        }
    } else if (warp >= 4) {
        const int ew = warp - 4;       // == warp % 4: TMEM lanes 32*ew .. 32*ew+31
        const int rl = ew * 32 + lane;
        mbar_wait(tfull, 0);
        tc_fence_after();
        float* P = reinterpret_cast<float*>(smem);   // partial tile [col][128] (stages are idle now)
        for (int j = 0; j < nb; ++j) {
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tbase + (static_cast<uint32_t>(ew * 32) << 16) + j * SUB_N + h * 32, r);
                tc_wait_ld();
                const int cl0 = j * SUB_N + h * 32;
                if (S == 1) {
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (cl0 + c < ncols) epilogue_any(p, m0 + rl, col0 + cl0 + c, __uint_as_float(r[c]));
                } else {
#pragma unroll
                    for (int c = 0; c < 32; ++c)
                        if (cl0 + c < ncols) P[(cl0 + c) * BM + rl] = __uint_as_float(r[c]);
                }
            }
        }
    }
    if (S > 1) {
        cluster_sync_all();   // partial tiles of all segments visible cluster-wide
        if (warp >= 4) {
            const int rl = (warp - 4) * 32 + lane;
            const uint32_t pbase = smem_u32(smem);
            for (int cl = seg; cl < ncols; cl += S) {
                float v[8];
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    v[s] = s < S ? ld_dsmem_f32(mapa_shared(pbase + 4u * static_cast<uint32_t>(cl * BM + rl), s))
                                 : kNegZero;
                epilogue_any(p, m0 + rl, col0 + cl, local_tree_sum<8>(v));
            }
        }
        cluster_sync_all();   // peers keep their shared memory until every reader is done
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, C::TMEM);
    }
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
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<NSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.ksplit, p.n_out / BM, (p.ncols + NSUB * SUB_N - 1) / (NSUB * SUB_N));
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
    if (p.ncols <= 64) return launch_nsub<1>(tmW, tmX, p, stream, pdl);
    if (p.ncols <= 128) return launch_nsub<2>(tmW, tmX, p, stream, pdl);
    return launch_nsub<4>(tmW, tmX, p, stream, pdl);
}

}  // namespace detgpu
