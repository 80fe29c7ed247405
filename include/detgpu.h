/*
 * detgpu — C-ABI of the B200-native deterministic inference engine.
 *
 * This is the drop-in boundary for the reference's deterministic compute core
 * (reference proj/include/verinf/detcore.hpp:151-163, proj/src/detcore.cpp:380-410) and the
 * receipt output hash (proj/src/receipts.cpp:119-120). Plain pointers and sizes only; no torch or
 * C++ types cross it. Callers own every buffer. All functions are thread-safe across handles;
 * calls on one handle are serialised by the caller (one handle per GPU = one replica).
 *
 * Errors: functions return DETGPU_OK or a DETGPU_E* code; detgpu_last_error(h) (or
 * detgpu_global_error() when no handle exists) gives the diagnostic. DETGPU_EINVAL is the
 * counterpart of the reference's std::invalid_argument (unknown arch, malformed policy,
 * out-of-vocabulary prompt token, batch_size == 0, non-finite values).
 */
#ifndef DETGPU_H
#define DETGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DETGPU_OK 0
#define DETGPU_EINVAL 1      /* std::invalid_argument in the reference */
#define DETGPU_ECUDA 2       /* CUDA runtime / launch failure */
#define DETGPU_ENOMEM 3      /* device or host allocation failed */
#define DETGPU_ENONFINITE 4  /* non-finite logits (reference check_finite, detcore.cpp:127-133) */
#define DETGPU_ENODEV 5      /* no sm_100 device */

/* DecodeKind (detcore.hpp:50). */
#define DETGPU_GREEDY 0
#define DETGPU_TOP_K 1
#define DETGPU_NUCLEUS 2

/* DecodePolicy (detcore.hpp:52-66): k present iff top_k, p present iff nucleus. */
typedef struct detgpu_policy {
    uint8_t kind;
    uint8_t has_k;
    uint8_t has_p;
    uint8_t reserved;
    uint32_t k;
    float p;
    uint32_t max_tokens;
} detgpu_policy;

typedef struct detgpu_model_info {
    uint32_t n_layers;
    uint32_t d_model;
    uint32_t n_heads;
    uint32_t n_kv_heads;
    uint32_t head_dim;
    uint32_t ffn;
    uint32_t vocab;
    uint32_t toy; /* 1: the reference ToyModel (detcore.hpp:139-149) run on the GPU */
    float rope_theta;
    float rms_eps;
    uint64_t n_params;
    uint64_t weight_bytes;
} detgpu_model_info;

/* Per-call device timings (CUDA events on the engine stream) and byte counts. */
typedef struct detgpu_stats {
    float prefill_ms;
    float decode_ms;       /* decode loop: steps 1..T-1 forward + all sampling */
    float d2h_ms;          /* device->host copies of tokens and logits */
    float hash_ms;         /* host SHA-256 of canonical bytes (wall) */
    uint64_t decode_steps; /* forward passes in the decode loop */
    uint64_t tokens;       /* generated tokens (sum over requests) */
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t kernel_launches;
} detgpu_stats;

/* Flags for detgpu_generate. */
#define DETGPU_F_DEVICE_ONLY 1u /* keep tokens/logits in HBM: no D2H, no out_hash (bench `value`) */
#define DETGPU_F_RECEIPT_V2 2u  /* out_hash = receipt v2 digest (per-step Merkle roots computed on the
                                   GPU, see detgpu_hash_canonical_v2); logits D2H only if requested */
#define DETGPU_F_CONTINUOUS 4u  /* continuous batching: batch_size decode slots stay busy, each
                                   request admitted as soon as a slot frees (same bytes per request) */

typedef struct detgpu_engine detgpu_engine;

const char* detgpu_version(void);
const char* detgpu_global_error(void);

/* Approved architecture profiles (ArchRegistry::defaults, detcore.cpp:12-20, plus "b200"). */
int detgpu_arch_supported(const char* arch);

/*
 * Create an engine on `device` for `model_id` under `arch`:
 *   arch "archA" / "archB": the reference ToyModel with that accumulation profile, any model_id
 *                           (weights from fnv1a64(model_id), detcore.cpp:275-296);
 *   arch "b200": a Llama-style transformer whose shape is named by the model_id prefix
 *                ("llama-tiny" | "llama-mid" | "llama3-8b", optionally ":tag"), weights
 *                counter-generated from fnv1a64(model_id).
 * max_batch: requests decoded together (1..256); max_context: prompt + generated tokens.
 * Replaces ToyModel::from_model_id + ArchRegistry::find (detcore.cpp:288, 333).
 */
int detgpu_create(int device, const char* model_id, const char* arch, uint32_t max_batch,
                  uint32_t max_context, detgpu_engine** out);
void detgpu_destroy(detgpu_engine* h);
int detgpu_get_model_info(const detgpu_engine* h, detgpu_model_info* out);
const char* detgpu_last_error(const detgpu_engine* h);

/*
 * Run n_req requests (reference infer_batch, detcore.cpp:387-410; infer == n_req 1).
 * Requests are decoded in groups of at most batch_size (0 -> DETGPU_EINVAL, detcore.cpp:389);
 * the bytes of each request do not depend on the grouping.
 *   prompts[i][0..prompt_lens[i]) token ids; seeds[i] seeds the request's xoshiro256++ stream.
 *                    An empty prompt is accepted as the reference accepts it (detcore.cpp:340-352):
 *                    for "b200" it means the one-token prompt [0] (BOS), for the ToyModel the
 *                    zero state.
 *   tokens_out[i]  : policies[i].max_tokens u32 (may be NULL with DETGPU_F_DEVICE_ONLY)
 *   logits_out     : NULL, or an array of n_req pointers each NULL or max_tokens*vocab f32
 *   out_hash       : NULL or n_req*32 bytes: SHA-256 of the canonical output bytes
 *                    (detcore.cpp:73-84 layout, receipts.cpp:120 commitment)
 *   stats          : NULL or filled with timings
 */
int detgpu_generate(detgpu_engine* h, uint32_t n_req, const uint32_t* const* prompts,
                    const uint32_t* prompt_lens, const detgpu_policy* policies, const uint64_t* seeds,
                    uint32_t batch_size, uint32_t* const* tokens_out, float* const* logits_out,
                    uint8_t* out_hash, uint32_t flags, detgpu_stats* stats);

/* The engine's CUDA stream (so callers can bracket work with their own events). */
void* detgpu_stream(const detgpu_engine* h);
/* One un-graphed decode step (forward + lm_head + sample) for ncols slots at context ctx with an
 * event after every launch: mean ms per step by kernel class (0 norm, 1 qkv, 2 attention, 3 o,
 * 4 gate/up, 5 down, 6 lm_head, 7 sample) and launches per step by class. Measurement hook for
 * bench.py's roofline; never used on the serving path. */
int detgpu_profile_decode_step(detgpu_engine* h, uint32_t ncols, uint32_t ctx, uint32_t reps,
                               float* ms_by_class, uint32_t* launches_by_class);

/* Scheduling knobs that never change a result bit (timing experiments / deployment tuning):
 *   "l2pf_mask"   which decode kernels warm the next kernel's weights into L2 (bit 0 attention->o,
 *                 1 o->gate/up, 2 gate/up->down, 3 down->next QKV, 4 QKV->o)
 *   "l2pf_cap_mb" cap on the bytes one kernel warms
 *   "pdl"         programmatic dependent launch on (1) / off (0)
 *   "prefill_blocks" prefill attention on query blocks sharing each K/V chunk (1, default) or
 *                 one query per CTA (0)
 *   "attn_cluster_max_cols" decode attention combines chunks in a cluster up to this many
 *                 columns (default 8), in the workspace/ticket path above (0: always cluster)
 *   "attn_sep_recv_max_cols" up to this many columns the cluster combine's leader receives the
 *                 chunk partials in a buffer of its own (no push handshake; default 2, 0: never)
 *   "attn_stream_min_cols" decode attention from this many columns on runs the streamed kernel
 *                 (persistent CTAs, TMA ring of K/V chunks; default 9; 0: never)
 *   "fuse_max_cols" decode RMSNorm folded into the consuming GEMMs up to this many columns
 *                 (default and maximum 8; 0: separate RMSNorm kernels)
 *   "max_nsub"    GEMM tiles above 64 columns: at most 2 or 4 64-column sub-tiles per CTA
 *   "gemm_persist" GEMMs above 64 columns as persistent clusters with double-buffered TMEM and a
 *                 push combine (bit-identical; 1: K-segment count S <= 2 only, 2: every S;
 *                 default 0: measured slower inside the decode / prefill pipeline)
 *   "gemm_pair"   GEMMs above 64 columns as CTA pairs (tcgen05 cta_group::2, 256 x 128 tiles;
 *                 bit-identical; default 0: measured no faster than two one-CTA tiles per SM)
 *   "self_pf_kb"  GEMM CTAs warm this many of their own weight k-blocks (16 KB each) beyond the
 *                 shared-memory ring into L2 before waiting on their predecessor
 *   "self_pf_kb_qkv" / "_o" / "_gate_up" / "_down" / "_lm_head": the same for one GEMM class
 *                 (-1: self_pf_kb; default -1 except the o and down projections: 0)
 *   "trace"       > 0: record a per-CTA timeline of the decode kernels (capacity in records), 0: off
 * Cached decode graphs are dropped. Returns DETGPU_EINVAL for an unknown name. */
int detgpu_set_option(detgpu_engine* h, const char* name, int64_t value);

/* Copy up to max_records timeline records (32 bytes each: u32 tag = class << 24 | CTA, u32 sm,
 * u64 t_start, t_wait_released, t_end in globaltimer ns) and reset the buffer. */
int detgpu_trace_read(detgpu_engine* h, void* out, uint32_t max_records, uint32_t* n_records);

/* Timing experiment: mean ms of a captured decode-step graph with the kernel classes of skip_mask
 * left out (results meaningless when skip_mask != 0). Measurement hook only. */
int detgpu_profile_graph(detgpu_engine* h, uint32_t ncols, uint32_t ctx, uint32_t skip_mask, uint32_t reps,
                         float* ms_per_step);

/* Out-of-bounds-write check (compute-sanitizer substitute): every engine device buffer is followed
 * by a 4 KiB canary; counts the live buffers and those whose canary changed. */
int detgpu_debug_check_canaries(uint64_t* n_checked, uint64_t* n_bad);

/* ---- host-side helpers of the receipt path (no GPU needed) ---- */

/* SHA-256 (receipts.hpp:53-54 hash_commit; sha256.cpp:32-37). */
void detgpu_sha256(const uint8_t* data, size_t n, uint8_t out[32]);
/* Canonical output size and encoding (detcore.cpp:73-84). */
size_t detgpu_canonical_size(uint32_t n_tokens, uint32_t vocab);
void detgpu_encode_canonical(const uint32_t* tokens, uint32_t n_tokens, const float* logits,
                             uint32_t vocab, uint8_t* out);
/* SHA-256 of the canonical bytes without materialising them. */
void detgpu_hash_canonical(const uint32_t* tokens, uint32_t n_tokens, const float* logits,
                           uint32_t vocab, uint8_t out[32]);
/* Receipt v2: root_t = Merkle root of step t's f32 logits (little-endian
 * bytes) in 4 KiB leaves with the reference DA tree rules (da.hpp:16-20: leaf H(0x00||blob),
 * node H(0x01||l||r), odd level pairs the last node with itself); out_hash_v2 =
 * SHA-256("RCPTv2\0\0" || [u32 T][T tokens][u32 T][(u32 V, root_t) x T]). Host reference of what
 * DETGPU_F_RECEIPT_V2 computes on the GPU. */
void detgpu_step_root(const float* logits, uint32_t vocab, uint8_t out[32]);
void detgpu_hash_canonical_v2(const uint32_t* tokens, uint32_t n_tokens, const float* logits,
                              uint32_t vocab, uint8_t out[32]);
/* ExecutionTuple encoding (codec.cpp:67-104, big-endian, length-prefixed); returns the size,
 * writes when out != NULL. req_hash = SHA-256 of these bytes (receipts.cpp:119). */
size_t detgpu_encode_exec_tuple(const char* model_id, const uint8_t container_digest[32], const char* arch,
                                const char* driver_tag, const detgpu_policy* policy, uint64_t seed,
                                const uint32_t* prompt, uint32_t prompt_len, uint8_t* out);
/* Strict decoder (rejects has_k/has_p outside {0,1}, payload on absent fields and trailing
 * bytes — the reference decoder's malleability, codec.cpp:76-91, is not inherited).
 * Returns DETGPU_OK and fills the outputs, or DETGPU_EINVAL. String outputs are NUL-terminated
 * into caller buffers of *_cap bytes; prompt_out has prompt_cap entries. */
int detgpu_decode_exec_tuple(const uint8_t* bytes, size_t n, char* model_id, size_t model_id_cap,
                             uint8_t container_digest[32], char* arch, size_t arch_cap, char* driver_tag,
                             size_t driver_cap, detgpu_policy* policy, uint64_t* seed, uint32_t* prompt_out,
                             uint32_t prompt_cap, uint32_t* prompt_len);

/* ---- kernel-level entry points (device pointers; used by the parity tests and the bench) ---- */

/* Y[col*ldy + n] = sum_k X[col*K + k] * W[n*K + k]; W [n_out,K] bf16, X [ncols,K] bf16. */
int detgpu_k_gemm(const void* W, const void* X, float* Y, int n_out, int K, int ncols, int64_t ldy,
                  void* stream);
/* Same with an explicit number of fixed K-segments (1..8; 0 = the engine's shape rule). Changes the
 * numeric definition: measurement hook only. Test hooks: -1 = the engine's rule with the wide-N MMA
 * form; 200 + S = the CTA-pair (cta_group::2) kernel above 64 columns (same bits). */
int detgpu_k_gemm_split(const void* W, const void* X, float* Y, int n_out, int K, int ncols, int64_t ldy,
                        int ksplit, void* stream);
/* out[col][i] = bf16(x[col][i] * rstd * gamma[i]); x f32 [ncols,d]; canonical-tree sum of squares. */
int detgpu_k_rmsnorm(const float* x, const void* gamma, void* out, int ncols, int d, float eps, void* stream);
/* f32 exp of n values with the engine's det_expf. */
int detgpu_k_expf(const float* x, float* y, int64_t n, void* stream);
/* Canonical tree sum of each of `rows` rows of length n (f32) -> out[rows]. */
int detgpu_k_tree_sum(const float* x, float* out, int rows, int n, void* stream);
/* Deterministic weight generation of one logical tensor into bf16. */
int detgpu_k_init_tensor(void* dst, uint64_t seed, int64_t rows, int64_t cols, int scale_exp, int is_gamma,
                         int row_mul, int row_add, void* stream);
/* Softmax + decode step on f32 logits rows (device). probs_out may be NULL. prng_state [rows][4]
 * is advanced once per row. tokens_out [rows]. Policies host array of `rows`. */
int detgpu_k_sample(const float* logits, int rows, int vocab, const detgpu_policy* policies, uint64_t* prng_state,
                    uint32_t* tokens_out, float* probs_out, int32_t* status_out, void* stream);
/* Receipt v2 roots of n_steps rows of `vocab` f32 logits: roots [n_steps][32]. */
int detgpu_k_step_roots(const float* trace, int n_steps, int vocab, uint8_t* roots, void* stream);
/* Decode attention (the engine's cluster / streamed kernels) for `ncols` query columns over the
 * PAGED cache: q [ncols][hq*hd] bf16; kcache / vcache [page][hkv][page positions][hd] bf16;
 * block_table [req][max_pages] page ids; col_pos[c] = the column's position (it attends to
 * [0, col_pos[c]]); col_req[c] its request row of block_table; out [ncols][hq*hd] bf16. */
int detgpu_k_attention(const void* q, const void* kcache, const void* vcache, const int32_t* block_table,
                       const int32_t* col_pos, const int32_t* col_req, void* out, int ncols, int hq, int hkv,
                       int hd, int page, int max_pages, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DETGPU_H */
