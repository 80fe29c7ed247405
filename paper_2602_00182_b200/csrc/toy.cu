// ToyModel engine: one warp per request, lane i owns output row i of every matvec. Bit-exact with
// the reference's detcore::infer (detcore.cpp:298-385): same weight stream (host, PrngState seeded
// from fnv1a64(model_id), detcore.cpp:275-296), products rounded then tree- (archA) or left-
// (archB) reduced (detcore.cpp:165-185), softsign, det_softmax with the glibc-exact det_expf and a
// 32-wide canonical tree, one PRNG draw per token, and the reference decode rules.
#include <cmath>
#include <cstring>
#include <vector>

#include "detmath.cuh"
#include "kernels.cuh"
#include "model.h"
#include "receipt.h"
#include "toy.cuh"

namespace detgpu {

namespace {

constexpr int kEmbed = 0, kRecur = 512, kHidden = 768, kProject = 1024, kTotal = 1536;

struct HostPrng {
    uint64_t s[4];
    uint64_t next() {
        const uint64_t result = ((s[0] + s[3]) << 23 | (s[0] + s[3]) >> 41) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = (s[3] << 45) | (s[3] >> 19);
        return result;
    }
    uint64_t below(uint64_t bound) {
        const uint64_t limit = bound * ((~uint64_t{0}) / bound);
        for (;;) {
            const uint64_t x = next();
            if (x < limit) return x % bound;
        }
    }
};

__device__ __forceinline__ float softsign(float x) { return __fdiv_rn(x, __fadd_rn(1.0f, fabsf(x))); }

// row . vec over 16 entries; arch 0: products rounded, canonical tree; arch 1: left fold.
__device__ __forceinline__ float toy_dot(const float* row, const float* vec, int arch, int* bad) {
    float p[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        p[j] = __fmul_rn(row[j], vec[j]);
        if (!isfinite(p[j])) *bad = 1;
    }
    if (arch == 0) return local_tree_sum<16>(p);
    float acc = p[0];
#pragma unroll
    for (int j = 1; j < 16; ++j) acc = __fadd_rn(acc, p[j]);
    return acc;
}

// The reference tree (level loop, odd tail promoted) over n <= 32 values.
__device__ float ref_tree(float* lv, int n) {
    if (n == 0) return 0.0f;
    while (n > 1) {
        const int half = n / 2;
        for (int i = 0; i < half; ++i) lv[i] = __fadd_rn(lv[2 * i], lv[2 * i + 1]);
        if (n % 2 != 0) {
            lv[half] = lv[n - 1];
            n = half + 1;
        } else {
            n = half;
        }
    }
    return lv[0];
}

__global__ void __launch_bounds__(32) toy_kernel(const float* __restrict__ W, int arch,
                                                 const uint32_t* __restrict__ prompts, const int* __restrict__ poff,
                                                 const int* __restrict__ plen, const DevPolicy* pols,
                                                 const uint64_t* __restrict__ seeds, int tcap, uint32_t* tok_out,
                                                 float* logits_out, int* status) {
    __shared__ float w[kTotal];
    __shared__ float state[16], hb[16], probs[32];
    const int r = blockIdx.x, lane = threadIdx.x;
    for (int i = lane; i < kTotal; i += 32) w[i] = W[i];
    if (lane < 16) state[lane] = 0.0f;
    __syncwarp();
    int bad = 0;
    auto advance = [&](uint32_t tok) {
        float nx = 0.0f;
        if (lane < 16) {
            nx = toy_dot(w + kRecur + lane * 16, state, arch, &bad);
            nx = softsign(__fadd_rn(nx, w[kEmbed + tok * 16 + lane]));
        }
        __syncwarp();
        if (lane < 16) state[lane] = nx;
        __syncwarp();
    };
    const uint32_t* pr = prompts + poff[r];
    for (int t = 0; t < plen[r]; ++t) advance(pr[t]);
    const DevPolicy pol = pols[r];
    uint64_t s[4];
    {
        uint64_t x = seeds[r];
        for (int i = 0; i < 4; ++i) {
            uint64_t z = (x += 0x9E3779B97F4A7C15ull);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            s[i] = z ^ (z >> 31);
        }
        if ((s[0] | s[1] | s[2] | s[3]) == 0) s[0] = 0x9E3779B97F4A7C15ull;
    }
    for (int t = 0; t < pol.max_tokens; ++t) {
        if (lane < 16) hb[lane] = softsign(toy_dot(w + kHidden + lane * 16, state, arch, &bad));
        __syncwarp();
        const float logit = toy_dot(w + kProject + lane * 16, hb, arch, &bad);
        logits_out[(static_cast<int64_t>(r) * tcap + t) * 32 + lane] = logit;
        // det_softmax (detcore.cpp:187-198): max, exp(x - max), canonical tree sum, divide
        if (!isfinite(logit)) bad = 1;
        const float mx = warp_max(logit);
        const float e = det_expf(__fsub_rn(logit, mx));
        const float sum = warp_tree_sum(e);
        probs[lane] = __fdiv_rn(e, sum);
        bad = __any_sync(0xffffffffu, bad);
        __syncwarp();
        uint32_t token = 0;
        if (lane == 0 && !bad) {
            const uint64_t u = xoshiro_next(s);
            const float rdraw = __fmul_rn(static_cast<float>(u >> 40), 0x1.0p-24f);
            if (pol.kind == DETGPU_GREEDY) {
                int best = 0;
                for (int i = 1; i < 32; ++i)
                    if (probs[i] > probs[best]) best = i;
                token = best;
            } else {
                int order[32];
                for (int i = 0; i < 32; ++i) order[i] = i;
                for (int i = 1; i < 32; ++i) {   // insertion sort by (p desc, idx asc)
                    const int v = order[i];
                    int j = i - 1;
                    while (j >= 0 && (probs[order[j]] < probs[v] || (probs[order[j]] == probs[v] && order[j] > v))) {
                        order[j + 1] = order[j];
                        --j;
                    }
                    order[j + 1] = v;
                }
                int kept = 32;
                if (pol.kind == DETGPU_TOP_K) {
                    kept = pol.k < 32u ? static_cast<int>(pol.k) : 32;
                } else {
                    float cum = 0.0f;
                    for (int i = 0; i < 32; ++i) {
                        cum = __fadd_rn(cum, probs[order[i]]);
                        if (cum >= pol.p) {
                            kept = i + 1;
                            break;
                        }
                    }
                }
                float kp[32], lv[32];
                for (int i = 0; i < kept; ++i) kp[i] = lv[i] = probs[order[i]];
                const float mass = ref_tree(lv, kept);
                if (!(mass > 0.0f)) {
                    bad = 2;
                } else {
                    token = order[kept - 1];
                    float cum = 0.0f;
                    for (int i = 0; i < kept; ++i) {
                        cum = __fadd_rn(cum, __fdiv_rn(kp[i], mass));
                        if (cum >= rdraw) {
                            token = order[i];
                            break;
                        }
                    }
                }
            }
        }
        bad = __shfl_sync(0xffffffffu, bad, 0);
        if (bad) {
            if (lane == 0) status[r] = bad == 2 ? DETGPU_EINVAL : DETGPU_ENONFINITE;
            return;
        }
        token = __shfl_sync(0xffffffffu, token, 0);
        if (lane == 0) tok_out[static_cast<int64_t>(r) * tcap + t] = token;
        advance(token);
    }
}

}  // namespace

int toy_init(ToyWeights& tw, const char* model_id, int arch, cudaStream_t stream) {
    // ToyModel::from_model_id (detcore.cpp:288-296): sequential stream, ldexp(u, below(7) - 3)
    HostPrng prng;
    prng_seeded(fnv1a64(model_id), prng.s);
    std::vector<float> w(kTotal);
    for (int i = 0; i < kTotal; ++i) {
        const float u = static_cast<float>(prng.next() >> 40) * 0x1.0p-23f - 1.0f;
        const int e = static_cast<int>(prng.below(7)) - 3;
        w[i] = std::ldexp(u, e);
    }
    tw.arch = arch;
    if (cudaMalloc(reinterpret_cast<void**>(&tw.w), sizeof(float) * kTotal) != cudaSuccess) return DETGPU_ENOMEM;
    if (cudaMemcpyAsync(tw.w, w.data(), sizeof(float) * kTotal, cudaMemcpyHostToDevice, stream) != cudaSuccess)
        return DETGPU_ECUDA;
    return cudaStreamSynchronize(stream) == cudaSuccess ? DETGPU_OK : DETGPU_ECUDA;
}

void toy_free(ToyWeights& tw) {
    if (tw.w) cudaFree(tw.w);
    tw.w = nullptr;
}

int toy_generate(ToyWeights& tw, uint32_t n, const uint32_t* const* prompts, const uint32_t* lens,
                 const detgpu_policy* pols, const uint64_t* seeds, uint32_t /*batch_size*/,
                 uint32_t* const* tokens_out, float* const* logits_out, uint8_t* out_hash, uint32_t flags,
                 detgpu_stats* st, cudaStream_t s, std::string* err) {
    // every request is an independent warp, so any grouping gives identical bytes
    int tcap = 1;
    std::vector<int> poff(n), plen(n);
    std::vector<uint32_t> flat;
    std::vector<DevPolicy> dp(n);
    for (uint32_t i = 0; i < n; ++i) {
        tcap = std::max<int>(tcap, static_cast<int>(pols[i].max_tokens));
        poff[i] = static_cast<int>(flat.size());
        plen[i] = static_cast<int>(lens[i]);
        flat.insert(flat.end(), prompts[i], prompts[i] + lens[i]);
        dp[i].kind = pols[i].kind;
        dp[i].k = pols[i].has_k ? pols[i].k : 0;
        dp[i].p = pols[i].has_p ? pols[i].p : 0.0f;
        dp[i].max_tokens = static_cast<int>(pols[i].max_tokens);
    }
    if (flat.empty()) flat.push_back(0);
    uint32_t *d_prompts = nullptr, *d_tok = nullptr;
    int *d_poff = nullptr, *d_plen = nullptr, *d_status = nullptr;
    DevPolicy* d_pol = nullptr;
    uint64_t* d_seed = nullptr;
    float* d_logits = nullptr;
    auto cleanup = [&] {
        cudaFree(d_prompts);
        cudaFree(d_tok);
        cudaFree(d_poff);
        cudaFree(d_plen);
        cudaFree(d_status);
        cudaFree(d_pol);
        cudaFree(d_seed);
        cudaFree(d_logits);
    };
    bool ok = cudaMalloc(&d_prompts, sizeof(uint32_t) * flat.size()) == cudaSuccess &&
              cudaMalloc(&d_tok, sizeof(uint32_t) * size_t(n) * tcap) == cudaSuccess &&
              cudaMalloc(&d_poff, sizeof(int) * n) == cudaSuccess && cudaMalloc(&d_plen, sizeof(int) * n) == cudaSuccess &&
              cudaMalloc(&d_status, sizeof(int) * n) == cudaSuccess &&
              cudaMalloc(&d_pol, sizeof(DevPolicy) * n) == cudaSuccess &&
              cudaMalloc(&d_seed, sizeof(uint64_t) * n) == cudaSuccess &&
              cudaMalloc(&d_logits, sizeof(float) * size_t(n) * tcap * 32) == cudaSuccess;
    if (!ok) {
        cleanup();
        *err = "toy: device allocation failed";
        return DETGPU_ENOMEM;
    }
    cudaMemcpyAsync(d_prompts, flat.data(), sizeof(uint32_t) * flat.size(), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_poff, poff.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_plen, plen.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(d_status, 0, sizeof(int) * n, s);
    cudaMemcpyAsync(d_pol, dp.data(), sizeof(DevPolicy) * n, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(d_seed, seeds, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    toy_kernel<<<n, 32, 0, s>>>(tw.w, tw.arch, d_prompts, d_poff, d_plen, d_pol, d_seed, tcap, d_tok, d_logits, d_status);
    cudaEventRecord(e1, s);
    cudaError_t ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) {
        cleanup();
        *err = std::string("toy kernel: ") + cudaGetErrorString(ce);
        return DETGPU_ECUDA;
    }
    if (st) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        st->decode_ms += ms;
        st->kernel_launches += 1;
        for (uint32_t i = 0; i < n; ++i) st->tokens += pols[i].max_tokens;
        st->h2d_bytes += sizeof(uint32_t) * flat.size() + n * (8 + sizeof(int) * 2 + sizeof(DevPolicy));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::vector<int> status(n);
    cudaMemcpy(status.data(), d_status, sizeof(int) * n, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < n; ++i)
        if (status[i] != 0) {
            cleanup();
            *err = status[i] == DETGPU_ENONFINITE ? "canonical_reduce: non-finite value"
                                                  : "decode: zero probability mass after truncation";
            return DETGPU_EINVAL;
        }
    if (!(flags & DETGPU_F_DEVICE_ONLY)) {
        std::vector<uint32_t> toks(size_t(n) * tcap);
        std::vector<float> lg(size_t(n) * tcap * 32);
        cudaMemcpy(toks.data(), d_tok, sizeof(uint32_t) * toks.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(lg.data(), d_logits, sizeof(float) * lg.size(), cudaMemcpyDeviceToHost);
        if (st) st->d2h_bytes += sizeof(uint32_t) * toks.size() + sizeof(float) * lg.size();
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t T = pols[i].max_tokens;
            if (tokens_out && tokens_out[i] && T) std::memcpy(tokens_out[i], &toks[size_t(i) * tcap], 4 * size_t(T));
            if (logits_out && logits_out[i] && T)
                std::memcpy(logits_out[i], &lg[size_t(i) * tcap * 32], 4 * size_t(T) * 32);
            if (out_hash && (flags & DETGPU_F_RECEIPT_V2)) {   // v2 on the host: 32 logits = one leaf per step
                std::vector<uint8_t> roots(32 * size_t(T));
                for (uint32_t t = 0; t < T; ++t)
                    step_root(&lg[(size_t(i) * tcap + t) * 32], 32, roots.data() + 32 * size_t(t));
                hash_canonical_v2_roots(&toks[size_t(i) * tcap], T, roots.data(), 32, out_hash + 32 * size_t(i));
            } else if (out_hash) {
                hash_canonical(&toks[size_t(i) * tcap], T, &lg[size_t(i) * tcap * 32], 32, out_hash + 32 * size_t(i));
            }
        }
    }
    cleanup();
    return DETGPU_OK;
}

}  // namespace detgpu
