// gate.cu — K1 gate epilogue: top-K selection, top-K softmax weights and the
// per-(source GPU, expert) token histogram, i.e. the load-matrix columns
// input_e^g the scheduler consumes (reference LoadMatrix, core.py:229-268).
//
// One warp per token: each lane scans E/32 logits (+ selection bias), K rounds
// of a warp arg-max (ties -> lower expert id) pick K distinct experts; the
// weights are softmax over the K selected logits, computed in fp32 in pick
// order.  Histogram: per-block shared-memory counters for the (at most two)
// sources a block's token range touches, flushed with one integer atomic per
// (source, expert) — integer sums, so the result is order-independent.
#include "common.cuh"

namespace hep {

constexpr int kGateWarps = 8;
constexpr int kGateTokensPerWarp = 16;
constexpr int kMaxTopK = 16;
constexpr int kMaxGateExperts = 1024;

__global__ void __launch_bounds__(kGateWarps * 32) gate_topk_kernel(const float *__restrict__ logits, int64_t ld,
                                                                    const float *__restrict__ bias, int64_t T, int E,
                                                                    int K, int64_t tps, int n_src,
                                                                    int32_t *__restrict__ topk_idx,
                                                                    float *__restrict__ topk_w, int64_t *hist) {
    extern __shared__ int32_t sh_hist[];  // [2][E]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t_block = (int64_t)blockIdx.x * kGateWarps * kGateTokensPerWarp;
    const int src0 = (int)(t_block / tps < (int64_t)(n_src - 1) ? t_block / tps : (int64_t)(n_src - 1));
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    for (int it = 0; it < kGateTokensPerWarp; ++it) {
        const int64_t t = t_block + (int64_t)warp * kGateTokensPerWarp + it;
        if (t >= T) break;
        const float *row = logits + t * ld;
        // lane-local candidate list: experts lane, lane+32, ...
        float best_s = -INFINITY, best_l = 0.f;
        int best_e = 0x7fffffff;
        int32_t picked_e[kMaxTopK];
        float picked_l[kMaxTopK];
        for (int k = 0; k < K; ++k) {
            best_s = -INFINITY;
            best_e = 0x7fffffff;
            for (int e = lane; e < E; e += 32) {
                bool taken = false;
                for (int j = 0; j < k; ++j) taken |= (picked_e[j] == e);
                if (taken) continue;
                const float l = row[e];
                const float s = bias ? l + bias[e] : l;
                if (s > best_s || (s == best_s && e < best_e)) { best_s = s; best_e = e; best_l = l; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float os = __shfl_xor_sync(0xffffffffu, best_s, o);
                const int oe = __shfl_xor_sync(0xffffffffu, best_e, o);
                const float ol = __shfl_xor_sync(0xffffffffu, best_l, o);
                if (os > best_s || (os == best_s && oe < best_e)) { best_s = os; best_e = oe; best_l = ol; }
            }
            picked_e[k] = best_e;
            picked_l[k] = best_l;
        }
        if (lane == 0) {
            float mx = picked_l[0];
            for (int k = 1; k < K; ++k) mx = fmaxf(mx, picked_l[k]);
            float den = 0.f;
            float ex[kMaxTopK];
            for (int k = 0; k < K; ++k) { ex[k] = expf(picked_l[k] - mx); den += ex[k]; }
            const int src = (int)(t / tps < (int64_t)(n_src - 1) ? t / tps : (int64_t)(n_src - 1));
            const int slot = src - src0;
            for (int k = 0; k < K; ++k) {
                topk_idx[t * K + k] = picked_e[k];
                topk_w[t * K + k] = ex[k] / den;
                if (slot < 2) atomicAdd(&sh_hist[slot * E + picked_e[k]], 1);
                else atomicAdd((unsigned long long *)&hist[(int64_t)src * E + picked_e[k]], 1ull);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) {
        const int c = sh_hist[i];
        const int src = src0 + i / E;
        if (c && src < n_src) atomicAdd((unsigned long long *)&hist[(int64_t)src * E + i % E], (unsigned long long)c);
    }
}

}  // namespace hep

using namespace hep;

extern "C" int hep_gate_topk(const float *d_logits, int64_t ld_logits, const float *d_bias, int64_t T, int E, int K,
                             int64_t tokens_per_src, int n_src, int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist,
                             void *stream) {
    HEP_REQUIRE(d_logits && d_topk_idx && d_topk_w && d_hist, HEP_E_CONTRACT, "hep_gate_topk: null pointer");
    HEP_REQUIRE(E >= 1 && E <= kMaxGateExperts && K >= 1 && K <= kMaxTopK && K <= E, HEP_E_DIMENSION,
                "hep_gate_topk: E=%d K=%d", E, K);
    HEP_REQUIRE(tokens_per_src >= 1 && n_src >= 1 && ld_logits >= E, HEP_E_DIMENSION, "hep_gate_topk: bad shape");
    cudaStream_t s = (cudaStream_t)stream;
    HEP_CHECK_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(int64_t) * (size_t)n_src * E, s));
    if (T <= 0) return HEP_OK;
    const int64_t per_block = kGateWarps * kGateTokensPerWarp;
    const int64_t grid = (T + per_block - 1) / per_block;
    gate_topk_kernel<<<(unsigned)grid, kGateWarps * 32, 2 * E * sizeof(int32_t), s>>>(
        d_logits, ld_logits, d_bias, T, E, K, tokens_per_src, n_src, d_topk_idx, d_topk_w, d_hist);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}
