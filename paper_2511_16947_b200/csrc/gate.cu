// gate.cu — K1 gate epilogue: top-K selection, top-K softmax weights and the
// per-(source GPU, expert) token histogram, i.e. the load-matrix columns
// input_e^g the scheduler consumes (reference LoadMatrix, core.py:229-268).
//
// Selection: top-K of (logit + bias_e), ties -> lower expert id; weights:
// softmax over the K selected logits in pick order (fp32).
//   E <= 32 : one thread per token, the row lives in registers.
//   E  > 32 : one warp per token, E/32 scores per lane in registers; each of
//             the K rounds is a lane-local arg-max plus two warp reductions
//             (redux.sync max over an order-preserving uint32 key of the
//             score, then redux.sync min over expert ids holding that key).
// Histogram: per-block shared-memory counters for the (at most two) sources a
// block's token range touches, flushed with one integer atomic per (source,
// expert) — integer sums, so the result is order-independent.
#include "common.cuh"

namespace hep {

constexpr int kMaxTopK = 16;
constexpr int kMaxGateExperts = 1024;

__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0: equal scores must tie
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int src_of(int64_t t, int64_t tps, int n_src) {
    const int64_t s = t / tps;
    return (int)(s < n_src - 1 ? s : n_src - 1);
}

__device__ __forceinline__ void write_token(int64_t t, int K, const int *pe, const float *pl, int32_t *topk_idx,
                                            float *topk_w, int src, int src0, int E, int32_t *sh_hist,
                                            int64_t *hist) {
    float mx = pl[0];
    for (int k = 1; k < K; ++k) mx = fmaxf(mx, pl[k]);
    float ex[kMaxTopK], den = 0.f;
    for (int k = 0; k < K; ++k) {
        ex[k] = expf(pl[k] - mx);
        den += ex[k];
    }
    const int slot = src - src0;
    for (int k = 0; k < K; ++k) {
        topk_idx[t * K + k] = pe[k];
        topk_w[t * K + k] = ex[k] / den;
        if (slot < 2) atomicAdd(&sh_hist[slot * E + pe[k]], 1);
        else atomicAdd((unsigned long long *)&hist[(int64_t)src * E + pe[k]], 1ull);
    }
}

__device__ __forceinline__ void flush_hist(const int32_t *sh_hist, int E, int src0, int n_src, int64_t *hist) {
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) {
        const int c = sh_hist[i];
        const int src = src0 + i / E;
        if (c && src < n_src) atomicAdd((unsigned long long *)&hist[(int64_t)src * E + i % E], (unsigned long long)c);
    }
}

// one thread per token, E <= EMAX (<= 32)
template <int EMAX>
__global__ void __launch_bounds__(128) gate_topk_thread(const float *__restrict__ logits, int64_t ld,
                                                        const float *__restrict__ bias, int64_t T, int E, int K,
                                                        int64_t tps, int n_src, int32_t *__restrict__ topk_idx,
                                                        float *__restrict__ topk_w, int64_t *hist) {
    extern __shared__ int32_t sh_hist[];  // [2][E]
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x;
    const int src0 = src_of(t0, tps, n_src);
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    const int64_t t = t0 + threadIdx.x;
    if (t < T) {
        float sc[EMAX], lg[EMAX];
        const float *row = logits + t * ld;
#pragma unroll
        for (int e = 0; e < EMAX; ++e) {
            lg[e] = e < E ? row[e] : 0.f;
            sc[e] = e < E ? (bias ? lg[e] + bias[e] : lg[e]) : -INFINITY;
        }
        int pe[kMaxTopK];
        float pl[kMaxTopK];
        for (int k = 0; k < K; ++k) {
            int be = 0;
            float bs = -INFINITY, bl = 0.f;
            bool found = false;
#pragma unroll
            for (int e = 0; e < EMAX; ++e) {
                if (e < E && sc[e] != -INFINITY && (!found || sc[e] > bs)) {
                    found = true;
                    bs = sc[e];
                    be = e;
                    bl = lg[e];
                }
            }
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                if (e == be) sc[e] = -INFINITY;
            pe[k] = be;
            pl[k] = bl;
        }
        write_token(t, K, pe, pl, topk_idx, topk_w, src_of(t, tps, n_src), src0, E, sh_hist, hist);
    }
    __syncthreads();
    flush_hist(sh_hist, E, src0, n_src, hist);
}

// one warp per token, E <= 32*PER
template <int PER>
__global__ void __launch_bounds__(256) gate_topk_warp(const float *__restrict__ logits, int64_t ld,
                                                      const float *__restrict__ bias, int64_t T, int E, int K,
                                                      int64_t tps, int n_src, int tokens_per_warp,
                                                      int32_t *__restrict__ topk_idx, float *__restrict__ topk_w,
                                                      int64_t *hist) {
    extern __shared__ int32_t sh_hist[];  // [2][E]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t_block = (int64_t)blockIdx.x * (blockDim.x >> 5) * tokens_per_warp;
    const int src0 = src_of(t_block, tps, n_src);
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) sh_hist[i] = 0;
    __syncthreads();
    for (int it = 0; it < tokens_per_warp; ++it) {
        const int64_t t = t_block + (int64_t)warp * tokens_per_warp + it;
        if (t >= T) break;
        const float *row = logits + t * ld;
        float lg[PER];
        uint32_t key[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int e = lane + 32 * j;
            lg[j] = e < E ? row[e] : 0.f;
            key[j] = e < E ? order_key(bias ? lg[j] + bias[e] : lg[j]) : 0u;  // 0 = below every real score
        }
        int pe[kMaxTopK];
        float pl[kMaxTopK];
        for (int k = 0; k < K; ++k) {
            uint32_t bk = 0;
            int bj = -1;
#pragma unroll
            for (int j = 0; j < PER; ++j)
                if (key[j] > bk) { bk = key[j]; bj = j; }  // ascending e: first max = lowest id
            const uint32_t wk = __reduce_max_sync(0xffffffffu, bk);
            const uint32_t mine = (bj >= 0 && bk == wk) ? (uint32_t)(lane + 32 * bj) : 0xffffffffu;
            const uint32_t we = __reduce_min_sync(0xffffffffu, mine);
            float l = 0.f;
#pragma unroll
            for (int j = 0; j < PER; ++j)
                if ((uint32_t)(lane + 32 * j) == we) { l = lg[j]; key[j] = 0u; }
            const int owner = (int)(we & 31u);
            pe[k] = (int)we;
            pl[k] = __shfl_sync(0xffffffffu, l, owner);
        }
        if (lane == 0)
            write_token(t, K, pe, pl, topk_idx, topk_w, src_of(t, tps, n_src), src0, E, sh_hist, hist);
    }
    __syncthreads();
    flush_hist(sh_hist, E, src0, n_src, hist);
}

}  // namespace hep

using namespace hep;

extern "C" int hep_gate_topk(const float *d_logits, int64_t ld_logits, const float *d_bias, int64_t T, int E, int K,
                             int64_t tokens_per_src, int n_src, int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist,
                             void *stream) {
    HEP_NVTX("hep_gate_topk");
    HEP_REQUIRE(d_logits && d_topk_idx && d_topk_w && d_hist, HEP_E_CONTRACT, "hep_gate_topk: null pointer");
    HEP_REQUIRE(E >= 1 && E <= kMaxGateExperts && K >= 1 && K <= kMaxTopK && K <= E, HEP_E_DIMENSION,
                "hep_gate_topk: E=%d K=%d", E, K);
    HEP_REQUIRE(tokens_per_src >= 1 && n_src >= 1 && ld_logits >= E, HEP_E_DIMENSION, "hep_gate_topk: bad shape");
    cudaStream_t s = (cudaStream_t)stream;
    HEP_CHECK_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(int64_t) * (size_t)n_src * E, s));
    if (T <= 0) return HEP_OK;
    const size_t sm = 2 * (size_t)E * sizeof(int32_t);
    if (E <= 32) {
        const unsigned grid = (unsigned)((T + 127) / 128);
        if (E <= 8)
            gate_topk_thread<8><<<grid, 128, sm, s>>>(d_logits, ld_logits, d_bias, T, E, K, tokens_per_src, n_src,
                                                      d_topk_idx, d_topk_w, d_hist);
        else if (E <= 16)
            gate_topk_thread<16><<<grid, 128, sm, s>>>(d_logits, ld_logits, d_bias, T, E, K, tokens_per_src, n_src,
                                                       d_topk_idx, d_topk_w, d_hist);
        else
            gate_topk_thread<32><<<grid, 128, sm, s>>>(d_logits, ld_logits, d_bias, T, E, K, tokens_per_src, n_src,
                                                       d_topk_idx, d_topk_w, d_hist);
    } else {
        const int tpw = 8;
        const unsigned grid = (unsigned)((T + 8 * tpw - 1) / (8 * tpw));
#define HEP_GATE_WARP(P)                                                                                 \
    gate_topk_warp<P><<<grid, 256, sm, s>>>(d_logits, ld_logits, d_bias, T, E, K, tokens_per_src, n_src, tpw, \
                                            d_topk_idx, d_topk_w, d_hist)
        if (E <= 64) HEP_GATE_WARP(2);
        else if (E <= 128) HEP_GATE_WARP(4);
        else if (E <= 256) HEP_GATE_WARP(8);
        else if (E <= 512) HEP_GATE_WARP(16);
        else HEP_GATE_WARP(32);
#undef HEP_GATE_WARP
    }
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}
