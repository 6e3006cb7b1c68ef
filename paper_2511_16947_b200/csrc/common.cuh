// common.cuh — shared helpers for the HarmonyEP sm_100a kernels (error
// plumbing for the C ABI, warp/block reductions, PTX wrappers).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hep.h"

namespace hep {

// thread-local message behind hep_last_error()
void set_error(const char *fmt, ...);
// process-wide launch tuning (hep_tuning_set); never read from the environment
extern hep_tuning g_tuning;

#define HEP_CHECK_CUDA(expr)                                                          \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            ::hep::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return HEP_E_CUDA;                                                        \
        }                                                                             \
    } while (0)

// NVTX range around every hot C-ABI entry point (header-only NVTX3: a no-op unless a
// tool such as ncu --nvtx is attached), so profiles attribute launches to their stage
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define HEP_NVTX(name) ::hep::NvtxRange hep_nvtx_range_(name)

#define HEP_CHECK_LAUNCH() HEP_CHECK_CUDA(cudaGetLastError())

#define HEP_REQUIRE(cond, code, ...)        \
    do {                                    \
        if (!(cond)) {                      \
            ::hep::set_error(__VA_ARGS__);  \
            return (code);                  \
        }                                   \
    } while (0)

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// inclusive warp scan
__device__ __forceinline__ int64_t warp_incl_scan_i64(int64_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t w = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += w;
    }
    return v;
}

// Block-wide exclusive scan of one int64 per thread; returns exclusive prefix,
// writes the block total to *total.  `sm` needs (blockDim/32 + 1) int64.
__device__ __forceinline__ int64_t block_excl_scan_i64(int64_t v, int64_t *sm, int64_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    int64_t inc = warp_incl_scan_i64(v);
    if (lane == 31) sm[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int64_t s = lane < nw ? sm[lane] : 0;
        int64_t si = warp_incl_scan_i64(s);
        if (lane < nw) sm[lane] = si - s;
        if (lane == nw - 1) sm[nw] = si;
    }
    __syncthreads();
    int64_t res = sm[wid] + inc - v;
    *total = sm[nw];
    __syncthreads();
    return res;
}

__device__ __forceinline__ int64_t block_sum_i64(int64_t v, int64_t *sm) {
    int64_t t;
    block_excl_scan_i64(v, sm, &t);
    return t;
}

__device__ __forceinline__ void set_status(int32_t *st, int code) {
    if (st) atomicCAS(st, 0, code);
}

}  // namespace hep
