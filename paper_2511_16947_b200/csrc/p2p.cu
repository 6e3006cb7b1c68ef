// p2p.cu — expert-parallel exchange over NVLink peer memory (no NCCL on the data path).
//
// Every rank computes the identical schedule, hence the identical transfer matrix
// pair[s][d] (rows source s sends to destination d), so each rank knows, without
// any exchange, where its rows land in every peer's buffers:
//   send layout of rank s:   [dst][expert][rank]      chunk d starts at sbase_s(d) = sum_{d'<d} pair[s][d']
//   receive layout of rank d: [src][hosted expert]    chunk s starts at rbase_d(s) = sum_{s'<s} pair[s'][d]
// Dispatch (K5 fused with the all-to-all): rank s writes x[t] for assignment (t,k) with
// send position p (chunk d) straight to peer d's receive buffer at rbase_d(s) + p - sbase_s(d).
// Combine all-to-all fused into the down-projection GEMM's epilogue: receive row i of
// rank d (chunk s) goes back to rank s's return buffer at its send position
// sbase_s(d) + i - rbase_d(s); hep_moe_return_addr writes that per-row address table.
// Peer buffers are CUDA IPC mappings (one process per GPU) or plain device pointers
// (all ranks in one process); the kernels only see 64-bit addresses.
#include <cuda.h>
#include <string.h>

#include "common.cuh"

namespace hep {

__device__ __forceinline__ void chunk_bases(const int64_t *pair, int G, int me, int64_t *sbase, int64_t *rbase) {
    // sbase[d] = sum_{d'<d} pair[me][d'] (send chunks of this rank); rbase[d] = sum_{s'<me} pair[s'][d]
    int64_t run = 0;
    for (int d = 0; d < G; ++d) {
        sbase[d] = run;
        run += pair[me * G + d];
        int64_t r = 0;
        for (int s = 0; s < me; ++s) r += pair[s * G + d];
        rbase[d] = r;
    }
    sbase[G] = run;
}

__global__ void __launch_bounds__(256) dispatch_p2p_kernel(const int4 *__restrict__ x, const int32_t *__restrict__ tok_row,
                                                           int64_t T, int K, int64_t nvec, int me, int G,
                                                           const int64_t *__restrict__ pair,
                                                           const uint64_t *__restrict__ peer_recv,
                                                           int64_t recv_capacity, const int32_t *status) {
    __shared__ int64_t sbase[HEP_MAX_GPUS + 1], rbase[HEP_MAX_GPUS];
    __shared__ uint64_t peer[HEP_MAX_GPUS];
    __shared__ int skip;
    if (threadIdx.x == 0) {
        chunk_bases(pair, G, me, sbase, rbase);
        // no valid schedule, or some destination would receive more rows than its buffer
        // holds (every rank evaluates all destinations on the identical plan: they agree)
        int f = status != nullptr && *status != 0;
        for (int d = 0; d < G && !f; ++d) {
            int64_t r = 0;
            for (int s2 = 0; s2 < G; ++s2) r += pair[s2 * G + d];
            f = recv_capacity > 0 && r > recv_capacity;
        }
        skip = f;
    }
    if (threadIdx.x < G) peer[threadIdx.x] = peer_recv[threadIdx.x];
    __syncthreads();
    if (skip) return;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < T; t += nwarps) {
        int4 *dst[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (k >= K) break;
            const int64_t p = tok_row[t * K + k];
            int d = 0;
            while (d + 1 < G && p >= sbase[d + 1]) ++d;
            dst[k] = reinterpret_cast<int4 *>(peer[d]) + (rbase[d] + p - sbase[d]) * nvec;
        }
        const int4 *src = x + t * nvec;
        for (int64_t v0 = lane; v0 < nvec; v0 += 32 * 4) {
            int4 buf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v0 + 32 * u < nvec) buf[u] = __ldg(src + v0 + 32 * u);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k >= K) break;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v0 + 32 * u < nvec) dst[k][v0 + 32 * u] = buf[u];
            }
        }
    }
}

__global__ void return_addr_kernel(const int64_t *__restrict__ pair, int me, int G, const uint64_t *__restrict__ peer_back,
                                   int64_t row_bytes, int64_t cap, uint64_t *__restrict__ addr,
                                   const int32_t *__restrict__ row_map = nullptr) {
    __shared__ int64_t rb[HEP_MAX_GPUS + 1], sb[HEP_MAX_GPUS];
    if (threadIdx.x == 0) {
        // this rank as destination: receive chunk s starts at rb[s]; source s sent it from
        // its send chunk `me`, which starts at sb[s] = sum_{d'<me} pair[s][d']
        int64_t run = 0;
        for (int s = 0; s < G; ++s) {
            rb[s] = run;
            run += pair[s * G + me];
            int64_t b = 0;
            for (int d = 0; d < me; ++d) b += pair[s * G + d];
            sb[s] = b;
        }
        rb[G] = run;
    }
    __syncthreads();
    const int64_t n = rb[G] < cap ? rb[G] : cap;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int s = 0;
        while (s + 1 < G && i >= rb[s + 1]) ++s;
        const uint64_t a = peer_back[s] + (uint64_t)((sb[s] + i - rb[s]) * row_bytes);
        if (row_map) {  // receive row i now sits at row_map[i] (rows regrouped per weight slot); -1 =
            const int32_t j = row_map[i];  // no such row (an empty exchange after a capacity overflow)
            if (j >= 0) addr[j] = a;
        } else {
            addr[i] = a;
        }
    }
}

// ---------------------------------------------------------------------------
// Device-side group barrier (and all-gather) through peer memory, so an EP forward
// needs no host synchronisation: every rank owns flags[world + 1] (uint32) mapped by
// every peer; slot r holds the last epoch rank r arrived with, slot `world` this rank's
// own epoch counter (advanced by the kernel itself, so the launch is graph-capturable).
// Arrival is a release store at system scope into every peer's slot `rank`, made after
// the optional payload stores; waiting is an acquire load per peer slot.  Stream order
// puts the peer stores of earlier kernels (dispatch, the GEMM epilogue) before the
// release (cumulativity), and every later kernel after the acquire.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(256) p2p_barrier_kernel(const uint64_t *__restrict__ peer_flags, uint32_t *my_flags,
                                                          int rank, int world, const int4 *__restrict__ src,
                                                          int64_t nvec, const uint64_t *__restrict__ peer_dst) {
    __shared__ uint32_t epoch;
    if (src)  // all-gather payload: this rank's block into slot `rank` of every peer's buffer
        for (int i = 0; i < world; ++i) {
            int4 *dst = reinterpret_cast<int4 *>(peer_dst[i]) + (int64_t)rank * nvec;
            for (int64_t v = threadIdx.x; v < nvec; v += blockDim.x) dst[v] = src[v];
        }
    if (threadIdx.x == 0) {
        epoch = my_flags[world] + 1;
        my_flags[world] = epoch;
    }
    __syncthreads();  // payload stores of every thread precede thread i's release below
    __threadfence_system();
    if (threadIdx.x < world)
        st_release_sys(reinterpret_cast<uint32_t *>(peer_flags[threadIdx.x]) + rank, epoch);
    if (threadIdx.x < world) {
        // a peer that never arrives (dead rank, broken mapping) must not hang the GPU: give up
        // after ~10 s and raise the sticky flag in slot world + 1 (checked by the host)
        uint64_t t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while ((int32_t)(ld_acquire_sys(my_flags + threadIdx.x) - epoch) < 0) {
            __nanosleep(64);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 10000000000ull) {
                atomicExch(my_flags + world + 1, 1u);
                break;
            }
        }
    }
    __syncthreads();
}

}  // namespace hep

using namespace hep;

extern "C" int hep_p2p_barrier(const uint64_t *d_peer_flags, uint32_t *d_my_flags, int rank, int world, void *stream) {
    HEP_NVTX("hep_p2p_barrier");
    HEP_REQUIRE(d_peer_flags && d_my_flags, HEP_E_CONTRACT, "hep_p2p_barrier: null pointer");
    HEP_REQUIRE(world >= 1 && world <= HEP_MAX_GPUS && rank >= 0 && rank < world, HEP_E_DIMENSION,
                "hep_p2p_barrier: rank %d of %d", rank, world);
    p2p_barrier_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_peer_flags, d_my_flags, rank, world, nullptr, 0, nullptr);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_p2p_allgather(const void *d_src, int64_t bytes, const uint64_t *d_peer_dst,
                                 const uint64_t *d_peer_flags, uint32_t *d_my_flags, int rank, int world,
                                 void *stream) {
    HEP_NVTX("hep_p2p_allgather");
    HEP_REQUIRE(d_src && d_peer_dst && d_peer_flags && d_my_flags, HEP_E_CONTRACT, "hep_p2p_allgather: null pointer");
    HEP_REQUIRE(world >= 1 && world <= HEP_MAX_GPUS && rank >= 0 && rank < world && bytes >= 0 && bytes % 16 == 0,
                HEP_E_DIMENSION, "hep_p2p_allgather: rank %d of %d, %lld bytes (multiple of 16)", rank, world,
                (long long)bytes);
    p2p_barrier_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(d_peer_flags, d_my_flags, rank, world,
                                                            (const int4 *)d_src, bytes / 16, d_peer_dst);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_dispatch_p2p(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model,
                                    int rank, int num_gpus, const int64_t *d_pair, const uint64_t *d_peer_recv,
                                    int64_t recv_capacity, const int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_dispatch_p2p");
    HEP_REQUIRE(d_x && d_tok_row && d_pair && d_peer_recv, HEP_E_CONTRACT, "hep_moe_dispatch_p2p: null pointer");
    HEP_REQUIRE(d_model % 8 == 0 && K >= 1 && K <= 16 && num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS && rank >= 0 &&
                    rank < num_gpus,
                HEP_E_DIMENSION, "hep_moe_dispatch_p2p: d_model %% 8, K <= 16, 1 <= G <= %d", HEP_MAX_GPUS);
    if (T <= 0) return HEP_OK;
    const int64_t warps = T < 148 * 64 ? T : 148 * 64;
    dispatch_p2p_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const int4 *)d_x, d_tok_row, T, K, d_model / 8, rank, num_gpus, d_pair, d_peer_recv, recv_capacity, d_status);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

namespace hep {
// received rows -> their source ranks: rows[i] (or rows[row_map[i]]) -> the address addr[i]
// (a peer's buffer over NVLink, or local), i < this rank's received count from the transfer
// plan (at most capacity); one warp per row, 16-byte vector copies
__global__ void __launch_bounds__(256) rows_to_addr_kernel(const int4 *__restrict__ src, const int32_t *__restrict__ row_map,
                                                           const int64_t *__restrict__ pair, int me, int G,
                                                           int64_t cap, int64_t nvec, const uint64_t *__restrict__ addr,
                                                           const int32_t *status) {
    if (status && *status) return;
    int64_t n = 0;
    for (int s = 0; s < G; ++s) n += pair[s * G + me];
    if (n > cap) n = cap;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nwarps) {
        const int64_t r = row_map ? row_map[i] : i;
        const int4 *s = src + r * nvec;
        int4 *d = reinterpret_cast<int4 *>(addr[i]);
        for (int64_t v = lane; v < nvec; v += 32) d[v] = __ldg(s + v);
    }
}
}  // namespace hep

extern "C" int hep_moe_rows_to_addr(const void *d_src, const int32_t *d_row_map, const int64_t *d_pair, int rank,
                                    int num_gpus, int64_t capacity, int64_t d_model, const uint64_t *d_addr,
                                    const int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_rows_to_addr");
    HEP_REQUIRE(d_src && d_pair && d_addr, HEP_E_CONTRACT, "hep_moe_rows_to_addr: null pointer");
    HEP_REQUIRE(d_model % 8 == 0 && num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS && rank >= 0 && rank < num_gpus,
                HEP_E_DIMENSION, "hep_moe_rows_to_addr: d_model %% 8, rank / G");
    if (capacity <= 0) return HEP_OK;
    const int64_t warps = capacity < 148 * 64 ? capacity : 148 * 64;
    rows_to_addr_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        (const int4 *)d_src, d_row_map, d_pair, rank, num_gpus, capacity, d_model / 8, d_addr, d_status);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_return_addr_map(const int64_t *d_pair, int rank, int num_gpus, const uint64_t *d_peer_back,
                                       int64_t row_bytes, int64_t capacity, const int32_t *d_row_map, uint64_t *d_addr,
                                       void *stream) {
    HEP_NVTX("hep_moe_return_addr");
    HEP_REQUIRE(d_pair && d_peer_back && d_addr, HEP_E_CONTRACT, "hep_moe_return_addr: null pointer");
    HEP_REQUIRE(num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS && rank >= 0 && rank < num_gpus && row_bytes % 16 == 0,
                HEP_E_DIMENSION, "hep_moe_return_addr: G, rank, row_bytes %% 16");
    if (capacity <= 0) return HEP_OK;
    const int64_t blocks = (capacity + 255) / 256 < 148 * 4 ? (capacity + 255) / 256 : 148 * 4;
    return_addr_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_pair, rank, num_gpus, d_peer_back,
                                                                           row_bytes, capacity, d_addr, d_row_map);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_return_addr(const int64_t *d_pair, int rank, int num_gpus, const uint64_t *d_peer_back,
                                   int64_t row_bytes, int64_t capacity, uint64_t *d_addr, void *stream) {
    HEP_NVTX("hep_moe_return_addr");
    HEP_REQUIRE(d_pair && d_peer_back && d_addr, HEP_E_CONTRACT, "hep_moe_return_addr: null pointer");
    HEP_REQUIRE(num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS && rank >= 0 && rank < num_gpus && row_bytes % 16 == 0,
                HEP_E_DIMENSION, "hep_moe_return_addr: G, rank, row_bytes %% 16");
    if (capacity <= 0) return HEP_OK;
    const int64_t blocks = (capacity + 255) / 256 < 148 * 4 ? (capacity + 255) / 256 : 148 * 4;
    return_addr_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_pair, rank, num_gpus, d_peer_back,
                                                                           row_bytes, capacity, d_addr);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_ipc_handle(const void *d_ptr, void *handle_out, int64_t *offset_out) {
    HEP_REQUIRE(d_ptr && handle_out && offset_out, HEP_E_CONTRACT, "hep_ipc_handle: null pointer");
    // the handle names the whole allocation; report where d_ptr sits inside it
    using range_fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    static range_fn fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<range_fn>(ptr);
    }
    HEP_REQUIRE(fn, HEP_E_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    HEP_REQUIRE(fn(&base, &size, (CUdeviceptr)d_ptr) == CUDA_SUCCESS, HEP_E_CUDA, "cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    HEP_CHECK_CUDA(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((CUdeviceptr)d_ptr - base);
    return HEP_OK;
}

extern "C" int hep_ipc_open(const void *handle, void **d_ptr) {
    HEP_REQUIRE(handle && d_ptr, HEP_E_CONTRACT, "hep_ipc_open: null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    HEP_CHECK_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return HEP_OK;
}

extern "C" int hep_ipc_close(void *d_ptr) {
    HEP_REQUIRE(d_ptr, HEP_E_CONTRACT, "hep_ipc_close: null pointer");
    HEP_CHECK_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return HEP_OK;
}
