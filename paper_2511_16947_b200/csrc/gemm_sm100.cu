// gemm_sm100.cu — K6 expert FFN (grouped GEMM) and the K1 router GEMM on
// 5th-generation tensor cores.
//
// One persistent, warp-specialised kernel template (one CTA per SM):
//   warp 0      TMA producer: A tile [128 x 64] + B tile [BN x 64] per stage,
//               128-byte swizzle, STAGES-deep mbarrier ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M=128, N=BN, K=16 per instruction, fp32 accumulator in TMEM,
//               two accumulator buffers so the epilogue of tile i overlaps
//               the MMAs of tile i+1)
//   warps 2..9  epilogue, two warps per TMEM lane quarter (column halves):
//               tcgen05.ld TMEM -> registers -> fused op -> global
//               (EPI_SWIGLU: silu(gate) * up -> bf16 H, the first expert GEMM;
//                EPI_BF16: plain bf16 store, the down projection / dgrad;
//                EPI_F32: fp32 output, the weight gradients;
//                EPI_SWIGLU_BWD: the SwiGLU backward fused into the dgrad;
//                EPI_GATE: the router GEMM with top-K / softmax / histogram fused)
// plus the CTA-pair variant (gemm2sm_kernel, cta_group::2, M = 256 per pair).
// Grouped mode walks a device-resident m-tile list built from the scheduler's
// segments (no host sync): tiles are ordered expert-major, then in raster bands of
// m-tiles swept across the N-blocks, so an expert's weight panels and rows are reused
// from L2 within a wave; long-K tiles start each wave together (wave counters).
// Weight gradients (mode 2) walk the shorter tile dimension fastest.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace hep {
namespace gemm {

using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle atom row
#ifndef HEP_EPI_SPLIT
#define HEP_EPI_SPLIT 2
#endif
constexpr int kEpiSplit = HEP_EPI_SPLIT;  // epilogue warps per TMEM lane quarter (column slices)
constexpr int kEpiWarps = 4 * kEpiSplit;
constexpr int kThreads = 64 + 32 * kEpiWarps;

enum Epi { EPI_SWIGLU = 0, EPI_BF16 = 1, EPI_F32 = 2, EPI_SWIGLU_BWD = 3, EPI_GATE = 4 };

// EPI_GATE (router GEMM with the gate fused into its epilogue): the accumulator tile
// holds 128 tokens x all E_pad <= 256 logits, so one TMEM lane = one token's whole
// logit row and the epilogue thread selects its top-K, the softmax weights and
// counts the load-matrix histogram without the logits ever leaving the SM.
constexpr int kGateMaxK = 8;
constexpr int kGateMaxSrc = HEP_MAX_GPUS;
constexpr int kGateMaxE = 256;
// [n_src][E] histogram, [3][E] chunk counters of a tile (a tile of <= 128 rows touches at
// most 3 aligned 64-token chunks), [E] bias, and the column-half merge buffers
// (128 rows x KG x (key, expert, logit))
constexpr int kGateSmemBytes = 4 * (kGateMaxSrc * kGateMaxE + 4 * kGateMaxE) + 128 * (kGateMaxK * 12 + 16);
struct GateParams {
    const float *bias;   // [E] selection bias or null
    int K, E;            // top-K, experts (columns >= E are padding)
    int64_t tps;         // tokens per source GPU (token t belongs to source t / tps)
    int n_src;
    int ncs;             // 64-token chunks per source (chunk counts; 0 = none)
    int32_t *topk_idx;   // [T][K]
    float *topk_w;       // [T][K]
    int64_t *hist;       // [n_src][E], zeroed by the caller's launch sequence
    int32_t *chunk_cnt;  // [n_src][ncs][E] or null
    // in-kernel histogram zeroing (hep_router_topk_ws): {flag, ticket}, zero between launches.
    // CTA 0 zeroes hist, then raises flag; every CTA flushes its counts once flag is up and
    // takes a ticket; the last ticket lowers flag and ticket again (self-resetting, so a
    // captured graph can replay it).  null: the caller's launch sequence zeroes hist.
    unsigned int *sync;
};

struct Params {
    int grouped;             // 0: dense M rows; 1: m-tile list; 2: per-expert K-ragged (weight gradients)
    int64_t M;               // dense rows
    int n_tiles;             // N / BN
    int kblocks;             // K / 64
    int64_t b_rows_per_exp;  // rows of B per expert (N_total)
    const int32_t *mt_row0;  // [n_mtiles] first row of each m-tile
    const int32_t *mt_rows;  // [n_mtiles] valid rows (<= 128)
    const int32_t *exp_mt_off;  // [n_exp+1] m-tile offsets per expert
    int n_exp;
    void *out;
    int64_t ld_out;          // elements per output row
    int64_t out_cols;        // valid output columns (EPI_F32 masking)
    // mode 2 (weight gradients): expert e contracts over rows [exp_rows[e], exp_rows[e+1])
    // (64-row padded blocks), output tile grid m_tiles x n_tiles per expert
    const int64_t *exp_rows;
    const int32_t *exp_perm;  // grouped == 2: expert visit order (staged in s_off), or null
    int m_tiles;
    int64_t out_exp_stride;  // elements between consecutive experts' outputs
    // EPI_SWIGLU: optional pre-activation store; EPI_SWIGLU_BWD: pre-activation input
    void *aux;
    int64_t ld_aux;
    int raster_gm;  // grouped mode: m-tiles per raster band (0 = whole expert)
    int pol_mode;  // 0: defaults; else (A policy | B policy << 2), 1 normal, 2 last, 3 first (tuning)
    // EPI_BF16: optional per-row destination addresses (row r -> row_addr[r]); the fused
    // combine all-to-all stores each expert output row straight into its source GPU's
    // buffer over NVLink (peer pointers), instead of into `out`
    const uint64_t *row_addr;
    GateParams gate;  // EPI_GATE only
    // grouped mode, A operand gathered by row (the permute fused into the GEMM): receive
    // row r is token gather_idx[r] of the A tensor map (box {64, 1}), rows past an m-tile's
    // valid rows read gather_oob (outside the map: TMA zero fill)
    const int32_t *gather_idx;
    int32_t gather_oob;
    int tile_m;    // modes 0 / 2: rows per m-tile (0 = BM; 256 on the CTA pair)
    int light_first;  // grouped: weights of single-m-tile experts loaded evict-first
    int k_split;      // mode 0: contraction split into k_split ranges, partial s -> out + s*out_exp_stride
    int wait_cluster;
    int st256;  // epilogue rows 32-B aligned: one 256-bit store per 16 bf16 / 8 fp32 columns (full L2 sectors)
    int clk_slot;
    unsigned int *wave_ctr;  // pair kernel: producers' wave counter (zeroed before the launch) or null
    int a_box_rows;  // mode 0, K-major A: rows per A TMA box (= tile_m when < 128; 0 = BM)  // > 0: CTA 0 stamps (clock64, globaltimer) at entry and exit into g_gemm_clk[clk_slot - 1]
    // mode 0 (the router GEMM): > 1 = the launch's thread-block cluster size; every CTA of a
    // cluster TMA-loads 1/b_mc of each B (Wg) tile and multicasts it to all of them, so B
    // crosses L2 -> SM once per cluster.  The cluster's CTAs walk their tiles in lockstep
    // (tiles past the last one are empty: B only, no MMAs, no epilogue work)
    int b_mc;
};

// Diagnostics (hep_tuning.ffn_clock = 1): SM clock cycles and wall nanoseconds of CTA 0 across
// the two expert GEMMs, i.e. the SM clock the tensor cores actually ran at (the
// power-capped clock of a long GEMM is not what nvidia-smi samples between kernels).
__device__ long long g_gemm_clk[2][4];
__device__ __forceinline__ void clk_stamp(const Params &p, int at) {
    if (p.clk_slot > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
        long long ns;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
        g_gemm_clk[p.clk_slot - 1][2 * at] = clock64();
        g_gemm_clk[p.clk_slot - 1][2 * at + 1] = ns;
    }
}

// Diagnostics build only (-DHEP_ROUTER_STAMPS, tools/router_stamps.py): %globaltimer of every
// router CTA at entry, last MMA issued, epilogue start / end, exit
#ifdef HEP_ROUTER_STAMPS
__device__ unsigned long long g_router_stamps[256][8];
#define ROUTER_STAMP(i)                                                                   \
    do {                                                                                 \
        if (EPI == EPI_GATE && blockIdx.x < 256) g_router_stamps[blockIdx.x][i] = globaltimer_ns(); \
    } while (0)
#define GATE_STAMP(i)                                                                              \
    do {                                                                                           \
        if (row_in_tile == 0 && half == 0 && blockIdx.x < 256) g_router_stamps[blockIdx.x][i] = globaltimer_ns(); \
    } while (0)
#else
#define GATE_STAMP(i) \
    do {              \
    } while (0)
#define ROUTER_STAMP(i) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ uint64_t pick_policy(int k) {
    return k == 2 ? sm100::policy_evict_last() : (k == 3 ? sm100::policy_evict_first() : sm100::policy_evict_normal());
}

// grouped mode: p.exp_mt_off staged in shared memory (the per-tile binary search over
// experts would otherwise be a chain of dependent global loads in every warp role)
constexpr int kMaxExpSmem = 1024;
constexpr int kOffBytes = 4 * (kMaxExpSmem + 4);

template <int BN, int STAGES>
struct Smem {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
    static constexpr size_t BYTES = 1024 + (size_t)STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4) + 16 + kOffBytes;
};

struct Tile {
    int expert, n_blk;
    int32_t row0, rows;
    int64_t k0;  // first contraction row (mode 2)
    int kb;      // contraction blocks of 64
};

__device__ __forceinline__ int64_t total_tiles(const Params &p) {
    const int tm = p.tile_m ? p.tile_m : BM;
    if (p.grouped == 0) return ((p.M + tm - 1) / tm) * p.n_tiles * (p.k_split > 1 ? p.k_split : 1);
    if (p.grouped == 2) return (int64_t)p.n_exp * p.m_tiles * p.n_tiles;
    return (int64_t)p.exp_mt_off[p.n_exp] * p.n_tiles;
}

__device__ __forceinline__ Tile decode(const Params &p, int64_t t, const int32_t *off) {
    Tile tl;
    tl.k0 = 0;
    tl.kb = p.kblocks;
    const int tm = p.tile_m ? p.tile_m : BM;
    if (p.grouped == 2) {
        const int64_t per = (int64_t)p.m_tiles * p.n_tiles;
        const int slot = (int)(t / per);
        const int64_t rem = t - (int64_t)slot * per;
        const int e = p.exp_perm ? off[slot] : slot;
        tl.expert = e;
        // the shorter tile dimension runs fastest: a wave of tiles then spans a few panels of
        // the long dimension and ALL panels of the short one, which stay in L2 (m fastest
        // at dW13 = dA13^T X, 112 x 16 tiles at the Mixtral shape, streamed every dA13 panel
        // from DRAM once per N block: 27 GB per launch)
        if (p.raster_gm == -2 && p.n_tiles < p.m_tiles) {
            tl.n_blk = (int)(rem % p.n_tiles);
            tl.row0 = (int32_t)((rem / p.n_tiles) * tm);
        } else {
            tl.n_blk = (int)(rem / p.m_tiles);
            tl.row0 = (int32_t)((rem % p.m_tiles) * tm);
        }
        tl.rows = (int32_t)(p.M - tl.row0 < tm ? p.M - tl.row0 : tm);
        tl.k0 = p.exp_rows[e];
        tl.kb = (int)((p.exp_rows[e + 1] - tl.k0) / BK);
        return tl;
    }
    if (p.grouped == 0) {
        const int64_t mt = (p.M + tm - 1) / tm;
        tl.expert = 0;
        if (p.k_split > 1) {  // split-K: partial s of every output tile, over k-blocks [s*kps, ...)
            const int64_t per = mt * p.n_tiles;
            const int sp = (int)(t / per);
            t -= (int64_t)sp * per;
            const int kps = (p.kblocks + p.k_split - 1) / p.k_split;
            tl.expert = sp;
            tl.k0 = (int64_t)sp * kps * BK;
            tl.kb = min(kps, p.kblocks - sp * kps);
            if (tl.kb < 0) tl.kb = 0;
        }
        tl.n_blk = (int)(t / mt);
        const int64_t m = t % mt;
        tl.row0 = (int32_t)(m * tm);
        const int64_t left = p.M - m * tm;
        tl.rows = (int32_t)(left < tm ? left : tm);
        return tl;
    }
    // expert e owns tiles [off[e]*n_tiles, off[e+1]*n_tiles)
    int lo = 0, hi = p.n_exp - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if ((int64_t)off[mid] * p.n_tiles <= t) lo = mid; else hi = mid - 1;
    }
    const int e = lo;
    const int64_t base = (int64_t)off[e];
    const int64_t mt_e = (int64_t)off[e + 1] - base;
    const int64_t local = t - base * p.n_tiles;
    tl.expert = e;
    int64_t m;
    if (p.raster_gm > 0 && mt_e > p.raster_gm) {
        // grouped raster: bands of raster_gm m-tiles, each swept across all N-blocks, so the
        // operands live in L2 for one band instead of the whole expert
        const int64_t band = local / ((int64_t)p.raster_gm * p.n_tiles);
        const int64_t within = local - band * p.raster_gm * p.n_tiles;
        const int64_t gm = (mt_e - band * p.raster_gm) < p.raster_gm ? (mt_e - band * p.raster_gm) : p.raster_gm;
        tl.n_blk = (int)(within / gm);
        m = base + band * p.raster_gm + within % gm;
    } else {
        tl.n_blk = (int)(local / mt_e);
        m = base + local % mt_e;
    }
    tl.row0 = p.mt_row0[m];
    tl.rows = p.mt_rows[m];
    return tl;
}

// fast reciprocal (MUFU.RCP + FMUL, ~2 ulp fp32) instead of IEEE division (FCHK + Newton
// + slow-path call): far below the bf16 rounding of every output it feeds
__device__ __forceinline__ float silu(float x) { return __fdividef(x, 1.0f + __expf(-x)); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&v);
}

// Epilogue of one accumulator tile row (this thread's TMEM lane): TMEM ->
// registers -> fused op -> global.  t_row = TMEM address of the row's first
// column, grow = global output row.
__device__ __forceinline__ float sigmoid(float x) { return __fdividef(1.0f, 1.0f + __expf(-x)); }

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

template <int BN, int EPI>
__device__ __forceinline__ void store_tile(const Params &p, uint32_t t_row, int64_t grow, bool valid, int n_blk,
                                           uint64_t pol_out, int expert, bool zero, int half) {
    // this warp's share of the tile's columns: half 0 / 1 of the accumulator
    // (spans under 16 columns per slice are not split: slice 0 takes them all)
    constexpr int SPAN = EPI == EPI_SWIGLU ? BN / 2 : BN;
    constexpr bool SPLIT = SPAN / kEpiSplit >= 16;
    static_assert(EPI != EPI_BF16 || (SPAN / kEpiSplit) % 32 == 0, "bf16 epilogue stores 32 columns per step");
    const int c_begin = SPLIT ? half * (SPAN / kEpiSplit) : 0;
    const int c_end = SPLIT ? c_begin + SPAN / kEpiSplit : (half == 0 ? SPAN : 0);
    if constexpr (EPI == EPI_SWIGLU_BWD) {
        // accumulator = dH for ffn columns [n_blk*BN, +BN); the pre-activations
        // (gate a, up b) live in aux with the W13 interleave (128-blocks: gate j, up j).
        // dA_gate = dH * b * silu'(a), dA_up = dH * silu(a); written in the same interleave.
        const __nv_bfloat16 *pre = reinterpret_cast<const __nv_bfloat16 *>(p.aux) + grow * p.ld_aux;
        __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.out) + grow * p.ld_out;
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 16) {
            const int64_t f = (int64_t)n_blk * BN + c;       // first ffn column of this chunk
            const int64_t gcol = (f / 128) * 256 + (f % 128);  // gate column; up = gcol + 128
            // the pre-activation loads go out before the TMEM load so the two latencies overlap
            uint32_t gw[8], uw[8];
            if (valid) {
                if (p.st256) {  // aux rows are 32-B aligned too (with_store_width)
                    ld_global_v8(pre + gcol, gw);
                    ld_global_v8(pre + gcol + 128, uw);
                } else {
                    const uint4 *ga = reinterpret_cast<const uint4 *>(pre + gcol);
                    const uint4 *ua = reinterpret_cast<const uint4 *>(pre + gcol + 128);
                    *reinterpret_cast<uint4 *>(gw) = ga[0];
                    *reinterpret_cast<uint4 *>(gw + 4) = ga[1];
                    *reinterpret_cast<uint4 *>(uw) = ua[0];
                    *reinterpret_cast<uint4 *>(uw + 4) = ua[1];
                }
            }
            uint32_t v[16];
            tmem_ld16(t_row + c, v);
            tmem_ld_wait();
            if (!valid) continue;
            uint32_t dg[8], du[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float d0 = __uint_as_float(v[2 * i]), d1 = __uint_as_float(v[2 * i + 1]);
                float a0 = bf16lo(gw[i]), a1 = bf16hi(gw[i]), b0 = bf16lo(uw[i]), b1 = bf16hi(uw[i]);
                float s0 = sigmoid(a0), s1 = sigmoid(a1);
                float ds0 = s0 * (1.0f + a0 * (1.0f - s0)), ds1 = s1 * (1.0f + a1 * (1.0f - s1));
                dg[i] = pack_bf16(d0 * b0 * ds0, d1 * b1 * ds1);
                du[i] = pack_bf16(d0 * a0 * s0, d1 * a1 * s1);
            }
            if (p.st256) {
                st_global_v8_hint(out + gcol, dg, pol_out);
                st_global_v8_hint(out + gcol + 128, du, pol_out);
            } else {
                st_global_v4_hint(out + gcol, make_uint4(dg[0], dg[1], dg[2], dg[3]), pol_out);
                st_global_v4_hint(out + gcol + 8, make_uint4(dg[4], dg[5], dg[6], dg[7]), pol_out);
                st_global_v4_hint(out + gcol + 128, make_uint4(du[0], du[1], du[2], du[3]), pol_out);
                st_global_v4_hint(out + gcol + 136, make_uint4(du[4], du[5], du[6], du[7]), pol_out);
            }
        }
    } else if constexpr (EPI == EPI_SWIGLU) {
        // columns [0, BN/2) = gate (W1 block), [BN/2, BN) = up (W3 block)
        __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(p.out) + grow * p.ld_out +
                             (int64_t)n_blk * (BN / 2);
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 16) {
            uint32_t g[16], u[16];
            tmem_ld16(t_row + c, g);
            tmem_ld16(t_row + BN / 2 + c, u);
            tmem_ld_wait();
            uint32_t packed[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float g0 = __uint_as_float(g[2 * i]), g1 = __uint_as_float(g[2 * i + 1]);
                float u0 = __uint_as_float(u[2 * i]), u1 = __uint_as_float(u[2 * i + 1]);
                packed[i] = pack_bf16(silu(g0) * u0, silu(g1) * u1);
            }
            if (valid && p.aux) {  // training: keep the pre-activations for the backward pass
                __nv_bfloat16 *pre = reinterpret_cast<__nv_bfloat16 *>(p.aux) + grow * p.ld_aux + (int64_t)n_blk * BN + c;
                uint32_t pg[8], pu[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    pg[i] = pack_bf16(__uint_as_float(g[2 * i]), __uint_as_float(g[2 * i + 1]));
                    pu[i] = pack_bf16(__uint_as_float(u[2 * i]), __uint_as_float(u[2 * i + 1]));
                }
                if (p.st256) {
                    st_global_v8_hint(pre, pg, pol_out);
                    st_global_v8_hint(pre + BN / 2, pu, pol_out);
                } else {
                    st_global_v4_hint(pre, make_uint4(pg[0], pg[1], pg[2], pg[3]), pol_out);
                    st_global_v4_hint(pre + 8, make_uint4(pg[4], pg[5], pg[6], pg[7]), pol_out);
                    st_global_v4_hint(pre + BN / 2, make_uint4(pu[0], pu[1], pu[2], pu[3]), pol_out);
                    st_global_v4_hint(pre + BN / 2 + 8, make_uint4(pu[4], pu[5], pu[6], pu[7]), pol_out);
                }
            }
            if (valid) {
                if (p.st256) {
                    st_global_v8_hint(out + c, packed, pol_out);
                } else {
                    st_global_v4_hint(out + c, make_uint4(packed[0], packed[1], packed[2], packed[3]), pol_out);
                    st_global_v4_hint(out + c + 8, make_uint4(packed[4], packed[5], packed[6], packed[7]), pol_out);
                }
            }
        }
    } else if constexpr (EPI == EPI_BF16) {
        const bool remote = p.row_addr != nullptr;
        __nv_bfloat16 *out =
            (remote ? (valid ? reinterpret_cast<__nv_bfloat16 *>(p.row_addr[grow]) : nullptr)
                    : reinterpret_cast<__nv_bfloat16 *>(p.out) + grow * p.ld_out) +
            (int64_t)n_blk * BN;
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 32) {  // two TMEM loads in flight per wait
            uint32_t v[16], w[16];
            tmem_ld16(t_row + c, v);
            tmem_ld16(t_row + c + 16, w);
            tmem_ld_wait();
            uint32_t packed[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                packed[i] = pack_bf16(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
                packed[8 + i] = pack_bf16(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1]));
            }
            if (valid && p.st256) {
                st_global_v8_hint(out + c, packed, pol_out);
                st_global_v8_hint(out + c + 16, packed + 8, pol_out);
            } else if (valid) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 val = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
                    if (remote)  // peer (NVLink) or local destination row: plain 16-byte stores
                        reinterpret_cast<uint4 *>(out + c)[q] = val;
                    else
                        st_global_v4_hint(out + c + 8 * q, val, pol_out);
                }
            }
        }
    } else {
        float *out = reinterpret_cast<float *>(p.out) + (int64_t)expert * p.out_exp_stride + grow * p.ld_out +
                     (int64_t)n_blk * BN;
        const int64_t col0 = (int64_t)n_blk * BN;
#pragma unroll 1
        for (int c = c_begin; c < c_end; c += 16) {
            uint32_t v[16];
            tmem_ld16(t_row + c, v);
            tmem_ld_wait();
            if (zero)  // empty contraction (expert without rows): the accumulator was never written
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = 0u;
            if (valid) {
                if (p.st256 && col0 + c + 16 <= p.out_cols) {
                    st_global_v8_hint(out + c, v, pol_out);
                    st_global_v8_hint(out + c + 8, v + 8, pol_out);
                } else if (col0 + c + 16 <= p.out_cols) {
                    float4 *dst = reinterpret_cast<float4 *>(out + c);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                             __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (col0 + c + i < p.out_cols) out[c + i] = __uint_as_float(v[i]);
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(f + 0.0f);  // -0 -> +0: equal scores must tie
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// order_key of a value known not to be -0 (SHF + LOP3)
__device__ __forceinline__ uint32_t order_key_nz(float f) {
    const uint32_t u = __float_as_uint(f);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}

// EPI_GATE epilogue of one accumulator tile (<= 128 tokens), run by all 8 epilogue
// warps: warp pair (q, q+4) shares TMEM lane quarter q; with E_pad % 32 == 0 the two
// warps scan one column half each (nhalf = 2), else half 0 scans every column (nhalf =
// 1).  Named barrier 1 spans the 128 * nhalf participating threads.
// Selection and weights are exactly hep_gate_topk's (gate.cu): top-K of the order key
// of (logit + bias) with ties to the lower expert id, softmax over the K selected
// logits in pick order (key descending, ties by expert id).  Two passes over the
// thread's row, so the per-column work is a handful of instructions:
//   1. the K largest KEYS (a multiset: ties kept) by a min/max network -- slot j takes
//      min(slot j-1, max(key, slot j)), 2 IMNMX per slot, no expert/logit tracking;
//      half 1 hands its K keys to half 0, which merges them and fixes the threshold
//      vK = the K-th key and how many vK-keyed experts each half contributes (the lower
//      expert ids -- half 0's -- first);
//   2. a rescan selects exactly those experts (key > vK, or key == vK within the
//      half's quota) in ascending expert order into a shared K-entry list; half 0 then
//      orders the K entries with the strict insertion network (the same list a full
//      sequential scan keeps) and computes the weights.
// Histogram counts go to shared memory (flushed once per CTA); the per-64-token
// chunk counts (chunks aligned to 64 tokens) are stored directly when the tile is made
// of whole chunks, else added with integer atomics into the zeroed global counts.
template <int KG>
__device__ __forceinline__ void gate_insert(uint32_t key, int e, float l, uint32_t (&tk)[KG], int (&te)[KG],
                                            float (&tv)[KG]) {
#pragma unroll
    for (int j = KG - 1; j >= 0; --j) {
        const bool up = j > 0 && key > tk[j > 0 ? j - 1 : 0];  // slot j takes slot j-1's entry
        const bool here = key > tk[j];                          // ... or the new one
        tk[j] = up ? tk[j > 0 ? j - 1 : 0] : (here ? key : tk[j]);
        te[j] = up ? te[j > 0 ? j - 1 : 0] : (here ? e : te[j]);
        tv[j] = up ? tv[j > 0 ? j - 1 : 0] : (here ? l : tv[j]);
    }
}

// top-KG key multiset, sorted descending: tk[j] <- min(tk[j-1], max(key, tk[j]))
template <int KG>
__device__ __forceinline__ void key_insert(uint32_t key, uint32_t (&tk)[KG]) {
#pragma unroll
    for (int j = KG - 1; j > 0; --j) tk[j] = min(tk[j - 1], max(key, tk[j]));
    tk[0] = max(key, tk[0]);
}

// descending compare-exchange, the optimal 19-comparator sorting network for 8 keys, and the
// top-8 merge of two descending 8-lists (bitonic: max(a[i], b[7-i]), then a half-cleaner cascade)
__device__ __forceinline__ void cx_desc(uint32_t &a, uint32_t &b) {
    const uint32_t hi = max(a, b), lo = min(a, b);
    a = hi;
    b = lo;
}
__device__ __forceinline__ void sort8_desc(uint32_t (&k)[8]) {
    cx_desc(k[0], k[1]); cx_desc(k[2], k[3]); cx_desc(k[4], k[5]); cx_desc(k[6], k[7]);
    cx_desc(k[0], k[2]); cx_desc(k[1], k[3]); cx_desc(k[4], k[6]); cx_desc(k[5], k[7]);
    cx_desc(k[1], k[2]); cx_desc(k[5], k[6]); cx_desc(k[0], k[4]); cx_desc(k[3], k[7]);
    cx_desc(k[1], k[5]); cx_desc(k[2], k[6]);
    cx_desc(k[1], k[4]); cx_desc(k[3], k[6]);
    cx_desc(k[2], k[4]); cx_desc(k[3], k[5]);
    cx_desc(k[3], k[4]);
}
__device__ __forceinline__ void merge8_top(uint32_t (&a)[8], const uint32_t (&b)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = max(a[i], b[7 - i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) cx_desc(a[i], a[i + 4]);
    cx_desc(a[0], a[2]); cx_desc(a[1], a[3]); cx_desc(a[4], a[6]); cx_desc(a[5], a[7]);
    cx_desc(a[0], a[1]); cx_desc(a[2], a[3]); cx_desc(a[4], a[5]); cx_desc(a[6], a[7]);
}

__device__ __forceinline__ void gate_bar(int nthr) { asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory"); }
// v[i] for a runtime i < 16 without local memory: a 4-level select tree
__device__ __forceinline__ uint32_t pick16(const uint32_t (&v)[16], int i) {
    uint32_t a[8], b[4], c[2];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = (i & 8) ? v[j + 8] : v[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = (i & 4) ? a[j + 4] : a[j];
#pragma unroll
    for (int j = 0; j < 2; ++j) c[j] = (i & 2) ? b[j + 2] : b[j];
    return (i & 1) ? c[1] : c[0];
}
// named barrier 1 that also ORs a predicate over its nthr threads
__device__ __forceinline__ bool gate_bar_or(int nthr, bool v) {
    uint32_t r;
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.u32 p, %1, 0;\n\t"
        "bar.red.or.pred q, 1, %2, p;\n\t"
        "selp.u32 %0, 1, 0, q;\n}"
        : "=r"(r)
        : "r"((uint32_t)v), "r"(nthr)
        : "memory");
    return r != 0;
}

template <int KG, int SPAN>
__device__ __forceinline__ void gate_tile(const Params &p, uint32_t t_row, int64_t row0, int rows, int row_in_tile,
                                          int half, int nhalf, int32_t *s_hist, int32_t *s_chunk,
                                          const float *s_bias, uint8_t *s_merge) {
    // SPAN = columns per thread (E_pad / nhalf); TMEM is read CW columns per wait (64
    // columns per wait -- four loads in flight -- measured slower: Qwen3 45.3 -> 53.7 µs)
    constexpr int CW = 16;
    constexpr int NJ = CW / 16;
    static_assert(SPAN % CW == 0 && CW % 16 == 0, "gate column span");
    const GateParams &g = p.gate;
    const int E = g.E;
    const int nthr = 128 * nhalf;
    const int tid = half * 128 + row_in_tile;
    // chunk counters: aligned 64-token chunks [c0, c0 + 3) relative to this tile
    const int64_t c0 = row0 >> 6;
    const bool whole = (row0 & 63) == 0 && ((rows & 63) == 0 || row0 + rows == p.M);
    if (g.chunk_cnt) {
        gate_bar(nthr);  // previous tile's chunk counts are out
        for (int i = tid; i < 3 * E; i += nthr) s_chunk[i] = 0;
        gate_bar(nthr);
    }
    const bool valid = row_in_tile < rows;
    const int64_t t = row0 + row_in_tile;
    // shared buffers: half 1's keys [128][KG] | (vK, quota, offset) [128][4] | list e / logit [128][KG]
    uint32_t *mk = reinterpret_cast<uint32_t *>(s_merge) + row_in_tile * KG;
    int32_t *bc = reinterpret_cast<int32_t *>(s_merge + 128 * KG * 4) + row_in_tile * 4;
    int32_t *le = reinterpret_cast<int32_t *>(s_merge + 128 * KG * 4 + 128 * 16) + row_in_tile * KG;
    float *lv = reinterpret_cast<float *>(s_merge + 128 * KG * 8 + 128 * 16) + row_in_tile * KG;
    const int c_lo = half * SPAN;
    const int c_hi = c_lo + SPAN;
    // ---- pass 1: logits out, top-KG keys -------------------------------------------
    // two independent networks (even / odd columns), merged after the scan: the per-column
    // min/max chain is latency-bound at two warps per scheduler, so this doubles its ILP.
    // s_bias holds bias + 0.0f (never -0) and -inf on padding columns, so logit + bias is
    // never -0 and order_key needs no normalising add; padding keys (of -inf) stay below
    // every finite score
    uint32_t tk[KG], tk2[KG];
#pragma unroll
    for (int i = 0; i < KG; ++i) tk[i] = tk2[i] = 0u;
    float *lrow = (valid && p.out) ? reinterpret_cast<float *>(p.out) + t * p.ld_out : nullptr;
#pragma unroll 1
    for (int c = c_lo; c < c_hi; c += CW) {
        uint32_t v[NJ][16];
#pragma unroll
        for (int j = 0; j < NJ; ++j) tmem_ld16(t_row + c + 16 * j, v[j]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int cj = c + 16 * j;
            if (lrow && cj < p.out_cols) {  // logits buffer is [T][e_pad]; BN may be wider
                float4 *dst = reinterpret_cast<float4 *>(lrow + cj);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    dst[i] = make_float4(__uint_as_float(v[j][4 * i]), __uint_as_float(v[j][4 * i + 1]),
                                         __uint_as_float(v[j][4 * i + 2]), __uint_as_float(v[j][4 * i + 3]));
            }
            if constexpr (KG == 8) {
                // batches of 8 columns: sort the batch (19 comparators), keep the top 8 of
                // list + batch (8 max of the list against the reversed batch = a bitonic
                // sequence), re-sort it (12 comparators): 70 IMNMX per 8 columns instead of 120
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t bk[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        bk[i] = order_key_nz(__uint_as_float(v[j][8 * h + i]) + s_bias[cj + 8 * h + i]);
                    sort8_desc(bk);
                    merge8_top(tk, bk);
                }
            } else {
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    key_insert<KG>(order_key_nz(__uint_as_float(v[j][i]) + s_bias[cj + i]), tk);
                    key_insert<KG>(order_key_nz(__uint_as_float(v[j][i + 1]) + s_bias[cj + i + 1]), tk2);
                }
            }
        }
    }
    if constexpr (KG != 8) {
#pragma unroll
        for (int k = 0; k < KG; ++k) key_insert<KG>(tk2[k], tk);
    }
    GATE_STAMP(5);
    // ---- threshold and per-half quotas ------------------------------------------------
    uint32_t vK;
    int quota, offset, lim;  // lim: one past this half's last slot in the K-entry list
    if (nhalf == 2) {
        if (half == 1)
#pragma unroll
            for (int k = 0; k < KG; ++k) mk[k] = tk[k];
        gate_bar(nthr);
        if (half == 0) {
            uint32_t tm[KG];
#pragma unroll
            for (int k = 0; k < KG; ++k) tm[k] = tk[k];
#pragma unroll
            for (int k = 0; k < KG; ++k) key_insert<KG>(mk[k], tm);
            vK = tm[KG - 1];
            int need = 0, gt0 = 0, c0h = 0;
#pragma unroll
            for (int k = 0; k < KG; ++k) {
                need += tm[k] == vK;
                gt0 += tk[k] > vK;
                c0h += tk[k] == vK;
            }
            quota = c0h < need ? c0h : need;  // the lower expert ids take the ties first
            offset = 0;
            lim = gt0 + quota;
            bc[0] = (int32_t)vK;
            bc[1] = need - quota;
            bc[2] = gt0 + quota;
        }
        gate_bar(nthr);
        if (half == 1) {
            vK = (uint32_t)bc[0];
            quota = bc[1];
            offset = bc[2];
            lim = KG;
        }
    } else {
        vK = tk[KG - 1];
        quota = 0;
#pragma unroll
        for (int k = 0; k < KG; ++k) quota += tk[k] == vK;
        offset = 0;
        lim = KG;
    }
    GATE_STAMP(6);
    // ---- pass 2: the selected experts, ascending, into the shared list -----------------
    // Fast path: one compare per column into a 16-bit mask of the columns with key >= vK;
    // their expert ids and logits (pick16) go to the list.  That set is exactly the
    // selection unless a half holds more vK-keyed columns than its quota (exact score ties
    // at the K-th place): then its count overshoots `lim`, and the whole tile reruns the
    // exact scan below.
    int cnt = offset;
    bool exact = false;
    {
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += 16) {
            uint32_t v[16];
            tmem_ld16(t_row + c, v);
            tmem_ld_wait();
            uint32_t m = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (order_key_nz(__uint_as_float(v[i]) + s_bias[c + i]) >= vK) m |= 1u << i;
            while (m) {
                const int i = __ffs(m) - 1;
                m &= m - 1;
                if (cnt < KG) {
                    le[cnt] = c + i;
                    lv[cnt] = __uint_as_float(pick16(v, i));
                }
                ++cnt;
            }
        }
        exact = gate_bar_or(nthr, valid && cnt != lim);  // also: both halves' entries are in
        cnt = offset;
    }
    if (exact) {
#pragma unroll 1
        for (int c = c_lo; c < c_hi; c += CW) {
            uint32_t v[NJ][16];
#pragma unroll
            for (int j = 0; j < NJ; ++j) tmem_ld16(t_row + c + 16 * j, v[j]);
            tmem_ld_wait();
            if (valid) {
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int e = c + 16 * j + i;
                        const float l = __uint_as_float(v[j][i]);
                        const uint32_t key = e < E ? order_key(l + s_bias[e]) : 0u;
                        const bool tie = key == vK && quota > 0;
                        if (e < E && (key > vK || tie)) {
                            le[cnt] = e;
                            lv[cnt] = l;
                            ++cnt;
                            quota -= tie;
                        }
                    }
                }
            }
        }
        if (nhalf == 2) gate_bar(nthr);  // half 1's entries are in the list
    }
    GATE_STAMP(7);
    if (half == 0 && valid) {
        uint32_t tkf[KG];
        int te[KG];
        float tv[KG];
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            tkf[k] = 0u;
            te[k] = 0;
            tv[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            const int e = le[k];
            const float l = lv[k];
            gate_insert<KG>(order_key(l + s_bias[e]), e, l, tkf, te, tv);
        }
        float mx = tv[0];
#pragma unroll
        for (int k = 1; k < KG; ++k) mx = fmaxf(mx, tv[k]);
        float ex[KG], den = 0.f;
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            ex[k] = expf(tv[k] - mx);
            den += ex[k];
        }
        const int64_t s64 = t / g.tps;
        const int src = (int)(s64 < g.n_src - 1 ? s64 : g.n_src - 1);
        const int ch = (int)((t >> 6) - c0);
#pragma unroll
        for (int k = 0; k < KG; ++k) {
            g.topk_idx[t * KG + k] = te[k];
            g.topk_w[t * KG + k] = ex[k] / den;
            atomicAdd(&s_hist[src * E + te[k]], 1);
            if (g.chunk_cnt) atomicAdd(&s_chunk[ch * E + te[k]], 1);
        }
    }
    if (nhalf == 2) gate_bar(nthr);  // the merge buffers are free for the next tile
    if (g.chunk_cnt) {
        gate_bar(nthr);
        // chunk j of the tile is global chunk c0 + j = (src * ncs + c) in the [n_src][ncs][E]
        // layout (the launch guarantees tps % 64 == 0, so chunks never straddle sources)
        const int64_t n_chunks = ((row0 + rows - 1) >> 6) - c0 + 1;
        for (int i = tid; i < n_chunks * E; i += nthr) {
            const int j = i / E, e = i - j * E;
            int32_t *dst = g.chunk_cnt + (c0 + j) * E + e;
            if (whole)
                *dst = s_chunk[i];
            else if (s_chunk[i])
                atomicAdd(dst, s_chunk[i]);
        }
    }
}

// hist zeroing by CTA 0 (GateParams::sync), at kernel entry
__device__ __forceinline__ void gate_hist_zero(const GateParams &g) {
    if (!g.sync || blockIdx.x != 0) return;
    for (int i = threadIdx.x; i < g.n_src * g.E; i += blockDim.x) g.hist[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(&g.sync[0], 1u);
    }
}

// the CTA's histogram counts into hist (integer sums: order-free, deterministic); with
// GateParams::sync, after CTA 0's zeroing and followed by the self-reset of the sync words
__device__ __forceinline__ void gate_hist_flush(const GateParams &g, const int32_t *s_hist) {
    if (g.sync) {
        // CTA 0 is dispatched first and zeroes at entry, long before any CTA gets here; the
        // wait is bounded anyway (a grid that cannot run its CTA 0 fails loudly, not silently)
        if (threadIdx.x == 0) {
            const uint64_t t0 = globaltimer_ns();
            while (ld_acquire_gpu_u32(&g.sync[0]) == 0u) {
                __nanosleep(32);
                if (globaltimer_ns() - t0 > 200000000ull) __trap();
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < g.n_src * g.E; i += blockDim.x)
        if (s_hist[i]) atomicAdd(reinterpret_cast<unsigned long long *>(g.hist) + i, (unsigned long long)s_hist[i]);
    if (g.sync) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&g.sync[1], 1u) == gridDim.x - 1) {  // every CTA has flushed
                atomicExch(&g.sync[0], 0u);
                atomicExch(&g.sync[1], 0u);
            }
        }
    }
}

// A_MN / B_MN: operand stored MN-major in global memory (the contraction index
// is the row index, e.g. activations [rows][d] contracted over rows for weight
// gradients, or weights [K][N] used untransposed).  Such an operand is staged as
// (extent/64) TMA boxes of 64(MN) x 64(K) — 128-byte rows along MN, k-groups of
// 8 rows 1024 B apart (SBO), MN blocks 8 KB apart (LBO) — and each 16-deep MMA
// step advances 2 KB.
template <int BN, int STAGES, int EPI, bool A_MN = false, bool B_MN = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Params p) {
    using S = Smem<BN, STAGES>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align within the array (not through uintptr_t) so s_off etc. stay LDS, not generic loads
    uint8_t *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = base;
    uint8_t *sB = base + STAGES * S::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(base + STAGES * S::STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    int32_t *s_off = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(tmem_slot) + 16);
    if (p.grouped == 1)
        for (int i = threadIdx.x; i <= p.n_exp; i += blockDim.x) s_off[i] = p.exp_mt_off[i];
    else if (p.grouped == 2 && p.exp_perm)
        for (int i = threadIdx.x; i < p.n_exp; i += blockDim.x) s_off[i] = p.exp_perm[i];
    int32_t *s_hist = s_off + kMaxExpSmem + 4;             // EPI_GATE: [n_src][E] counts
    int32_t *s_chunk = s_hist + kGateMaxSrc * kGateMaxE;  // EPI_GATE: [3][E] tile chunk counts
    float *s_bias = reinterpret_cast<float *>(s_chunk + 3 * kGateMaxE);  // EPI_GATE: [E_pad] bias
    uint8_t *s_merge = reinterpret_cast<uint8_t *>(s_bias + kGateMaxE);   // EPI_GATE: column-half merge
    if constexpr (EPI == EPI_GATE) {
        for (int i = threadIdx.x; i < p.gate.n_src * p.gate.E; i += blockDim.x) s_hist[i] = 0;
        for (int i = threadIdx.x; i < BN; i += blockDim.x)  // + 0.0f: -0 -> +0 (see gate_tile)
            s_bias[i] = i >= p.gate.E ? -__int_as_float(0x7f800000) : (p.gate.bias ? p.gate.bias[i] + 0.0f : 0.f);
        gate_hist_zero(p.gate);
    }

    if (threadIdx.x == 0) ROUTER_STAMP(0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mc = (EPI == EPI_GATE && !A_MN && !B_MN && p.grouped == 0) ? p.b_mc : 0;  // router only
    const uint32_t mc_rank = mc > 1 ? cluster_ctarank() : 0u;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], mc > 1 ? mc : 1);  // multicast B: every cluster CTA's MMAs release the slot
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);
        }
        fence_barrier_init();
        fence_proxy_async_smem();
    }
    if (warp == 1) tmem_alloc(tmem_slot, S::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    if (mc > 1) cluster_sync();  // peers multicast into this CTA's smem / barriers only after init
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    clk_stamp(p, 0);

    const int64_t n_total = total_tiles(p);
    const int kb = p.kblocks;
    // multicast B: a cluster's CTAs walk tiles in lockstep, so a CTA runs while its cluster's
    // first tile exists (t - rank < n_total); tiles >= n_total are empty (rows = 0)
    const int64_t t_end = n_total + (mc > 1 ? (int64_t)mc_rank : 0);

    if (warp == 0 && p.gather_idx) {
        // ============ TMA producer, A rows gathered by token (the fused permute) ============
        // lane l gathers tile rows 4l..4l+3 with one tile::gather4; lane 0 owns the barriers
        // and the weight tile
        const uint64_t pol_a = policy_evict_last();
        const uint64_t pol_b = p.pol_mode ? pick_policy((p.pol_mode >> 2) & 3) : policy_evict_normal();
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = blockIdx.x; t < n_total; t += gridDim.x) {
            const Tile tl = decode(p, t, s_off);
            const int32_t b_row = (int32_t)(tl.expert * p.b_rows_per_exp + (int64_t)tl.n_blk * BN);
            int r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int local = 4 * lane + j;
                r[j] = local < tl.rows ? p.gather_idx[tl.row0 + local] : p.gather_oob;
            }
            const int4 rows = make_int4(r[0], r[1], r[2], r[3]);
            for (int k = 0; k < tl.kb; ++k) {
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
                }
                __syncwarp();
                tma_gather4(sA + stage * S::A_BYTES + 512 * lane, &tmA, &full[stage], k * BK, rows, pol_a);
                if (lane == 0) tma_load_2d_hint(sB + stage * S::B_BYTES, &tmB, &full[stage], k * BK, b_row, pol_b);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ===================== TMA producer =====================
            int stage = 0;
            // grouped expert GEMMs reuse A (token rows) across N-blocks and stream B (weights);
            // the router GEMM streams A (x) and reuses B (Wg)
            const uint64_t pol_a = p.pol_mode ? pick_policy(p.pol_mode & 3) : (p.grouped ? policy_evict_last() : policy_evict_first());
            // weights are re-read by every m-tile of their expert: evict-last (single-m-tile experts:
            // evict-first, below); measured DSv3 FFN 13.26 -> 12.16 ms, Mixtral neutral
            const uint64_t pol_b = p.pol_mode ? pick_policy((p.pol_mode >> 2) & 3) : policy_evict_last();
            const uint64_t pol_first = policy_evict_first();
            uint32_t phase = 0;
            int64_t wave_target = 0;
            const uint16_t mc_mask = (uint16_t)((1u << (mc > 1 ? mc : 1)) - 1u);
            for (int64_t t = blockIdx.x; t < t_end; t += gridDim.x) {
                if (p.wave_ctr && t >= gridDim.x) {  // as in gemm2sm_kernel: waves start together
                    const int64_t w = t / gridDim.x;
                    const int64_t in_wave = n_total - w * gridDim.x < gridDim.x ? n_total - w * gridDim.x : gridDim.x;
                    wave_target += in_wave;
                    atomicAdd(p.wave_ctr, 1u);
                    const uint64_t t_start = globaltimer_ns();
                    while ((int64_t)ld_acquire_gpu_u32(p.wave_ctr) < wave_target && globaltimer_ns() - t_start < 200000)
                        __nanosleep(64);
                }
                const bool empty_tile = t >= n_total;  // multicast B only
                const Tile tl = decode(p, empty_tile ? 0 : t, s_off);
                const int32_t b_row = (int32_t)(tl.expert * p.b_rows_per_exp + (int64_t)tl.n_blk * BN);
                // contraction offsets: mode 2 contracts over the expert's rows; an MN-major
                // weight (mode 1) is [K][N] per expert, stacked along K
                const int32_t a_k0 = (int32_t)tl.k0;
                const int32_t b_k0 = (p.grouped == 2 || p.k_split > 1) ? (int32_t)tl.k0
                                                                       : (B_MN ? b_row - tl.n_blk * BN : 0);
                // an expert with a single m-tile streams its weights once: keep them out of L2's way
                const bool light = p.light_first && p.grouped == 1 && s_off[tl.expert + 1] - s_off[tl.expert] == 1;
                // A boxes of a_box_rows rows (router tiles of < 128 tokens): the MMA still reads
                // 128 rows, the rows past the box are stale and land only in ignored accumulator rows
                const uint32_t tx = empty_tile ? (uint32_t)S::B_BYTES
                                    : (!A_MN && p.a_box_rows > 0) ? (uint32_t)(p.a_box_rows * BK * 2) + S::B_BYTES
                                                                  : (uint32_t)S::STAGE_BYTES;
                for (int k = 0; k < tl.kb; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], tx);
                    if (!A_MN && !B_MN && mc > 1) {
                        // B slice mc_rank (BN / mc rows, a multiple of the 8-row swizzle atom) to
                        // every CTA of the cluster; A (this CTA's tokens) locally
                        if (!empty_tile)
                            tma_load_2d_hint(sA + stage * S::A_BYTES, &tmA, &full[stage], a_k0 + k * BK, tl.row0, pol_a);
                        const int slice = BN / mc;
                        tma_load_2d_mc(sB + stage * S::B_BYTES + mc_rank * slice * (BK * 2), &tmB, &full[stage], k * BK,
                                       b_row + (int32_t)mc_rank * slice, mc_mask, pol_b);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    if constexpr (A_MN) {
#pragma unroll
                        for (int i = 0; i < BM / 64; ++i)
                            tma_load_2d_hint(sA + stage * S::A_BYTES + i * 8192, &tmA, &full[stage], tl.row0 + 64 * i,
                                             a_k0 + k * BK, pol_a);
                    } else {
                        tma_load_2d_hint(sA + stage * S::A_BYTES, &tmA, &full[stage], a_k0 + k * BK, tl.row0, pol_a);
                    }
                    if constexpr (B_MN) {
#pragma unroll
                        for (int i = 0; i < BN / 64; ++i)
                            tma_load_2d_hint(sB + stage * S::B_BYTES + i * 8192, &tmB, &full[stage],
                                             tl.n_blk * BN + 64 * i, b_k0 + k * BK, pol_b);
                    } else {
                        tma_load_2d_hint(sB + stage * S::B_BYTES, &tmB, &full[stage], k * BK, b_row,
                                         light ? pol_first : pol_b);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
            if (mc > 1)  // producer tail: every cluster CTA's release of every slot has landed here
                for (int i = 0; i < STAGES; ++i) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===================== MMA issuer =====================
            constexpr uint32_t idesc = idesc_bf16_f32(BM, BN) | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint16_t mc_mask = (uint16_t)((1u << (mc > 1 ? mc : 1)) - 1u);
            for (int64_t t = blockIdx.x; t < t_end; t += gridDim.x) {
                const int tkb = (p.grouped == 2 || p.k_split > 1) ? decode(p, t, s_off).kb : kb;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int k = 0; k < tkb; ++k) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (mc > 1) {  // the slot's B slices came from every CTA: release it in all of them
                        if (t < n_total) {
                            const uint32_t a_addr = smem_u32(sA + stage * S::A_BYTES);
                            const uint32_t b_addr = smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
                            for (int kk = 0; kk < BK / 16; ++kk)
                                mma_bf16(d_tmem, desc_kmajor_sw128(a_addr + kk * 32), desc_kmajor_sw128(b_addr + kk * 32),
                                         idesc_bf16_f32(BM, BN), (k | kk) ? 1u : 0u);
                        }
                        mma_commit_mc(&empty[stage], mc_mask);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        continue;
                    }
                    const uint32_t a_addr = smem_u32(sA + stage * S::A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t ad = A_MN ? desc_mnmajor_sw128(a_addr + kk * 2048) : desc_kmajor_sw128(a_addr + kk * 32);
                        const uint64_t bd = B_MN ? desc_mnmajor_sw128(b_addr + kk * 2048) : desc_kmajor_sw128(b_addr + kk * 32);
                        mma_bf16(d_tmem, ad, bd, idesc, (k | kk) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);  // frees the smem slot when these MMAs finish
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);  // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
            ROUTER_STAMP(1);
        }
    } else {
        // ===================== epilogue (warps 2..9) =====================
        const uint64_t pol_out = policy_evict_first();  // outputs are not re-read from L2 soon
        const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
        const int half = (warp - 2) >> 2;  // which column slice
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = blockIdx.x; t < t_end; t += gridDim.x) {
            const Tile tl = decode(p, t < n_total ? t : 0, s_off);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) ROUTER_STAMP(2);
            const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
            if constexpr (EPI == EPI_GATE) {
                // both column halves when E_pad splits into 16-column steps, else half 0 alone
                constexpr int NH = (BN % 32 == 0 && kEpiSplit == 2) ? 2 : 1;
                if (half < NH && t < n_total) {
#define HEP_GATE_K(KK) \
    case KK: gate_tile<KK, BN / NH>(p, t_row, tl.row0, tl.rows, row_in_tile, half, NH, s_hist, s_chunk, s_bias, s_merge); break;
                    switch (p.gate.K) {  // the insertion network is unrolled per K
                        HEP_GATE_K(1) HEP_GATE_K(2) HEP_GATE_K(3) HEP_GATE_K(4)
                        HEP_GATE_K(5) HEP_GATE_K(6) HEP_GATE_K(7)
                        default: gate_tile<8, BN / NH>(p, t_row, tl.row0, tl.rows, row_in_tile, half, NH, s_hist, s_chunk, s_bias, s_merge); break;
                    }
#undef HEP_GATE_K
                }
            } else {
                const bool valid = row_in_tile < tl.rows;
                const int64_t grow = (int64_t)tl.row0 + row_in_tile;
                store_tile<BN, EPI>(p, t_row, grow, valid, tl.n_blk, pol_out, tl.expert, tl.kb == 0, half);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_relaxed(&tempty[acc]);
            if (warp == 2 && lane == 0) ROUTER_STAMP(3);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    // multicast B: peers' last commits arrive on this CTA's barriers; nobody exits before them
    if (mc > 1) cluster_sync();
    clk_stamp(p, 1);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, S::TMEM_COLS);
    }
    if constexpr (EPI == EPI_GATE) {
        gate_hist_flush(p.gate, s_hist);
#ifdef HEP_ROUTER_STAMPS
        __syncthreads();
        if (threadIdx.x == 0) ROUTER_STAMP(4);
#endif
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x 256
// tile.  Each CTA TMA-loads its own 128 rows of A and its 128-row half of the
// 256-wide weight tile into its own smem (the bytes complete on the leader's
// barrier); the leader's single MMA thread issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16), whose operands come from both
// CTAs' smem, and each CTA's TMEM receives its 128 accumulator rows.  Weights
// cross L2->SM once per pair instead of once per CTA and the per-CTA stage is
// 32 KB (6 stages).  Commits are multicast to both CTAs; the peer's epilogue
// releases TMEM through a remote arrive on the leader's barrier.
// ---------------------------------------------------------------------------
constexpr int kPairRows = 256;

// Pair-kernel mbarrier wait.  Every consumer of these barriers reads its data through
// the async proxy (TMA -> MMA smem operands, MMA -> tcgen05.ld of TMEM, ordered by the
// tcgen05 fences), so a CTA-scope wait suffices; an .acquire.cluster wait compiles to
// an L1 invalidate (CCTL.IVALL) after every completed wait.
__device__ __forceinline__ void pair_wait(const Params &p, uint64_t *bar, uint32_t parity) {
    if (p.wait_cluster)
        mbar_wait_cluster(bar, parity);
    else
        mbar_wait(bar, parity);
}

template <int STAGES, int BN = 256>
struct Smem2 {
    static constexpr int A_BYTES = 128 * BK * 2;
    static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the B tile
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr size_t BYTES = 1024 + (size_t)STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4) + 16 + kOffBytes;
};

// A_MN / B_MN as in gemm_kernel (the backward GEMMs): an MN-major operand half of 128
// rows is two 64 x 64 boxes per stage, 8 KB apart (the descriptor's LBO).
// BN_ = N of the pair MMA (256; 128 for the router+gate of <= 128 experts): each CTA stages
// BN_ / 2 rows of the B tile.
template <int STAGES, int EPI, bool A_MN = false, bool B_MN = false, int BN_ = 256>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, const Params p) {
    constexpr int BN = BN_;
    constexpr int BH = BN / 2;  // B rows per CTA
    static_assert(BN == 256 || (!A_MN && !B_MN), "MN-major operands: BN = 256 only");
    constexpr uint32_t TMEM_COLS = 2 * BN;
    using S = Smem2<STAGES, BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // align within the array (not through uintptr_t) so s_off etc. stay LDS, not generic loads
    uint8_t *base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sA = base;
    uint8_t *sB = base + STAGES * S::A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(base + STAGES * S::STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    int32_t *s_off = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(tmem_slot) + 16);
    if (p.grouped == 1)
        for (int i = threadIdx.x; i <= p.n_exp; i += blockDim.x) s_off[i] = p.exp_mt_off[i];
    else if (p.grouped == 2 && p.exp_perm)
        for (int i = threadIdx.x; i < p.n_exp; i += blockDim.x) s_off[i] = p.exp_perm[i];

    int32_t *s_hist = s_off + kMaxExpSmem + 4;             // EPI_GATE: as in gemm_kernel
    int32_t *s_chunk = s_hist + kGateMaxSrc * kGateMaxE;
    float *s_bias = reinterpret_cast<float *>(s_chunk + 3 * kGateMaxE);
    uint8_t *s_merge = reinterpret_cast<uint8_t *>(s_bias + kGateMaxE);
    if constexpr (EPI == EPI_GATE) {
        for (int i = threadIdx.x; i < p.gate.n_src * p.gate.E; i += blockDim.x) s_hist[i] = 0;
        for (int i = threadIdx.x; i < BN; i += blockDim.x)  // + 0.0f: -0 -> +0 (see gate_tile)
            s_bias[i] = i >= p.gate.E ? -__int_as_float(0x7f800000) : (p.gate.bias ? p.gate.bias[i] + 0.0f : 0.f);
        gate_hist_zero(p.gate);
    }

    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * kEpiWarps);  // epilogue warps of both CTAs
        }
        fence_barrier_init();
        fence_proxy_async_smem();
    }
    if (warp == 1) tmem_alloc_2sm(tmem_slot, TMEM_COLS);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    clk_stamp(p, 0);

    const int64_t n_total = total_tiles(p);
    const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int kb = p.kblocks;

    if (warp == 0 && p.gather_idx) {
        // ===== TMA producer (both CTAs), A rows gathered by token (the fused permute) =====
        // lane l gathers this CTA's tile rows 4l..4l+3 (tile::gather4 completing on the
        // leader's barrier); lane 0 owns the barrier and the weight half
        const uint64_t pol_a = policy_evict_last();
        const uint64_t pol_b = p.pol_mode ? pick_policy((p.pol_mode >> 2) & 3) : policy_evict_normal();
        const uint32_t full_l = mapa_shared(smem_u32(&full[0]), 0);
        int stage = 0;
        uint32_t phase = 0;
        for (int64_t t = cid; t < n_total; t += ncl) {
            const Tile tl = decode(p, t, s_off);
            const int32_t b_row = (int32_t)(tl.expert * p.b_rows_per_exp + (int64_t)tl.n_blk * BN) + (int32_t)rank * BH;
            int r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int local = (int)rank * 128 + 4 * lane + j;
                r[j] = local < tl.rows ? p.gather_idx[tl.row0 + local] : p.gather_oob;
            }
            const int4 rows = make_int4(r[0], r[1], r[2], r[3]);
            for (int k = 0; k < kb; ++k) {
                if (lane == 0) {
                    pair_wait(p, &empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE_BYTES);
                }
                __syncwarp();
                tma_gather4_2sm(sA + stage * S::A_BYTES + 512 * lane, &tmA, full_l + 8 * stage, k * BK, rows, pol_a);
                if (lane == 0)
                    tma_load_2d_2sm(sB + stage * S::B_BYTES, &tmB, full_l + 8 * stage, k * BK, b_row, pol_b);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            // ===================== TMA producer (both CTAs) =====================
            const uint64_t pol_a = p.pol_mode ? pick_policy(p.pol_mode & 3) : policy_evict_last();
            const uint64_t pol_b = p.pol_mode ? pick_policy((p.pol_mode >> 2) & 3) : policy_evict_last();  // see gemm_kernel
            const uint64_t pol_first = policy_evict_first();
            const uint32_t full_l = mapa_shared(smem_u32(&full[0]), 0);  // leader's full[0]
            int stage = 0;
            uint32_t phase = 0;
            int64_t wave_target = 0;
            for (int64_t t = cid; t < n_total; t += ncl) {
                if (p.wave_ctr && t >= ncl) {
                    // every producer of the grid starts wave w = t / ncl together: arrive once
                    // per wave, wait for the arrivals of every CTA that has a tile in it
                    const int64_t w = t / ncl;
                    const int64_t in_wave = n_total - w * ncl < ncl ? n_total - w * ncl : ncl;
                    wave_target += 2 * in_wave;
                    atomicAdd(p.wave_ctr, 1u);
                    // bounded: the counter only paces the producers, so a CTA that is not
                    // resident (another kernel holds its SM) delays the wave by 200 µs at most
                    const uint64_t t_start = globaltimer_ns();
                    while ((int64_t)ld_acquire_gpu_u32(p.wave_ctr) < wave_target && globaltimer_ns() - t_start < 200000)
                        __nanosleep(64);
                }
                const Tile tl = decode(p, t, s_off);
                const int32_t a_row = tl.row0 + (int32_t)rank * 128;
                const int32_t b_row = (int32_t)(tl.expert * p.b_rows_per_exp + (int64_t)tl.n_blk * BN) + (int32_t)rank * BH;
                // contraction offsets (gemm_kernel's): mode 2 contracts over the expert's rows;
                // an MN-major weight is [K][N] per expert, stacked along K
                const int32_t a_k0 = (int32_t)tl.k0;
                const int32_t b_k0 = p.grouped == 2 ? (int32_t)tl.k0 : (int32_t)(tl.expert * p.b_rows_per_exp);
                const int32_t b_mn = tl.n_blk * BN + (int32_t)rank * 128;
                // an expert with a single m-tile streams its weights once: keep them out of L2's way
                const bool light = p.light_first && p.grouped == 1 && s_off[tl.expert + 1] - s_off[tl.expert] == 1;
                for (int k = 0; k < tl.kb; ++k) {
                    pair_wait(p, &empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE_BYTES);
                    if constexpr (A_MN) {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
                            tma_load_2d_2sm(sA + stage * S::A_BYTES + i * 8192, &tmA, full_l + 8 * stage, a_row + 64 * i,
                                            a_k0 + k * BK, pol_a);
                    } else {
                        tma_load_2d_2sm(sA + stage * S::A_BYTES, &tmA, full_l + 8 * stage, a_k0 + k * BK, a_row, pol_a);
                    }
                    if constexpr (B_MN) {
#pragma unroll
                        for (int i = 0; i < 2; ++i)
                            tma_load_2d_2sm(sB + stage * S::B_BYTES + i * 8192, &tmB, full_l + 8 * stage, b_mn + 64 * i,
                                            b_k0 + k * BK, pol_b);
                    } else {
                        tma_load_2d_2sm(sB + stage * S::B_BYTES, &tmB, full_l + 8 * stage, k * BK, b_row,
                                        light ? pol_first : pol_b);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            // ===================== MMA issuer (leader CTA) =====================
            constexpr uint32_t idesc =
                idesc_bf16_f32(kPairRows, BN) | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = cid; t < n_total; t += ncl) {
                const int tkb = (p.grouped == 2 || p.k_split > 1) ? decode(p, t, s_off).kb : kb;
                pair_wait(p, &tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int k = 0; k < tkb; ++k) {
                    pair_wait(p, &full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(sA + stage * S::A_BYTES);
                    const uint32_t b_addr = smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk) {
                        const uint64_t ad = A_MN ? desc_mnmajor_sw128(a_addr + kk * 2048) : desc_kmajor_sw128(a_addr + kk * 32);
                        const uint64_t bd = B_MN ? desc_mnmajor_sw128(b_addr + kk * 2048) : desc_kmajor_sw128(b_addr + kk * 32);
                        mma_bf16_2sm(d_tmem, ad, bd, idesc, (k | kk) ? 1u : 0u);
                    }
                    mma_commit_2sm_mc(&empty[stage], 0x3);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm_mc(&tfull[acc], 0x3);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue (warps 2..9, both CTAs) =====================
        const uint64_t pol_out = policy_evict_first();
        const uint32_t tempty_l = mapa_shared(smem_u32(&tempty[0]), 0);
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const int row_in_cta = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t t = cid; t < n_total; t += ncl) {
            const Tile tl = decode(p, t, s_off);
            pair_wait(p, &tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t t_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
            const int local_row = (int)rank * 128 + row_in_cta;
            if constexpr (EPI == EPI_GATE) {
                // this CTA's 128 accumulator rows are tokens [row0 + 128 rank, ...): the 1-CTA
                // kernel's gate epilogue on them
                const int sub_rows = tl.rows - (int)rank * 128;
                if (sub_rows > 0) {
                    const int32_t sub0 = tl.row0 + (int32_t)rank * 128;
                    const int nr = sub_rows < 128 ? sub_rows : 128;
                    switch (p.gate.K) {
#define HEP_GATE2_K(KK) \
    case KK: gate_tile<KK, BN / 2>(p, t_row, sub0, nr, row_in_cta, half, 2, s_hist, s_chunk, s_bias, s_merge); break;
                        HEP_GATE2_K(1) HEP_GATE2_K(2) HEP_GATE2_K(3) HEP_GATE2_K(4)
                        HEP_GATE2_K(5) HEP_GATE2_K(6) HEP_GATE2_K(7)
#undef HEP_GATE2_K
                        default: gate_tile<8, BN / 2>(p, t_row, sub0, nr, row_in_cta, half, 2, s_hist, s_chunk, s_bias, s_merge); break;
                    }
                }
            } else {
                store_tile<BN, EPI>(p, t_row, (int64_t)tl.row0 + local_row, local_row < tl.rows, tl.n_blk, pol_out, tl.expert,
                                    tl.kb == 0, half);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(tempty_l + 8 * acc);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    clk_stamp(p, 1);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2sm(tmem_base, TMEM_COLS);
    }
    if constexpr (EPI == EPI_GATE) gate_hist_flush(p.gate, s_hist);
}

// ---------------------------------------------------------------------------
// m-tile list from segments (row_start, rows, expert, dst): expert-major.
// Consecutive segments of one expert that are contiguous in rows are merged
// (the receive layout keeps all replicas of an expert adjacent), so an m-tile
// may span several destination GPUs' rows of the same expert.  One CTA; one
// thread per expert chunk, deterministic block scan.
// ---------------------------------------------------------------------------
// Tiles of expert e: its segments in list order, contiguous ones (next row_start = end
// of the previous) merged into runs, each run cut into tile_rows-row m-tiles.  One warp
// per expert: lanes test 32 segments at a time, matches are merged in list order from
// a ballot (all lanes keep the same run state), tile rows are written lane-parallel.
template <bool WRITE>
__device__ int64_t expert_tiles_warp(const int32_t *seg, int n_seg, int e, int32_t *mt_row0, int32_t *mt_rows,
                                     int64_t pos, int tile_rows, int lane) {
    int64_t cnt = 0;
    int32_t r0 = 0, n = 0;
    bool open = false;
    auto flush = [&]() {
        const int32_t nt = (n + tile_rows - 1) / tile_rows;
        if (WRITE)
            for (int32_t j = lane; j < nt; j += 32) {
                mt_row0[pos + cnt + j] = r0 + j * tile_rows;
                mt_rows[pos + cnt + j] = min(tile_rows, n - j * tile_rows);
            }
        cnt += nt;
    };
    for (int base = 0; base < n_seg; base += 32) {
        const int s = base + lane;
        int32_t a = 0, b = 0;
        bool m = false;
        if (s < n_seg) {
            a = seg[4 * s];
            b = seg[4 * s + 1];
            m = seg[4 * s + 2] == e && b != 0;
        }
        uint32_t mask = __ballot_sync(0xffffffffu, m);
        while (mask) {
            const int l = __ffs(mask) - 1;
            mask &= mask - 1;
            const int32_t sa = __shfl_sync(0xffffffffu, a, l), sb = __shfl_sync(0xffffffffu, b, l);
            if (open && sa == r0 + n) {
                n += sb;
            } else {
                if (open) flush();
                r0 = sa;
                n = sb;
                open = true;
            }
        }
    }
    if (open) flush();
    return cnt;
}

// total rows of expert e over its segments (warp-uniform result)
__device__ int64_t expert_rows_warp(const int32_t *seg, int n_seg, int e, int lane) {
    int64_t n = 0;
    for (int s = lane; s < n_seg; s += 32)
        if (seg[4 * s + 2] == e) n += seg[4 * s + 1];
#pragma unroll
    for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    return n;
}

constexpr int kTileSegSmem = 2048;  // segments staged in shared memory (16 B each)
constexpr int kTileWarps = 8;       // experts per block (one warp each)

__device__ __forceinline__ const int32_t *stage_segments(const int32_t *seg_g, int n_seg, int4 *st) {
    if (n_seg > kTileSegSmem) return seg_g;
    for (int i = threadIdx.x; i < n_seg; i += blockDim.x) st[i] = reinterpret_cast<const int4 *>(seg_g)[i];
    __syncthreads();
    return reinterpret_cast<const int32_t *>(st);
}

// pass 1: m-tiles per expert (one warp per expert, experts spread over blocks/SMs)
__global__ void __launch_bounds__(32 * kTileWarps) tile_count_kernel(const int32_t *seg_g, int n_seg, int n_exp,
                                                                     int32_t *exp_cnt, int tile_rows, int light_max,
                                                                     int light_sel) {
    extern __shared__ int4 st[];
    const int32_t *seg = stage_segments(seg_g, n_seg, st);
    const int lane = threadIdx.x & 31, e = blockIdx.x * kTileWarps + (threadIdx.x >> 5);
    if (e >= n_exp) return;
    // light_max > 0: this list holds only the experts with (rows <= light_max) == light_sel
    const bool keep = light_max <= 0 || ((expert_rows_warp(seg, n_seg, e, lane) <= light_max) == (light_sel != 0));
    const int64_t c = keep ? expert_tiles_warp<false>(seg, n_seg, e, nullptr, nullptr, 0, tile_rows, lane) : 0;
    if (lane == 0) exp_cnt[e] = (int32_t)c;
}

// pass 2: every block scans the per-expert counts (n_exp <= 1024) and writes its experts'
// m-tiles at their offsets; block 0 publishes the offsets.
__global__ void __launch_bounds__(32 * kTileWarps) tile_write_kernel(const int32_t *seg_g, int n_seg, int n_exp,
                                                                     const int32_t *exp_cnt, int32_t *mt_row0,
                                                                     int32_t *mt_rows, int32_t *exp_mt_off,
                                                                     int64_t cap, int32_t *status, int tile_rows,
                                                                     unsigned int *zero2) {
    extern __shared__ int4 st[];
    if (zero2 && blockIdx.x == 0 && threadIdx.x < 8) zero2[threadIdx.x] = 0u;  // the expert GEMMs' wave counters
    __shared__ int64_t scan[64];
    __shared__ int64_t off_sm[kTileWarps];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, w = tid >> 5;
    const int e_first = blockIdx.x * kTileWarps;
    const int chunk = (n_exp + nt - 1) / nt;
    const int e0 = min(n_exp, tid * chunk), e1 = min(n_exp, e0 + chunk);
    int64_t mine = 0;
    for (int e = e0; e < e1; ++e) mine += exp_cnt[e];
    int64_t total;
    int64_t pos = block_excl_scan_i64(mine, scan, &total);
    for (int e = e0; e < e1; ++e) {
        if (e >= e_first && e < e_first + kTileWarps) off_sm[e - e_first] = pos;
        if (blockIdx.x == 0 && total <= cap) exp_mt_off[e] = (int32_t)pos;
        pos += exp_cnt[e];
    }
    if (total > cap) {
        if (blockIdx.x == 0 && tid == 0 && status) atomicCAS(status, 0, HEP_E_CAPACITY);
        if (blockIdx.x == 0)
            for (int e = tid; e <= n_exp; e += nt) exp_mt_off[e] = 0;
        return;
    }
    if (blockIdx.x == 0 && tid == 0) exp_mt_off[n_exp] = (int32_t)total;
    __syncthreads();  // off_sm (stage_segments only synchronises when it stages)
    const int32_t *seg = stage_segments(seg_g, n_seg, st);
    const int e = e_first + w;
    if (e < n_exp && exp_cnt[e] > 0) expert_tiles_warp<true>(seg, n_seg, e, mt_row0, mt_rows, off_sm[w], tile_rows, lane);
}

// build the device m-tile list of a grouped GEMM from its segments (2 launches)
static int build_tiles(const int32_t *d_seg, int n_seg, int n_exp, int32_t *mt_row0, int32_t *mt_rows,
                       int32_t *exp_off, int32_t *exp_cnt, int64_t cap, int32_t *d_status, int tile_rows,
                       cudaStream_t s, int light_max = 0, int light_sel = 0, unsigned int *wave_ctr = nullptr) {
    const size_t sm = n_seg <= kTileSegSmem ? 16 * (size_t)n_seg : 0;
    const int blocks = n_exp > 0 ? (n_exp + kTileWarps - 1) / kTileWarps : 1;
    tile_count_kernel<<<blocks, 32 * kTileWarps, sm, s>>>(d_seg, n_seg, n_exp, exp_cnt, tile_rows, light_max,
                                                          light_sel);
    HEP_CHECK_LAUNCH();
    tile_write_kernel<<<blocks, 32 * kTileWarps, sm, s>>>(d_seg, n_seg, n_exp, exp_cnt, mt_row0, mt_rows, exp_off, cap,
                                                          d_status, tile_rows, wave_ctr);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// 2D bf16 row-major [rows][cols] tensor, box [box_rows][64], 128B swizzle
static int make_tmap(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
    auto fn = encode_fn();
    HEP_REQUIRE(fn, HEP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    HEP_REQUIRE(((uintptr_t)ptr & 15) == 0 && (cols * 2) % 16 == 0, HEP_E_CONTRACT,
                "TMA needs 16-byte aligned base and row pitch");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HEP_REQUIRE(r == CUDA_SUCCESS, HEP_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return HEP_OK;
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// MN-major operand: global [k_rows][mn_cols] bf16 (mn contiguous), 64 x 64 boxes
static int make_tmap_mn(CUtensorMap *m, const void *ptr, uint64_t k_rows, uint64_t mn_cols) {
    auto fn = encode_fn();
    HEP_REQUIRE(fn, HEP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    HEP_REQUIRE(((uintptr_t)ptr & 15) == 0 && (mn_cols * 2) % 16 == 0, HEP_E_CONTRACT,
                "TMA needs 16-byte aligned base and row pitch");
    cuuint64_t dims[2] = {mn_cols, k_rows};
    cuuint64_t strides[1] = {mn_cols * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HEP_REQUIRE(r == CUDA_SUCCESS, HEP_E_CUDA, "cuTensorMapEncodeTiled (MN-major) failed (%d)", (int)r);
    return HEP_OK;
}

// 256-bit epilogue stores when every output row (and the training pre-activation
// rows) starts 32-B aligned; peer-row (NVLink) destinations keep 16-B stores.
// hep_tuning.st256 = 0 disables.
template <int EPI>
static Params with_store_width(const Params &p0) {
    Params p = p0;
    const int64_t esz = (EPI == EPI_F32) ? 4 : 2;
    auto al = [](const void *q, int64_t stride_bytes) {
        return q == nullptr || (reinterpret_cast<uintptr_t>(q) % 32 == 0 && stride_bytes % 32 == 0);
    };
    p.st256 = g_tuning.st256 != 0 && EPI != EPI_GATE && p.row_addr == nullptr && p.out != nullptr &&
              al(p.out, p.ld_out * esz) && (EPI != EPI_F32 || (p.out_exp_stride * esz) % 32 == 0) &&
              al(p.aux, p.ld_aux * 2);
    return p;
}

template <int BN, int STAGES, int EPI, bool A_MN, bool B_MN>
static int launch_maps(const CUtensorMap &ta, const CUtensorMap &tb, const Params &p0, int64_t max_tiles,
                       cudaStream_t stream) {
    using S = Smem<BN, STAGES>;
    Params p = with_store_width<EPI>(p0);
    if (g_tuning.pair_wave_sync <= 0 || p.kblocks < g_tuning.pair_wave_sync || p.grouped != 1 || p.gather_idx ||
        g_tuning.light_wave_sync == 0)
        p.wave_ctr = nullptr;
    auto kern = gemm_kernel<BN, STAGES, EPI, A_MN, B_MN>;
    HEP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES));
    int grid = sm_count();
    if (max_tiles > 0 && max_tiles < grid) grid = (int)max_tiles;
    if (grid < 1) grid = 1;
    kern<<<grid, kThreads, S::BYTES, stream>>>(ta, tb, p);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

template <int BN, int STAGES, int EPI>
static int launch(const void *A, int64_t a_rows, int64_t K, const void *B, int64_t b_rows, const Params &p,
                  int64_t max_tiles, cudaStream_t stream) {
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, A, (uint64_t)a_rows, (uint64_t)K, p.gather_idx ? 1 : BM);  // gather: {64, 1} rows
    if (rc) return rc;
    rc = make_tmap(&tb, B, (uint64_t)b_rows, (uint64_t)K, BN);
    if (rc) return rc;
    return launch_maps<BN, STAGES, EPI, false, false>(ta, tb, p, max_tiles, stream);
}

template <int STAGES, int EPI, bool A_MN, bool B_MN>
static int launch2sm_maps(const CUtensorMap &ta, const CUtensorMap &tb, const Params &p0, cudaStream_t stream) {
    using S = Smem2<STAGES>;
    Params p = with_store_width<EPI>(p0);
    p.wait_cluster = g_tuning.pair_wait_cluster == 1;
    // wave-synchronised producers only for long tiles (hep_tuning.pair_wave_sync k-blocks)
    // (grouped == 2, the K-ragged weight gradients: only when the caller set the counter,
    // hep_tuning.wgrad_wave_sync)
    if (p.grouped != 2 &&
        (g_tuning.pair_wave_sync <= 0 || p.kblocks < g_tuning.pair_wave_sync || p.grouped != 1 || p.gather_idx))
        p.wave_ctr = nullptr;
    auto kern = gemm2sm_kernel<STAGES, EPI, A_MN, B_MN>;
    HEP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES));
    const int grid = sm_count() & ~1;
    kern<<<grid, kThreads, S::BYTES, stream>>>(ta, tb, p);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

template <int STAGES, int EPI>
static int launch2sm(const void *A, int64_t a_rows, int64_t K, const void *B, int64_t b_rows, const Params &p,
                     cudaStream_t stream) {
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, A, (uint64_t)a_rows, (uint64_t)K, p.gather_idx ? 1 : 128);  // gather: {64, 1} rows
    if (rc) return rc;
    rc = make_tmap(&tb, B, (uint64_t)b_rows, (uint64_t)K, 128);
    if (rc) return rc;
    return launch2sm_maps<STAGES, EPI, false, false>(ta, tb, p, stream);
}

// CTA pairs unless experts carry so few rows that 256-row tiles waste more than
// the pair's halved operand traffic saves: measured in-process (tools/ffn_ab.py,
// profiles/r01/ffn_ab_r01d.txt) the pair wins at 512 rows per expert (DeepSeek-V3
// shape) and above.  hep_tuning.ffn_pair = 0 / 1 forces it.
static bool use_pairs(int64_t R, int n_experts) {
    if (g_tuning.ffn_pair == 0 || g_tuning.ffn_pair == 1) return g_tuning.ffn_pair == 1;
    return n_experts > 0 && R / n_experts >= 512;
}

}  // namespace gemm
}  // namespace hep

using namespace hep;
using namespace hep::gemm;

extern "C" int hep_gemm_bf16(const void *d_A, const void *d_B, void *d_D, int64_t M, int64_t N, int64_t K, int out_kind,
                             void *stream) {
    HEP_NVTX("hep_gemm_bf16");
    HEP_REQUIRE(d_A && d_B && d_D, HEP_E_CONTRACT, "hep_gemm_bf16: null pointer");
    HEP_REQUIRE(M > 0 && N > 0 && K > 0 && K % BK == 0, HEP_E_DIMENSION, "hep_gemm_bf16: need K %% 64 == 0 (K=%lld)",
                (long long)K);
    Params p{};
    p.grouped = 0;
    p.M = M;
    p.kblocks = (int)(K / BK);
    p.b_rows_per_exp = 0;
    p.out = d_D;
    p.ld_out = N;
    p.out_cols = N;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t mt = (M + BM - 1) / BM;
    if (out_kind == HEP_OUT_F32) {
        HEP_REQUIRE(N % 16 == 0, HEP_E_DIMENSION, "fp32 GEMM needs N %% 16 == 0");
        int bn = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
        p.n_tiles = (int)((N + bn - 1) / bn);
        HEP_REQUIRE(N <= 256 || N % 256 == 0, HEP_E_DIMENSION, "fp32 GEMM: N=%lld", (long long)N);
        switch (bn) {
            case 16: return launch<16, 8, EPI_F32>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
            case 32: return launch<32, 8, EPI_F32>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
            case 64: return launch<64, 6, EPI_F32>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
            case 128: return launch<128, 5, EPI_F32>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
            default: return launch<256, 4, EPI_F32>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
        }
    }
    HEP_REQUIRE(N % 256 == 0, HEP_E_DIMENSION, "bf16 GEMM needs N %% 256 == 0");
    p.n_tiles = (int)(N / 256);
    return launch<256, 4, EPI_BF16>(d_A, M, K, d_B, N, p, mt * p.n_tiles, s);
}

#ifndef HEP_ROUTER_STAGES_128
#define HEP_ROUTER_STAGES_128 5  // TMA ring depth of the 128-expert router+gate (diagnostics builds vary it)
#endif

// Router tile height (hep_tuning.router_tile_rows, multiple of 16, <= 128; 0 = 128).  Shorter
// tiles that fill every SM (16384 tokens: 147 tiles of 112 rows instead of 128 of 128) were
// measured SLOWER (Mixtral 31.1 vs 28.7 us, Qwen3 48.7 vs 47.4, DSv3 75.5 vs 72.0,
// profiles/r02/router_ab_r02c.txt): the kernel's time is one tile's DRAM-bound mainloop plus
// its exposed gate epilogue, both per CTA, and the epilogue costs the same for a short tile
// (every TMEM lane runs the scan), so the 128-row tiling stays the default.
static int router_tile_rows(int64_t T) {
    (void)T;
    if (g_tuning.router_tile_rows > 0) return g_tuning.router_tile_rows < BM ? (g_tuning.router_tile_rows + 15) / 16 * 16 : BM;
    return BM;
}

template <int BN, int STAGES>
static int launch_gate(const void *x, const void *wg, int64_t T, int64_t d_model, int e_pad, const Params &p,
                       cudaStream_t s) {
    using S = Smem<BN, STAGES>;
    static_assert(S::BYTES + kGateSmemBytes <= 232448, "router+gate kernel shared memory");
    CUtensorMap ta, tb;
    const int tm = p.tile_m > 0 ? p.tile_m : BM;
    // Wg multicast cluster size (hep_tuning.router_mc; 0 = auto): the B tile is split into
    // mc slices of BN / mc rows, each a whole number of 8-row swizzle atoms
    int mc = g_tuning.router_mc > 0 ? g_tuning.router_mc : 1;  // auto: off (measured slower, router_ab_r02i)
    if (mc != 2 && mc != 4) mc = 1;
    while (mc > 1 && BN / mc < 8) mc >>= 1;
    int rc = make_tmap(&ta, x, (uint64_t)T, (uint64_t)d_model, (uint32_t)tm);
    if (rc) return rc;
    rc = make_tmap(&tb, wg, (uint64_t)e_pad, (uint64_t)d_model, (uint32_t)(BN / mc));  // rows past e_pad: zero fill
    if (rc) return rc;
    auto kern = gemm_kernel<BN, STAGES, EPI_GATE>;
    const int bytes = (int)S::BYTES + kGateSmemBytes;
    HEP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int64_t tiles = (T + tm - 1) / tm;
    int grid = (int)(tiles < sm_count() ? tiles : sm_count());
    Params q = p;
    q.b_mc = mc;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = s;
    if (mc > 1) {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = mc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // whole clusters, no more than can be co-resident (a cluster lives on one GPC)
        static int max_clusters[5] = {};  // per <BN, STAGES> instance
        int &mcl = max_clusters[mc];
        if (mcl == 0) {
            cfg.gridDim = dim3((unsigned)(sm_count() / mc * mc));
            HEP_CHECK_CUDA(cudaOccupancyMaxActiveClusters(&mcl, (void *)kern, &cfg));
            if (mcl < 1) mcl = 1;
        }
        const int64_t want = (tiles + mc - 1) / mc;
        grid = (int)(want < mcl ? want : mcl) * mc;
    }
    cfg.gridDim = dim3((unsigned)grid);
    HEP_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, q));
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

// Router+gate on CTA pairs (cta_group::2, M = 256 tokens per pair): each CTA stages its 128
// token rows and HALF of the Wg tile, so a stage is 16 KB + BN * 64 B instead of 16 KB +
// BN * 128 B and the ring keeps 1.5x (BN = 256) / 1.6x (BN = 128) more token bytes in
// flight per SM; each CTA's TMEM holds its 128 tokens x BN logits and runs the same gate
// epilogue.  hep_tuning.router_pair: 0 auto (E_pad > 64), 1 off, 2 on.
template <int BN, int STAGES>
static int launch_gate2(const void *x, const void *wg, int64_t T, int64_t d_model, int e_pad, const Params &p0,
                        cudaStream_t s) {
    using S = Smem2<STAGES, BN>;
    static_assert(S::BYTES + kGateSmemBytes <= 232448, "pair router+gate kernel shared memory");
    CUtensorMap ta, tb;
    int rc = make_tmap(&ta, x, (uint64_t)T, (uint64_t)d_model, 128);
    if (rc) return rc;
    rc = make_tmap(&tb, wg, (uint64_t)e_pad, (uint64_t)d_model, BN / 2);  // rows past e_pad: TMA zero fill
    if (rc) return rc;
    Params p = p0;
    p.tile_m = kPairRows;
    p.wait_cluster = g_tuning.pair_wait_cluster == 1;
    auto kern = gemm2sm_kernel<STAGES, EPI_GATE, false, false, BN>;
    const int bytes = (int)S::BYTES + kGateSmemBytes;
    HEP_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int64_t tiles = (T + kPairRows - 1) / kPairRows;
    const int64_t pairs = sm_count() / 2;
    const int grid = 2 * (int)(tiles < pairs ? tiles : pairs);
    kern<<<grid, kThreads, bytes, s>>>(ta, tb, p);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_gate_chunk_counts(const int32_t *d_topk_idx, int64_t T, int K, int E, int64_t tokens_per_src,
                                     int n_src, int32_t *d_chunk_cnt, void *stream);

#ifdef HEP_ROUTER_STAMPS
extern "C" int hep_diag_router_stamps(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, hep::gemm::g_router_stamps, sizeof(hep::gemm::g_router_stamps)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int hep_router_topk_ws(const void *d_x, const void *d_wg, int64_t T, int64_t d_model, int E, int e_pad,
                                  const float *d_bias, int K, int64_t tokens_per_src, int n_src, float *d_logits,
                                  int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist, int32_t *d_chunk_cnt,
                                  unsigned int *d_sync, void *stream);

extern "C" int hep_router_topk(const void *d_x, const void *d_wg, int64_t T, int64_t d_model, int E, int e_pad,
                               const float *d_bias, int K, int64_t tokens_per_src, int n_src, float *d_logits,
                               int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist, int32_t *d_chunk_cnt,
                               void *stream) {
    return hep_router_topk_ws(d_x, d_wg, T, d_model, E, e_pad, d_bias, K, tokens_per_src, n_src, d_logits, d_topk_idx,
                              d_topk_w, d_hist, d_chunk_cnt, nullptr, stream);
}

extern "C" size_t hep_router_sync_bytes(void) { return 16; }

extern "C" int hep_router_topk_ws(const void *d_x, const void *d_wg, int64_t T, int64_t d_model, int E, int e_pad,
                                  const float *d_bias, int K, int64_t tokens_per_src, int n_src, float *d_logits,
                                  int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist, int32_t *d_chunk_cnt,
                                  unsigned int *d_sync, void *stream) {
    HEP_NVTX("hep_router_topk");
    HEP_REQUIRE(d_x && d_wg && d_topk_idx && d_topk_w && d_hist, HEP_E_CONTRACT, "hep_router_topk: null pointer");
    HEP_REQUIRE(E >= 1 && K >= 1 && K <= E && e_pad >= E && e_pad % 16 == 0 && d_model % BK == 0, HEP_E_DIMENSION,
                "hep_router_topk: E=%d e_pad=%d K=%d d=%lld", E, e_pad, K, (long long)d_model);
    HEP_REQUIRE(tokens_per_src >= 1 && n_src >= 1 && tokens_per_src * n_src >= T, HEP_E_DIMENSION,
                "hep_router_topk: tokens_per_src * n_src < T");
    cudaStream_t s = (cudaStream_t)stream;
    const bool fused = e_pad <= kGateMaxE && K <= kGateMaxK && n_src <= kGateMaxSrc;
    if (!fused) {  // unfused: logits through HBM, then the gate kernel (both still on the device)
        HEP_REQUIRE(d_logits, HEP_E_CONTRACT, "hep_router_topk: E_pad > 256 / K > 8 needs d_logits");
        int rc = hep_gemm_bf16(d_x, d_wg, d_logits, T, e_pad, d_model, HEP_OUT_F32, stream);
        if (rc) return rc;
        rc = hep_gate_topk(d_logits, e_pad, d_bias, T, E, K, tokens_per_src, n_src, d_topk_idx, d_topk_w, d_hist, stream);
        if (rc || !d_chunk_cnt) return rc;
        return hep_gate_chunk_counts(d_topk_idx, T, K, E, tokens_per_src, n_src, d_chunk_cnt, stream);
    }
    // the fused kernel zeroes hist itself when given the sync words (and tokens to launch for)
    const bool zero_in_kernel = d_sync != nullptr && T > 0;
    if (!zero_in_kernel) HEP_CHECK_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(int64_t) * (size_t)n_src * E, s));
    if (T <= 0) return HEP_OK;
    // chunk counts come out of the epilogue when every 64-token chunk lies inside one tile
    const bool chunks_fused = d_chunk_cnt && tokens_per_src % 64 == 0 && tokens_per_src * n_src == T;
    Params p{};
    p.grouped = 0;
    p.M = T;
    p.kblocks = (int)(d_model / BK);
    p.n_tiles = 1;
    p.out = d_logits;
    p.ld_out = e_pad;
    p.out_cols = e_pad;
    p.gate.bias = d_bias;
    p.gate.K = K;
    p.gate.E = E;
    p.gate.tps = tokens_per_src;
    p.gate.n_src = n_src;
    p.gate.ncs = (int)((tokens_per_src + 63) / 64);
    p.gate.topk_idx = d_topk_idx;
    p.gate.topk_w = d_topk_w;
    p.gate.hist = d_hist;
    p.gate.chunk_cnt = chunks_fused ? d_chunk_cnt : nullptr;
    p.gate.sync = zero_in_kernel ? d_sync : nullptr;
    const int tm = router_tile_rows(T);
    if (tm < BM) {
        p.tile_m = tm;
        p.a_box_rows = tm;
        // tiles no longer hold whole 64-token chunks: the epilogue adds its chunk counts
        // with integer atomics (order-free) into zeroed counters
        if (chunks_fused && tm % 64 != 0)
            HEP_CHECK_CUDA(cudaMemsetAsync(d_chunk_cnt, 0, sizeof(int32_t) * (size_t)n_src * p.gate.ncs * E, s));
    }
    int rc;
    const bool pair = tm == BM && e_pad > 64 && (g_tuning.router_pair == 2 || (g_tuning.router_pair == 0 && e_pad > 128));
    if (pair && e_pad <= 128) rc = launch_gate2<128, 8>(d_x, d_wg, T, d_model, e_pad, p, s);
    else if (pair) rc = launch_gate2<256, 6>(d_x, d_wg, T, d_model, e_pad, p, s);
    else if (e_pad <= 16) rc = launch_gate<16, 8>(d_x, d_wg, T, d_model, e_pad, p, s);
    else if (e_pad <= 32) rc = launch_gate<32, 8>(d_x, d_wg, T, d_model, e_pad, p, s);
    else if (e_pad <= 64) rc = launch_gate<64, 6>(d_x, d_wg, T, d_model, e_pad, p, s);
    else if (e_pad <= 128) rc = launch_gate<128, HEP_ROUTER_STAGES_128>(d_x, d_wg, T, d_model, e_pad, p, s);
    else rc = launch_gate<256, 4>(d_x, d_wg, T, d_model, e_pad, p, s);
    if (rc || !d_chunk_cnt || chunks_fused) return rc;
    return hep_gate_chunk_counts(d_topk_idx, T, K, E, tokens_per_src, n_src, d_chunk_cnt, stream);
}

extern "C" size_t hep_moe_ffn_workspace(int n_seg, int64_t R, int n_experts) {
    const int64_t cap = R / BM + n_seg + 1;
    // two tile lists (CTA-pair tiles of the heavy experts, 1-CTA tiles of the light ones),
    // each: m-tile rows / sizes [cap] x2, expert tile offsets [E+1], per-expert tile counts [E+1]
    // + the weight-gradient expert order [E]; the 64-byte tail holds the forward pair GEMMs'
    // two wave counters (ffn_wave_ctr)
    return (2 * (size_t)(2 * cap + 2 * (int64_t)n_experts + 2) + (size_t)n_experts) * sizeof(int32_t) + 64;
}

static unsigned int *ffn_wave_ctr(void *ws, int64_t cap, int n_experts) {
    return reinterpret_cast<unsigned int *>(ws) + 2 * (2 * cap + 2 * (int64_t)n_experts + 2) + n_experts;
}

static int expert_ffn_fwd(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg, int n_seg,
                          int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h, void *d_y, void *d_pre,
                          void *d_workspace, size_t workspace_bytes, int32_t *d_status, void *stream,
                          const uint64_t *d_y_addr = nullptr, int64_t rows_hint = -1, const int32_t *d_row_tok = nullptr,
                          int64_t T = 0);

// heavy/light split of the forward FFN (see expert_ffn_fwd): light_max rows or 0
static int ffn_light_max(int64_t R, int n_experts, bool gather) {
    // experts up to one pair tile (256 rows) run as 128-row tiles: DeepSeek-V3 shape FFN
    // 14.18 -> 12.95 ms (threshold 128: 13.08) (profiles/r01/ab_light_r01k.txt).  Only when
    // experts average under 1024 rows (many light experts): at the Qwen3 shape (2048 rows
    // per expert, a few dozen light ones) the two extra GEMM launches cost more than the
    // half-empty pair tiles, 1.95 -> 1.88 ms without the split (profiles/r02/ab_light_r02l.txt)
    return (use_pairs(R, n_experts) && n_experts >= 32 && !gather && R < 1024 * (int64_t)n_experts)
               ? g_tuning.ffn_light_rows
               : 0;
}

extern "C" int hep_moe_ffn_launches(int64_t R, int n_experts, int gather) {
    return ffn_light_max(R, n_experts, gather != 0) > 0 ? 8 : 4;
}

extern "C" int hep_moe_ffn_bwd_launches(int64_t Rcap, int n_experts) {
    // zero padding x2, tile list x2, 4 GEMMs, weight-gradient expert order; + tile list x2
    // and 2 dgrad GEMMs when split
    const int order = g_tuning.wgrad_order != 0 ? 1 : 0;
    return (ffn_light_max(Rcap, n_experts, false) > 0 ? 12 : 8) + order;
}

extern "C" int hep_moe_expert_ffn_gather(const void *d_x, int64_t T, const int32_t *d_row_tok, const void *d_w13,
                                         const void *d_w2, const int32_t *d_seg, int n_seg, int64_t R, int64_t d_model,
                                         int64_t ffn, int n_experts, void *d_h, void *d_y, void *d_workspace,
                                         size_t workspace_bytes, int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_expert_ffn_gather");
    HEP_REQUIRE(d_x && d_row_tok, HEP_E_CONTRACT, "hep_moe_expert_ffn_gather: null pointer");
    HEP_REQUIRE(T > 0 && T < ((int64_t)1 << 31), HEP_E_DIMENSION, "hep_moe_expert_ffn_gather: T=%lld", (long long)T);
    return expert_ffn_fwd(d_x, d_w13, d_w2, d_seg, n_seg, R, d_model, ffn, n_experts, d_h, d_y, nullptr, d_workspace,
                          workspace_bytes, d_status, stream, nullptr, -1, d_row_tok, T);
}

extern "C" int hep_moe_expert_ffn_p2p(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg,
                                      int n_seg, int64_t R, int64_t rows_hint, int64_t d_model, int64_t ffn,
                                      int n_experts, void *d_h, const uint64_t *d_y_addr, void *d_workspace,
                                      size_t workspace_bytes, int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_expert_ffn_p2p");
    HEP_REQUIRE(d_y_addr, HEP_E_CONTRACT, "hep_moe_expert_ffn_p2p: d_y_addr required");
    return expert_ffn_fwd(d_rows, d_w13, d_w2, d_seg, n_seg, R, d_model, ffn, n_experts, d_h, (void *)d_y_addr,
                          nullptr, d_workspace, workspace_bytes, d_status, stream, d_y_addr, rows_hint);
}

extern "C" int hep_moe_expert_ffn(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg,
                                  int n_seg, int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h,
                                  void *d_y, void *d_workspace, size_t workspace_bytes, int32_t *d_status,
                                  void *stream) {
    HEP_NVTX("hep_moe_expert_ffn");
    return expert_ffn_fwd(d_rows, d_w13, d_w2, d_seg, n_seg, R, d_model, ffn, n_experts, d_h, d_y, nullptr,
                          d_workspace, workspace_bytes, d_status, stream);
}

extern "C" int hep_moe_expert_ffn_train(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg,
                                        int n_seg, int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h,
                                        void *d_y, void *d_pre, void *d_workspace, size_t workspace_bytes,
                                        int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_expert_ffn_train");
    HEP_REQUIRE(d_pre, HEP_E_CONTRACT, "hep_moe_expert_ffn_train: d_pre required");
    return expert_ffn_fwd(d_rows, d_w13, d_w2, d_seg, n_seg, R, d_model, ffn, n_experts, d_h, d_y, d_pre, d_workspace,
                          workspace_bytes, d_status, stream);
}

static int expert_ffn_fwd(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg, int n_seg,
                          int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h, void *d_y, void *d_pre,
                          void *d_workspace, size_t workspace_bytes, int32_t *d_status, void *stream,
                          const uint64_t *d_y_addr, int64_t rows_hint, const int32_t *d_row_tok, int64_t T) {
    HEP_REQUIRE(d_rows && d_w13 && d_w2 && d_seg && d_h && d_y && d_workspace, HEP_E_CONTRACT,
                "hep_moe_expert_ffn: null pointer");
    HEP_REQUIRE(d_model % 256 == 0 && ffn % 128 == 0 && d_model % BK == 0, HEP_E_DIMENSION,
                "expert FFN needs d_model %% 256 == 0 and ffn %% 128 == 0 (d=%lld F=%lld)", (long long)d_model,
                (long long)ffn);
    HEP_REQUIRE(workspace_bytes >= hep_moe_ffn_workspace(n_seg, R, n_experts), HEP_E_CAPACITY, "workspace too small");
    HEP_REQUIRE(n_experts <= kMaxExpSmem, HEP_E_CAPACITY, "expert FFN: at most %d experts (slots)", kMaxExpSmem);
    if (R <= 0) return HEP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cap = R / BM + n_seg + 1;
    int32_t *mt_row0 = reinterpret_cast<int32_t *>(d_workspace);
    int32_t *mt_rows = mt_row0 + cap;
    int32_t *exp_off = mt_rows + cap;
    const bool pairs = use_pairs(rows_hint >= 0 ? rows_hint : R, n_experts);
    const int pol_mode = g_tuning.l2_policy;
    // Light experts (<= light_max rows: one 128-row tile) leave the CTA-pair kernel, whose
    // 256-row tiles would issue twice their useful MMA work, for a second launch of the
    // 1-CTA kernel on their own tile list.  Only with many experts (HEP_FFN_LIGHT_ROWS,
    // hep_tuning.ffn_light_rows, 0 disables; the gather variant keeps one list).
    const int light_max = ffn_light_max(rows_hint >= 0 ? rows_hint : R, n_experts, d_row_tok != nullptr);
    int32_t *mt_row0_l = exp_off + 2 * (n_experts + 1);
    int32_t *mt_rows_l = mt_row0_l + cap;
    int32_t *exp_off_l = mt_rows_l + cap;
    unsigned int *wave_ctr = ffn_wave_ctr(d_workspace, cap, n_experts);
    int rc0 = build_tiles(d_seg, n_seg, n_experts, mt_row0, mt_rows, exp_off, exp_off + n_experts + 1, cap, d_status,
                          pairs ? kPairRows : BM, s, light_max, 0, wave_ctr);
    if (rc0) return rc0;
    if (light_max > 0) {
        rc0 = build_tiles(d_seg, n_seg, n_experts, mt_row0_l, mt_rows_l, exp_off_l, exp_off_l + n_experts + 1, cap,
                          d_status, BM, s, light_max, 1);
        if (rc0) return rc0;
    }
    auto light_list = [&](Params q) {
        q.mt_row0 = mt_row0_l;
        q.mt_rows = mt_rows_l;
        q.exp_mt_off = exp_off_l;
        q.clk_slot = 0;
        q.wave_ctr = q.wave_ctr ? q.wave_ctr + 2 : nullptr;  // counters 2 / 3: the light GEMMs
        return q;
    };
    Params p{};
    p.grouped = 1;
    p.pol_mode = pol_mode;
    // experts whose rows fit one m-tile stream their weights exactly once: load them
    // evict-first so they do not push the reused panels of the other experts out of L2
    // (DeepSeek-V3 shape 13.36 -> 12.87 ms, Qwen3 2.06 -> 2.00 ms; hep_tuning.light_first = 0 disables)
    p.light_first = g_tuning.light_first;
    const bool clk = g_tuning.ffn_clock == 1;
    p.clk_slot = clk ? 1 : 0;
    // raster bands (m-tiles swept across all N-blocks before the next band): 16 for the
    // SwiGLU GEMM, 8 for the down projection (profiles/r01/raster*.txt)
    p.raster_gm = g_tuning.raster_gm1;
    p.mt_row0 = mt_row0;
    p.mt_rows = mt_rows;
    p.exp_mt_off = exp_off;
    p.n_exp = n_experts;
    // GEMM 1: H = silu(X W1^T) * (X W3^T), B = W13 [E][2F][d]
    p.kblocks = (int)(d_model / BK);
    p.n_tiles = (int)(2 * ffn / 256);
    p.b_rows_per_exp = 2 * ffn;
    p.out = d_h;
    p.ld_out = ffn;
    p.out_cols = ffn;
    p.aux = d_pre;  // training: store the pre-activations A13 (W13 interleave)
    p.ld_aux = 2 * ffn;
    // fused permute: A = x [T][d] gathered through row_tok instead of the permuted rows
    p.gather_idx = d_row_tok;
    p.gather_oob = (int32_t)T;
    const int64_t a_rows = d_row_tok ? T : R;
    p.wave_ctr = wave_ctr;
    int rc = pairs ? launch2sm<6, EPI_SWIGLU>(d_rows, a_rows, d_model, d_w13, (int64_t)n_experts * 2 * ffn, p, s)
                   : launch<256, 4, EPI_SWIGLU>(d_rows, a_rows, d_model, d_w13, (int64_t)n_experts * 2 * ffn, p, 0, s);
    if (rc) return rc;
    if (light_max > 0 &&
        (rc = launch<256, 4, EPI_SWIGLU>(d_rows, a_rows, d_model, d_w13, (int64_t)n_experts * 2 * ffn, light_list(p), 0,
                                         s)))
        return rc;
    // GEMM 2: Y = H W2^T, B = W2 [E][d][F]
    p.aux = nullptr;
    p.gather_idx = nullptr;
    p.clk_slot = clk ? 2 : 0;
    p.row_addr = d_y_addr;
    p.raster_gm = g_tuning.raster_gm2;
    p.wave_ctr = wave_ctr + 1;
    p.kblocks = (int)(ffn / BK);
    p.n_tiles = (int)(d_model / 256);
    p.b_rows_per_exp = d_model;
    p.out = d_y;
    p.ld_out = d_model;
    p.out_cols = d_model;
    rc = pairs ? launch2sm<6, EPI_BF16>(d_h, R, ffn, d_w2, (int64_t)n_experts * d_model, p, s)
               : launch<256, 4, EPI_BF16>(d_h, R, ffn, d_w2, (int64_t)n_experts * d_model, p, 0, s);
    if (rc || light_max <= 0) return rc;
    return launch<256, 4, EPI_BF16>(d_h, R, ffn, d_w2, (int64_t)n_experts * d_model, light_list(p), 0, s);
}

// ===========================================================================
// Backward of the expert FFN (training).  Layout as in the forward; the receive
// rows are in 64-row aligned expert blocks (hep_moe_assign row_align = 64) and
// the forward kept the pre-activations A13 = [x W1^T | x W3^T] (W13 interleave).
//   dA13    = swiglu'(A13) * (dY W2)      dgrad GEMM, W2 MN-major, fused epilogue
//   dX_rows = dA13 W13                    dgrad GEMM, W13 MN-major
//   dW2_e   = dY_e^T H_e                  wgrad GEMM, both operands MN-major, K = the
//   dW13_e  = dA13_e^T X_e                expert's rows (K-ragged per expert)
// ===========================================================================
// Weight-gradient visit order: experts by descending row count (ties: lower id first),
// so the long-K tiles of the heavy experts all start with the launch and stream their
// operand panels together instead of drifting apart behind a mix of short tiles.
__global__ void expert_order_kernel(const int64_t *exp_rows, int E, int32_t *perm) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int64_t n = exp_rows[e + 1] - exp_rows[e];
        int rank = 0;
        for (int j = 0; j < E; ++j) {
            const int64_t m = exp_rows[j + 1] - exp_rows[j];
            rank += (m > n) || (m == n && j < e);
        }
        perm[rank] = e;
    }
}

extern "C" int hep_moe_expert_ffn_bwd(const void *d_rows, const void *d_pre, const void *d_h, void *d_dy,
                                      const void *d_w13, const void *d_w2, const int32_t *d_seg, int n_seg,
                                      const int64_t *d_expert_rows, int64_t Rcap, int64_t d_model, int64_t ffn,
                                      int n_experts, void *d_da13, void *d_dx_rows, float *d_dw13, float *d_dw2,
                                      void *d_workspace, size_t workspace_bytes, int32_t *d_status, void *stream) {
    HEP_NVTX("hep_moe_expert_ffn_bwd");
    HEP_REQUIRE(d_rows && d_pre && d_h && d_dy && d_w13 && d_w2 && d_seg && d_expert_rows && d_da13 && d_dx_rows &&
                    d_dw13 && d_dw2 && d_workspace,
                HEP_E_CONTRACT, "hep_moe_expert_ffn_bwd: null pointer");
    HEP_REQUIRE(d_model % 256 == 0 && ffn % 256 == 0, HEP_E_DIMENSION,
                "FFN backward needs d_model %% 256 == 0 and ffn %% 256 == 0");
    HEP_REQUIRE(workspace_bytes >= hep_moe_ffn_workspace(n_seg, Rcap, n_experts), HEP_E_CAPACITY, "workspace too small");
    HEP_REQUIRE(n_experts <= kMaxExpSmem, HEP_E_CAPACITY, "expert FFN backward: at most %d experts", kMaxExpSmem);
    if (Rcap <= 0) return HEP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    int rc = hep_moe_zero_padding(d_expert_rows, d_seg, n_seg, n_experts, d_dy, d_model, stream);
    if (rc) return rc;
    const int64_t cap = Rcap / BM + n_seg + 1;
    int32_t *mt_row0 = reinterpret_cast<int32_t *>(d_workspace);
    int32_t *mt_rows = mt_row0 + cap;
    int32_t *exp_off = mt_rows + cap;
    // CTA pairs (256-row tiles, half the operand traffic per SM) on the same rule as the
    // forward; MN-major operands are two 64-wide boxes per CTA half
    const bool pairs = use_pairs(Rcap, n_experts) && d_model % 256 == 0 && (2 * ffn) % 256 == 0;
    // light experts on a 1-CTA tile list, as in the forward (the weight-gradient GEMMs
    // contract over the rows, so only the two dgrad GEMMs have row tiles to split)
    const int light_max = pairs ? ffn_light_max(Rcap, n_experts, false) : 0;
    // wave counters 4 / 5 of the workspace tail: the weight-gradient pair GEMMs (hep_tuning.wgrad_wave_sync)
    unsigned int *wave_ctr = ffn_wave_ctr(d_workspace, cap, n_experts);
    if ((rc = build_tiles(d_seg, n_seg, n_experts, mt_row0, mt_rows, exp_off, exp_off + n_experts + 1, cap, d_status,
                          pairs ? kPairRows : BM, s, light_max, 0, wave_ctr)))
        return rc;
    int32_t *mt_row0_l = exp_off + 2 * (n_experts + 1);
    int32_t *mt_rows_l = mt_row0_l + cap;
    int32_t *exp_off_l = mt_rows_l + cap;
    if (light_max > 0 && (rc = build_tiles(d_seg, n_seg, n_experts, mt_row0_l, mt_rows_l, exp_off_l,
                                           exp_off_l + n_experts + 1, cap, d_status, BM, s, light_max, 1)))
        return rc;
    auto light_list = [&](Params q) {
        q.mt_row0 = mt_row0_l;
        q.mt_rows = mt_rows_l;
        q.exp_mt_off = exp_off_l;
        return q;
    };
    CUtensorMap ta, tb;  // A boxes are 128 rows for both kernels (a CTA's half of a pair tile)
    Params p{};
    // --- dA13 = swiglu'(A13) * (dY W2)
    p.grouped = 1;
    p.mt_row0 = mt_row0;
    p.mt_rows = mt_rows;
    p.exp_mt_off = exp_off;
    p.n_exp = n_experts;
    p.kblocks = (int)(d_model / BK);
    p.n_tiles = (int)(ffn / 256);
    p.b_rows_per_exp = d_model;  // W2[e] is [d][F]: K rows per expert
    p.out = d_da13;
    p.ld_out = 2 * ffn;
    p.out_cols = 2 * ffn;
    p.aux = const_cast<void *>(d_pre);
    p.ld_aux = 2 * ffn;
    // the two dgrad pair GEMMs start their waves together like the forward's (counters 6 / 7;
    // launch2sm_maps keeps the counter only for tiles of >= pair_wave_sync k-blocks)
    p.wave_ctr = wave_ctr + 6;
    if ((rc = make_tmap(&ta, d_dy, (uint64_t)Rcap, (uint64_t)d_model, pairs ? 128 : BM))) return rc;
    if ((rc = make_tmap_mn(&tb, d_w2, (uint64_t)n_experts * d_model, (uint64_t)ffn))) return rc;
    if ((rc = pairs ? launch2sm_maps<6, EPI_SWIGLU_BWD, false, true>(ta, tb, p, s)
                    : launch_maps<256, 4, EPI_SWIGLU_BWD, false, true>(ta, tb, p, 0, s)))
        return rc;
    if (light_max > 0 && (rc = launch_maps<256, 4, EPI_SWIGLU_BWD, false, true>(ta, tb, light_list(p), 0, s)))
        return rc;
    p.wave_ctr = wave_ctr + 7;
    if ((rc = hep_moe_zero_padding(d_expert_rows, d_seg, n_seg, n_experts, d_da13, 2 * ffn, stream))) return rc;
    // --- dX_rows = dA13 W13
    p.kblocks = (int)(2 * ffn / BK);
    p.n_tiles = (int)(d_model / 256);
    p.b_rows_per_exp = 2 * ffn;  // W13[e] is [2F][d]
    p.out = d_dx_rows;
    p.ld_out = d_model;
    p.out_cols = d_model;
    p.aux = nullptr;
    if ((rc = make_tmap(&ta, d_da13, (uint64_t)Rcap, (uint64_t)(2 * ffn), pairs ? 128 : BM))) return rc;
    if ((rc = make_tmap_mn(&tb, d_w13, (uint64_t)n_experts * 2 * ffn, (uint64_t)d_model))) return rc;
    if ((rc = pairs ? launch2sm_maps<6, EPI_BF16, false, true>(ta, tb, p, s)
                    : launch_maps<256, 4, EPI_BF16, false, true>(ta, tb, p, 0, s)))
        return rc;
    if (light_max > 0 && (rc = launch_maps<256, 4, EPI_BF16, false, true>(ta, tb, light_list(p), 0, s))) return rc;
    // --- dW2_e = dY_e^T H_e   (fp32, [E][d][F])
    Params q{};
    q.grouped = 2;
    q.exp_rows = d_expert_rows;
    if (g_tuning.wgrad_order != 0) {
        int32_t *perm = exp_off_l + 2 * (n_experts + 1);  // after the two tile lists
        expert_order_kernel<<<1, 1024, 0, s>>>(d_expert_rows, n_experts, perm);
        HEP_CHECK_LAUNCH();
        q.exp_perm = perm;
    }
    q.n_exp = n_experts;
    q.raster_gm = g_tuning.wgrad_raster ? -2 : 0;  // mode 2: the shorter tile dimension fastest
    const int tm = pairs ? kPairRows : BM;
    q.tile_m = pairs ? kPairRows : 0;
    q.M = d_model;
    q.m_tiles = (int)(d_model / tm);
    q.n_tiles = (int)(ffn / 256);
    q.out = d_dw2;
    q.ld_out = ffn;
    q.out_cols = ffn;
    q.out_exp_stride = d_model * ffn;
    if (g_tuning.wgrad_wave_sync) q.wave_ctr = wave_ctr + 4;
    if ((rc = make_tmap_mn(&ta, d_dy, (uint64_t)Rcap, (uint64_t)d_model))) return rc;
    if ((rc = make_tmap_mn(&tb, d_h, (uint64_t)Rcap, (uint64_t)ffn))) return rc;
    if ((rc = pairs ? launch2sm_maps<6, EPI_F32, true, true>(ta, tb, q, s)
                    : launch_maps<256, 4, EPI_F32, true, true>(ta, tb, q, 0, s)))
        return rc;
    // --- dW13_e = dA13_e^T X_e  (fp32, [E][2F][d], W13 interleave)
    q.M = 2 * ffn;
    q.m_tiles = (int)(2 * ffn / tm);
    q.n_tiles = (int)(d_model / 256);
    q.out = d_dw13;
    q.ld_out = d_model;
    q.out_cols = d_model;
    q.out_exp_stride = 2 * ffn * d_model;
    if (g_tuning.wgrad_wave_sync) q.wave_ctr = wave_ctr + 5;
    if ((rc = make_tmap_mn(&ta, d_da13, (uint64_t)Rcap, (uint64_t)(2 * ffn)))) return rc;
    if ((rc = make_tmap_mn(&tb, d_rows, (uint64_t)Rcap, (uint64_t)d_model))) return rc;
    return pairs ? launch2sm_maps<6, EPI_F32, true, true>(ta, tb, q, s)
                 : launch_maps<256, 4, EPI_F32, true, true>(ta, tb, q, 0, s);
}

// split-K reduction: out[i] = sum_s part[s][i], s ascending (deterministic)
__global__ void splitk_reduce_kernel(const float4 *__restrict__ part, int S, int64_t n4, float4 *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = part[i];
        for (int sp = 1; sp < S; ++sp) {
            const float4 b = part[(int64_t)sp * n4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        out[i] = a;
    }
}

// Router backward: dWg = dlogits^T x (fp32 [E64][d]) and dx_gate = dlogits Wg (bf16 [T][d]);
// dlogits is bf16 [T][E64], Wg is [E64][d] (E64 = experts padded to 64), T % 64 == 0.
extern "C" int hep_router_bwd(const void *d_x, const void *d_wg, const void *d_dlogits, int64_t T, int64_t d_model,
                              int E64, float *d_dwg, void *d_dxg, void *stream) {
    HEP_NVTX("hep_router_bwd");
    HEP_REQUIRE(d_x && d_wg && d_dlogits && d_dwg && d_dxg, HEP_E_CONTRACT, "hep_router_bwd: null pointer");
    HEP_REQUIRE(T % 64 == 0 && E64 % 64 == 0 && d_model % 256 == 0, HEP_E_DIMENSION,
                "hep_router_bwd: T %% 64, E64 %% 64, d %% 256");
    if (T <= 0) return HEP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    CUtensorMap ta, tb;
    int rc;
    Params p{};
    p.grouped = 0;
    p.M = E64;
    p.kblocks = (int)(T / BK);
    p.n_tiles = (int)(d_model / 256);
    p.out = d_dwg;
    p.ld_out = d_model;
    p.out_cols = d_model;
    // dWg has only ceil(E64/128) x d/256 output tiles but a T-long contraction: split the
    // contraction so every SM works (fp32 partials staged in the dx_gate buffer, which the
    // second GEMM overwrites afterwards, then summed in split order — deterministic)
    const int64_t tiles = (E64 + BM - 1) / BM * p.n_tiles;
    int S = (int)(sm_count() / (tiles > 0 ? tiles : 1));
    const int64_t cap_split = T / (2 * (int64_t)E64);  // S x E64 x d fp32 must fit in T x d bf16
    if (S > cap_split) S = (int)cap_split;
    if (S > p.kblocks) S = p.kblocks;
    if (S > 1) {
        p.k_split = S;
        p.out = d_dxg;
        p.out_exp_stride = (int64_t)E64 * d_model;
    }
    if ((rc = make_tmap_mn(&ta, d_dlogits, (uint64_t)T, (uint64_t)E64))) return rc;
    if ((rc = make_tmap_mn(&tb, d_x, (uint64_t)T, (uint64_t)d_model))) return rc;
    if ((rc = launch_maps<256, 4, EPI_F32, true, true>(ta, tb, p, tiles * (S > 1 ? S : 1), s))) return rc;
    if (S > 1) {
        const int64_t n4 = (int64_t)E64 * d_model / 4;
        splitk_reduce_kernel<<<(unsigned)((n4 + 255) / 256 < 4 * 148 ? (n4 + 255) / 256 : 4 * 148), 256, 0, s>>>(
            reinterpret_cast<const float4 *>(d_dxg), S, n4, reinterpret_cast<float4 *>(d_dwg));
        HEP_CHECK_LAUNCH();
    }
    Params q{};
    q.grouped = 0;
    q.M = T;
    q.kblocks = E64 / BK;
    q.n_tiles = (int)(d_model / 256);
    q.out = d_dxg;
    q.ld_out = d_model;
    q.out_cols = d_model;
    if ((rc = make_tmap(&ta, d_dlogits, (uint64_t)T, (uint64_t)E64, BM))) return rc;
    if ((rc = make_tmap_mn(&tb, d_wg, (uint64_t)E64, (uint64_t)d_model))) return rc;
    return launch_maps<256, 4, EPI_BF16, false, true>(ta, tb, q, (T + BM - 1) / BM * q.n_tiles, s);
}

// [gemm][start cycles, start ns, end cycles, end ns] of CTA 0 in the last FFN launched
// with hep_tuning.ffn_clock = 1 (diagnostic: the effective SM clock of the expert GEMMs)
extern "C" int hep_ffn_debug_clock(int64_t *host_out8) {
    HEP_REQUIRE(host_out8, HEP_E_CONTRACT, "null output");
    long long tmp[8];
    HEP_CHECK_CUDA(cudaMemcpyFromSymbol(tmp, hep::gemm::g_gemm_clk, sizeof(tmp)));
    for (int i = 0; i < 8; ++i) host_out8[i] = tmp[i];
    return HEP_OK;
}
