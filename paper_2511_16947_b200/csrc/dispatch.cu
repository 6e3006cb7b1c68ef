// dispatch.cu — K4 per-assignment slot assignment, K5 permute/dispatch and
// K7 combine/un-permute.
//
// Receive layout ("rows"): [expert ascending][dst GPU ascending][src GPU
// ascending][rank within (src, expert)] — every expert's rows are contiguous
// (one grouped-GEMM segment per expert, whichever GPUs its replicas live on;
// on a real rank the same rule restricted to dst = this rank).  The routing table
// (reference RoutingTable, router.py:38-46) says, for every (expert, src), how
// its tokens are split into consecutive ranges in sequence order; K4 turns
// that into a row for every (token, k) assignment with a deterministic stable
// counting pass (no atomics decide positions):
//   plan_prep    one CTA: segment table, row bases, per-(expert, src) range lists
//   chunk_count  per 64-token chunk: per-expert assignment counts
//   chunk_scan   per (src, expert): exclusive prefix over chunks (sequence order)
//   chunk_map    per chunk: walk tokens in order -> rank -> range -> row
// K5/K7 are HBM-bound row copies with 128-bit vector loads/stores, one warp
// per token (K5 reads each token once and writes its K rows; K7 reads K rows
// and sums them in fixed k order with fp32 accumulation).
#include "common.cuh"
#include "sched_internal.cuh"

namespace hep {

constexpr int kChunk = 64;
constexpr int kPrepSmemMax = 160 * 1024;  // plan_prep: routing table staged in shared memory up to this size

struct AssignWs {
    int32_t *row_base;  // [nnz] first row of segment (dst, e) per nnz entry
    int32_t *es_cnt;    // [E*G] number of ranges of (e, src)
    int32_t *es_end;    // [E*G*G] rank end (exclusive) of each range, table order
    int32_t *es_delta;  // [E*G*G] row - rank of each range
    int32_t *first;     // [E+1] first range index of expert e (-1 = none)
    int32_t *chunk_cnt; // [n_src * n_chunks * E] per-chunk expert counts (router-written when precounted)
    int32_t *chunk_pre; // [n_src * n_chunks * E] their exclusive prefix over chunks (the counts stay intact)
    int32_t *cnt3;      // [E*G*G] range count of (expert, src, dst)   (EP rank view)
    int32_t *sbase;     // [E*G]   send-buffer base of (expert, dst)   (EP rank view)
    int32_t *es_lo;     // [E*G]   first rank of (e, src) in this phase (pipelined split)
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t assign_ws_bytes(const hep_sched *h, int64_t T, int n_src, int64_t tps) {
    const int64_t E = h->E, G = h->G;
    const int64_t ncs = (tps + kChunk - 1) / kChunk;
    size_t b = 0;
    b += align256(4 * (size_t)h->nnz + 4);
    b += align256(4 * (size_t)(E * G));
    b += align256(4 * (size_t)(E * G * G));
    b += align256(4 * (size_t)(E * G * G));
    b += align256(4 * (size_t)(E + 1));
    b += 2 * align256(4 * (size_t)(n_src * ncs * E));
    b += align256(4 * (size_t)(E * G * G));
    b += align256(4 * (size_t)(E * G));
    b += align256(4 * (size_t)(E * G));
    return b;
}

static AssignWs carve_ws(const hep_sched *h, void *ws, int n_src, int64_t tps) {
    const int64_t E = h->E, G = h->G;
    const int64_t ncs = (tps + kChunk - 1) / kChunk;
    char *p = (char *)ws;
    AssignWs w;
    w.row_base = (int32_t *)p; p += align256(4 * (size_t)h->nnz + 4);
    w.es_cnt = (int32_t *)p; p += align256(4 * (size_t)(E * G));
    w.es_end = (int32_t *)p; p += align256(4 * (size_t)(E * G * G));
    w.es_delta = (int32_t *)p; p += align256(4 * (size_t)(E * G * G));
    w.first = (int32_t *)p; p += align256(4 * (size_t)(E + 1));
    w.chunk_cnt = (int32_t *)p; p += align256(4 * (size_t)(n_src * ((tps + kChunk - 1) / kChunk) * E));
    w.chunk_pre = (int32_t *)p; p += align256(4 * (size_t)(n_src * ((tps + kChunk - 1) / kChunk) * E));
    w.cnt3 = (int32_t *)p; p += align256(4 * (size_t)(E * G * G));
    w.sbase = (int32_t *)p; p += align256(4 * (size_t)(E * G));
    w.es_lo = (int32_t *)p;
    return w;
}

// ---------------------------------------------------------------------------
__global__ void plan_prep_kernel(int G, int E, int nnz, const int32_t *grp_off, const int32_t *grp_gpu,
                                 const int32_t *sorted, const int32_t *nnz_exp, const int64_t *xi,
                                 const int64_t *ranges, const int64_t *n_ranges_p, int64_t *expert_rows,
                                 int32_t *seg, AssignWs w, int32_t *status, int row_align,
                                 const int64_t *split, int phase, int64_t stage_cap, int meta_staged) {
    __shared__ int64_t scan[64];
    const int tid = threadIdx.x, nt = blockDim.x;
    // pipelined split: split = [2][E][G] (static share, scheduled share); this phase's ranks of
    // (e, src) start after the static share's in the scheduled phase
    const int64_t *rank_base = (split && phase == 1) ? split : nullptr;
    const int64_t row_off = 0;
    if (*status) {  // the scheduler failed (and left an empty plan): no segments, no rows
        for (int p = tid; p < nnz; p += nt) {
            seg[4 * p + 0] = (int32_t)row_off;
            seg[4 * p + 1] = 0;
            seg[4 * p + 2] = -1;
            seg[4 * p + 3] = -1;
        }
        for (int e = tid; e <= E; e += nt) expert_rows[e] = row_off;
        for (int i = tid; i < E * G; i += nt) w.es_cnt[i] = 0;
        return;
    }
    const int64_t n_ranges = *n_ranges_p;
    // dynamic smem: [E*G] per-(expert, src) range counters, then the staged routing table
    extern __shared__ int4 s_dyn[];
    int32_t *s_cnt = reinterpret_cast<int32_t *>(s_dyn);
    int4 *s_rng = s_dyn + (E * G + 3) / 4;
    if (meta_staged) {
        // one CTA walks chains of dependent reads (sorted -> xi, grp_off -> grp_gpu) below:
        // stage the small plan arrays in shared memory first, all loads in flight at once
        int64_t *s_xi = reinterpret_cast<int64_t *>(s_rng + stage_cap);
        int32_t *s_off = reinterpret_cast<int32_t *>(s_xi + nnz);
        int32_t *s_sorted = s_off + E + 1;
        int32_t *s_gpu = s_sorted + nnz;
        for (int i = tid; i < nnz; i += nt) {
            s_xi[i] = xi[i];
            s_sorted[i] = sorted[i];
            s_gpu[i] = grp_gpu[i];
        }
        for (int i = tid; i <= E; i += nt) s_off[i] = grp_off[i];
        xi = s_xi;
        grp_off = s_off;
        sorted = s_sorted;
        grp_gpu = s_gpu;
    }
    for (int i = tid; i < E * G; i += nt) {
        s_cnt[i] = 0;
        w.es_lo[i] = rank_base ? (int32_t)rank_base[i] : 0;
    }
    for (int i = tid; i <= E; i += nt) w.first[i] = -1;
    if (meta_staged) __syncthreads();
    // expert blocks ([expert][dst asc][src][rank]), each starting on a row_align boundary
    // (64 in training so weight-gradient GEMMs contract over whole 64-row blocks).  Pipelined
    // split: [expert][phase][dst][src][rank] -- expert e's block holds both phases (its size
    // is the expert's total load, known from the split before the scheduled phase is solved),
    // the static rows first, so the grouped GEMM sees ONE contiguous run per expert and the
    // two phases' assignments can run on different streams
    const int chunk = (E + nt - 1) / nt;
    const int e0 = min(E, tid * chunk), e1 = min(E, e0 + chunk);
    int64_t mine = 0;
    for (int e = e0; e < e1; ++e) {
        int64_t n = 0;
        if (split)
            for (int g = 0; g < G; ++g) n += split[(int64_t)e * G + g] + split[((int64_t)E + e) * G + g];
        else
            for (int p = grp_off[e]; p < grp_off[e + 1]; ++p) n += xi[sorted[p]];
        mine += (n + row_align - 1) / row_align * row_align;
    }
    int64_t total;
    int64_t row = block_excl_scan_i64(mine, scan, &total) + row_off;
    total += row_off;
    for (int e = e0; e < e1; ++e) {
        int64_t skip = 0;  // the static phase's rows of e precede the scheduled phase's
        if (split && phase == 1)
            for (int g = 0; g < G; ++g) skip += split[(int64_t)e * G + g];
        const int64_t blk = row;
        row += skip;
        expert_rows[e] = row;
        int64_t r = row;
        for (int p = grp_off[e]; p < grp_off[e + 1]; ++p) {  // segments in the scheduler's sorted arc order
            const int i = sorted[p];
            seg[4 * p + 0] = (int32_t)r;
            seg[4 * p + 1] = (int32_t)xi[i];
            seg[4 * p + 2] = e;
            seg[4 * p + 3] = grp_gpu[i];
            w.row_base[i] = (int32_t)r;
            r += xi[i];
        }
        if (split) {  // next expert block: after both phases' rows of e
            int64_t n = 0;
            for (int g = 0; g < G; ++g) n += split[(int64_t)e * G + g] + split[((int64_t)E + e) * G + g];
            row = blk + n;
        } else {
            row += (r - row + row_align - 1) / row_align * row_align;
        }
    }
    if (tid == 0) {
        expert_rows[E] = total;
        if (total >= (int64_t)1 << 31) atomicCAS(status, 0, HEP_E_CAPACITY);
    }
    // the routing table as int4 (expert, src, dst, count) in shared memory when it fits
    // (the per-expert passes below re-read each expert's ranges O(ranges^2) times)
    const bool staged = n_ranges <= stage_cap;
    if (staged)
        for (int64_t r = tid; r < n_ranges; r += nt)
            s_rng[r] = make_int4((int)ranges[4 * r], (int)ranges[4 * r + 1], (int)ranges[4 * r + 2],
                                 (int)ranges[4 * r + 3]);
    __syncthreads();
    auto rng = [&](int64_t j) -> int4 {
        return staged ? s_rng[j]
                      : make_int4((int)ranges[4 * j], (int)ranges[4 * j + 1], (int)ranges[4 * j + 2],
                                  (int)ranges[4 * j + 3]);
    };
    for (int64_t r = tid; r < n_ranges; r += nt) {
        const int e = rng(r).x;
        if (r == 0 || rng(r - 1).x != e) w.first[e] = (int)r;
    }
    __syncthreads();
    // one thread per range j (a thread per expert walked its ranges serially: E = 8 left
    // 504 of the 512 threads idle): row and rank offsets from the expert's ranges before j,
    // and j's slot among its (expert, src) ranges = how many of them precede it
    for (int64_t j = tid; j < n_ranges; j += nt) {
        const int4 rj = rng(j);
        const int e = rj.x, src = rj.y, dst = rj.z;
        const int64_t cnt = rj.w;
        int nz = -1;
        for (int i = grp_off[e]; i < grp_off[e + 1]; ++i)
            if (grp_gpu[i] == dst) nz = i;
        if (nz < 0) { atomicCAS(status, 0, HEP_E_CONTRACT); continue; }
        int64_t row = w.row_base[nz], rank = rank_base ? rank_base[e * G + src] : 0;
        int slot = 0;
        for (int64_t k = w.first[e]; k < n_ranges; ++k) {
            const int4 rk = rng(k);
            if (rk.x != e) break;
            if (rk.z == dst && rk.y < src) row += rk.w;
            if (k < j && rk.y == src) { rank += rk.w; ++slot; }
        }
        const int es = e * G + src;
        atomicAdd(&s_cnt[es], 1);
        w.es_end[es * G + slot] = (int32_t)(rank + cnt);
        w.es_delta[es * G + slot] = (int32_t)(row - rank);
    }
    __syncthreads();
    for (int i = tid; i < E * G; i += nt) w.es_cnt[i] = s_cnt[i];
}

__global__ void chunk_count_kernel(const int32_t *topk_idx, int K, int E, int64_t tps, int64_t T, int ncs,
                                   int32_t *chunk_cnt) {
    extern __shared__ int32_t cnt[];
    const int src = blockIdx.x / ncs, c = blockIdx.x % ncs;
    const int64_t t0 = (int64_t)src * tps + (int64_t)c * kChunk;
    int64_t t1 = (int64_t)src * tps + tps;
    if (t0 + kChunk < t1) t1 = t0 + kChunk;
    if (T < t1) t1 = T;
    for (int i = threadIdx.x; i < E; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    for (int64_t a = t0 * K + threadIdx.x; a < t1 * K; a += blockDim.x) atomicAdd(&cnt[topk_idx[a]], 1);
    __syncthreads();
    int32_t *out = chunk_cnt + (int64_t)blockIdx.x * E;
    for (int i = threadIdx.x; i < E; i += blockDim.x) out[i] = cnt[i];
}

// exclusive prefix over a source's chunks, one warp per (src, expert): 32 chunks per
// step, all loads of a step in flight together (the serial walk was a chain of
// dependent L2 round trips)
__global__ void chunk_scan_kernel(int n_src, int ncs, int E, const int32_t *chunk_cnt, int32_t *chunk_pre) {
    const int id = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (id >= n_src * E) return;
    const int src = id / E, e = id % E;
    int32_t run = 0;
    for (int c0 = 0; c0 < ncs; c0 += 32) {
        const int c = c0 + lane;
        const int64_t at = ((int64_t)src * ncs + c) * E + e;
        const int32_t v = c < ncs ? chunk_cnt[at] : 0;
        int32_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (c < ncs) chunk_pre[at] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
}

// one warp per chunk; lanes k < K own pick k of each token (distinct experts)
__global__ void chunk_map_kernel(const int32_t *topk_idx, int K, int E, int G, int64_t tps, int64_t T, int ncs,
                                 const int32_t *chunk_pre, AssignWs w, int32_t *tok_row, int32_t *row_tok,
                                 int src_base, bool windowed, const int32_t *status, int32_t *tok_row_phase) {
    extern __shared__ int32_t sm[];
    int32_t *ctr = sm;                // [E]
    int32_t *l_cnt = ctr + E;         // [E]
    int32_t *l_end = l_cnt + E;       // [E*G]
    int32_t *l_delta = l_end + E * G; // [E*G]
    int32_t *l_lo = l_delta + E * G;  // [E] (windowed: first rank of this phase)
    int32_t *l_idx = l_lo + E;        // [kChunk * K] this chunk's top-K picks
    const int src = blockIdx.x / ncs, c = blockIdx.x % ncs;
    const int lane = threadIdx.x;
    if (*status) {
        // no valid schedule for this micro-batch: identity map, (t, k) -> row t*K + k, so the
        // permute / dispatch / combine queued behind stay inside their [T*K] buffers (the
        // layer raises the status; the outputs of this micro-batch are not defined)
        const int64_t ta = (int64_t)src * tps + (int64_t)c * kChunk;
        int64_t tb = (int64_t)src * tps + tps;
        if (ta + kChunk < tb) tb = ta + kChunk;
        if (T < tb) tb = T;
        for (int64_t i = ta * K + threadIdx.x; i < tb * K; i += blockDim.x) {
            tok_row[i] = (int32_t)i;
            if (tok_row_phase) tok_row_phase[i] = -1;
            if (row_tok) row_tok[i] = (int32_t)(i / K);
        }
        return;
    }
    // stage this source's range lists with the whole block, independent loads (all G
    // slots of every expert; slots past es_cnt are never read)
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        ctr[e] = chunk_pre[(int64_t)blockIdx.x * E + e];
        const int es = e * G + src_base + src;
        l_cnt[e] = w.es_cnt[es];
        if (windowed) l_lo[e] = w.es_lo[es];
    }
    for (int i = threadIdx.x; i < E * G; i += blockDim.x) {
        const int e = i / G, j = i - e * G;
        const int64_t es = (int64_t)e * G + src_base + src;
        l_end[i] = w.es_end[es * G + j];
        l_delta[i] = w.es_delta[es * G + j];
    }
    const int64_t t0 = (int64_t)src * tps + (int64_t)c * kChunk;
    int64_t t1 = (int64_t)src * tps + tps;
    if (t0 + kChunk < t1) t1 = t0 + kChunk;
    if (T < t1) t1 = T;
    // the chunk's picks, so the sequential walk below reads shared memory only
    for (int64_t i = threadIdx.x; i < (t1 - t0) * K; i += blockDim.x) l_idx[i] = topk_idx[t0 * K + i];
    __syncthreads();
    if (threadIdx.x >= 32) return;
    // 32 assignments (token-major, k minor = sequence order: a token's picks are distinct
    // experts) per step: lanes with the same expert find each other with match.any, their
    // ranks are the running counter plus the number of earlier peers; the lowest peer
    // advances the counter
    const int n_asg = (int)(t1 - t0) * K;
    for (int a0 = 0; a0 < n_asg; a0 += 32) {
        const int a = a0 + lane;
        const int e = a < n_asg ? l_idx[a] : -1 - lane;
        const uint32_t peers = __match_any_sync(0xffffffffu, e);
        if (e >= 0) {
            const int q = ctr[e] + __popc(peers & ((1u << lane) - 1u));
            int j = 0;
            const int n = l_cnt[e];
            // pipelined split: this phase owns ranks [lo, end of its last range) of (e, src)
            const bool mine = !windowed || (n > 0 && q >= l_lo[e] && q < l_end[e * G + n - 1]);
            const int64_t t = t0 + a / K;
            const int64_t tk = t * K + (a - (a / K) * K);
            if (mine) {
                while (j + 1 < n && q >= l_end[e * G + j]) ++j;
                const int row = q + l_delta[e * G + j];
                tok_row[tk] = row;
                if (tok_row_phase) tok_row_phase[tk] = row;
                if (row_tok) row_tok[row] = (int32_t)t;
            } else if (tok_row_phase) {
                tok_row_phase[tk] = -1;  // the other phase's assignment: this phase's permute skips it
            }
        }
        __syncwarp();
        if (e >= 0 && (__ffs(peers) - 1) == lane) ctr[e] += __popc(peers);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// EP rank view (one process per GPU).  Rank r is source r of its own T tokens
// and destination r of its replicas.  Send buffer: [dst][expert asc][rank];
// receive buffer (what NCCL all-to-all-v delivers): [src][expert asc][rank],
// one grouped-GEMM segment per (src, hosted expert) carrying the expert's
// local weight slot.  Every rank derives all offsets from the same routing
// table, so both sides agree without exchanging anything but the rows.
// ---------------------------------------------------------------------------
// Pipelined split (split != null): this phase's plan covers ranks [lo, lo + share) of every
// (expert, source) token sequence, lo = 0 (phase 0, the static share) or the static share
// split[e][src] (phase 1); send rows start at row_off (the two phases' send layouts share one
// buffer, phase 1 after phase 0's worst case).
__global__ void ep_prep_kernel(int G, int E, int rank, const int64_t *ranges, const int64_t *n_ranges_p,
                               const int64_t *transfer, const int32_t *hosted, int n_hosted, const int32_t *nnz_exp,
                               const int32_t *slots, int64_t *counts, int32_t *seg, AssignWs w, int32_t *status,
                               int64_t recv_capacity, const int64_t *split = nullptr, int phase = 0,
                               int64_t row_off = 0) {
    const int tid = threadIdx.x, nt = blockDim.x;
    __shared__ int fail;
    if (tid == 0) {
        // receive capacity (NVLink path: fixed buffers peers store into): every rank checks
        // EVERY destination's total from the identical transfer plan, so all ranks agree
        int f = *status != 0;
        if (!f && recv_capacity > 0)
            for (int d = 0; d < G; ++d) {
                int64_t r = 0;
                for (int s2 = 0; s2 < G; ++s2) r += transfer[s2 * G + d];
                if (r > recv_capacity) f = 1;
            }
        if (f) atomicCAS(status, 0, HEP_E_CAPACITY);
        fail = f;
    }
    __syncthreads();
    if (fail) {  // empty exchange: nothing sent, nothing received, no FFN tiles
        for (int i = tid; i < 2 * G; i += nt) counts[i] = 0;
        for (int i = tid; i < G * n_hosted; i += nt) {
            int32_t *sg = seg + 4 * (int64_t)i;
            sg[0] = 0;
            sg[1] = 0;
            sg[2] = 0;
            sg[3] = i / (n_hosted > 0 ? n_hosted : 1);
        }
        for (int i = tid; i < E * G; i += nt) w.es_cnt[i] = 0;
        return;
    }
    const int64_t n_ranges = *n_ranges_p;
    for (int i = tid; i < E * G * G; i += nt) w.cnt3[i] = 0;
    for (int i = tid; i < E * G; i += nt) {
        w.es_cnt[i] = 0;
        w.es_lo[i] = (split && phase == 1) ? (int32_t)split[i] : 0;  // the phase's first rank of (e, src)
    }
    for (int i = tid; i <= E; i += nt) w.first[i] = -1;
    __syncthreads();
    for (int64_t r = tid; r < n_ranges; r += nt) {
        const int64_t *q = ranges + 4 * r;
        const int e = (int)q[0];
        w.cnt3[((int64_t)e * G + q[1]) * G + q[2]] = (int32_t)q[3];
        if (r == 0 || ranges[4 * (r - 1)] != e) w.first[e] = (int)r;
    }
    __syncthreads();
    if (tid < G) {
        const int d = tid;
        counts[d] = transfer[rank * G + d];      // rows this rank sends to d
        counts[G + d] = transfer[d * G + rank];  // rows this rank receives from d
        int64_t run = 0;
        for (int dd = 0; dd < d; ++dd) run += transfer[rank * G + dd];
        for (int e = 0; e < E; ++e) {
            w.sbase[e * G + d] = (int32_t)(run + row_off);
            run += w.cnt3[((int64_t)e * G + rank) * G + d];
        }
        // receive segments of source d: [src][hosted expert asc]
        int64_t row = 0;
        for (int ss = 0; ss < d; ++ss) row += transfer[ss * G + rank];
        for (int h = 0; h < n_hosted; ++h) {
            const int e = nnz_exp[hosted[h]];
            const int32_t c = w.cnt3[((int64_t)e * G + d) * G + rank];
            int32_t *sg = seg + 4 * ((int64_t)d * n_hosted + h);
            sg[0] = (int32_t)row;
            sg[1] = c;
            sg[2] = slots[e];
            sg[3] = d;
            row += c;
        }
        if (row >= ((int64_t)1 << 31)) atomicCAS(status, 0, HEP_E_CAPACITY);
    }
    __syncthreads();
    // per (expert, this source): ranges in table order -> send positions, one thread per
    // range of this source (its slot and first rank from the expert's earlier ranges)
    for (int64_t j = tid; j < n_ranges; j += nt) {
        if (ranges[4 * j + 1] != rank) continue;
        const int e = (int)ranges[4 * j];
        const int dst = (int)ranges[4 * j + 2];
        const int64_t c = ranges[4 * j + 3];
        const int es = e * G + rank;
        int64_t rank_start = w.es_lo[es];
        int slot = 0;
        for (int64_t k = w.first[e]; k < j; ++k)
            if (ranges[4 * k + 1] == rank) {
                rank_start += ranges[4 * k + 3];
                ++slot;
            }
        atomicAdd(&w.es_cnt[es], 1);
        w.es_end[es * G + slot] = (int32_t)(rank_start + c);
        w.es_delta[es * G + slot] = (int32_t)(w.sbase[e * G + dst] - rank_start);
    }
}

// ---------------------------------------------------------------------------
// K5: rows[tok_row[t][k]] = x[t]
__global__ void __launch_bounds__(256) permute_kernel(const int4 *__restrict__ x, const int32_t *__restrict__ tok_row,
                                                      int64_t T, int K, int64_t nvec, int4 *__restrict__ rows) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < T; t += nwarps) {
        int32_t r[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < K) r[k] = tok_row[t * K + k];
        bool any = false;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < K) any |= r[k] >= 0;
        if (!any) continue;  // no assignment of this token in this phase: x[t] is not read
        const int4 *src = x + t * nvec;
        for (int64_t v0 = lane; v0 < nvec; v0 += 32 * 4) {
            int4 buf[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (v0 + 32 * u < nvec) buf[u] = __ldg(src + v0 + 32 * u);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k >= K) break;
                if (r[k] < 0) continue;  // not this phase's assignment (pipelined split)
                int4 *dst = rows + (int64_t)r[k] * nvec;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v0 + 32 * u < nvec) dst[v0 + 32 * u] = buf[u];
            }
        }
    }
}

// 32-byte LSU accesses (sm_100 LDG/STG .256): half the load/store instructions of the
// 128-bit kernel for the same bytes in flight; rows 32-B aligned (d_model % 16).  The
// permute gains 2-4 % (5.82-5.92 -> 6.01-6.09 TB/s, tools/lsu_ab.py); the same change
// made the combine 5-10 % slower, so it keeps 128-bit loads.
struct alignas(32) V8 {
    uint32_t w[8];
};
__device__ __forceinline__ V8 ldg_v8(const V8 *p) {
    V8 v;
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v.w[0]), "=r"(v.w[1]), "=r"(v.w[2]), "=r"(v.w[3]), "=r"(v.w[4]), "=r"(v.w[5]), "=r"(v.w[6]),
                   "=r"(v.w[7])
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void stg_v8(V8 *p, const V8 &v) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                 "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

__global__ void __launch_bounds__(256) permute_v8_kernel(const V8 *__restrict__ x, const int32_t *__restrict__ tok_row,
                                                         int64_t T, int K, int64_t nv8, V8 *__restrict__ rows) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < T; t += nwarps) {
        int32_t r[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < K) r[k] = tok_row[t * K + k];
        bool any = false;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < K) any |= r[k] >= 0;
        if (!any) continue;  // no assignment of this token in this phase: x[t] is not read
        const V8 *src = x + t * nv8;
        for (int64_t v0 = lane; v0 < nv8; v0 += 32 * 2) {
            V8 buf[2];
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (v0 + 32 * u < nv8) buf[u] = ldg_v8(src + v0 + 32 * u);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if (k >= K) break;
                if (r[k] < 0) continue;  // not this phase's assignment (pipelined split)
                V8 *dst = rows + (int64_t)r[k] * nv8;
#pragma unroll
                for (int u = 0; u < 2; ++u)
                    if (v0 + 32 * u < nv8) stg_v8(dst + v0 + 32 * u, buf[u]);
            }
        }
    }
}

static bool use_lsu256(const void *a, const void *b, const void *c, int64_t d_model) {
    if (g_tuning.lsu256 == 0) return false;
    auto al = [](const void *p) { return p == nullptr || reinterpret_cast<uintptr_t>(p) % 32 == 0; };
    return d_model % 16 == 0 && al(a) && al(b) && al(c);
}

// K7: out[t] = sum_k w[t][k] * y[tok_row[t][k]], fp32 accumulation in k order.
// One warp per token; each lane keeps 2 x K 128-bit loads in flight.
template <int K>
__global__ void __launch_bounds__(256) combine_kernel(const int4 *__restrict__ y, const int32_t *__restrict__ tok_row,
                                                      const float *__restrict__ topk_w, int64_t T, int64_t nvec,
                                                      int4 *__restrict__ out, const int4 *__restrict__ add) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < T; t += nwarps) {
        const int4 *src[K];
        float wk[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            src[k] = y + (int64_t)tok_row[t * K + k] * nvec;
            wk[k] = topk_w ? topk_w[t * K + k] : 1.0f;  // unit weights: the permute's transpose
        }
        for (int64_t v0 = lane; v0 < nvec; v0 += 64) {
            int4 in[2][K];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    if (v0 + 32 * u < nvec) in[u][k] = __ldg(src[k] + v0 + 32 * u);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (v0 + 32 * u >= nvec) break;
                float acc[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[i] = 0.f;
                if (add) {  // e.g. the router's contribution to dx
                    const int4 av = add[t * nvec + v0 + 32 * u];
                    const __nv_bfloat162 *ah = reinterpret_cast<const __nv_bfloat162 *>(&av);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 f = __bfloat1622float2(ah[i]);
                        acc[2 * i] = f.x;
                        acc[2 * i + 1] = f.y;
                    }
                }
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&in[u][k]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 f = __bfloat1622float2(h[i]);
                        acc[2 * i] = fmaf(wk[k], f.x, acc[2 * i]);
                        acc[2 * i + 1] = fmaf(wk[k], f.y, acc[2 * i + 1]);
                    }
                }
                int4 o;
                __nv_bfloat162 *oh = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                for (int i = 0; i < 4; ++i) oh[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
                out[t * nvec + v0 + 32 * u] = o;
            }
        }
    }
}

static int grid_for_warps(int64_t T, int blocks_per_sm = 8) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (T + 7) / 8;  // 8 warps per block
    const int64_t cap = (int64_t)sms * blocks_per_sm;
    const int64_t g = want < cap ? want : cap;
    return (int)(g > 1 ? g : 1);
}

}  // namespace hep

using namespace hep;

extern "C" size_t hep_moe_assign_workspace(hep_sched_t h, int64_t T, int K) {
    (void)K;
    if (!h) return 0;
    const int n_src = h->G;
    const int64_t tps = (T + n_src - 1) / n_src;
    return assign_ws_bytes(h, T, n_src, tps > 0 ? tps : 1);
}

static int assign_impl(hep_sched_t h, const hep_sched_out *sched, bool windowed, bool precounted,
                       const int64_t *d_split, int phase, const int32_t *d_topk_idx, int64_t T, int K,
                       int64_t tokens_per_src, int row_align, int32_t *d_tok_row, int32_t *d_row_tok, int32_t *d_seg,
                       int64_t *d_expert_rows, void *workspace, size_t workspace_bytes, void *stream,
                       int32_t *d_tok_row_phase = nullptr) {
    HEP_REQUIRE(row_align >= 1 && row_align <= 1024, HEP_E_DIMENSION, "row_align=%d", row_align);
    HEP_REQUIRE(h && sched && d_topk_idx && d_tok_row && d_row_tok && d_seg && d_expert_rows && workspace,
                HEP_E_CONTRACT, "hep_moe_assign: null argument");
    HEP_REQUIRE(K >= 1 && K <= 16 && tokens_per_src >= 1, HEP_E_DIMENSION, "hep_moe_assign: K=%d", K);
    const int n_src = h->G;
    HEP_REQUIRE(tokens_per_src * n_src >= T, HEP_E_DIMENSION, "tokens_per_src * G < T");
    HEP_REQUIRE(workspace_bytes >= assign_ws_bytes(h, T, n_src, tokens_per_src), HEP_E_CAPACITY,
                "hep_moe_assign: workspace too small (%zu < %zu)", workspace_bytes,
                assign_ws_bytes(h, T, n_src, tokens_per_src));
    cudaStream_t s = (cudaStream_t)stream;
    AssignWs w = carve_ws(h, workspace, n_src, tokens_per_src);
    const int E = h->E, G = h->G;
    const size_t cnt_sm = 16 * (size_t)((E * G + 3) / 4);
    HEP_REQUIRE(cnt_sm <= kPrepSmemMax, HEP_E_CAPACITY, "plan_prep: E*G too large");
    int64_t stage_cap = h->max_ranges;
    if (cnt_sm + 16 * stage_cap > kPrepSmemMax) stage_cap = 0;  // too large to stage: read the table from global
    // + the plan arrays (xi, grp_off, sorted, grp_gpu) when they fit too
    const size_t meta_sm = 16 * (((size_t)h->nnz * 16 + 4 * ((size_t)E + 1) + 15) / 16);
    const int meta_staged = cnt_sm + 16 * (size_t)stage_cap + meta_sm <= kPrepSmemMax;
    const size_t prep_sm = cnt_sm + 16 * (size_t)stage_cap + (meta_staged ? meta_sm : 0);
    if (prep_sm + 512 > 48 * 1024)  // + the kernel's static scan buffer
        HEP_CHECK_CUDA(cudaFuncSetAttribute(plan_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPrepSmemMax));
    plan_prep_kernel<<<1, 512, prep_sm, s>>>(G, E, h->nnz, h->d_grp_off, h->d_grp_gpu, h->d_sorted, h->d_nnz_exp,
                                             sched->d_xi, sched->d_ranges, sched->d_n_ranges, d_expert_rows, d_seg, w,
                                             sched->d_status, row_align, d_split, phase, stage_cap, meta_staged);
    HEP_CHECK_LAUNCH();
    if (T <= 0) return HEP_OK;
    const int ncs = (int)((tokens_per_src + kChunk - 1) / kChunk);
    const int nblk = n_src * ncs;
    if (!precounted) {
        chunk_count_kernel<<<nblk, 128, E * sizeof(int32_t), s>>>(d_topk_idx, K, E, tokens_per_src, T, ncs,
                                                                  w.chunk_cnt);
        HEP_CHECK_LAUNCH();
    }
    chunk_scan_kernel<<<(n_src * E + 7) / 8, 256, 0, s>>>(n_src, ncs, E, w.chunk_cnt, w.chunk_pre);
    HEP_CHECK_LAUNCH();
    const size_t sm = sizeof(int32_t) * (3 * (size_t)E + 2 * (size_t)E * G + (size_t)kChunk * K);
    HEP_REQUIRE(sm <= 200 * 1024, HEP_E_CAPACITY, "chunk_map smem %zu", sm);
    if (sm > 48 * 1024) HEP_CHECK_CUDA(cudaFuncSetAttribute(chunk_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    chunk_map_kernel<<<nblk, 256, sm, s>>>(d_topk_idx, K, E, G, tokens_per_src, T, ncs, w.chunk_pre, w, d_tok_row,
                                           d_row_tok, 0, windowed, sched->d_status, d_tok_row_phase);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_assign(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K,
                              int64_t tokens_per_src, int row_align, int32_t *d_tok_row, int32_t *d_row_tok,
                              int32_t *d_seg, int64_t *d_expert_rows, void *workspace, size_t workspace_bytes,
                              void *stream) {
    HEP_NVTX("hep_moe_assign");
    return assign_impl(h, sched, false, false, nullptr, 0, d_topk_idx, T, K, tokens_per_src, row_align, d_tok_row,
                       d_row_tok, d_seg, d_expert_rows, workspace, workspace_bytes, stream);
}

extern "C" size_t hep_moe_assign_chunk_offset(hep_sched_t h, int64_t T, int K) {
    (void)T;
    (void)K;
    if (!h) return 0;
    const int64_t E = h->E, G = h->G;
    return align256(4 * (size_t)h->nnz + 4) + align256(4 * (size_t)(E * G)) + 2 * align256(4 * (size_t)(E * G * G)) +
           align256(4 * (size_t)(E + 1));
}

extern "C" int hep_moe_assign_precounted(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx,
                                         int64_t T, int K, int64_t tokens_per_src, int row_align, int32_t *d_tok_row,
                                         int32_t *d_row_tok, int32_t *d_seg, int64_t *d_expert_rows, void *workspace,
                                         size_t workspace_bytes, void *stream) {
    HEP_NVTX("hep_moe_assign_precounted");
    return assign_impl(h, sched, false, true, nullptr, 0, d_topk_idx, T, K, tokens_per_src, row_align, d_tok_row,
                       d_row_tok, d_seg, d_expert_rows, workspace, workspace_bytes, stream);
}

extern "C" int hep_gate_chunk_counts(const int32_t *d_topk_idx, int64_t T, int K, int E, int64_t tokens_per_src,
                                     int n_src, int32_t *d_chunk_cnt, void *stream) {
    HEP_REQUIRE(d_topk_idx && d_chunk_cnt, HEP_E_CONTRACT, "hep_gate_chunk_counts: null pointer");
    HEP_REQUIRE(E >= 1 && K >= 1 && tokens_per_src >= 1 && n_src >= 1, HEP_E_DIMENSION, "hep_gate_chunk_counts");
    if (T <= 0) return HEP_OK;
    const int ncs = (int)((tokens_per_src + kChunk - 1) / kChunk);
    chunk_count_kernel<<<n_src * ncs, 128, E * sizeof(int32_t), (cudaStream_t)stream>>>(d_topk_idx, K, E,
                                                                                       tokens_per_src, T, ncs,
                                                                                       d_chunk_cnt);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_assign_phase(hep_sched_t h, const hep_sched_out *sched, const int64_t *d_split, int phase,
                                    const int32_t *d_topk_idx, int64_t T, int K, int64_t tokens_per_src,
                                    int32_t *d_tok_row, int32_t *d_tok_row_phase, int32_t *d_row_tok, int32_t *d_seg,
                                    int64_t *d_expert_rows, void *workspace, size_t workspace_bytes, void *stream) {
    HEP_NVTX("hep_moe_assign_phase");
    HEP_REQUIRE(d_split && (phase == 0 || phase == 1), HEP_E_CONTRACT, "hep_moe_assign_phase: split and phase 0/1");
    return assign_impl(h, sched, true, false, d_split, phase, d_topk_idx, T, K, tokens_per_src, 1, d_tok_row,
                       d_row_tok, d_seg, d_expert_rows, workspace, workspace_bytes, stream, d_tok_row_phase);
}

extern "C" int hep_moe_permute_ex(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model,
                                  void *d_rows, int blocks_per_sm, void *stream) {
    HEP_NVTX("hep_moe_permute");
    HEP_REQUIRE(d_x && d_tok_row && d_rows, HEP_E_CONTRACT, "hep_moe_permute: null pointer");
    HEP_REQUIRE(d_model % 8 == 0 && K >= 1 && K <= 16, HEP_E_DIMENSION, "hep_moe_permute: d_model %% 8, K<=16");
    HEP_REQUIRE(blocks_per_sm >= 1 && blocks_per_sm <= 8, HEP_E_CONTRACT, "hep_moe_permute: blocks_per_sm 1..8");
    if (T <= 0) return HEP_OK;
    const int grid = grid_for_warps(T, blocks_per_sm);
    if (use_lsu256(d_x, d_rows, nullptr, d_model))
        permute_v8_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const V8 *)d_x, d_tok_row, T, K, d_model / 16,
                                                                   (V8 *)d_rows);
    else
        permute_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const int4 *)d_x, d_tok_row, T, K, d_model / 8,
                                                                (int4 *)d_rows);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_permute(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model,
                               void *d_rows, void *stream) {
    return hep_moe_permute_ex(d_x, d_tok_row, T, K, d_model, d_rows, 8, stream);
}

extern "C" int hep_moe_combine(const void *d_y, const int32_t *d_tok_row, const float *d_topk_w, int64_t T, int K,
                               int64_t d_model, void *d_out, void *stream) {
    HEP_NVTX("hep_moe_combine");
    return hep_moe_gather_sum(d_y, d_tok_row, d_topk_w, nullptr, T, K, d_model, d_out, stream);
}

extern "C" int hep_moe_gather_sum(const void *d_y, const int32_t *d_tok_row, const float *d_topk_w, const void *d_add,
                                  int64_t T, int K, int64_t d_model, void *d_out, void *stream) {
    HEP_NVTX("hep_moe_gather_sum");
    HEP_REQUIRE(d_y && d_tok_row && d_out, HEP_E_CONTRACT, "hep_moe_gather_sum: null pointer");
    HEP_REQUIRE(d_model % 8 == 0 && K >= 1 && K <= 16, HEP_E_DIMENSION, "hep_moe_combine: d_model %% 8, K<=16");
    if (T <= 0) return HEP_OK;
    const int grid = grid_for_warps(T);
    cudaStream_t st = (cudaStream_t)stream;
    const int4 *yv = (const int4 *)d_y;
    int4 *ov = (int4 *)d_out;
    const int4 *av = (const int4 *)d_add;
    const int64_t nv = d_model / 8;
    switch (K) {
#define HEP_COMBINE(KK) \
        case KK: combine_kernel<KK><<<grid, 256, 0, st>>>(yv, d_tok_row, d_topk_w, T, nv, ov, av); break;
        HEP_COMBINE(1) HEP_COMBINE(2) HEP_COMBINE(3) HEP_COMBINE(4) HEP_COMBINE(5) HEP_COMBINE(6) HEP_COMBINE(7)
        HEP_COMBINE(8) HEP_COMBINE(9) HEP_COMBINE(10) HEP_COMBINE(11) HEP_COMBINE(12) HEP_COMBINE(13)
        HEP_COMBINE(14) HEP_COMBINE(15) HEP_COMBINE(16)
#undef HEP_COMBINE
    }
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" size_t hep_moe_assign_ep_workspace(hep_sched_t h, int64_t T, int K) {
    (void)K;
    if (!h) return 0;
    return assign_ws_bytes(h, T, 1, T > 0 ? T : 1);
}

extern "C" int hep_sched_hosted(hep_sched_t h, int rank, int *n_hosted, int *n_slots) {
    HEP_REQUIRE(h && rank >= 0 && rank < h->G, HEP_E_DIMENSION, "hep_sched_hosted: rank %d", rank);
    const int b = h->h_hosted_off[rank], n = h->h_hosted_off[rank + 1] - b;
    if (n_hosted) *n_hosted = n;
    if (n_slots) {
        int mx = 0;
        for (int e = 0; e < h->E; ++e)
            for (int i = h->h_grp_off[e]; i < h->h_grp_off[e + 1]; ++i)
                if (h->h_grp_gpu[i] == rank && h->h_slots[e] + 1 > mx) mx = h->h_slots[e] + 1;
        *n_slots = mx;
    }
    return HEP_OK;
}

static int assign_ep_impl(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K,
                          int rank, int64_t recv_capacity, int32_t *d_tok_row, int32_t *d_seg, int64_t *d_counts,
                          void *workspace, size_t workspace_bytes, void *stream, const int64_t *d_split, int phase,
                          int64_t row_off, int32_t *d_tok_row_phase) {
    HEP_REQUIRE(h && sched && d_topk_idx && d_tok_row && d_seg && d_counts && workspace, HEP_E_CONTRACT,
                "hep_moe_assign_ep: null argument");
    HEP_REQUIRE(rank >= 0 && rank < h->G && K >= 1 && K <= 16, HEP_E_DIMENSION, "hep_moe_assign_ep: rank/K");
    const int64_t tps = T > 0 ? T : 1;
    HEP_REQUIRE(workspace_bytes >= assign_ws_bytes(h, T, 1, tps), HEP_E_CAPACITY, "hep_moe_assign_ep: workspace");
    cudaStream_t s = (cudaStream_t)stream;
    AssignWs w = carve_ws(h, workspace, 1, tps);
    const int E = h->E, G = h->G;
    const int n_hosted = h->h_hosted_off[rank + 1] - h->h_hosted_off[rank];
    ep_prep_kernel<<<1, 512, 0, s>>>(G, E, rank, sched->d_ranges, sched->d_n_ranges, sched->d_transfer,
                                     h->d_seg_nnz + h->h_hosted_off[rank], n_hosted, h->d_nnz_exp, h->d_slots,
                                     d_counts, d_seg, w, sched->d_status, recv_capacity, d_split, phase, row_off);
    HEP_CHECK_LAUNCH();
    if (T <= 0) return HEP_OK;
    const int ncs = (int)((tps + kChunk - 1) / kChunk);
    chunk_count_kernel<<<ncs, 128, E * sizeof(int32_t), s>>>(d_topk_idx, K, E, tps, T, ncs, w.chunk_cnt);
    HEP_CHECK_LAUNCH();
    chunk_scan_kernel<<<(E + 7) / 8, 256, 0, s>>>(1, ncs, E, w.chunk_cnt, w.chunk_pre);
    HEP_CHECK_LAUNCH();
    const size_t sm = sizeof(int32_t) * (3 * (size_t)E + 2 * (size_t)E * G + (size_t)kChunk * K);
    HEP_REQUIRE(sm <= 200 * 1024, HEP_E_CAPACITY, "chunk_map smem %zu", sm);
    if (sm > 48 * 1024)
        HEP_CHECK_CUDA(cudaFuncSetAttribute(chunk_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    chunk_map_kernel<<<ncs, 256, sm, s>>>(d_topk_idx, K, E, G, tps, T, ncs, w.chunk_pre, w, d_tok_row, nullptr, rank,
                                          d_split != nullptr, sched->d_status, d_tok_row_phase);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_assign_ep(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K,
                                 int rank, int64_t recv_capacity, int32_t *d_tok_row, int32_t *d_seg, int64_t *d_counts,
                                 void *workspace, size_t workspace_bytes, void *stream) {
    HEP_NVTX("hep_moe_assign_ep");
    return assign_ep_impl(h, sched, d_topk_idx, T, K, rank, recv_capacity, d_tok_row, d_seg, d_counts, workspace,
                          workspace_bytes, stream, nullptr, 0, 0, nullptr);
}

extern "C" int hep_moe_assign_ep_phase(hep_sched_t h, const hep_sched_out *sched, const int64_t *d_split, int phase,
                                       const int32_t *d_topk_idx, int64_t T, int K, int rank, int64_t send_row_offset,
                                       int32_t *d_tok_row, int32_t *d_tok_row_phase, int32_t *d_seg, int64_t *d_counts,
                                       void *workspace, size_t workspace_bytes, void *stream) {
    HEP_NVTX("hep_moe_assign_ep_phase");
    HEP_REQUIRE(d_split && (phase == 0 || phase == 1) && send_row_offset >= 0, HEP_E_CONTRACT,
                "hep_moe_assign_ep_phase: split, phase 0/1, row offset >= 0");
    return assign_ep_impl(h, sched, d_topk_idx, T, K, rank, 0, d_tok_row, d_seg, d_counts, workspace, workspace_bytes,
                          stream, d_split, phase, send_row_offset, d_tok_row_phase);
}

// ===========================================================================
// Backward data-path kernels
// ===========================================================================
namespace hep {

// K7^T: dY[row(t,k)] = w[t,k] * dout[t] (bf16 rows), dw[t,k] = <dout[t], Y[row(t,k)]> (fp32).
// One warp per token; the dot products reduce with shuffles in a fixed order.
template <int K>
__global__ void __launch_bounds__(256) combine_bwd_kernel(const int4 *__restrict__ dout, const int4 *__restrict__ y,
                                                          const int32_t *__restrict__ tok_row,
                                                          const float *__restrict__ topk_w, int64_t T, int64_t nvec,
                                                          int4 *__restrict__ dy, float *__restrict__ dw) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < T; t += nwarps) {
        int32_t r[K];
        float wk[K], dot[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            r[k] = tok_row[t * K + k];
            wk[k] = topk_w[t * K + k];
            dot[k] = 0.f;
        }
        for (int64_t v = lane; v < nvec; v += 32) {
            const int4 g = __ldg(dout + t * nvec + v);
            const __nv_bfloat162 *gh = reinterpret_cast<const __nv_bfloat162 *>(&g);
            float gf[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(gh[i]);
                gf[2 * i] = f.x;
                gf[2 * i + 1] = f.y;
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int4 yv = __ldg(y + (int64_t)r[k] * nvec + v);
                const __nv_bfloat162 *yh = reinterpret_cast<const __nv_bfloat162 *>(&yv);
                int4 o;
                __nv_bfloat162 *oh = reinterpret_cast<__nv_bfloat162 *>(&o);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f = __bfloat1622float2(yh[i]);
                    dot[k] = fmaf(gf[2 * i], f.x, dot[k]);
                    dot[k] = fmaf(gf[2 * i + 1], f.y, dot[k]);
                    oh[i] = __floats2bfloat162_rn(wk[k] * gf[2 * i], wk[k] * gf[2 * i + 1]);
                }
                dy[(int64_t)r[k] * nvec + v] = o;
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            float v = dot[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) dw[t * K + k] = v;
        }
    }
}

// zero the alignment padding rows of each expert block: [start + n_e, next start)
__global__ void zero_pad_rows_kernel(const int64_t *expert_rows, const int32_t *seg, int n_seg, int E, int64_t nvec,
                                     int4 *buf) {
    const int e = blockIdx.x;
    if (e >= E) return;
    int64_t n = 0;
    for (int s = 0; s < n_seg; ++s)
        if (seg[4 * s + 2] == e) n += seg[4 * s + 1];
    const int64_t r0 = expert_rows[e] + n, r1 = expert_rows[e + 1];
    const int4 z = make_int4(0, 0, 0, 0);
    for (int64_t i = (int64_t)threadIdx.x; i < (r1 - r0) * nvec; i += blockDim.x) buf[r0 * nvec + i] = z;
}

// router backward: weights w = softmax(selected logits), so
// dlogit[t, idx_k] = w_k (dw_k - sum_j w_j dw_j); other columns 0.  bf16 [T][ld] out.
__global__ void gate_bwd_kernel(const int32_t *topk_idx, const float *topk_w, const float *dw, int64_t T, int K,
                                int64_t ld, __nv_bfloat16 *dlogits) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    __nv_bfloat16 *row = dlogits + t * ld;
    for (int64_t c = 0; c < ld; ++c) row[c] = __float2bfloat16(0.f);
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += topk_w[t * K + k] * dw[t * K + k];
    for (int k = 0; k < K; ++k) {
        const float w = topk_w[t * K + k];
        row[topk_idx[t * K + k]] = __float2bfloat16(w * (dw[t * K + k] - s));
    }
}

}  // namespace hep

extern "C" int hep_moe_combine_bwd(const void *d_dout, const void *d_y, const int32_t *d_tok_row, const float *d_topk_w,
                                   int64_t T, int K, int64_t d_model, void *d_dy, float *d_dw, void *stream) {
    HEP_NVTX("hep_moe_combine_bwd");
    HEP_REQUIRE(d_dout && d_y && d_tok_row && d_topk_w && d_dy && d_dw, HEP_E_CONTRACT, "hep_moe_combine_bwd: null");
    HEP_REQUIRE(d_model % 8 == 0 && K >= 1 && K <= 16, HEP_E_DIMENSION, "hep_moe_combine_bwd: d_model %% 8, K<=16");
    if (T <= 0) return HEP_OK;
    const int grid = grid_for_warps(T);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nv = d_model / 8;
    switch (K) {
#define HEP_CB(KK)                                                                                                 \
        case KK:                                                                                                   \
            combine_bwd_kernel<KK><<<grid, 256, 0, st>>>((const int4 *)d_dout, (const int4 *)d_y, d_tok_row,       \
                                                         d_topk_w, T, nv, (int4 *)d_dy, d_dw);                     \
            break;
        HEP_CB(1) HEP_CB(2) HEP_CB(3) HEP_CB(4) HEP_CB(5) HEP_CB(6) HEP_CB(7) HEP_CB(8)
        HEP_CB(9) HEP_CB(10) HEP_CB(11) HEP_CB(12) HEP_CB(13) HEP_CB(14) HEP_CB(15) HEP_CB(16)
#undef HEP_CB
    }
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

namespace hep {
// EP training layout: the receive buffer is [src][hosted expert] (what the dispatch
// all-to-all delivers); the weight-gradient GEMMs need every local slot's rows as one
// block starting on a multiple of `align`.  Block b handles receive segment b = (src, h):
// it recomputes the per-slot totals and their aligned prefix (n_slots <= 1024, G <= 10:
// a few hundred adds) and writes row_map for the segment's rows; block 0 also writes
// the per-slot segments and the slot row offsets.
__global__ void __launch_bounds__(256) ep_layout_kernel(const int32_t *seg, int n_hosted, int G, int n_slots,
                                                        int align, int32_t *row_map, int64_t row_map_len,
                                                        int32_t *seg_out, int64_t *slot_rows) {
    extern __shared__ int64_t sm_tot[];  // [n_slots] totals, then aligned starts
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < n_slots; i += nt) sm_tot[i] = 0;
    __syncthreads();
    for (int h = tid; h < n_hosted; h += nt) {
        int64_t n = 0;
        for (int d = 0; d < G; ++d) n += seg[4 * (d * n_hosted + h) + 1];
        sm_tot[seg[4 * h + 2]] = n;
    }
    __syncthreads();
    if (tid == 0) {
        int64_t run = 0;
        for (int s = 0; s < n_slots; ++s) {
            const int64_t n = sm_tot[s];
            sm_tot[s] = run;
            if (blockIdx.x == 0) {
                slot_rows[s] = run;
                seg_out[4 * s] = (int32_t)run;
                seg_out[4 * s + 1] = (int32_t)n;
                seg_out[4 * s + 2] = s;
                seg_out[4 * s + 3] = 0;
            }
            run += (n + align - 1) / align * align;
        }
        if (blockIdx.x == 0) slot_rows[n_slots] = run;
    }
    __syncthreads();
    if (row_map_len > 0) {  // received rows past this micro-batch's count map to -1 (skipped)
        int64_t R = 0;
        for (int i = 0; i < G * n_hosted; ++i) R += seg[4 * i + 1];
        for (int64_t i = R + (int64_t)blockIdx.x * nt + tid; i < row_map_len; i += (int64_t)gridDim.x * nt)
            row_map[i] = -1;
    }
    if (n_hosted == 0) return;
    const int b = blockIdx.x, src = b / n_hosted, h = b % n_hosted;
    const int32_t *sg = seg + 4 * b;
    int64_t dst = sm_tot[sg[2]];
    for (int d = 0; d < src; ++d) dst += seg[4 * (d * n_hosted + h) + 1];
    const int32_t r0 = sg[0], n = sg[1];
    for (int i = tid; i < n; i += nt) row_map[r0 + i] = (int32_t)(dst + i);
}
}  // namespace hep

extern "C" int hep_moe_ep_train_layout(const int32_t *d_seg, int n_hosted, int G, int n_slots, int row_align,
                                       int32_t *d_row_map, int64_t row_map_len, int32_t *d_seg_out,
                                       int64_t *d_slot_rows, void *stream) {
    HEP_NVTX("hep_moe_ep_train_layout");
    HEP_REQUIRE(d_seg && d_row_map && d_seg_out && d_slot_rows, HEP_E_CONTRACT, "hep_moe_ep_train_layout: null");
    // G = the [src] blocks of d_seg: the group size, or twice it (the pipelined split's two phases)
    HEP_REQUIRE(G >= 1 && G <= 2 * HEP_MAX_GPUS && n_hosted >= 0 && n_slots >= n_hosted && n_slots <= 1024 &&
                    row_align >= 1,
                HEP_E_DIMENSION, "hep_moe_ep_train_layout: G %d n_hosted %d n_slots %d align %d", G, n_hosted,
                n_slots, row_align);
    if (n_slots == 0) return HEP_OK;
    const int blocks = n_hosted > 0 ? G * n_hosted : 1;
    ep_layout_kernel<<<blocks, 256, sizeof(int64_t) * n_slots, (cudaStream_t)stream>>>(
        d_seg, n_hosted, G, n_slots, row_align, d_row_map, row_map_len, d_seg_out, d_slot_rows);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_moe_zero_padding(const int64_t *d_expert_rows, const int32_t *d_seg, int n_seg, int E, void *d_buf,
                                    int64_t width, void *stream) {
    HEP_REQUIRE(d_expert_rows && d_seg && d_buf && width % 8 == 0, HEP_E_CONTRACT, "hep_moe_zero_padding");
    if (E <= 0) return HEP_OK;
    zero_pad_rows_kernel<<<E, 256, 0, (cudaStream_t)stream>>>(d_expert_rows, d_seg, n_seg, E, width / 8, (int4 *)d_buf);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_gate_bwd(const int32_t *d_topk_idx, const float *d_topk_w, const float *d_dw, int64_t T, int K,
                            int64_t ld, void *d_dlogits, void *stream) {
    HEP_NVTX("hep_gate_bwd");
    HEP_REQUIRE(d_topk_idx && d_topk_w && d_dw && d_dlogits && K >= 1 && K <= ld, HEP_E_CONTRACT, "hep_gate_bwd");
    if (T <= 0) return HEP_OK;
    gate_bwd_kernel<<<(unsigned)((T + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_topk_idx, d_topk_w, d_dw, T, K, ld,
                                                                                   (__nv_bfloat16 *)d_dlogits);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}
