// sched.cu — K3: the per-micro-batch balanced token scheduler on one CTA.
//
// Replaces, bit-exactly, the reference chain (paths under
// /root/reference/pkg/src/harmonyep/):
//   solve_replica_loads / warm_solve    scheduler.py:337-461  (exact m + lex-min plan)
//   integerize_plan                     scheduler.py:697-735
//   route_tokens / route_topology_aware router.py:114-175     (Algorithm 1)
//   build_transfer_plan                 router.py:178-226
//
// Device algorithm (not a port of the reference's Dinic max-flow): the
// subset (Gale/Hall) formulation of SURVEY.md Appendix B.
//   1. stage the load matrix in shared memory; totals[e] = row sums   (core.py:261)
//   2. W[S] = summed totals of experts whose EDP group ⊆ S: zeta transform
//      over the 2^G GPU subsets (placement.py:131-143's transform)
//   3. m = max_S (W[S] + base(S)) / |S| — the exact min-max GPU load (Eq. 3;
//      the fixpoint of the reference's probe / min-cut loop :354-371)
//   4. lex-min canonical plan (scheduler.py:295-321): for arcs (e, g) in
//      (expert, gpu) order the minimum feasible replica load is
//        v = max(0, max_{S ⊇ need, g ∉ S} r + Wf[S] - C[S])
//      with need = remaining group \ {g}, Wf = not-yet-processed load inside
//      S, C = remaining capacity of S.  One warp holds all 2^G subsets in
//      registers (SPL per lane); when every value fits 31 bits the per-arc
//      reduction is a single redux.sync (int32 path), else int64 shuffles.
//   5. integerize (largest remainder, ties -> lowest GPU id), one thread per
//      expert, shared-memory plan
//   6. Algorithm 1 routing, one thread per contiguous expert chunk, two passes
//      (count, block scan, emit) so the table comes out in expert order; the
//      pairwise transfer counts are accumulated with integer shared-memory
//      atomics during emission (order-independent, deterministic)
//   7. transfer plan vectors from the pair matrix
// Everything is exact integer arithmetic in units of 1/Q, Q = lcm(1..G)
// (scheduler.py:184).
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"
#include "sched_internal.cuh"

namespace hep {

constexpr int kSchedThreads = 256;
constexpr int kSchedSmemMax = 227 * 1024 - 1024;  // opt-in dynamic shared memory per block, minus the static arrays
constexpr int kProfSlots = 16;
__device__ long long g_sched_prof[kProfSlots];

struct SchedArgs {
    int G, E, nnz, gpn, flags;
    int64_t Q, max_ranges, den;  // den: denominator of the input plan (Q when solved here)
    const int32_t *grp_off, *grp_gpu, *sorted;
    const uint32_t *mask;
    const int8_t *kidx;
    const int64_t *loads;
    int64_t se, sg;
    const int64_t *base;
    const int64_t *xi_in;  // route-only: caller plan (global)
    int status_in;         // keep an error already in out.d_status (set by a preceding kernel)
    int lexmin_warps;      // warps on the lex-min arc chain (8 = whole block, 4)
    int route_serial;      // Algorithm 1 as per-thread merges only (no route_lanes)
    hep_sched_out out;
};

struct SchedSmem {
    int64_t *totals;    // [E]
    int64_t *W;         // [2^G]
    int64_t *C;         // [2^G] capacity of each GPU subset at the optimum
    int64_t *loads;     // [E*G]
    int64_t *xq;        // [nnz]
    int64_t *xi;        // [nnz]
    int64_t *gpu_load;  // [G]
    unsigned long long *pair;  // [G*G]
    int64_t *scan;      // [kSchedThreads/32 + 2]
    int64_t *misc;      // [8]
    int32_t *grp_off;   // [E+1]
    int32_t *grp_gpu;   // [nnz] list order
    int32_t *arc_idx;   // [nnz] arcs in (e, gpu id) order: nnz index
    int32_t *arc_gpu;   // [nnz] arcs in (e, gpu id) order: gpu
    uint32_t *mask;     // [E]
    int4 *emeta;        // [E] (arc base, #arcs, group mask, load*Q when it fits 32 bits)
    int8_t *kidx;       // [E*G] list position of GPU g in expert e's group, -1 if absent
    int16_t *rc;        // [2*E*G] per-(expert, source) range counts: phase 1, final merge (<= 3d + 2G)
};

__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }

// Row stride (int64 elements) of the staged load matrix: odd, so the per-expert rows that
// one warp reads together (thread = expert in the routing passes) fall into different
// shared-memory banks instead of the 16-way conflict of a G = 8 stride.
__host__ __device__ inline int loads_stride(int G) { return G | 1; }

__host__ __device__ inline size_t sched_smem_bytes(int G, int E, int nnz) {
    const size_t ns = size_t(1) << G;
    return align8(8 * (size_t)E) + 2 * align8(8 * ns) + align8(8 * (size_t)E * loads_stride(G)) +
           2 * align8(8 * (size_t)nnz) +
           align8(8 * (size_t)G) + align8(8 * (size_t)G * G) + align8(8 * (kSchedThreads / 32 + 2)) + 64 +
           align8(4 * (size_t)(E + 1)) + 3 * align8(4 * (size_t)nnz) + align8(4 * (size_t)E) + 16 * (size_t)E +
           align8((size_t)E * G) + 4 * (size_t)E * G;
}

__device__ inline SchedSmem carve(char *p, int G, int E, int nnz) {
    SchedSmem s;
    const size_t ns = size_t(1) << G;
    s.emeta = (int4 *)p; p += 16 * (size_t)E;  // first: 16-byte aligned
    s.totals = (int64_t *)p; p += align8(8 * (size_t)E);
    s.W = (int64_t *)p; p += align8(8 * ns);
    s.C = (int64_t *)p; p += align8(8 * ns);
    s.loads = (int64_t *)p; p += align8(8 * (size_t)E * loads_stride(G));
    s.xq = (int64_t *)p; p += align8(8 * (size_t)nnz);
    s.xi = (int64_t *)p; p += align8(8 * (size_t)nnz);
    s.gpu_load = (int64_t *)p; p += align8(8 * (size_t)G);
    s.pair = (unsigned long long *)p; p += align8(8 * (size_t)G * G);
    s.scan = (int64_t *)p; p += align8(8 * (kSchedThreads / 32 + 2));
    s.misc = (int64_t *)p; p += 64;
    s.grp_off = (int32_t *)p; p += align8(4 * (size_t)(E + 1));
    s.grp_gpu = (int32_t *)p; p += align8(4 * (size_t)nnz);
    s.arc_idx = (int32_t *)p; p += align8(4 * (size_t)nnz);
    s.arc_gpu = (int32_t *)p; p += align8(4 * (size_t)nnz);
    s.mask = (uint32_t *)p; p += align8(4 * (size_t)E);
    s.kidx = (int8_t *)p; p += align8((size_t)E * G);
    s.rc = (int16_t *)p;
    return s;
}

// a/b > c/d with denominators |S| <= HEP_MAX_GPUS and numerators < 2^56
// (capacity-checked), so the cross products fit int64
__device__ __forceinline__ bool frac_gt(int64_t a, int64_t b, int64_t c, int64_t d) { return a * d > c * b; }

__device__ __forceinline__ int64_t gcd_i64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

__device__ __forceinline__ void prof_mark(int flags, int slot) {
    if ((flags & HEP_SCHED_PROFILE) && threadIdx.x == 0 && slot < kProfSlots) g_sched_prof[slot] = clock64();
}

// warp min of non-negative values
__device__ __forceinline__ uint32_t wmin(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint64_t wmin(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// floor(v / d) for d > 0 without the 64-bit division routine: a double
// estimate corrected to the exact quotient (|v| < 2^62 capacity-checked)
__device__ __forceinline__ int64_t floordiv(int64_t v, int64_t d) {
    int64_t q = (int64_t)floor((double)v / (double)d);
    int64_t r = v - q * d;
    while (r < 0) { --q; r += d; }
    while (r >= d) { ++q; r -= d; }
    return q;
}

// ---------------------------------------------------------------------------
// step 4: lex-min canonical plan, whole block.  Every thread keeps the slack
// C[S] - Wf[S] >= 0 of its SPB subsets (S = tid + 256 j); the minimum feasible
// load of arc (e, g) is v = max(0, r - min{slack[S] : S ⊇ need, g ∉ S}): a
// warp redux.sync per warp, the 8 warp minima through shared memory (double
// buffered by arc parity, one barrier per arc), then every thread applies the
// same decision to its subsets.  Result of arc p (position in (expert, gpu id)
// order) goes to vtmp[p].  U = uint32_t when every slack and load fits 32 bits.
// ---------------------------------------------------------------------------
template <typename U, int NW = kSchedThreads / 32>
__device__ __forceinline__ U block_min(U v, U (*red)[kSchedThreads / 32], int &par) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = wmin(v);
    if (lane == 0) red[par][w] = v;
    if constexpr (NW == kSchedThreads / 32) __syncthreads();
    else asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
    U m;
    if constexpr (sizeof(U) == 4 && NW == 4) {  // the four partials in one 16-byte load
        const uint4 q = *reinterpret_cast<const uint4 *>(red[par]);
        m = (U)min(min(q.x, q.y), min(q.z, q.w));
    } else {
        m = red[par][0];
#pragma unroll
        for (int i = 1; i < NW; ++i) m = red[par][i] < m ? red[par][i] : m;
    }
    par ^= 1;
    return m;
}

template <int SPB, typename U, int NT = kSchedThreads>
__device__ void lexmin_block(const SchedArgs &a, SchedSmem &s, int64_t *vtmp) {
    __shared__ __align__(16) U red[2][kSchedThreads / 32];
    const int tid = threadIdx.x;
    const int E = a.E;
    const uint32_t NS = 1u << a.G;
    const int64_t Q = a.Q;
    const U UMAX = ~(U)0;
    U sl[SPB];
    uint32_t valid = 0;
#pragma unroll
    for (int j = 0; j < SPB; ++j) {
        const uint32_t S = tid + NT * j;
        sl[j] = S < NS ? (U)(s.C[S] - s.W[S] * Q) : (U)0;
        valid |= (S < NS) << j;
    }
    int par = 0;
    int4 nxt = s.emeta[0];
    for (int e = 0; e < E; ++e) {
        const int b = nxt.x, n = nxt.y & 0xff, ga2 = (nxt.y >> 8) & 0xff, gc2 = (nxt.y >> 16) & 0xff;
        uint32_t R = (uint32_t)nxt.z;
        U r = sizeof(U) == 4 ? (U)(uint32_t)nxt.w : (U)(s.totals[e] * Q);
        if (e + 1 < E) nxt = s.emeta[e + 1];  // prefetch the next expert
        if (n == 0) continue;
        if (n == 1) {  // single replica: v = r; +r on S ⊇ {g} and -r on S ∋ g cancel
            if (tid == 0) vtmp[b] = (int64_t)r;
            continue;
        }
        if (n == 2) {
            // Two replicas a < c (the d=2 common case), folded into one reduction:
            // arc a's family {S : c ∈ S, a ∉ S} never contains R, so it sees the slack
            // before the "+r on S ⊇ R" step; the net update afterwards is -v_a on
            // S ∋ a, S ∌ c and -v_c on S ∋ c, S ∌ a (S ⊇ R: +r - v_a - v_c = 0).
            const int ga = ga2, gc = gc2;
            U mn = UMAX;
#pragma unroll
            for (int j = 0; j < SPB; ++j) {
                const uint32_t S = tid + NT * j;
                const bool ok = ((valid >> j) & 1) && ((S >> gc) & 1) && !((S >> ga) & 1);
                mn = (ok && sl[j] < mn) ? sl[j] : mn;
            }
            mn = block_min<U, NT / 32>(mn, red, par);
            const U v_a = r > mn ? r - mn : (U)0;
            const U v_c = r - v_a;
            if (tid == 0) {
                vtmp[b] = (int64_t)v_a;
                vtmp[b + 1] = (int64_t)v_c;
            }
#pragma unroll
            for (int j = 0; j < SPB; ++j) {
                const uint32_t S = tid + NT * j;
                const uint32_t ha = (S >> ga) & 1, hc = (S >> gc) & 1;
                sl[j] -= (ha & ~hc) ? v_a : ((hc & ~ha) ? v_c : (U)0);
            }
            continue;
        }
        if (r) {
#pragma unroll
            for (int j = 0; j < SPB; ++j) {
                const uint32_t S = tid + NT * j;
                sl[j] += ((S & R) == R) ? r : (U)0;  // expert e leaves the not-yet-processed set
            }
        }
        for (int k = 0; k < n; ++k) {
            const int g = s.arc_gpu[b + k];
            const uint32_t gbit = 1u << g;
            const uint32_t need = R & ~gbit;
            U v;
            if (r == 0) {
                v = 0;  // every bound r - slack is <= 0
            } else if (need == 0) {
                v = r;  // S = {} has slack 0; every other bound is <= r
            } else {
                U mn = UMAX;
#pragma unroll
                for (int j = 0; j < SPB; ++j) {
                    const uint32_t S = tid + NT * j;
                    const bool ok = ((valid >> j) & 1) && ((S & need) == need) && !(S & gbit);
                    mn = (ok && sl[j] < mn) ? sl[j] : mn;
                }
                mn = block_min<U, NT / 32>(mn, red, par);
                v = r > mn ? r - mn : (U)0;
            }
            if (tid == 0) vtmp[b + k] = (int64_t)v;
            r -= v;
            R = need;
            if (v) {
#pragma unroll
                for (int j = 0; j < SPB; ++j) {
                    const uint32_t S = tid + NT * j;
                    sl[j] -= (S & gbit) ? v : (U)0;  // capacity of every subset holding g drops by v
                }
            }
        }
    }
}

// 64-bit shared-memory accumulation (pair matrix, W[S], GPU loads) with native 32-bit
// atomics (the 64-bit atomicAdd on shared memory is a CAS spin loop, slow under the
// same-address contention of E experts adding into 2^G or G*G slots):
// the low word's returned old value gives this add's carry, so the high word receives
// exactly the carries of every add -- the little-endian u64 view holds the exact sum.
__device__ __forceinline__ void pair_add(unsigned long long *p, int64_t y) {
    uint32_t *w = reinterpret_cast<uint32_t *>(p);
    const uint32_t lo = (uint32_t)y, hi = (uint32_t)((uint64_t)y >> 32);
    const uint32_t old = atomicAdd(w, lo);
    const uint32_t up = hi + (uint32_t)(old + lo < old);
    if (up) atomicAdd(w + 1, up);
}

// One routing-table row (expert, src, dst, count) as a single 256-bit store when the table
// is 32-byte aligned (every row then is): a quarter of the store instructions the table
// costs otherwise -- they queue ahead of the kernel's later global accesses.
__device__ __forceinline__ void put_range(int64_t *r_, int64_t e, int64_t src, int64_t dst, int64_t y) {
    if (((uintptr_t)r_ & 31) == 0) {
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(r_),
                     "r"((uint32_t)e), "r"((uint32_t)(e >> 32)), "r"((uint32_t)src), "r"((uint32_t)(src >> 32)),
                     "r"((uint32_t)dst), "r"((uint32_t)(dst >> 32)), "r"((uint32_t)y), "r"((uint32_t)(y >> 32))
                     : "memory");
    } else {
        r_[0] = e; r_[1] = src; r_[2] = dst; r_[3] = y;
    }
}

// Non-topology routing, one thread per (expert e, source src): the phase-1
// range of src (if it hosts e) and src's ranges of the final merge, whose
// offset A_src is the prefix of the remaining source amounts and whose
// replica intervals start at the prefix B_k of the remaining quotas.  c1/c2
// return the counts; EMIT writes them at pos1 / pos2.
template <bool EMIT>
__device__ void route_pair(const SchedArgs &a, SchedSmem &s, int e, int src, int *c1, int *c2, int64_t pos1,
                           int64_t pos2) {
    const int G = a.G;
    const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
    const int64_t *L = s.loads + (size_t)e * loads_stride(G);
    const int8_t *kx = s.kidx + (size_t)e * G;
    auto rem_of = [&](int g) -> int64_t {
        const int kk = kx[g];
        if (kk < 0) return L[g];
        const int64_t d = L[g] - s.xi[b + kk];
        return d > 0 ? d : 0;
    };
    const int kk = kx[src];
    const int64_t in = L[src];
    const int64_t y1 = kk >= 0 ? (in < s.xi[b + kk] ? in : s.xi[b + kk]) : 0;
    *c1 = y1 > 0;
    if (EMIT && y1 > 0) {
        int64_t *r_ = a.out.d_ranges + 4 * pos1;
        put_range(r_, e, src, src, y1);
        pair_add(&s.pair[src * G + src], y1);
    }
    const int64_t rem = rem_of(src);
    int cnt = 0;
    if (rem > 0) {
        int64_t A = 0;
        for (int g = 0; g < src; ++g) A += rem_of(g);
        int64_t B = 0;
        for (int k = 0; k < n && B < A + rem; ++k) {
            const int dst = s.grp_gpu[b + k];
            const int64_t qd = s.xi[b + k] - L[dst];
            const int64_t q = qd > 0 ? qd : 0;
            const int64_t lo = A > B ? A : B, hi = (A + rem) < (B + q) ? (A + rem) : (B + q);
            if (hi > lo) {
                if (EMIT) {
                    int64_t *r_ = a.out.d_ranges + 4 * (pos2 + cnt);
                    put_range(r_, e, src, dst, hi - lo);
                    pair_add(&s.pair[src * G + dst], hi - lo);
                }
                ++cnt;
            }
            B += q;
        }
    }
    *c2 = cnt;
}

// Segmented scans over W-lane groups (W = 8 / 16, one group per expert).
template <typename T>
__device__ __forceinline__ T seg_incl_scan(T v, int idx, int W) {
#pragma unroll
    for (int d = 1; d < 16; d <<= 1) {
        if (d >= W) break;
        const T t = __shfl_up_sync(0xffffffffu, v, d, W);
        if (idx >= d) v += t;
    }
    return v;
}

// Algorithm 1 with one lane per (expert, source): W lanes per expert (W = 8 for G <= 8,
// else 16), 32 / W experts per warp per step.  The same table as route_pair (phase-1 range
// of src, then src's pieces of the final sweep, whose offset A_src is the segmented prefix
// of the remaining source amounts), but the per-expert prefixes -- A_src and the table
// positions -- are warp shuffles instead of per-thread loops.  COUNT pass: ecount[e] =
// the expert's number of ranges; EMIT pass: ranges from ecount[e] (scanned) on.
template <bool EMIT>
__device__ void route_lanes(const SchedArgs &a, SchedSmem &s, int64_t *ecount) {
    const int G = a.G, E = a.E;
    const int W = G <= 8 ? 8 : 16;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int epw = 32 / W, sub = lane / W, src = lane % W;
    for (int e0 = warp * epw; e0 < E; e0 += nw * epw) {  // uniform per warp: shuffles see all lanes
        const int e = e0 + sub;
        const bool ok = e < E && src < G;
        int b = 0, n = 0;
        const int64_t *L = nullptr;
        int64_t y1 = 0, rem = 0;
        if (ok) {
            b = s.grp_off[e];
            n = s.grp_off[e + 1] - b;
            L = s.loads + (size_t)e * loads_stride(G);
            const int kk = s.kidx[(size_t)e * G + src];
            const int64_t in = L[src];
            if (kk >= 0) {
                const int64_t xk = s.xi[b + kk];
                y1 = in < xk ? in : xk;
                rem = in > xk ? in - xk : 0;
            } else {
                rem = in;
            }
        }
        const int64_t A = seg_incl_scan<int64_t>(rem, src, W) - rem;
        int c2 = 0;
        int64_t pos2 = 0;
        int c1 = y1 > 0;
        const int i1 = seg_incl_scan<int>(c1, src, W);
        const int n1 = __shfl_sync(0xffffffffu, i1, W - 1, W);
        int pass_c2 = 0;
        if (ok && rem > 0) {  // count this source's pieces of the sweep
            int64_t B = 0;
            for (int k = 0; k < n && B < A + rem; ++k) {
                const int64_t qd = s.xi[b + k] - L[s.grp_gpu[b + k]];
                const int64_t q = qd > 0 ? qd : 0;
                const int64_t lo = A > B ? A : B, hi = (A + rem) < (B + q) ? (A + rem) : (B + q);
                pass_c2 += hi > lo;
                B += q;
            }
        }
        const int i2 = seg_incl_scan<int>(pass_c2, src, W);
        const int n2 = __shfl_sync(0xffffffffu, i2, W - 1, W);
        if (!EMIT) {
            if (ok && src == 0) ecount[e] = (int64_t)n1 + n2;
            continue;
        }
        if (!ok) continue;
        const int64_t base = ecount[e];
        if (y1 > 0) {
            int64_t *r_ = a.out.d_ranges + 4 * (base + i1 - 1);
            put_range(r_, e, src, src, y1);
            pair_add(&s.pair[src * G + src], y1);
        }
        if (rem > 0) {
            pos2 = base + n1 + (i2 - pass_c2);
            int64_t B = 0;
            for (int k = 0; k < n && B < A + rem; ++k) {
                const int dst = s.grp_gpu[b + k];
                const int64_t qd = s.xi[b + k] - L[dst];
                const int64_t q = qd > 0 ? qd : 0;
                const int64_t lo = A > B ? A : B, hi = (A + rem) < (B + q) ? (A + rem) : (B + q);
                if (hi > lo) {
                    int64_t *r_ = a.out.d_ranges + 4 * (pos2 + c2);
                    put_range(r_, e, src, dst, hi - lo);
                    pair_add(&s.pair[src * G + dst], hi - lo);
                    ++c2;
                }
                B += q;
            }
        }
    }
}

// One thread per expert (used when E is large enough to fill the block):
// phase 1 in sorted(group) order, then the final sweep as the two-pointer
// merge of the remaining source amounts (src order) with the remaining
// quotas (list order) — each emitting step of the reference sweep exhausts
// either the current source or the current replica.
template <bool EMIT>
__device__ int route_expert_merge(const SchedArgs &a, SchedSmem &s, int e, int64_t pos) {
    const int G = a.G;
    const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
    const int64_t *L = s.loads + (size_t)e * loads_stride(G);
    const int8_t *kx = s.kidx + (size_t)e * G;
    int cnt = 0;
    auto emit = [&](int src, int dst, int64_t y) {
        if (EMIT) {
            int64_t *r_ = a.out.d_ranges + 4 * (pos + cnt);
            put_range(r_, e, src, dst, y);
            pair_add(&s.pair[src * G + dst], y);
        }
        ++cnt;
    };
    for (int k = 0; k < n; ++k) {
        const int g = s.arc_gpu[b + k];
        const int64_t x = s.xi[s.arc_idx[b + k]];
        const int64_t y = L[g] < x ? L[g] : x;
        if (y > 0) emit(g, g, y);
    }
    auto rem_of = [&](int g) -> int64_t {
        const int kk = kx[g];
        if (kk < 0) return L[g];
        const int64_t d = L[g] - s.xi[b + kk];
        return d > 0 ? d : 0;
    };
    auto quota_of = [&](int kk) -> int64_t {
        const int64_t d = s.xi[b + kk] - L[s.grp_gpu[b + kk]];
        return d > 0 ? d : 0;
    };
    int src = 0, k = 0;
    int64_t rem = rem_of(0), q = n > 0 ? quota_of(0) : 0;
    while (true) {
        while (rem == 0) {
            if (++src >= G) return cnt;
            rem = rem_of(src);
        }
        while (q == 0) {
            if (++k >= n) return cnt;
            q = quota_of(k);
        }
        const int64_t y = rem < q ? rem : q;
        emit(src, s.grp_gpu[b + k], y);
        rem -= y;
        q -= y;
    }
}

// Topology-aware variant (router.py:136-147): sequential per expert, one thread.
template <bool EMIT>
__device__ int route_expert_topo(const SchedArgs &a, SchedSmem &s, int e, int64_t pos, int32_t *status) {
    const int G = a.G;
    const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
    int64_t rin[HEP_MAX_GPUS], rx[HEP_MAX_GPUS];
    int64_t tot = 0, xs = 0;
    for (int g = 0; g < G; ++g) { rin[g] = s.loads[e * loads_stride(G) + g]; rx[g] = 0; tot += rin[g]; }
    if (n == 0 && tot == 0) return 0;
    bool neg = false;
    for (int k = 0; k < n; ++k) {
        const int64_t v = s.xi[b + k];
        neg |= v < 0;
        xs += v;
        rx[s.grp_gpu[b + k]] = v;
    }
    if (neg || xs != tot) { set_status(status, HEP_E_CONTRACT); return 0; }
    int cnt = 0;
    auto emit = [&](int src, int dst, int64_t y) {
        if (EMIT) {
            int64_t *r_ = a.out.d_ranges + 4 * (pos + cnt);
            put_range(r_, e, src, dst, y);
            pair_add(&s.pair[src * G + dst], y);
        }
        ++cnt;
    };
    for (int k = 0; k < n; ++k) {  // phase 1, sorted(group)
        const int g = s.arc_gpu[b + k];
        const int64_t y = rin[g] < rx[g] ? rin[g] : rx[g];
        if (y > 0) { emit(g, g, y); rin[g] -= y; rx[g] -= y; }
    }
    for (int src = 0; src < G; ++src) {  // phase 2: same node
        if (rin[src] == 0) continue;
        for (int k = 0; k < n; ++k) {
            const int dst = s.grp_gpu[b + k];
            if (dst == src || dst / a.gpn != src / a.gpn) continue;
            const int64_t y = rin[src] < rx[dst] ? rin[src] : rx[dst];
            if (y > 0) { emit(src, dst, y); rin[src] -= y; rx[dst] -= y; }
        }
    }
    for (int src = 0; src < G; ++src) {  // final phase
        if (rin[src] == 0) continue;
        for (int k = 0; k < n; ++k) {
            const int dst = s.grp_gpu[b + k];
            const int64_t y = rin[src] < rx[dst] ? rin[src] : rx[dst];
            if (y > 0) { emit(src, dst, y); rin[src] -= y; rx[dst] -= y; }
        }
    }
    return cnt;
}

// On a device-detected error the kernel leaves an EMPTY plan instead of the previous
// micro-batch's: no integerized rows, no ranges, zero GPU loads and transfer counts, so
// the kernels queued behind it on the stream (assignment, dispatch, FFN) see no work
// rather than a stale schedule that no longer matches this micro-batch's top-K.
__device__ void clear_outputs(const SchedArgs &a, int tid, int nt) {
    const bool integ = a.flags & (HEP_SCHED_SOLVE | HEP_SCHED_INTEGERIZE);
    if (integ && a.out.d_xi && a.out.d_xi != a.xi_in)
        for (int i = tid; i < a.nnz; i += nt) a.out.d_xi[i] = 0;
    if (integ && a.out.d_gpu_load)
        for (int g = tid; g < a.G; g += nt) a.out.d_gpu_load[g] = 0;
    if ((a.flags & HEP_SCHED_ROUTE) && a.out.d_n_ranges && tid == 0) *a.out.d_n_ranges = 0;
    if ((a.flags & HEP_SCHED_ROUTE) && (a.flags & HEP_SCHED_TRANSFER) && a.out.d_transfer)
        for (int i = tid; i < a.G * a.G + 8 * a.G + 2; i += nt) a.out.d_transfer[i] = 0;
}

template <int SPL>
__global__ void __launch_bounds__(kSchedThreads, 1) sched_kernel(SchedArgs a) {
    extern __shared__ __align__(16) char smem_raw[];
    SchedSmem s = carve(smem_raw, a.G, a.E, a.nnz);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int G = a.G, E = a.E, nnz = a.nnz;
    const int NS = 1 << G;
    int32_t *status = a.out.d_status;
    const bool solve = a.flags & HEP_SCHED_SOLVE;
    const bool route = a.flags & HEP_SCHED_ROUTE;
    prof_mark(a.flags, 0);

    // ---- step 1: stage placement + loads (+ caller plan) in shared memory -------
    for (int i = tid; i <= E; i += nt) s.grp_off[i] = a.grp_off[i];
    for (int i = tid; i < E; i += nt) s.mask[i] = a.mask[i];
    for (int i = tid; i < E * G; i += nt) s.kidx[i] = a.kidx[i];
    for (int i = tid; i < nnz; i += nt) {
        const int idx = a.sorted[i];
        s.arc_idx[i] = idx;
        s.arc_gpu[i] = a.grp_gpu[idx];
        s.grp_gpu[i] = a.grp_gpu[i];
        if (!solve) s.xq[i] = a.out.d_xq[i];
        if (a.xi_in) s.xi[i] = a.xi_in[i];
    }
    const bool need_loads = solve || route;
    int bad = 0;
    if (need_loads) {
        for (int i = tid; i < E * G; i += nt) {
            const int e = i / G, g = i - e * G;
            const int64_t v = a.loads[(int64_t)e * a.se + (int64_t)g * a.sg];
            bad |= v < 0;
            s.loads[e * loads_stride(G) + g] = v;
        }
    }
    for (int i = tid; i < G * G; i += nt) s.pair[i] = 0;
    for (int g = tid; g < G; g += nt) s.gpu_load[g] = 0;
    if (tid == 0 && !a.status_in) *status = 0;
    __syncthreads();
    if (bad) set_status(status, HEP_E_CONTRACT);
    int64_t my_total = 0;
    if (need_loads) {
        for (int e = tid; e < E; e += nt) {
            int64_t t = 0;
            for (int g = 0; g < G; ++g) t += s.loads[e * loads_stride(G) + g];
            s.totals[e] = t;
            my_total += t;
            // scheduler.py:344-347: a loaded expert with an empty EDP group
            if (solve && t > 0 && s.grp_off[e + 1] == s.grp_off[e]) set_status(status, HEP_E_PLACEMENT);
        }
    }
    int64_t base_sum = 0;
    if (tid == 0 && a.base)
        for (int g = 0; g < G; ++g) base_sum += a.base[g];
    const int64_t total_all = block_sum_i64(my_total + base_sum, s.scan);
    if (solve && (__int128)total_all * a.Q >= ((__int128)1 << 56)) set_status(status, HEP_E_CAPACITY);
    __syncthreads();
    if (*status) { clear_outputs(a, tid, nt); return; }
    prof_mark(a.flags, 1);

    if (solve) {
        // ---- step 2: zeta transform over GPU subsets --------------------------
        for (int S = tid; S < NS; S += nt) s.W[S] = 0;
        __syncthreads();
        for (int e = tid; e < E; e += nt)
            if (s.totals[e] > 0 && s.mask[e])
                pair_add((unsigned long long *)&s.W[s.mask[e]], s.totals[e]);
        __syncthreads();
        for (int bit = 0; bit < G; ++bit) {
            for (int S = tid; S < NS; S += nt)
                if ((S >> bit) & 1) s.W[S] += s.W[S ^ (1 << bit)];
            __syncthreads();
        }
        // ---- step 3: m = max subset density (Eq. 3) ---------------------------
        int64_t bn = 0, bd = 1;
        if (tid == 0 && a.base)  // candidate max(base) (scheduler.py:357)
            for (int g = 0; g < G; ++g)
                if (a.base[g] > bn) bn = a.base[g];
        for (int S = tid + 1; S < NS; S += nt) {
            int64_t num = s.W[S];
            if (a.base)
                for (int g = 0; g < G; ++g)
                    if ((S >> g) & 1) num += a.base[g];
            const int64_t den = __popc(S);
            if (frac_gt(num, den, bn, bd)) { bn = num; bd = den; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int64_t on = __shfl_xor_sync(0xffffffffu, bn, o), od = __shfl_xor_sync(0xffffffffu, bd, o);
            if (frac_gt(on, od, bn, bd)) { bn = on; bd = od; }
        }
        __shared__ int64_t red_n[kSchedThreads / 32], red_d[kSchedThreads / 32];
        if ((tid & 31) == 0) { red_n[tid >> 5] = bn; red_d[tid >> 5] = bd; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nt / 32; ++w)
                if (frac_gt(red_n[w], red_d[w], bn, bd)) { bn = red_n[w]; bd = red_d[w]; }
            int64_t g = gcd_i64(bd, bn - floordiv(bn, bd) * bd);  // den <= G: one reduction step
            if (g == 0) g = 1;
            bn /= g;
            bd /= g;
            s.misc[0] = bn * (a.Q / bd);  // m scaled by Q (scheduler.py:267)
            a.out.d_m[0] = bn;
            a.out.d_m[1] = bd;
            a.out.d_m[2] = a.Q;
        }
        __syncthreads();
        // capacity of every GPU subset: C[S] = sum_{g in S} max(mQ - base_g*Q, 0)
        {
            const int64_t mQ = s.misc[0];
            for (int S = tid; S < NS; S += nt) {
                int64_t c = 0;
#pragma unroll 1
                for (int g = 0; g < G; ++g) {
                    if (!((S >> g) & 1)) continue;
                    const int64_t cg = mQ - (a.base ? a.base[g] * a.Q : 0);
                    c += cg > 0 ? cg : 0;
                }
                s.C[S] = c;
            }
        }
        for (int e = tid; e < E; e += nt) {
            // .y = #arcs | first two arc GPUs << 8 / << 16 (the d = 2 step reads no arc table)
            const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
            const int y = n | (n >= 2 ? (s.arc_gpu[b] << 8) | (s.arc_gpu[b + 1] << 16) : 0);
            s.emeta[e] = make_int4(b, y, (int)s.mask[e], (int)(uint32_t)(s.totals[e] * a.Q));
        }
        __syncthreads();
        prof_mark(a.flags, 2);
        // ---- step 4: lex-min canonical plan ------------------------------------
        {
            const int64_t mQ = s.misc[0];
            const bool fits32 = (__int128)G * (total_all + 1) * a.Q < ((__int128)1 << 31) &&
                                (__int128)G * (mQ + 1) < ((__int128)1 << 31);
            constexpr int SPB = SPL >= 8 ? SPL / 8 : 1;  // subsets per thread (2^G / 256)
            constexpr int SPB4 = SPL >= 4 ? SPL / 4 : 1;  // ... with 4 warps (2^G / 128)
            if (a.lexmin_warps == 4) {  // half the block: fewer warps meet at each arc's barrier
                if (threadIdx.x < 128) {
                    if (fits32) lexmin_block<SPB4, uint32_t, 128>(a, s, s.xi);
                    else lexmin_block<SPB4, uint64_t, 128>(a, s, s.xi);
                }
            } else if (fits32) {
                lexmin_block<SPB, uint32_t>(a, s, s.xi);
            } else {
                lexmin_block<SPB, uint64_t>(a, s, s.xi);
            }
        }
        __syncthreads();
        for (int p = tid; p < nnz; p += nt) {  // (expert, gpu id) order -> EDP list order
            const int64_t v = s.xi[p];
            s.xq[s.arc_idx[p]] = v;
            a.out.d_xq[s.arc_idx[p]] = v;
        }
        __syncthreads();
        prof_mark(a.flags, 3);
    }

    // ---- step 5: integerize (largest remainder, ties -> lowest GPU id) -----------
    if (a.flags & HEP_SCHED_INTEGERIZE) {
        const int64_t den = solve ? a.Q : a.den;
        for (int e = tid; e < E; e += nt) {
            const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
            int64_t total = 0, sum_floor = 0;
            for (int k = 0; k < n; ++k) {
                const int64_t v = s.xq[b + k];
                const int64_t fl = floordiv(v, den);
                s.xi[b + k] = fl;
                sum_floor += fl;
                total += v;
            }
            // round(total) must be an integer within 1e-6 (scheduler.py:706-713);
            // Python rounds half to even
            const int64_t t_fl = floordiv(total, den);
            const int64_t t_rem = total - t_fl * den;
            int64_t rounded = t_fl;
            if (t_rem > den - t_rem || (t_rem == den - t_rem && (t_fl & 1))) rounded = t_fl + 1;
            int64_t diff = total - rounded * den;
            if (diff < 0) diff = -diff;
            if ((__int128)diff * 1000000 > den) { set_status(status, HEP_E_CONTRACT); continue; }
            const int64_t units = rounded - sum_floor;
            for (int u = 0; u < units && u < n; ++u) {
                int best = -1, best_gpu = 0;
                int64_t best_rem = -1;
                for (int k = 0; k < n; ++k) {
                    const int64_t rem = s.xq[b + k] - s.xi[b + k] * den;
                    if (rem < 0) continue;  // already rounded up
                    const int gg = s.grp_gpu[b + k];
                    if (best < 0 || rem > best_rem || (rem == best_rem && gg < best_gpu)) {
                        best = k;
                        best_rem = rem;
                        best_gpu = gg;
                    }
                }
                if (best < 0) break;
                s.xi[b + best] += 1;
            }
            for (int k = 0; k < n; ++k)
                pair_add((unsigned long long *)&s.gpu_load[s.grp_gpu[b + k]], s.xi[b + k]);
        }
        __syncthreads();
        for (int i = tid; i < nnz; i += nt) a.out.d_xi[i] = s.xi[i];
        if (tid == 0) {
            int64_t mx = 0;
            for (int g = 0; g < G; ++g) {
                a.out.d_gpu_load[g] = s.gpu_load[g];
                if (g == 0 || s.gpu_load[g] > mx) mx = s.gpu_load[g];
            }
            a.out.d_m[3] = mx;
        }
        __syncthreads();
        prof_mark(a.flags, 4);
    }
    if (*status) { clear_outputs(a, tid, nt); return; }

    // ---- step 6: Algorithm 1 routing (router.py:114-158) --------------------------
    if (route) {
        const bool topo = (a.flags & HEP_SCHED_TOPO) && a.gpn > 0 && a.gpn < G;
        // pass 0: range counts (one thread per (expert, source); per expert for topology routing)
        int64_t *ecount = s.totals;  // totals are no longer needed once the plan exists
        int16_t *rc1 = s.rc, *rc2 = s.rc + E * G;
        // one lane per (expert, source) (route_lanes) while that is one step per warp
        // (E <= 32 at G <= 8): 6.1K vs 9.5K cycles at E = 8; from E = 128 on the per-thread
        // merges win (14.1K vs 15.6K at E = 128, profiles/r02/sched_ab_notes.md);
        // hep_tuning.sched_route_serial = 1 forces the per-thread merges
        const bool lanes = !topo && !a.route_serial && E * (G <= 8 ? 8 : 16) <= nt;
        const bool per_expert = !topo && !lanes && E >= nt / 4;  // enough experts to fill the block
        if (lanes) {
            route_lanes<false>(a, s, ecount);
            for (int e = tid; e < E; e += nt) {  // _check_plan (router.py:97-111)
                const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
                int64_t tot = 0, xs = 0;
                bool neg = false;
                for (int g = 0; g < G; ++g) tot += s.loads[e * loads_stride(G) + g];
                for (int k = 0; k < n; ++k) { xs += s.xi[b + k]; neg |= s.xi[b + k] < 0; }
                if (neg || xs != tot) set_status(status, HEP_E_CONTRACT);
            }
        } else if (!topo) {
            if (per_expert) {
                for (int e = tid; e < E; e += nt) rc1[e * G] = (int16_t)route_expert_merge<false>(a, s, e, 0);
            } else {
                for (int i = tid; i < E * G; i += nt) {
                    int c1, c2;
                    route_pair<false>(a, s, i / G, i % G, &c1, &c2, 0, 0);
                    rc1[i] = (int16_t)c1;
                    rc2[i] = (int16_t)c2;
                }
            }
            for (int e = tid; e < E; e += nt) {  // _check_plan (router.py:97-111)
                const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
                int64_t tot = 0, xs = 0;
                bool neg = false;
                for (int g = 0; g < G; ++g) tot += s.loads[e * loads_stride(G) + g];
                for (int k = 0; k < n; ++k) { xs += s.xi[b + k]; neg |= s.xi[b + k] < 0; }
                if (neg || xs != tot) set_status(status, HEP_E_CONTRACT);
            }
            __syncthreads();
            for (int e = tid; e < E; e += nt) {
                int64_t c = 0;
                if (per_expert) c = rc1[e * G];
                else
                    for (int g = 0; g < G; ++g) c += rc1[e * G + g] + rc2[e * G + g];
                ecount[e] = c;
            }
        } else {
            for (int e = tid; e < E; e += nt) ecount[e] = route_expert_topo<false>(a, s, e, 0, status);
        }
        __syncthreads();
        // exclusive scan over experts (contiguous chunk per thread) -> table positions
        const int chunk = (E + nt - 1) / nt;
        const int e0 = min(E, tid * chunk), e1 = min(E, e0 + chunk);
        int64_t mine = 0;
        for (int e = e0; e < e1; ++e) mine += ecount[e];
        int64_t total_ranges;
        int64_t pos = block_excl_scan_i64(mine, s.scan, &total_ranges);
        for (int e = e0; e < e1; ++e) {
            const int64_t c = ecount[e];
            ecount[e] = pos;
            pos += c;
        }
        if (tid == 0) *a.out.d_n_ranges = total_ranges;
        if (total_ranges > a.max_ranges) set_status(status, HEP_E_CAPACITY);
        __syncthreads();
        if (*status == 0) {
            if (lanes) {
                route_lanes<true>(a, s, ecount);
            } else if (per_expert) {
                for (int e = tid; e < E; e += nt) route_expert_merge<true>(a, s, e, ecount[e]);
            } else if (!topo) {
                for (int i = tid; i < E * G; i += nt) {
                    const int e = i / G, src = i % G;
                    int64_t p1 = ecount[e], n1 = 0, p2 = 0;
                    for (int g = 0; g < G; ++g) {
                        const int c = rc1[e * G + g];
                        n1 += c;
                        if (g < src) { p1 += c; p2 += rc2[e * G + g]; }
                    }
                    int d1, d2;
                    route_pair<true>(a, s, e, src, &d1, &d2, p1, ecount[e] + n1 + p2);
                }
            } else {
                for (int e = tid; e < E; e += nt) route_expert_topo<true>(a, s, e, ecount[e], status);
            }
        }
        __syncthreads();
        prof_mark(a.flags, 5);
    }
    if (*status) { clear_outputs(a, tid, nt); return; }

    // ---- step 7: transfer plan (router.py:178-226) from the pair matrix ----------
    if (route && (a.flags & HEP_SCHED_TRANSFER)) {
        int64_t *T = a.out.d_transfer;
        const int gpn = a.gpn > 0 ? a.gpn : G;
        for (int i = tid; i < G * G; i += nt) T[i] = (int64_t)s.pair[i];
        if (tid < 32) {
            int64_t send = 0, recv = 0, si = 0, ri = 0, sx = 0, rxv = 0;
            const int g = tid;
            if (g < G) {
                for (int o = 0; o < G; ++o) {
                    if (o == g) continue;
                    const int64_t oc = s.pair[g * G + o], ic = s.pair[o * G + g];
                    send += oc;
                    recv += ic;
                    if (o / gpn == g / gpn) { si += oc; ri += ic; } else { sx += oc; rxv += ic; }
                }
                T[G * G + 0 * G + g] = send;
                T[G * G + 1 * G + g] = recv;
                T[G * G + 2 * G + g] = (int64_t)s.pair[g * G + g];
                T[G * G + 3 * G + g] = si;
                T[G * G + 4 * G + g] = ri;
                T[G * G + 5 * G + g] = sx;
                T[G * G + 6 * G + g] = rxv;
            }
            const int64_t intra = warp_sum_i64(si), inter = warp_sum_i64(sx);
            if (tid == 0) {
                T[G * G + 7 * G] = intra;
                T[G * G + 7 * G + 1] = inter;
            }
        }
    }
    prof_mark(a.flags, 6);
}

// Standalone transfer plan over an arbitrary routing table (router.py:178-226)
__global__ void transfer_kernel(int G, int gpn, const int64_t *ranges, int64_t n, int64_t *T, int32_t *status) {
    __shared__ unsigned long long pair[HEP_MAX_GPUS * HEP_MAX_GPUS];
    const int tid = threadIdx.x;
    for (int i = tid; i < G * G; i += blockDim.x) pair[i] = 0;
    if (tid == 0) *status = 0;
    __syncthreads();
    for (int64_t i = tid; i < n; i += blockDim.x) {
        const int64_t *r = ranges + 4 * i;
        if (r[1] < 0 || r[1] >= G || r[2] < 0 || r[2] >= G) { set_status(status, HEP_E_DIMENSION); continue; }
        if (r[3] < 0) { set_status(status, HEP_E_CONTRACT); continue; }
        pair_add(&pair[r[1] * G + r[2]], r[3]);
    }
    __syncthreads();
    if (gpn <= 0) gpn = G;
    for (int i = tid; i < G * G; i += blockDim.x) T[i] = pair[i];
    for (int g = tid; g < G; g += blockDim.x) {
        int64_t send = 0, recv = 0, si = 0, ri = 0, sx = 0, rx = 0;
        for (int o = 0; o < G; ++o) {
            if (o == g) continue;
            const int64_t oc = pair[g * G + o], ic = pair[o * G + g];
            send += oc;
            recv += ic;
            if (o / gpn == g / gpn) { si += oc; ri += ic; } else { sx += oc; rx += ic; }
        }
        T[G * G + g] = send;
        T[G * G + G + g] = recv;
        T[G * G + 2 * G + g] = pair[g * G + g];
        T[G * G + 3 * G + g] = si;
        T[G * G + 4 * G + g] = ri;
        T[G * G + 5 * G + g] = sx;
        T[G * G + 6 * G + g] = rx;
    }
    if (tid == 0) {
        int64_t intra = 0, inter = 0;
        for (int x = 0; x < G; ++x)
            for (int y = 0; y < G; ++y)
                if (x != y) { if (x / gpn == y / gpn) intra += pair[x * G + y]; else inter += pair[x * G + y]; }
        T[G * G + 7 * G] = intra;
        T[G * G + 7 * G + 1] = inter;
    }
}

template <int SPL>
static int launch_spl(hep_sched *h, const SchedArgs &a, size_t smem, cudaStream_t stream) {
    // the opt-in is a property of the kernel (shared by every handle): only ever raise it
    static size_t granted = 0;
    (void)h;
    if (granted < smem) {
        HEP_CHECK_CUDA(cudaFuncSetAttribute(sched_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        granted = smem;
    }
    sched_kernel<SPL><<<1, kSchedThreads, smem, stream>>>(a);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

static int launch_sched(hep_sched *h, SchedArgs &a, cudaStream_t stream) {
    // lex-min arc chain on 4 warps (2 subsets per thread, named barrier): 93.4K vs 97.6K
    // cycles at E=256 (8 warps), 97.7K on 2 warps; hep_tuning.sched_lexmin_warps = 8 for the whole block
    a.lexmin_warps = g_tuning.sched_lexmin_warps;
    a.route_serial = g_tuning.sched_route_serial;
    a.G = h->G;
    a.E = h->E;
    a.nnz = h->nnz;
    a.gpn = h->gpn;
    a.Q = h->Q;
    a.max_ranges = h->max_ranges;
    a.grp_off = h->d_grp_off;
    a.grp_gpu = h->d_grp_gpu;
    a.sorted = h->d_sorted;
    a.mask = h->d_mask;
    a.kidx = h->d_kidx;
    const size_t smem = sched_smem_bytes(h->G, h->E, h->nnz);
    HEP_REQUIRE(smem <= kSchedSmemMax, HEP_E_CAPACITY, "scheduler shared memory %zu B exceeds %d B (E=%d G=%d)", smem,
                kSchedSmemMax, h->E, h->G);
    switch (h->G <= 5 ? 1 : (1 << (h->G - 5))) {
        case 1: return launch_spl<1>(h, a, smem, stream);
        case 2: return launch_spl<2>(h, a, smem, stream);
        case 4: return launch_spl<4>(h, a, smem, stream);
        case 8: return launch_spl<8>(h, a, smem, stream);
        case 16: return launch_spl<16>(h, a, smem, stream);
        case 32: return launch_spl<32>(h, a, smem, stream);
    }
    set_error("unsupported G=%d", h->G);
    return HEP_E_CAPACITY;
}

}  // namespace hep

using namespace hep;

extern "C" int hep_sched_create(int num_gpus, int num_experts, const int32_t *grp_off, const int32_t *grp_gpu,
                                const int32_t *slots, int gpus_per_node, hep_sched_t *out) {
    HEP_REQUIRE(out != nullptr, HEP_E_CONTRACT, "out is NULL");
    *out = nullptr;
    HEP_REQUIRE(num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS, HEP_E_CAPACITY,
                "num_gpus=%d outside the device scheduler range 1..%d", num_gpus, HEP_MAX_GPUS);
    HEP_REQUIRE(num_experts >= 0, HEP_E_DIMENSION, "num_experts=%d", num_experts);
    HEP_REQUIRE(grp_off && grp_off[0] == 0, HEP_E_CONTRACT, "grp_off must start at 0");
    const int E = num_experts, G = num_gpus;
    const int nnz = grp_off[E];
    std::vector<int32_t> off(grp_off, grp_off + E + 1), gpu(grp_gpu, grp_gpu + nnz), sorted(nnz), nnz_exp(nnz);
    std::vector<uint32_t> mask(E, 0);
    int64_t max_ranges = 0;
    for (int e = 0; e < E; ++e) {
        HEP_REQUIRE(off[e + 1] >= off[e], HEP_E_CONTRACT, "grp_off not monotone at %d", e);
        for (int i = off[e]; i < off[e + 1]; ++i) {
            HEP_REQUIRE(gpu[i] >= 0 && gpu[i] < G, HEP_E_PLACEMENT, "expert %d: GPU id %d out of range", e, gpu[i]);
            HEP_REQUIRE(!(mask[e] >> gpu[i] & 1u), HEP_E_PLACEMENT, "expert %d: duplicate GPU %d in EDP group", e,
                        gpu[i]);
            mask[e] |= 1u << gpu[i];
            nnz_exp[i] = e;
        }
        // arcs of expert e in (e, gpu id) order (scheduler.py:303 sorted(arc_edges))
        int k = off[e];
        for (int g = 0; g < G; ++g)
            for (int i = off[e]; i < off[e + 1]; ++i)
                if (gpu[i] == g) sorted[k++] = i;
        max_ranges += 3 * (off[e + 1] - off[e]) + 2 * G;
    }
    const int gpn = gpus_per_node <= 0 ? G : gpus_per_node;
    HEP_REQUIRE(G % gpn == 0, HEP_E_DIMENSION, "gpus_per_node=%d does not divide num_gpus=%d", gpn, G);
    int64_t Q = 1;
    for (int i = 2; i <= G; ++i) {
        int64_t x = Q, y = i;
        while (y) {
            const int64_t t = x % y;
            x = y;
            y = t;
        }
        Q = Q / x * i;
    }
    hep_sched *h = new hep_sched();
    h->G = G;
    h->E = E;
    h->nnz = nnz;
    h->gpn = gpn;
    h->Q = Q;
    h->max_ranges = max_ranges > 0 ? max_ranges : 1;
    h->h_grp_off = off;
    h->h_grp_gpu = gpu;
    if (slots) h->h_slots.assign(slots, slots + E); else h->h_slots.assign(E, 0);
    // per-destination hosted lists (expert ascending), for rank-local receive layouts
    std::vector<int32_t> hosted_off(G + 1, 0), seg_nnz(nnz);
    for (int i = 0; i < nnz; ++i) hosted_off[gpu[i] + 1]++;
    for (int g = 0; g < G; ++g) hosted_off[g + 1] += hosted_off[g];
    std::vector<int32_t> fill(G, 0);
    for (int e = 0; e < E; ++e)
        for (int i = off[e]; i < off[e + 1]; ++i) seg_nnz[hosted_off[gpu[i]] + fill[gpu[i]]++] = i;
    h->h_hosted_off = hosted_off;
    auto up = [&](void **dst, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, bytes > 0 ? bytes : 4);
        if (e != cudaSuccess) return e;
        if (bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    cudaError_t ce = cudaSuccess;
    if (ce == cudaSuccess) ce = up((void **)&h->d_grp_off, off.data(), sizeof(int32_t) * (E + 1));
    if (ce == cudaSuccess) ce = up((void **)&h->d_grp_gpu, gpu.data(), sizeof(int32_t) * nnz);
    if (ce == cudaSuccess) ce = up((void **)&h->d_sorted, sorted.data(), sizeof(int32_t) * nnz);
    if (ce == cudaSuccess) ce = up((void **)&h->d_mask, mask.data(), sizeof(uint32_t) * E);
    if (ce == cudaSuccess) ce = up((void **)&h->d_slots, h->h_slots.data(), sizeof(int32_t) * E);
    if (ce == cudaSuccess) ce = up((void **)&h->d_hosted_off, hosted_off.data(), sizeof(int32_t) * (G + 1));
    if (ce == cudaSuccess) ce = up((void **)&h->d_seg_nnz, seg_nnz.data(), sizeof(int32_t) * nnz);
    if (ce == cudaSuccess) ce = up((void **)&h->d_nnz_exp, nnz_exp.data(), sizeof(int32_t) * nnz);
    std::vector<int8_t> kidx((size_t)E * G, (int8_t)-1);
    for (int e = 0; e < E; ++e)
        for (int i = off[e]; i < off[e + 1]; ++i) kidx[(size_t)e * G + gpu[i]] = (int8_t)(i - off[e]);
    if (ce == cudaSuccess) ce = up((void **)&h->d_kidx, kidx.data(), (size_t)E * G);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
    if (ce != cudaSuccess) {
        set_error("hep_sched_create: %s", cudaGetErrorString(ce));
        hep_sched_destroy(h);
        return HEP_E_CUDA;
    }
    *out = h;
    return HEP_OK;
}

extern "C" int hep_sched_destroy(hep_sched_t h) {
    if (!h) return HEP_OK;
    cudaFree(h->d_grp_off);
    cudaFree(h->d_grp_gpu);
    cudaFree(h->d_sorted);
    cudaFree(h->d_mask);
    cudaFree(h->d_slots);
    cudaFree(h->d_hosted_off);
    cudaFree(h->d_seg_nnz);
    cudaFree(h->d_nnz_exp);
    cudaFree(h->d_kidx);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    delete h;
    return HEP_OK;
}

extern "C" int hep_sched_sizes(hep_sched_t h, int64_t *nnz, int64_t *max_ranges, int64_t *Q, int64_t *transfer_len) {
    HEP_REQUIRE(h, HEP_E_CONTRACT, "null handle");
    if (nnz) *nnz = h->nnz;
    if (max_ranges) *max_ranges = h->max_ranges;
    if (Q) *Q = h->Q;
    if (transfer_len) *transfer_len = (int64_t)h->G * h->G + 8 * h->G + 2;
    return HEP_OK;
}

extern "C" int hep_sched_solve(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                               const int64_t *d_base, int flags, const hep_sched_out *out, void *stream) {
    HEP_NVTX("hep_sched_solve");
    HEP_REQUIRE(h && out && d_loads, HEP_E_CONTRACT, "hep_sched_solve: null argument");
    HEP_REQUIRE(out->d_status, HEP_E_CONTRACT, "hep_sched_solve: d_status required");
    SchedArgs a{};
    a.flags = flags | HEP_SCHED_SOLVE;
    a.loads = d_loads;
    a.se = stride_e;
    a.sg = stride_g;
    a.base = d_base;
    a.xi_in = nullptr;
    a.den = h->Q;
    a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

extern "C" int hep_sched_integerize(hep_sched_t h, const int64_t *d_xnum, int64_t den, const hep_sched_out *out,
                                    void *stream) {
    HEP_NVTX("hep_sched_integerize");
    HEP_REQUIRE(h && out && d_xnum && out->d_xq == d_xnum, HEP_E_CONTRACT,
                "hep_sched_integerize: pass the numerators in out->d_xq");
    HEP_REQUIRE(den > 0, HEP_E_CONTRACT, "denominator must be positive");
    SchedArgs a{};
    a.flags = HEP_SCHED_INTEGERIZE;
    a.den = den;
    a.loads = nullptr;
    a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

extern "C" int hep_sched_route(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                               const int64_t *d_xi, int flags, const hep_sched_out *out, void *stream) {
    HEP_NVTX("hep_sched_route");
    HEP_REQUIRE(h && out && d_loads && d_xi, HEP_E_CONTRACT, "hep_sched_route: null argument");
    SchedArgs a{};
    a.flags = HEP_SCHED_ROUTE | (flags & (HEP_SCHED_TRANSFER | HEP_SCHED_TOPO | HEP_SCHED_PROFILE));
    a.loads = d_loads;
    a.se = stride_e;
    a.sg = stride_g;
    a.xi_in = d_xi;
    a.den = 1;
    a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

namespace hep {
// Pipelined split (simulator.py:291-322): former = floor(v * num / den), latter = v - former
// ([E][G] each, expert-major), and the static phase's even plan over each expert's replicas
// as numerators over Q (Q/n is integral: n <= G).  One thread per expert.
// Also the static phase's integerized per-GPU loads (integerize_plan of the even plan,
// scheduler.py:697-735: every replica gets floor(tot / n), the tot mod n remainder units go to
// the replicas with the lowest GPU ids -- all remainders tie), i.e. the scheduled phase's
// gpu_base, so its solve need not wait for the static phase's routing.  base[G] is zeroed
// by the launcher; integer atomics, order-free.
__global__ void split_kernel(const int64_t *loads, int64_t se, int64_t sg, int E, int G, int64_t num, int64_t den,
                             const int32_t *grp_off, const int32_t *grp_gpu, int64_t Q, int64_t *former,
                             int64_t *latter, int64_t *xq_former, int64_t *base, int32_t *status) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    int64_t tot = 0;
    for (int g = 0; g < G; ++g) {
        const int64_t v = loads[(int64_t)e * se + (int64_t)g * sg];
        if (v < 0) { atomicCAS(status, 0, HEP_E_CONTRACT); return; }
        const int64_t f = (int64_t)(((__int128)v * num) / den);
        former[(int64_t)e * G + g] = f;
        latter[(int64_t)e * G + g] = v - f;
        tot += f;
    }
    const int b = grp_off[e], n = grp_off[e + 1] - b;
    if (n == 0) {
        if (tot) atomicCAS(status, 0, HEP_E_CONTRACT);  // "expert has load but no replicas" (:312-314)
        return;
    }
    const int64_t x = tot * (Q / n);
    const int64_t q = tot / n, r = tot - q * n;
    for (int k = 0; k < n; ++k) {
        xq_former[b + k] = x;
        const int g = grp_gpu[b + k];
        int rank = 0;  // position of g among the group's GPU ids
        for (int j = 0; j < n; ++j) rank += grp_gpu[b + j] < g;
        const int64_t v = q + (rank < r ? 1 : 0);
        if (v) atomicAdd(reinterpret_cast<unsigned long long *>(base + g), (unsigned long long)v);
    }
}
}  // namespace hep

extern "C" int hep_sched_pipelined(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                                   int64_t share_num, int64_t share_den, int flags, int64_t *d_split,
                                   const hep_sched_out *former, const hep_sched_out *latter, void *stream,
                                   void *stream_static) {
    HEP_NVTX("hep_sched_pipelined");
    HEP_REQUIRE(h && d_loads && d_split && former && latter, HEP_E_CONTRACT, "hep_sched_pipelined: null argument");
    HEP_REQUIRE(former->d_status && latter->d_status && former->d_status != latter->d_status, HEP_E_CONTRACT,
                "hep_sched_pipelined: the two phases need distinct d_status words");
    HEP_REQUIRE(share_den > 0 && share_num >= 0 && share_num <= share_den, HEP_E_CONTRACT,
                "static share %lld/%lld outside [0, 1]", (long long)share_num, (long long)share_den);
    cudaStream_t s = (cudaStream_t)stream;
    const int E = h->E, G = h->G;
    int64_t *f_loads = d_split, *l_loads = d_split + (int64_t)E * G, *base = d_split + 2 * (int64_t)E * G;
    HEP_CHECK_CUDA(cudaMemsetAsync(former->d_status, 0, sizeof(int32_t), s));
    HEP_CHECK_CUDA(cudaMemsetAsync(base, 0, sizeof(int64_t) * (size_t)G, s));
    if (E > 0) {
        split_kernel<<<(E + 127) / 128, 128, 0, s>>>(d_loads, stride_e, stride_g, E, G, share_num, share_den,
                                                     h->d_grp_off, h->d_grp_gpu, h->Q, f_loads, l_loads, former->d_xq,
                                                     base, former->d_status);
        HEP_CHECK_LAUNCH();
    }
    // static phase: integerize the even plan, route, transfer (no solve) -- on stream_static when
    // given, forked after the split, so it runs concurrently with the scheduled phase's solve
    cudaStream_t ss = s;
    if (stream_static) {
        ss = (cudaStream_t)stream_static;
        HEP_CHECK_CUDA(cudaEventRecord(h->ev_fork, s));
        HEP_CHECK_CUDA(cudaStreamWaitEvent(ss, h->ev_fork, 0));
    }
    SchedArgs a{};
    a.flags = HEP_SCHED_INTEGERIZE | HEP_SCHED_ROUTE | (flags & (HEP_SCHED_TRANSFER | HEP_SCHED_TOPO));
    a.loads = f_loads;
    a.se = G;
    a.sg = 1;
    a.den = h->Q;
    a.status_in = 1;
    a.out = *former;
    int rc = launch_sched(h, a, ss);
    if (rc) return rc;
    // scheduled phase: exact solve with the static phase's GPU loads as gpu_base (from the split)
    SchedArgs b{};
    b.flags = (flags & HEP_SCHED_ALL) | HEP_SCHED_SOLVE;
    b.loads = l_loads;
    b.se = G;
    b.sg = 1;
    b.base = base;
    b.den = h->Q;
    b.out = *latter;
    return launch_sched(h, b, s);
}

extern "C" int hep_transfer_plan(int num_gpus, int gpus_per_node, const int64_t *d_ranges, int64_t n_ranges,
                                 int64_t *d_transfer, int32_t *d_status, void *stream) {
    HEP_NVTX("hep_transfer_plan");
    HEP_REQUIRE(num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS, HEP_E_CAPACITY, "num_gpus=%d", num_gpus);
    HEP_REQUIRE(d_transfer && d_status, HEP_E_CONTRACT, "null output");
    transfer_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(num_gpus, gpus_per_node, d_ranges, n_ranges, d_transfer,
                                                         d_status);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}

extern "C" int hep_sched_debug_timing(int64_t *host_out, int n) {
    HEP_REQUIRE(host_out && n > 0, HEP_E_CONTRACT, "null output");
    long long tmp[kProfSlots];
    HEP_CHECK_CUDA(cudaMemcpyFromSymbol(tmp, g_sched_prof, sizeof(tmp)));
    for (int i = 0; i < n && i < kProfSlots; ++i) host_out[i] = tmp[i];
    return HEP_OK;
}
