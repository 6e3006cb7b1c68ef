// sched.cu — K3: the per-micro-batch balanced token scheduler on one CTA.
//
// Replaces, bit-exactly, the reference chain (paths under
// /root/reference/pkg/src/harmonyep/):
//   solve_replica_loads / warm_solve   scheduler.py:337-461  (exact m + lex-min plan)
//   integerize_plan                    scheduler.py:697-735
//   route_tokens / route_topology_aware router.py:114-175    (Algorithm 1)
//   build_transfer_plan                router.py:178-226
//
// Device algorithm (not a port of the reference's Dinic max-flow): the
// subset (Gale/Hall) formulation of SURVEY.md Appendix B.
//   1. totals[e] = row sums of the load matrix                       (core.py:261)
//   2. W[S] = sum of totals of experts whose EDP group ⊆ S: zeta transform
//      over the 2^G GPU subsets (placement.py:131-143's transform)
//   3. m = max_S (W[S] + base(S)) / |S| — the exact min-max GPU load
//      (Eq. 3; equal to the reference's probe/min-cut fixpoint :354-371)
//   4. lex-min canonical plan (scheduler.py:295-321): for arcs (e, g) in
//      (expert, gpu) order the minimum feasible replica load is
//        v = max(0, max_{S ⊇ need, g ∉ S} r + Wf[S] - C[S])
//      with need = remaining group \ {g}, Wf = not-yet-processed load inside S,
//      C = remaining capacity of S.  One warp holds all 2^G subsets in
//      registers (SPL per lane) and reduces with shuffles — E·d sequential
//      steps, no block barriers inside the loop.
//   5-7. integerize / route / transfer: one thread per expert, deterministic
//      block scans, integer shared-memory atomics (order-independent sums).
// Everything is exact int64 in units of 1/Q, Q = lcm(1..G) (scheduler.py:184).
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"

#include "sched_internal.cuh"

namespace hep {

constexpr int kSchedThreads = 256;

struct SchedArgs {
    int G, E, nnz, gpn, flags;
    int64_t Q, max_ranges, den;  // den: denominator of d_xq (Q when solved here)
    const int32_t *grp_off, *grp_gpu, *sorted;
    const uint32_t *mask;
    const int64_t *loads;
    int64_t se, sg;
    const int64_t *base;
    const int64_t *xi_in;  // route-only: caller plan
    hep_sched_out out;
};

// Shared memory carve-up (dynamic): see sched_smem_bytes()
struct SchedSmem {
    int64_t *totals;  // [E]
    int64_t *W;       // [NS]
    int32_t *grp_off; // [E+1]
    uint32_t *mask;   // [E]
    int32_t *arc_idx; // [nnz] sorted arcs: nnz index
    int32_t *arc_gpu; // [nnz] sorted arcs: gpu
    int64_t *gpu_load;// [G]
    int64_t *pair;    // [G*G]
    int64_t *scan;    // [kSchedThreads/32 + 2]
    int64_t *misc;    // [8]
};

__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }

__host__ __device__ inline size_t sched_smem_bytes(int G, int E, int nnz) {
    size_t ns = size_t(1) << G;
    size_t b = 0;
    b += align8(sizeof(int64_t) * E);
    b += align8(sizeof(int64_t) * ns);
    b += align8(sizeof(int32_t) * (E + 1));
    b += align8(sizeof(uint32_t) * E);
    b += align8(sizeof(int32_t) * nnz);
    b += align8(sizeof(int32_t) * nnz);
    b += align8(sizeof(int64_t) * G);
    b += align8(sizeof(int64_t) * G * G);
    b += align8(sizeof(int64_t) * (kSchedThreads / 32 + 2));
    b += align8(sizeof(int64_t) * 8);
    return b;
}

__device__ inline SchedSmem carve(char *base, int G, int E, int nnz) {
    SchedSmem s;
    size_t ns = size_t(1) << G;
    char *p = base;
    s.totals = (int64_t *)p; p += align8(sizeof(int64_t) * E);
    s.W = (int64_t *)p; p += align8(sizeof(int64_t) * ns);
    s.grp_off = (int32_t *)p; p += align8(sizeof(int32_t) * (E + 1));
    s.mask = (uint32_t *)p; p += align8(sizeof(uint32_t) * E);
    s.arc_idx = (int32_t *)p; p += align8(sizeof(int32_t) * nnz);
    s.arc_gpu = (int32_t *)p; p += align8(sizeof(int32_t) * nnz);
    s.gpu_load = (int64_t *)p; p += align8(sizeof(int64_t) * G);
    s.pair = (int64_t *)p; p += align8(sizeof(int64_t) * G * G);
    s.scan = (int64_t *)p; p += align8(sizeof(int64_t) * (kSchedThreads / 32 + 2));
    s.misc = (int64_t *)p;
    return s;
}

__device__ __forceinline__ int64_t ld_load(const SchedArgs &a, int e, int g) {
    return a.loads[(int64_t)e * a.se + (int64_t)g * a.sg];
}

// frac a/b > c/d with small positive denominators (<= 64) and |num| < 2^56
__device__ __forceinline__ bool frac_gt(int64_t a, int64_t b, int64_t c, int64_t d) {
    return (__int128)a * d > (__int128)c * b;
}

__device__ __forceinline__ int64_t gcd_i64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// ---------------------------------------------------------------------------
// Step 4: lex-min canonical plan, warp 0 only.  SPL subsets per lane.
// ---------------------------------------------------------------------------
template <int SPL>
__device__ void lexmin_warp(const SchedArgs &a, SchedSmem &s, int64_t mQ) {
    const int lane = threadIdx.x & 31;
    const int G = a.G, E = a.E;
    const int NS = 1 << G;
    const int64_t Q = a.Q;
    int64_t Wf[SPL], C[SPL];
    int64_t cap[HEP_MAX_GPUS];
#pragma unroll
    for (int g = 0; g < HEP_MAX_GPUS; ++g) {
        int64_t bq = (g < G && a.base) ? a.base[g] * Q : 0;
        int64_t c = mQ - bq;
        cap[g] = (g < G && c > 0) ? c : 0;
    }
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
        const int S = lane + 32 * j;
        int64_t c = 0;
#pragma unroll
        for (int g = 0; g < HEP_MAX_GPUS; ++g)
            if ((S >> g) & 1) c += cap[g];
        C[j] = c;
        Wf[j] = S < NS ? s.W[S] * Q : 0;
    }
    for (int e = 0; e < E; ++e) {
        const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
        if (n == 0) continue;
        int64_t r = s.totals[e] * Q;
        uint32_t R = s.mask[e];
        if (r > 0) {
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const uint32_t S = lane + 32 * j;
                if ((S & R) == R) Wf[j] -= r;
            }
        }
        for (int k = 0; k < n; ++k) {
            const int g = s.arc_gpu[b + k];
            const uint32_t gbit = 1u << g;
            const uint32_t need = R & ~gbit;
            int64_t v;
            if (r == 0) {
                v = 0;  // Wf <= C everywhere (feasible state) => bound <= 0
            } else if (need == 0) {
                v = r;  // S = {} attains r; every other bound is <= r
            } else {
                int64_t best = 0;
#pragma unroll
                for (int j = 0; j < SPL; ++j) {
                    const uint32_t S = lane + 32 * j;
                    const bool ok = (S < (uint32_t)NS) && ((S & need) == need) && !(S & gbit);
                    const int64_t cand = r + Wf[j] - C[j];
                    if (ok && cand > best) best = cand;
                }
                v = __any_sync(0xffffffffu, best > 0) ? warp_max_i64(best) : 0;
            }
            if (lane == 0) a.out.d_xq[s.arc_idx[b + k]] = v;
            r -= v;
            R = need;
            if (v) {
#pragma unroll
                for (int j = 0; j < SPL; ++j) {
                    const uint32_t S = lane + 32 * j;
                    if (S & gbit) C[j] -= v;
                }
            }
        }
    }
}

template <int SPL>
__global__ void __launch_bounds__(kSchedThreads, 1) sched_kernel(SchedArgs a) {
    extern __shared__ __align__(16) char smem_raw[];
    SchedSmem s = carve(smem_raw, a.G, a.E, a.nnz);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int G = a.G, E = a.E, NS = 1 << G;
    int32_t *status = a.out.d_status;

    // placement tables -> smem (all stages read them in sequential loops)
    for (int i = tid; i <= E; i += nt) s.grp_off[i] = a.grp_off[i];
    for (int i = tid; i < E; i += nt) s.mask[i] = a.mask[i];
    for (int i = tid; i < a.nnz; i += nt) {
        int idx = a.sorted[i];
        s.arc_idx[i] = idx;
        s.arc_gpu[i] = a.grp_gpu[idx];
    }
    if (tid == 0) *status = 0;
    __syncthreads();

    // ---------------- step 1: expert totals (LoadMatrix.expert_totals) -------------
    const bool solve = a.flags & HEP_SCHED_SOLVE;
    const bool need_loads = solve || (a.flags & HEP_SCHED_ROUTE);
    int64_t my_total = 0, my_bad = 0;
    if (need_loads) {
        for (int e = tid; e < E; e += nt) {
            int64_t t = 0;
            for (int g = 0; g < G; ++g) {
                int64_t v = ld_load(a, e, g);
                if (v < 0) my_bad = 1;
                t += v;
            }
            s.totals[e] = t;
            my_total += t;
            // scheduler.py:344-347 loaded expert with an empty EDP group
            if (solve && t > 0 && s.grp_off[e + 1] == s.grp_off[e]) set_status(status, HEP_E_PLACEMENT);
        }
        if (my_bad) set_status(status, HEP_E_CONTRACT);
    }
    int64_t base_sum = 0;
    if (tid == 0 && a.base)
        for (int g = 0; g < G; ++g) base_sum += a.base[g];
    int64_t total_all = block_sum_i64(my_total + base_sum, s.scan);
    if (solve && (__int128)total_all * a.Q >= ((__int128)1 << 56)) set_status(status, HEP_E_CAPACITY);
    __syncthreads();
    if (*status) return;

    if (solve) {
        // ---------------- step 2: zeta transform over GPU subsets ----------------
        for (int S = tid; S < NS; S += nt) s.W[S] = 0;
        __syncthreads();
        for (int e = tid; e < E; e += nt)
            if (s.totals[e] > 0 && s.mask[e])
                atomicAdd((unsigned long long *)&s.W[s.mask[e]], (unsigned long long)s.totals[e]);
        __syncthreads();
        for (int bit = 0; bit < G; ++bit) {
            for (int S = tid; S < NS; S += nt)
                if ((S >> bit) & 1) s.W[S] += s.W[S ^ (1 << bit)];
            __syncthreads();
        }
        // ---------------- step 3: m = max density (Eq. 3) ------------------------
        int64_t bn = 0, bd = 1;
        if (tid == 0 && a.base) {  // candidate max(base) (scheduler.py:357)
            for (int g = 0; g < G; ++g)
                if (a.base[g] > bn) bn = a.base[g];
        }
        for (int S = tid + 1; S < NS; S += nt) {
            int64_t num = s.W[S];
            if (a.base)
                for (int g = 0; g < G; ++g)
                    if ((S >> g) & 1) num += a.base[g];
            int64_t den = __popc(S);
            if (frac_gt(num, den, bn, bd)) { bn = num; bd = den; }
        }
        // block argmax over fractions
        for (int o = 16; o > 0; o >>= 1) {
            int64_t on = __shfl_xor_sync(0xffffffffu, bn, o), od = __shfl_xor_sync(0xffffffffu, bd, o);
            if (frac_gt(on, od, bn, bd)) { bn = on; bd = od; }
        }
        __shared__ int64_t red_n[kSchedThreads / 32], red_d[kSchedThreads / 32];
        if ((tid & 31) == 0) { red_n[tid >> 5] = bn; red_d[tid >> 5] = bd; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nt / 32; ++w)
                if (frac_gt(red_n[w], red_d[w], bn, bd)) { bn = red_n[w]; bd = red_d[w]; }
            int64_t g = gcd_i64(bn, bd);
            if (g == 0) g = 1;
            bn /= g; bd /= g;
            s.misc[0] = bn;
            s.misc[1] = bd;
            s.misc[2] = bn * (a.Q / bd);  // m scaled by Q (scheduler.py:267)
            a.out.d_m[0] = bn;
            a.out.d_m[1] = bd;
            a.out.d_m[2] = a.Q;
        }
        __syncthreads();
        // ---------------- step 4: lex-min canonical plan -------------------------
        if (tid < 32) lexmin_warp<SPL>(a, s, s.misc[2]);
        __syncthreads();
    }

    const int64_t den = solve ? a.Q : a.den;
    // ---------------- step 5: integerize (largest remainder) ----------------------
    if (a.flags & HEP_SCHED_INTEGERIZE) {
        for (int g = tid; g < G; g += nt) s.gpu_load[g] = 0;
        __syncthreads();
        for (int e = tid; e < E; e += nt) {
            const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
            __int128 total = 0;
            int64_t sum_floor = 0;
            for (int k = 0; k < n; ++k) {
                int64_t v = a.out.d_xq[b + k];
                int64_t fl = v >= 0 ? v / den : -((-v + den - 1) / den);
                a.out.d_xi[b + k] = fl;
                sum_floor += fl;
                total += v;
            }
            // round(total) must be an integer within 1e-6 (scheduler.py:706-713)
            int64_t t_fl = (int64_t)(total >= 0 ? total / den : -((-total + den - 1) / den));
            int64_t t_rem = (int64_t)(total - (__int128)t_fl * den);
            int64_t rounded = t_fl;
            if (2 * (__int128)t_rem > den || (2 * (__int128)t_rem == den && (t_fl & 1))) rounded = t_fl + 1;
            __int128 diff = total - (__int128)rounded * den;
            if (diff < 0) diff = -diff;
            if (diff * 1000000 > den) { set_status(status, HEP_E_CONTRACT); continue; }
            int64_t units = rounded - sum_floor;
            // remainder desc, ties -> lowest GPU id (key :718-721)
            for (int u = 0; u < units && u < n; ++u) {
                int best = -1, best_gpu = 0;
                int64_t best_rem = -1;
                for (int k = 0; k < n; ++k) {
                    int64_t rem = a.out.d_xq[b + k] - a.out.d_xi[b + k] * den;
                    if (rem < 0) continue;  // already rounded up
                    int gg = a.grp_gpu[b + k];
                    if (best < 0 || rem > best_rem || (rem == best_rem && gg < best_gpu)) {
                        best = k; best_rem = rem; best_gpu = gg;
                    }
                }
                if (best < 0) break;
                a.out.d_xi[b + best] += 1;
            }
            for (int k = 0; k < n; ++k)
                atomicAdd((unsigned long long *)&s.gpu_load[a.grp_gpu[b + k]], (unsigned long long)a.out.d_xi[b + k]);
        }
        __syncthreads();
        if (tid == 0) {
            int64_t mx = 0;
            for (int g = 0; g < G; ++g) {
                a.out.d_gpu_load[g] = s.gpu_load[g];
                if (g == 0 || s.gpu_load[g] > mx) mx = s.gpu_load[g];
            }
            a.out.d_m[3] = mx;
        }
        __syncthreads();
    }
    if (*status) return;

    // ---------------- step 6: Algorithm 1 routing (router.py:114-158) ------------------
    if (a.flags & HEP_SCHED_ROUTE) {
        const int64_t *xi = a.xi_in ? a.xi_in : a.out.d_xi;
        const bool topo = (a.flags & HEP_SCHED_TOPO) && a.gpn > 0 && a.gpn < G;
        // contiguous expert chunk per thread keeps ranges in expert order
        const int chunk = (E + nt - 1) / nt;
        const int e0 = min(E, tid * chunk), e1 = min(E, e0 + chunk);
        int64_t rin[HEP_MAX_GPUS], rx[HEP_MAX_GPUS];
        int64_t my_count = 0;
        for (int pass = 0; pass < 2; ++pass) {
            int64_t pos = 0;
            if (pass == 1) {
                int64_t tot;
                pos = block_excl_scan_i64(my_count, s.scan, &tot);
                if (tid == 0) *a.out.d_n_ranges = tot;
                if (tot > a.max_ranges) { set_status(status, HEP_E_CAPACITY); break; }
            }
            for (int e = e0; e < e1; ++e) {
                const int b = s.grp_off[e], n = s.grp_off[e + 1] - b;
                int64_t tot = 0, xs = 0;
                for (int g = 0; g < G; ++g) { rin[g] = ld_load(a, e, g); rx[g] = 0; tot += rin[g]; }
                if (n == 0 && tot == 0) continue;  // :125-126
                bool bad = false;
                for (int k = 0; k < n; ++k) {
                    int64_t v = xi[b + k];
                    if (v < 0) bad = true;
                    xs += v;
                    rx[a.grp_gpu[b + k]] = v;
                }
                if (bad || xs != tot) { set_status(status, HEP_E_CONTRACT); continue; }  // _check_plan :97-111
#define HEP_EMIT(S_, D_, Y_)                                                   \
    do {                                                                       \
        if (pass == 0) {                                                       \
            ++my_count;                                                        \
        } else {                                                               \
            int64_t *r_ = a.out.d_ranges + 4 * pos;                            \
            r_[0] = e; r_[1] = (S_); r_[2] = (D_); r_[3] = (Y_);                \
            ++pos;                                                             \
        }                                                                      \
    } while (0)
                // phase 1: same GPU, sorted(group)
                for (int k = 0; k < n; ++k) {
                    const int g = s.arc_gpu[b + k];
                    int64_t y = rin[g] < rx[g] ? rin[g] : rx[g];
                    if (y > 0) { HEP_EMIT(g, g, y); rin[g] -= y; rx[g] -= y; }
                }
                // phase 2 (topology-aware): same node
                if (topo) {
                    for (int src = 0; src < G; ++src) {
                        if (rin[src] == 0) continue;
                        for (int k = 0; k < n; ++k) {
                            const int dst = a.grp_gpu[b + k];
                            if (dst == src || dst / a.gpn != src / a.gpn) continue;
                            int64_t y = rin[src] < rx[dst] ? rin[src] : rx[dst];
                            if (y > 0) { HEP_EMIT(src, dst, y); rin[src] -= y; rx[dst] -= y; }
                        }
                    }
                }
                // final phase: src ascending x EDP list order
                for (int src = 0; src < G; ++src) {
                    if (rin[src] == 0) continue;
                    for (int k = 0; k < n; ++k) {
                        const int dst = a.grp_gpu[b + k];
                        int64_t y = rin[src] < rx[dst] ? rin[src] : rx[dst];
                        if (y > 0) { HEP_EMIT(src, dst, y); rin[src] -= y; rx[dst] -= y; }
                    }
                }
#undef HEP_EMIT
            }
            __syncthreads();
            if (*status) break;
        }
        __syncthreads();
    }
    if (*status) return;

    // ---------------- step 7: transfer plan (router.py:178-226) ------------------------
    if (a.flags & HEP_SCHED_TRANSFER) {
        for (int i = tid; i < G * G; i += nt) s.pair[i] = 0;
        __syncthreads();
        const int64_t n = *a.out.d_n_ranges;
        for (int64_t i = tid; i < n; i += nt) {
            const int64_t *r = a.out.d_ranges + 4 * i;
            atomicAdd((unsigned long long *)&s.pair[r[1] * G + r[2]], (unsigned long long)r[3]);
        }
        __syncthreads();
        int64_t *T = a.out.d_transfer;
        const int gpn = a.gpn > 0 ? a.gpn : G;
        for (int i = tid; i < G * G; i += nt) T[i] = s.pair[i];
        for (int g = tid; g < G; g += nt) {
            int64_t send = 0, recv = 0, si = 0, ri = 0, sx = 0, rx = 0;
            for (int o = 0; o < G; ++o) {
                if (o == g) continue;
                int64_t out_c = s.pair[g * G + o], in_c = s.pair[o * G + g];
                send += out_c; recv += in_c;
                if (o / gpn == g / gpn) { si += out_c; ri += in_c; } else { sx += out_c; rx += in_c; }
            }
            T[G * G + 0 * G + g] = send;
            T[G * G + 1 * G + g] = recv;
            T[G * G + 2 * G + g] = s.pair[g * G + g];
            T[G * G + 3 * G + g] = si;
            T[G * G + 4 * G + g] = ri;
            T[G * G + 5 * G + g] = sx;
            T[G * G + 6 * G + g] = rx;
        }
        if (tid == 0) {
            int64_t intra = 0, inter = 0;
            for (int x = 0; x < G; ++x)
                for (int y = 0; y < G; ++y) {
                    if (x == y) continue;
                    if (x / gpn == y / gpn) intra += s.pair[x * G + y]; else inter += s.pair[x * G + y];
                }
            T[G * G + 7 * G] = intra;
            T[G * G + 7 * G + 1] = inter;
        }
    }
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
        atomicAdd(&pair[r[1] * G + r[2]], (unsigned long long)r[3]);
    }
    __syncthreads();
    if (gpn <= 0) gpn = G;
    for (int i = tid; i < G * G; i += blockDim.x) T[i] = pair[i];
    for (int g = tid; g < G; g += blockDim.x) {
        int64_t send = 0, recv = 0, si = 0, ri = 0, sx = 0, rx = 0;
        for (int o = 0; o < G; ++o) {
            if (o == g) continue;
            int64_t oc = pair[g * G + o], ic = pair[o * G + g];
            send += oc; recv += ic;
            if (o / gpn == g / gpn) { si += oc; ri += ic; } else { sx += oc; rx += ic; }
        }
        T[G * G + g] = send; T[G * G + G + g] = recv; T[G * G + 2 * G + g] = pair[g * G + g];
        T[G * G + 3 * G + g] = si; T[G * G + 4 * G + g] = ri; T[G * G + 5 * G + g] = sx; T[G * G + 6 * G + g] = rx;
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

static int launch_sched(hep_sched *h, SchedArgs &a, cudaStream_t stream) {
    a.G = h->G; a.E = h->E; a.nnz = h->nnz; a.gpn = h->gpn; a.Q = h->Q; a.max_ranges = h->max_ranges;
    a.grp_off = h->d_grp_off; a.grp_gpu = h->d_grp_gpu; a.sorted = h->d_sorted; a.mask = h->d_mask;
    size_t smem = sched_smem_bytes(h->G, h->E, h->nnz);
    HEP_REQUIRE(smem <= 200 * 1024, HEP_E_CAPACITY, "scheduler shared memory %zu B exceeds 200 KB (E=%d G=%d)", smem,
                h->E, h->G);
    const int spl = h->G <= 5 ? 1 : (1 << (h->G - 5));
#define HEP_LAUNCH_SPL(N)                                                                          \
    case N: {                                                                                      \
        HEP_CHECK_CUDA(cudaFuncSetAttribute(sched_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        sched_kernel<N><<<1, kSchedThreads, smem, stream>>>(a);                                    \
        break;                                                                                     \
    }
    switch (spl) {
        HEP_LAUNCH_SPL(1)
        HEP_LAUNCH_SPL(2)
        HEP_LAUNCH_SPL(4)
        HEP_LAUNCH_SPL(8)
        HEP_LAUNCH_SPL(16)
        HEP_LAUNCH_SPL(32)
        default:
            set_error("unsupported G=%d", h->G);
            return HEP_E_CAPACITY;
    }
#undef HEP_LAUNCH_SPL
    HEP_CHECK_LAUNCH();
    return HEP_OK;
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
    std::vector<int32_t> off(grp_off, grp_off + E + 1), gpu(grp_gpu, grp_gpu + nnz), sorted(nnz);
    std::vector<uint32_t> mask(E, 0);
    int64_t max_ranges = 0;
    for (int e = 0; e < E; ++e) {
        HEP_REQUIRE(off[e + 1] >= off[e], HEP_E_CONTRACT, "grp_off not monotone at %d", e);
        for (int i = off[e]; i < off[e + 1]; ++i) {
            HEP_REQUIRE(gpu[i] >= 0 && gpu[i] < G, HEP_E_PLACEMENT, "expert %d: GPU id %d out of range", e, gpu[i]);
            HEP_REQUIRE(!(mask[e] >> gpu[i] & 1u), HEP_E_PLACEMENT, "expert %d: duplicate GPU %d in EDP group", e,
                        gpu[i]);
            mask[e] |= 1u << gpu[i];
        }
        // arcs of expert e in (e, gpu id) order (scheduler.py:303 sorted(arc_edges))
        int k = off[e];
        for (int g = 0; g < G; ++g)
            for (int i = off[e]; i < off[e + 1]; ++i)
                if (gpu[i] == g) sorted[k++] = i;
        const int n = off[e + 1] - off[e];
        max_ranges += 3 * n + 2 * G;
    }
    int gpn = gpus_per_node <= 0 ? G : gpus_per_node;
    HEP_REQUIRE(G % gpn == 0, HEP_E_DIMENSION, "gpus_per_node=%d does not divide num_gpus=%d", gpn, G);
    int64_t Q = 1;
    for (int i = 2; i <= G; ++i) {
        int64_t a = Q, b = i;
        while (b) { int64_t t = a % b; a = b; b = t; }
        Q = Q / a * i;
    }
    hep_sched *h = new hep_sched();
    h->G = G; h->E = E; h->nnz = nnz; h->gpn = gpn; h->Q = Q; h->max_ranges = max_ranges > 0 ? max_ranges : 1;
    h->h_grp_off = off; h->h_grp_gpu = gpu;
    if (slots) h->h_slots.assign(slots, slots + E); else h->h_slots.assign(E, 0);
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
    // receive-row layout tables: segments ordered [dst GPU][expert ascending]
    {
        std::vector<int32_t> hosted_off(G + 1, 0), seg_nnz(nnz), nnz_exp(nnz);
        for (int e = 0; e < E; ++e)
            for (int i = off[e]; i < off[e + 1]; ++i) { hosted_off[gpu[i] + 1]++; nnz_exp[i] = e; }
        for (int g = 0; g < G; ++g) hosted_off[g + 1] += hosted_off[g];
        std::vector<int32_t> fill(G, 0);
        for (int e = 0; e < E; ++e)
            for (int i = off[e]; i < off[e + 1]; ++i) seg_nnz[hosted_off[gpu[i]] + fill[gpu[i]]++] = i;
        h->h_hosted_off = hosted_off;
        if (ce == cudaSuccess) ce = up((void **)&h->d_hosted_off, hosted_off.data(), sizeof(int32_t) * (G + 1));
        if (ce == cudaSuccess) ce = up((void **)&h->d_seg_nnz, seg_nnz.data(), sizeof(int32_t) * nnz);
        if (ce == cudaSuccess) ce = up((void **)&h->d_nnz_exp, nnz_exp.data(), sizeof(int32_t) * nnz);
    }
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
    HEP_REQUIRE(h && out && d_loads, HEP_E_CONTRACT, "hep_sched_solve: null argument");
    HEP_REQUIRE(out->d_status, HEP_E_CONTRACT, "hep_sched_solve: d_status required");
    SchedArgs a{};
    a.flags = flags | HEP_SCHED_SOLVE;
    a.loads = d_loads; a.se = stride_e; a.sg = stride_g; a.base = d_base;
    a.xi_in = nullptr; a.den = h->Q;
    a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

extern "C" int hep_sched_integerize(hep_sched_t h, const int64_t *d_xnum, int64_t den, const hep_sched_out *out,
                                    void *stream) {
    HEP_REQUIRE(h && out && d_xnum && out->d_xq == d_xnum, HEP_E_CONTRACT,
                "hep_sched_integerize: pass the numerators in out->d_xq");
    HEP_REQUIRE(den > 0, HEP_E_CONTRACT, "denominator must be positive");
    SchedArgs a{};
    a.flags = HEP_SCHED_INTEGERIZE;
    a.den = den; a.loads = nullptr; a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

extern "C" int hep_sched_route(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                               const int64_t *d_xi, int flags, const hep_sched_out *out, void *stream) {
    HEP_REQUIRE(h && out && d_loads && d_xi, HEP_E_CONTRACT, "hep_sched_route: null argument");
    SchedArgs a{};
    a.flags = HEP_SCHED_ROUTE | (flags & (HEP_SCHED_TRANSFER | HEP_SCHED_TOPO));
    a.loads = d_loads; a.se = stride_e; a.sg = stride_g; a.xi_in = d_xi; a.den = 1;
    a.out = *out;
    return launch_sched(h, a, (cudaStream_t)stream);
}

extern "C" int hep_transfer_plan(int num_gpus, int gpus_per_node, const int64_t *d_ranges, int64_t n_ranges,
                                 int64_t *d_transfer, int32_t *d_status, void *stream) {
    HEP_REQUIRE(num_gpus >= 1 && num_gpus <= HEP_MAX_GPUS, HEP_E_CAPACITY, "num_gpus=%d", num_gpus);
    HEP_REQUIRE(d_transfer && d_status, HEP_E_CONTRACT, "null output");
    transfer_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(num_gpus, gpus_per_node, d_ranges, n_ranges, d_transfer,
                                                         d_status);
    HEP_CHECK_LAUNCH();
    return HEP_OK;
}
