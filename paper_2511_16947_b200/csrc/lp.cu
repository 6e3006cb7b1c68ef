// lp.cu — dense two-phase primal simplex (Bland's rule) on one thread-block
// cluster: the device solver behind the communication-aware scheduling modes.
//
// Drop-in for the reference's `simplex_solve` (/root/reference/pkg/src/harmonyep/
// simplex.py:99-192), which `solve_comm_aware` (scheduler.py:622-689) calls on the
// LPs `_comm_aware_lp` (:480-547) and `_topology_aware_lp` (:550-619) build.  The
// arithmetic is the reference's, operation for operation, so a cold solve reproduces
// its pivot sequence, basis and solution bit for bit:
//   * tableau [m+1][total+1] (objective last, rhs last column), rows a_eq then a_ub
//     with one slack per a_ub row, rows with b < 0 negated (simplex.py:113-125);
//   * artificials on every row lacking a +1 slack, phase-1 objective = sum of the
//     artificial rows subtracted in row order (:146-167);
//   * entering = lowest allowed column with obj < -tol; leaving = the sequential
//     ratio scan with the tolerance tie rule on basis ids (_run_phase :61-92);
//   * pivot: row /= pivot element, then T[i][j] = T[i][j] - (col[i] * row[j]) with
//     separate multiply and subtract roundings (np.outer then -=, :53-58) -- no FMA;
//   * infeasible when the phase-1 optimum is < -1e-7; surviving artificials driven
//     out on their first |entry| > tol column (:169-177); phase-2 objective rebuilt
//     from c by eliminating the basic columns in basis-row order (:179-185).
// Warm start (:127-144): the previous basis is factorised here by Gauss-Jordan pivots
// with partial pivoting instead of LAPACK's dgesv, so a warm solve agrees with the
// reference to rounding (same basis sequence whenever no ratio/reduced cost sits
// within rounding of the tolerance), not bit for bit.
//
// Layout: the tableau lives in global memory (L2-resident; row-major, leading
// dimension ld = width + m + 1); every CTA of the cluster owns the rows i with
// i % cluster_size == rank, one warp per row.  Each pivot is two hardware cluster
// barriers: (A) every CTA has chosen the same entering/leaving pair redundantly (no
// extra barrier to broadcast them) and cached the pivot row in shared memory; (B)
// every owned row is updated.  Rows whose pivot-column entry is zero and columns
// whose pivot-row entry is zero are skipped: x - 0*y == x (value-equal; only the
// sign of a zero can differ, which no comparison or later product observes).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace hep {
namespace lp {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
// shared int scratch: reductions [kWarps + 8], then the warm start's assigned/want [2m]
// or the ratio test's warp counts [kWarps + 1] (never live together)
__host__ __device__ constexpr int64_t sint_count(int64_t m) {
    return kWarps + 8 + (2 * m + 2 > kWarps + 2 ? 2 * m + 2 : kWarps + 2);
}

enum : int { ST_OK = 0, ST_INFEASIBLE = 1, ST_UNBOUNDED = 2, ST_MAXITER = 3 };

struct Args {
    const double *c, *a_eq, *b_eq, *a_ub, *b_ub;
    const int64_t *basis_in;  // device [m] or null
    int64_t n, m_eq, m_ub;
    double tol;
    int64_t max_iter;
    double *T0, *T1;          // workspace tableaux [(m+1) * ld] (T1: warm-start staging)
    int64_t ld;
    int dsm;                  // 1: rows live in the cluster's shared memory (row i on CTA i % ncta)
    double *x_full;           // out [width] (reference x_full before the [:n] clip)
    int64_t *basis_out;       // out [m]
    int64_t *info;            // out [8]: pivots, status, warm_used, n_art, phase1_pivots, phase2_pivots
};


// one thread-block cluster; all CTAs run the same control flow on the same data
struct Ctx {
    cg::cluster_group cl;
    int rank, ncta;
    int m, width, total;  // rows (excl. objective), vars+slacks, columns excl. rhs
    int64_t ld;
    double *T;      // global tableau (dsm = 0)
    bool dsm;
    double *rows_local;  // dsm: this CTA's row block; CTA r's block = mapa(rows_local, r)
    int lg;              // log2(ncta)
    int *basis;     // smem copy, identical in every CTA
    double *prow;   // smem [total+1] normalised pivot row
    int *nz;        // smem [total+1] nonzero columns of the pivot row
    int *s_int;     // smem scratch ints
    double *scol;   // smem [m+1] pivot column T[i][col] of every row (incl. objective)
    double *sratio; // smem [m] rhs/col for eligible rows, +inf otherwise
    int *rows;      // smem [m+1] owned rows with a nonzero pivot-column entry / ratio candidates
    double *sdbl;   // smem [kWarps + 1] double scratch
    double tol;
};

// row i of the tableau: global row-major, or (dsm) row i / ncta of CTA i % ncta's
// shared-memory block, reached through its generic DSMEM address
__device__ __forceinline__ double *rp(const Ctx &c, int i) {
    if (!c.dsm) return c.T + (int64_t)i * c.ld;
    double *blk = static_cast<double *>(__cluster_map_shared_rank(c.rows_local, (unsigned)(i & (c.ncta - 1))));
    return blk + (int64_t)(i >> c.lg) * c.ld;
}
// a tableau element another CTA may have written before the last cluster barrier:
// global through L2 (ld.global.cg, never a stale L1 line), DSMEM directly
__device__ __forceinline__ double lda(const Ctx &c, const double *p) { return c.dsm ? *p : __ldcg(p); }

// barrier.cluster.arrive (.release) + barrier.cluster.wait (.acquire): orders every
// CTA's tableau writes (global or DSMEM) before the other CTAs' reads
__device__ __forceinline__ void cluster_sync(Ctx &c) { c.cl.sync(); }

// block-wide min of an int (INT_MAX = none); all threads get the result
__device__ int block_min_int(int v, int *scratch) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = __reduce_min_sync(0xffffffffu, v);
    __syncthreads();
    if (lane == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        int u = lane < kWarps ? scratch[lane] : INT_MAX;
        u = __reduce_min_sync(0xffffffffu, u);
        if (lane == 0) scratch[kWarps] = u;
    }
    __syncthreads();
    int r = scratch[kWarps];
    __syncthreads();
    return r;
}

// _run_phase's entering rule: lowest column j < allowed with obj[j] < -tol
__device__ int choose_entering(Ctx &c, int allowed) {
    const double *obj = rp(c, c.m);
    const double ntol = -c.tol;
    int best = INT_MAX;
    for (int j0 = threadIdx.x; j0 < allowed && best == INT_MAX; j0 += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = j0 + u * kThreads < allowed ? lda(c, obj + j0 + u * kThreads) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (best == INT_MAX && v[u] < ntol) best = j0 + u * kThreads;
    }
    return block_min_int(best, c.s_int);
}

// the pivot column of every row (and its ratios) into shared memory: one round of
// independent L2 loads instead of a dependent chain per row
__device__ void load_column(Ctx &c, int col) {
    const double tol = c.tol;
    for (int i0 = threadIdx.x; i0 <= c.m; i0 += 2 * kThreads) {
        double a[2], rhs[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = i0 + u * kThreads;
            a[u] = i <= c.m ? lda(c, rp(c, i) + col) : 0.0;
            rhs[u] = i < c.m ? lda(c, rp(c, i) + c.total) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = i0 + u * kThreads;
            if (i <= c.m) c.scol[i] = a[u];
            if (i < c.m) c.sratio[i] = a[u] > tol ? rhs[u] / a[u] : __longlong_as_double(0x7ff0000000000000LL);
        }
    }
    __syncthreads();
}

// _run_phase's leaving rule: the reference's sequential scan over rows 0..m-1
// (simplex.py:75-86) -- best ratio, a replacement when ratio < best - tol or, within
// tol, on a lower basis id.  Exact but cheap: a block-wide prefix minimum of the
// eligible ratios in row order marks the candidates (ratio <= min of the earlier rows
// + 64 tol); one thread then runs the sequential rule over the candidates alone.  A
// skipped row can only have been accepted if the running best had drifted more than
// ~63 tol above the running minimum through chains of tolerance ties; the scan checks
// that drift and falls back to the full sequential scan if it ever exceeds 32 tol.
// Returns -1 if unbounded.  Uses c.rows as the candidate list.
__device__ int seq_leaving(Ctx &c, const int *list, int n, bool all_rows, double *drift) {
    const double tol = c.tol;
    bool have = false;
    double best = 0.0, runmin = 0.0, dmax = 0.0;
    int leave = -1;
    for (int k = 0; k < n; ++k) {
        const int i = all_rows ? k : list[k];
        if (all_rows && !(c.scol[i] > tol)) continue;
        const double r = c.sratio[i];
        bool take;
        if (!have) take = true;
        else if (r < best - tol) take = true;
        else take = fabs(r - best) <= tol && c.basis[i] < c.basis[leave];
        runmin = have ? fmin(runmin, r) : r;
        if (take) {
            have = true;
            best = r;
            leave = i;
        }
        dmax = fmax(dmax, best - runmin - fabs(runmin) * 1e-12);
    }
    *drift = dmax;
    return leave;
}

__device__ int choose_leaving(Ctx &c) {
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const double tol = c.tol, W = 64.0 * tol;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *s_wmin = c.sdbl;            // [kWarps] warp minima -> exclusive prefix
    int *s_wcnt = c.s_int + kWarps + 8;  // [kWarps] warp candidate counts -> exclusive prefix
    __shared__ double s_carry;
    __shared__ int s_ncand, s_leave;
    if (threadIdx.x == 0) {
        s_carry = INF;
        s_ncand = 0;
    }
    __syncthreads();
    for (int base = 0; base < c.m; base += kThreads) {
        const int i = base + threadIdx.x;
        const bool el = i < c.m && c.scol[i] > tol;
        const double r = el ? c.sratio[i] : INF;
        double v = r;  // inclusive warp prefix minimum
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v = fmin(v, t);
        }
        double ex = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0) ex = INF;
        if (lane == 31) s_wmin[w] = v;
        __syncthreads();
        if (w == 0) {
            const double x = lane < kWarps ? s_wmin[lane] : INF;
            double y = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y = fmin(y, t);
            }
            double yx = __shfl_up_sync(0xffffffffu, y, 1);
            if (lane == 0) yx = INF;
            if (lane < kWarps) s_wmin[lane] = fmin(yx, s_carry);  // min of everything before warp `lane`
            if (lane == 31) s_wmin[kWarps] = fmin(y, s_carry);     // carry for the next tile
        }
        __syncthreads();
        const double before = fmin(s_wmin[w], ex);
        const bool cand = el && (before == INF || r <= before + W + fabs(before) * 4e-12);
        const unsigned bal = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) s_wcnt[w] = __popc(bal);
        __syncthreads();
        if (w == 0) {
            const int x = lane < kWarps ? s_wcnt[lane] : 0;
            int y = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += t;
            }
            if (lane < kWarps) s_wcnt[lane] = y - x;
            if (lane == 31) s_wcnt[kWarps] = y;
        }
        __syncthreads();
        if (cand) c.rows[s_ncand + s_wcnt[w] + __popc(bal & ((1u << lane) - 1))] = i;
        __syncthreads();
        if (threadIdx.x == 0) {
            s_ncand += s_wcnt[kWarps];
            s_carry = s_wmin[kWarps];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double drift;
        int l = seq_leaving(c, c.rows, s_ncand, false, &drift);
        if (drift > 32.0 * tol) l = seq_leaving(c, nullptr, c.m, true, &drift);  // tie chains: scan every row
        s_leave = l;
    }
    __syncthreads();
    const int r = s_leave;
    __syncthreads();
    return r;
}

// _pivot (simplex.py:53-58) on row r, column col, over columns [0, ncols); the
// pivot column must be in c.scol (load_column)
__device__ void pivot(Ctx &c, int r, int col, int ncols) {
    const double *Tr = rp(c, r);
    const double p = c.scol[r];
    // normalised pivot row (the reference divides the stored row by the scalar
    // pivot value first) and its nonzero pattern, in every CTA
    for (int j0 = threadIdx.x; j0 < ncols; j0 += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = j0 + u * kThreads < ncols ? lda(c, Tr + j0 + u * kThreads) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (j0 + u * kThreads < ncols) c.prow[j0 + u * kThreads] = __ddiv_rn(v[u], p);
    }
    __syncthreads();
    // compact the nonzero columns and the owned rows i != r with a nonzero pivot-column
    // entry (order is irrelevant to the result): every warp ballots 32 at a time and
    // reserves its slots with one shared-memory atomic
    if (threadIdx.x == 0) {
        c.s_int[kWarps + 2] = 0;
        c.s_int[kWarps + 4] = 0;
    }
    __syncthreads();
    {
        const int lane = threadIdx.x & 31;
        for (int j0 = threadIdx.x - lane; j0 < ncols; j0 += kThreads) {
            const int j = j0 + lane;
            const bool nzj = j < ncols && c.prow[j] != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, nzj);
            int at = 0;
            if (lane == 0 && bal) at = atomicAdd(&c.s_int[kWarps + 2], __popc(bal));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (nzj) c.nz[at + __popc(bal & ((1u << lane) - 1))] = j;
        }
        const int n_own = (c.m - c.rank) / c.ncta + 1;  // rows rank, rank + ncta, ... <= m
        for (int k0 = threadIdx.x - lane; k0 < n_own; k0 += kThreads) {
            const int i = c.rank + (k0 + lane) * c.ncta;
            const bool act = k0 + lane < n_own && i <= c.m && i != r && c.scol[i] != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            int at = 0;
            if (lane == 0 && bal) at = atomicAdd(&c.s_int[kWarps + 4], __popc(bal));
            at = __shfl_sync(0xffffffffu, at, 0);
            if (act) c.rows[at + __popc(bal & ((1u << lane) - 1))] = i;
        }
    }
    __syncthreads();
    const int nnz = c.s_int[kWarps + 2], nrows = c.s_int[kWarps + 4];
    cluster_sync(c);  // (A) every CTA holds row r; nobody has written yet
    // the pivot row itself (its owner)
    if (r % c.ncta == c.rank) {
        double *Tr_w = rp(c, r);
        for (int j = threadIdx.x; j < ncols; j += kThreads) Tr_w[j] = c.prow[j];
    }
    // T[i][j] -= f_i * prow[j] over (active rows) x (nonzero columns), flattened so
    // every thread has kU independent loads in flight
    constexpr int kU = 4;
    const int64_t work = (int64_t)nrows * nnz;
    for (int64_t base = threadIdx.x; base < work; base += (int64_t)kThreads * kU) {
        double v[kU];
        double *ptr[kU];
        double f[kU], pr[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int64_t idx = base + (int64_t)u * kThreads;
            ptr[u] = nullptr;
            if (idx < work) {
                const int ri = (int)(idx / nnz), k = (int)(idx - (int64_t)ri * nnz);
                const int i = c.rows[ri], j = c.nz[k];
                ptr[u] = rp(c, i) + j;
                f[u] = c.scol[i];
                pr[u] = c.prow[j];
                v[u] = lda(c, ptr[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (ptr[u]) *ptr[u] = __dsub_rn(v[u], __dmul_rn(f[u], pr[u]));
    }
    if (threadIdx.x == 0) c.basis[r] = col;
    cluster_sync(c);  // (B) the tableau is consistent again
}

// _run_phase: returns pivots done; *status set on unbounded / max_iter
__device__ int64_t run_phase(Ctx &c, int allowed, int ncols, int64_t max_iter, int *status) {
    int64_t iters = 0;
    while (true) {
        const int e = choose_entering(c, allowed);
        if (e == INT_MAX) return iters;
        load_column(c, e);
        const int l = choose_leaving(c);
        if (l < 0) {
            *status = ST_UNBOUNDED;
            return iters;
        }
        pivot(c, l, e, ncols);
        ++iters;
        if (iters > max_iter) {
            *status = ST_MAXITER;
            return iters;
        }
    }
}

// assemble [a | slacks | (artificials) | b] with the b < 0 rows negated, rhs at
// column ncols_rhs_at; the cluster's threads split the elements (any CTA may write any
// row: DSMEM stores in dsm mode)
__device__ void assemble(Ctx &c, const Args &a, int ncols_rhs_at) {
    const int n = (int)a.n, m_eq = (int)a.m_eq;
    const int tid = threadIdx.x + c.rank * kThreads, nth = kThreads * c.ncta;
    for (int64_t idx = tid; idx < (int64_t)(c.m + 1) * c.ld; idx += nth)
        rp(c, (int)(idx / c.ld))[idx % c.ld] = 0.0;
    cluster_sync(c);
    for (int64_t idx = tid; idx < (int64_t)c.m * n; idx += nth) {
        const int i = (int)(idx / n), j = (int)(idx % n);
        const double b = i < m_eq ? a.b_eq[i] : a.b_ub[i - m_eq];
        double v = i < m_eq ? a.a_eq[(int64_t)i * n + j] : a.a_ub[(int64_t)(i - m_eq) * n + j];
        rp(c, i)[j] = b < 0 ? -v : v;
    }
    for (int i = tid; i < c.m; i += nth) {
        const double b = i < m_eq ? a.b_eq[i] : a.b_ub[i - m_eq];
        if (i >= m_eq) rp(c, i)[n + (i - m_eq)] = b < 0 ? -1.0 : 1.0;
        rp(c, i)[ncols_rhs_at] = b < 0 ? -b : b;
    }
    cluster_sync(c);
}

__global__ void __launch_bounds__(kThreads, 1) lp_kernel(Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Ctx c{cg::this_cluster()};
    c.rank = (int)c.cl.block_rank();
    c.ncta = (int)c.cl.num_blocks();
    c.m = (int)(a.m_eq + a.m_ub);
    c.width = (int)(a.n + a.m_ub);
    c.ld = a.ld;
    c.tol = a.tol;
    // smem: sv[kThreads] doubles | prow[ld] doubles | si[kThreads] | nz[ld] | basis[m] | ints
    const int m1 = c.m > 0 ? c.m : 1;
    double *sv = reinterpret_cast<double *>(smem_raw);
    c.sdbl = sv;  // the argmax scratch of the warm start is not live at the same time
    c.prow = sv + kThreads;
    c.scol = c.prow + a.ld;
    c.sratio = c.scol + (c.m + 1);
    int *si = reinterpret_cast<int *>(c.sratio + m1);
    c.nz = si + kThreads;
    c.basis = c.nz + a.ld;
    c.rows = c.basis + m1;
    c.s_int = c.rows + (c.m + 1);
    c.T = a.T0;
    c.dsm = a.dsm != 0;
    c.rows_local = nullptr;
    c.lg = 0;
    while ((1 << c.lg) < c.ncta) ++c.lg;
    if (c.dsm) {
        // this CTA's rows follow the scratch arrays (16-byte aligned); peer[r] = CTA r's block
        uintptr_t off = reinterpret_cast<uintptr_t>(c.s_int + sint_count(c.m));
        c.rows_local = reinterpret_cast<double *>((off + 15) & ~(uintptr_t)15);
    }
    const int m = c.m, width = c.width, n = (int)a.n, m_eq = (int)a.m_eq;
    int status = ST_OK;
    int64_t iters = 0, p1 = 0, p2 = 0;
    int warm = 0, n_art = 0;

    // ---- warm start (simplex.py:127-144) ---------------------------------
    bool warm_ok = a.basis_in != nullptr;
    if (warm_ok) {
        for (int i = threadIdx.x; i < m; i += kThreads) c.basis[i] = (int)a.basis_in[i];
        __syncthreads();
        for (int i = 0; i < m; ++i)
            if (c.basis[i] < 0 || c.basis[i] >= width) warm_ok = false;
    }
    if (warm_ok) {
        // [a | b] with rhs at column `width`; Gauss-Jordan on the basis columns with
        // partial pivoting (first maximum |entry| among the unassigned rows, as idamax)
        c.total = width;
        assemble(c, a, width);
        int *assigned = c.s_int + kWarps + 8;  // [m] row -> basis position or -1
        for (int i = threadIdx.x; i < m; i += kThreads) assigned[i] = -1;
        __syncthreads();
        int *want = assigned + m;  // [m] copy of the requested basis
        for (int i = threadIdx.x; i < m; i += kThreads) want[i] = c.basis[i];
        __syncthreads();
        bool singular = false;
        for (int k = 0; k < m && !singular; ++k) {
            const int col = want[k];
            // argmax |T[i][col]| over unassigned rows, lowest row on ties
            load_column(c, col);
            double bv = -1.0;
            int bi = INT_MAX;
            for (int i = threadIdx.x; i < m; i += kThreads) {
                if (assigned[i] >= 0) continue;
                const double v = fabs(c.scol[i]);
                if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
            }
            // block argmax through shared memory (deterministic: value then row)
            sv[threadIdx.x] = bv;
            si[threadIdx.x] = bi;
            __syncthreads();
            for (int s = kThreads / 2; s > 0; s >>= 1) {
                if (threadIdx.x < s) {
                    const double v2 = sv[threadIdx.x + s];
                    const int i2 = si[threadIdx.x + s];
                    if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
                        sv[threadIdx.x] = v2;
                        si[threadIdx.x] = i2;
                    }
                }
                __syncthreads();
            }
            const double pv = sv[0];
            const int pr = si[0];
            __syncthreads();
            if (!(pv > 0.0)) {
                singular = true;  // LAPACK dgesv: exactly singular -> LinAlgError -> cold start
                break;
            }
            pivot(c, pr, col, width + 1);
            if (threadIdx.x == 0) assigned[pr] = k;
            __syncthreads();
        }
        if (!singular) {
            // rows into basis order (tableau row k <-> basis[k]) into T1, then check
            // primal feasibility of the new rhs
            const int tid = threadIdx.x + c.rank * kThreads, nth = kThreads * c.ncta;
            for (int64_t idx = tid; idx < (int64_t)m * (width + 1); idx += nth) {
                const int i = (int)(idx / (width + 1)), j = (int)(idx % (width + 1));
                a.T1[(int64_t)assigned[i] * c.ld + j] = lda(c, rp(c, i) + j);
            }
            cluster_sync(c);
            for (int64_t idx = tid; idx < (int64_t)m * (width + 1); idx += nth) {
                const int k = (int)(idx / (width + 1)), j = (int)(idx % (width + 1));
                rp(c, k)[j] = __ldcg(a.T1 + (int64_t)k * c.ld + j);
            }
            cluster_sync(c);
            for (int i = threadIdx.x; i < m; i += kThreads) c.basis[i] = want[i];
            __syncthreads();
            int infeas = INT_MAX;
            for (int i = threadIdx.x; i < m; i += kThreads)
                if (lda(c, rp(c, i) + width) < -c.tol) infeas = i;
            infeas = block_min_int(infeas, c.s_int);
            if (infeas == INT_MAX) {
                warm = 1;
                // objective row: c, then eliminate the basic columns in basis-row order
                // (basic columns are exact unit vectors here, so each column is independent)
                double *obj = rp(c, m);
                for (int j = threadIdx.x + c.rank * kThreads; j <= width; j += nth) {
                    double o = j < n ? a.c[j] : 0.0;
                    for (int i = 0; i < m; ++i) {
                        const int bvi = c.basis[i];
                        const double coeff = bvi < n ? a.c[bvi] : 0.0;
                        if (coeff != 0.0) o = __dsub_rn(o, __dmul_rn(coeff, lda(c, rp(c, i) + j)));
                    }
                    obj[j] = o;
                }
                cluster_sync(c);
                p2 = run_phase(c, width, width + 1, a.max_iter, &status);
                iters += p2;
            }
        }
        cluster_sync(c);
    }

    if (!warm) {
        // ---- cold start: phase 1 with artificials (simplex.py:146-177) ----
        iters = 0;
        p2 = 0;
        status = ST_OK;
        // which rows need an artificial: equality rows, and a_ub rows whose b < 0
        // (their slack was negated); identical in every CTA
        if (threadIdx.x == 0) {
            int k = 0;
            for (int i = 0; i < m; ++i) {
                const bool need = i < m_eq || a.b_ub[i - m_eq] < 0;
                c.basis[i] = need ? width + k++ : n + (i - m_eq);
            }
            c.s_int[kWarps + 3] = k;
        }
        __syncthreads();
        n_art = c.s_int[kWarps + 3];
        c.total = width + n_art;
        assemble(c, a, c.total);
        const int tid = threadIdx.x + c.rank * kThreads, nth = kThreads * c.ncta;
        for (int i = tid; i < m; i += nth)
            if (c.basis[i] >= width) rp(c, i)[c.basis[i]] = 1.0;
        cluster_sync(c);
        if (n_art) {
            // objective: 1 on the artificial columns, minus every artificial row in
            // row order (column-independent sequential subtraction)
            double *obj = rp(c, m);
            for (int j = tid; j <= c.total; j += nth) {
                double o = (j >= width && j < c.total) ? 1.0 : 0.0;
                for (int i = 0; i < m; ++i)
                    if (c.basis[i] >= width) o = __dsub_rn(o, lda(c, rp(c, i) + j));
                obj[j] = o;
            }
            cluster_sync(c);
            p1 = run_phase(c, c.total, c.total + 1, a.max_iter, &status);
            iters += p1;
            if (status == ST_OK && lda(c, obj + c.total) < -1e-7) status = ST_INFEASIBLE;
            if (status == ST_OK) {
                // drive surviving artificials out of the basis where possible
                for (int i = 0; i < m; ++i) {
                    if (c.basis[i] < width) continue;
                    int j0 = INT_MAX;
                    const double *Ti = rp(c, i);
                    for (int j = threadIdx.x; j < width; j += kThreads)
                        if (fabs(lda(c, Ti + j)) > c.tol) { j0 = j; break; }
                    j0 = block_min_int(j0, c.s_int);
                    if (j0 != INT_MAX) {
                        load_column(c, j0);
                        pivot(c, i, j0, c.total + 1);
                        ++iters;
                    }
                }
            }
        }
        if (status == ST_OK) {
            // phase-2 objective (simplex.py:179-185): row = c; for each basis row in
            // order, row -= obj[bv] * T[i].  Basic columns are exact unit vectors after
            // pivoting, so obj[bv_i] is still its initial value when row i is reached
            // and every column can be computed independently in the same order.
            double *obj = rp(c, m);
            for (int j = tid; j <= c.total; j += nth) {
                double o = j < n ? a.c[j] : 0.0;
                for (int i = 0; i < m; ++i) {
                    const int bvi = c.basis[i];
                    const double coeff = bvi < n ? a.c[bvi] : 0.0;
                    if (coeff != 0.0) o = __dsub_rn(o, __dmul_rn(coeff, lda(c, rp(c, i) + j)));
                }
                obj[j] = o;
            }
            cluster_sync(c);
            p2 = run_phase(c, width, c.total + 1, a.max_iter, &status);
            iters += p2;
        }
    }

    // ---- extract (simplex.py:195-208) -------------------------------------
    if (c.rank == 0) {
        for (int j = threadIdx.x; j < width; j += kThreads) a.x_full[j] = 0.0;
        __syncthreads();
        for (int i = threadIdx.x; i < m; i += kThreads) {
            const int bv = c.basis[i];
            if (bv < width) a.x_full[bv] = lda(c, rp(c, i) + c.total);
            a.basis_out[i] = bv;
        }
        if (threadIdx.x == 0) {
            a.info[0] = iters;
            a.info[1] = status;
            a.info[2] = warm;
            a.info[3] = n_art;
            a.info[4] = p1;
            a.info[5] = p2;
            a.info[6] = c.dsm ? c.ncta : 0;
        }
    }
    cluster_sync(c);  // dsm: rank 0 read the other CTAs' rows; they stay resident until here
}

static size_t smem_bytes(int64_t ld, int64_t m) {
    // sv/prow doubles, si/nz/basis ints, scratch ints (kWarps + 8 +
    // assigned[m] + want[m] + 1) + argmax scratch (kThreads doubles + ints)
    const size_t m1 = m > 0 ? (size_t)m : 1;
    size_t b = (size_t)(kThreads + ld + (m + 1) + m1) * sizeof(double) + (size_t)(kThreads + ld) * sizeof(int);
    b += (m1 + (size_t)(m + 1)) * sizeof(int) + (size_t)sint_count(m) * sizeof(int);
    return b;
}

}  // namespace lp
}  // namespace hep

using namespace hep;

extern "C" size_t hep_lp_workspace(int64_t n, int64_t m_eq, int64_t m_ub) {
    const int64_t m = m_eq + m_ub, ld = n + m_ub + m + 1;
    return 2 * (size_t)(m + 1) * (size_t)ld * sizeof(double);
}

extern "C" int hep_lp_solve(const double *d_c, const double *d_a_eq, const double *d_b_eq, const double *d_a_ub,
                            const double *d_b_ub, int64_t n, int64_t m_eq, int64_t m_ub, const int64_t *d_basis_in,
                            double tol, int64_t max_iter, void *d_work, size_t work_bytes, double *d_x_full,
                            int64_t *d_basis_out, int64_t *d_info, void *stream) {
    HEP_NVTX("hep_lp_solve");
    const int64_t m = m_eq + m_ub, ld = n + m_ub + m + 1;
    HEP_REQUIRE(n >= 0 && m_eq >= 0 && m_ub >= 0 && n + m_ub > 0, HEP_E_DIMENSION,
                "hep_lp_solve: bad sizes n=%lld m_eq=%lld m_ub=%lld", (long long)n, (long long)m_eq, (long long)m_ub);
    HEP_REQUIRE(d_c && d_x_full && d_basis_out && d_info && d_work, HEP_E_CONTRACT, "hep_lp_solve: null pointer");
    HEP_REQUIRE(work_bytes >= hep_lp_workspace(n, m_eq, m_ub), HEP_E_CAPACITY,
                "hep_lp_solve: workspace %zu B < %zu B", work_bytes, hep_lp_workspace(n, m_eq, m_ub));
    const size_t smem = lp::smem_bytes(ld, m);
    HEP_REQUIRE(smem <= 227 * 1024, HEP_E_CAPACITY,
                "hep_lp_solve: LP too large for the on-chip pivot row (%lld columns, %lld rows)", (long long)ld,
                (long long)m);
    HEP_REQUIRE(m < (1LL << 30) && ld < (1LL << 30), HEP_E_CAPACITY, "hep_lp_solve: LP too large");
    // cluster size: ~16+ rows per CTA, up to 8 CTAs (portable cluster size)
    int ncta = 1;
    while (ncta < 8 && (m + 1) > 16 * ncta) ncta *= 2;
    // distributed shared memory: the tableau's rows spread over the cluster's shared
    // memory when they fit (8 or, non-portable, 16 CTAs), else global memory (L2)
    int dsm = 0;
    size_t smem_launch = smem;
    if (g_tuning.lp_dsm != 0) {
        for (int nc = ncta < 8 ? 8 : ncta; nc <= 8 && !dsm; nc *= 2) {
            const int64_t rpc = (m + 1 + nc - 1) / nc;
            const size_t need = ((smem + 15) & ~(size_t)15) + 16 + (size_t)rpc * (size_t)ld * sizeof(double);
            if (need > 227 * 1024) continue;
            HEP_CHECK_CUDA(cudaFuncSetAttribute(lp::lp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
            if (nc > 8)
                HEP_CHECK_CUDA(cudaFuncSetAttribute(lp::lp_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(nc);
            q.blockDim = dim3(lp::kThreads);
            q.dynamicSmemBytes = need;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = nc;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            q.attrs = at;
            q.numAttrs = 1;
            int n_cl = 0;
            if (cudaOccupancyMaxActiveClusters(&n_cl, lp::lp_kernel, &q) == cudaSuccess && n_cl >= 1) {
                dsm = 1;
                ncta = nc;
                smem_launch = need;
            } else {
                (void)cudaGetLastError();
            }
        }
    }
    HEP_CHECK_CUDA(cudaFuncSetAttribute(lp::lp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_launch));
    lp::Args a;
    a.dsm = dsm;
    a.c = d_c;
    a.a_eq = d_a_eq;
    a.b_eq = d_b_eq;
    a.a_ub = d_a_ub;
    a.b_ub = d_b_ub;
    a.basis_in = d_basis_in;
    a.n = n;
    a.m_eq = m_eq;
    a.m_ub = m_ub;
    a.tol = tol;
    a.max_iter = max_iter;
    a.T0 = static_cast<double *>(d_work);
    a.T1 = a.T0 + (m + 1) * ld;
    a.ld = ld;
    a.x_full = d_x_full;
    a.basis_out = d_basis_out;
    a.info = d_info;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(lp::kThreads);
    cfg.dynamicSmemBytes = smem_launch;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HEP_CHECK_CUDA(cudaLaunchKernelEx(&cfg, lp::lp_kernel, a));
    return HEP_OK;
}
