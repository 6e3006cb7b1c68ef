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

enum : int { ST_OK = 0, ST_INFEASIBLE = 1, ST_UNBOUNDED = 2, ST_MAXITER = 3 };

struct Args {
    const double *c, *a_eq, *b_eq, *a_ub, *b_ub;
    const int64_t *basis_in;  // device [m] or null
    int64_t n, m_eq, m_ub;
    double tol;
    int64_t max_iter;
    double *T0, *T1;          // workspace tableaux [(m+1) * ld]
    int64_t ld;
    double *x_full;           // out [width] (reference x_full before the [:n] clip)
    int64_t *basis_out;       // out [m]
    int64_t *info;            // out [8]: pivots, status, warm_used, n_art, phase1_pivots, phase2_pivots
};

__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

// one thread-block cluster; all CTAs run the same control flow on the same data
struct Ctx {
    cg::cluster_group cl;
    int rank, ncta;
    int m, width, total;  // rows (excl. objective), vars+slacks, columns excl. rhs
    int64_t ld;
    double *T;
    int *basis;     // smem copy, identical in every CTA
    double *prow;   // smem [total+1] normalised pivot row
    int *nz;        // smem [total+1] nonzero columns of the pivot row
    int *s_int;     // smem scratch ints
    double *scol;   // smem [m+1] pivot column T[i][col] of every row (incl. objective)
    double *sratio; // smem [m] rhs/col for eligible rows, +inf otherwise
    int *rows;      // smem [m+1] owned rows with a nonzero pivot-column entry
    double tol;
};

// barrier.cluster.arrive (.release) + barrier.cluster.wait (.acquire): orders every
// CTA's global tableau writes before the other CTAs' (L2, ld.global.cg) reads
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
    const double *obj = c.T + (int64_t)c.m * c.ld;
    const double ntol = -c.tol;
    int best = INT_MAX;
    for (int j0 = threadIdx.x; j0 < allowed && best == INT_MAX; j0 += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = j0 + u * kThreads < allowed ? ldcg(obj + j0 + u * kThreads) : 0.0;
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
            a[u] = i <= c.m ? ldcg(c.T + (int64_t)i * c.ld + col) : 0.0;
            rhs[u] = i < c.m ? ldcg(c.T + (int64_t)i * c.ld + c.total) : 0.0;
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

// _run_phase's leaving rule, the reference's sequential scan over rows 0..m-1
// (simplex.py:75-86) on the ratios in shared memory: warp 0 walks the rows 32 at a
// time and skips a chunk in one step when none of its ratios can displace the current
// best (a replacement needs ratio <= best + tol).  Returns -1 if unbounded.
__device__ int choose_leaving(Ctx &c) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const double tol = c.tol;
        bool have = false;
        double best = 0.0;
        int leave = -1;
        for (int base = 0; base < c.m; base += 32) {
            const int i = base + lane;
            const bool el = i < c.m && c.scol[i] > tol;
            const double ratio = el ? c.sratio[i] : __longlong_as_double(0x7ff0000000000000LL);
            unsigned any = __ballot_sync(0xffffffffu, el);
            if (!any) continue;
            if (have) {
                double mn = ratio;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                // nobody here can be accepted (a replacement needs ratio <= best + tol;
                // the margin absorbs the rounding of best + tol and |ratio - best|)
                if (mn > best + 2.0 * tol + fabs(best) * 1e-12) continue;
            }
            const int bi = i < c.m ? c.basis[i] : 0;
            while (any) {
                const int l = __ffs(any) - 1;
                any &= any - 1;
                const double r = __shfl_sync(0xffffffffu, ratio, l);
                const int b = __shfl_sync(0xffffffffu, bi, l);
                bool take;
                if (!have) take = true;
                else if (r < best - tol) take = true;
                else take = fabs(r - best) <= tol && b < c.basis[leave];
                if (take) {
                    have = true;
                    best = r;
                    leave = base + l;
                }
            }
        }
        if (lane == 0) c.s_int[kWarps + 1] = leave;
    }
    __syncthreads();
    int r = c.s_int[kWarps + 1];
    __syncthreads();
    return r;
}

// _pivot (simplex.py:53-58) on row r, column col, over columns [0, ncols); the
// pivot column must be in c.scol (load_column)
__device__ void pivot(Ctx &c, int r, int col, int ncols) {
    const double *Tr = c.T + (int64_t)r * c.ld;
    const double p = c.scol[r];
    // normalised pivot row (the reference divides the stored row by the scalar
    // pivot value first) and its nonzero pattern, in every CTA
    for (int j0 = threadIdx.x; j0 < ncols; j0 += 4 * kThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = j0 + u * kThreads < ncols ? ldcg(Tr + j0 + u * kThreads) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (j0 + u * kThreads < ncols) c.prow[j0 + u * kThreads] = __ddiv_rn(v[u], p);
    }
    __syncthreads();
    // compact nonzero columns (warp 0) and owned rows i != r with a nonzero pivot-
    // column entry (warp 1); order is irrelevant to the result
    if (threadIdx.x < 32) {
        int cnt = 0;
        for (int base = 0; base < ncols; base += 32) {
            const int j = base + threadIdx.x;
            const bool nzj = j < ncols && c.prow[j] != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, nzj);
            if (nzj) c.nz[cnt + __popc(bal & ((1u << threadIdx.x) - 1))] = j;
            cnt += __popc(bal);
        }
        if (threadIdx.x == 0) c.s_int[kWarps + 2] = cnt;
    } else if (threadIdx.x < 64) {
        const int lane = threadIdx.x - 32;
        int cnt = 0;
        for (int base = c.rank; base <= c.m; base += 32 * c.ncta) {
            const int i = base + lane * c.ncta;
            const bool act = i <= c.m && i != r && c.scol[i] != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            if (act) c.rows[cnt + __popc(bal & ((1u << lane) - 1))] = i;
            cnt += __popc(bal);
        }
        if (lane == 0) c.s_int[kWarps + 4] = cnt;
    }
    __syncthreads();
    const int nnz = c.s_int[kWarps + 2], nrows = c.s_int[kWarps + 4];
    cluster_sync(c);  // (A) every CTA holds row r; nobody has written yet
    // the pivot row itself (its owner)
    if (r % c.ncta == c.rank) {
        double *Tr_w = c.T + (int64_t)r * c.ld;
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
                ptr[u] = c.T + (int64_t)i * c.ld + j;
                f[u] = c.scol[i];
                pr[u] = c.prow[j];
                v[u] = ldcg(ptr[u]);
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

// assemble [a | slacks | (artificials) | b] with the b < 0 rows negated
__device__ void assemble(Ctx &c, const Args &a, double *T, int ncols_rhs_at, bool with_slack_art, int n_art_max) {
    const int n = (int)a.n, m_eq = (int)a.m_eq;
    const int tid = threadIdx.x + c.rank * kThreads, nth = kThreads * c.ncta;
    for (int64_t idx = tid; idx < (int64_t)(c.m + 1) * c.ld; idx += nth) T[idx] = 0.0;
    cluster_sync(c);
    for (int64_t idx = tid; idx < (int64_t)c.m * n; idx += nth) {
        const int i = (int)(idx / n), j = (int)(idx % n);
        const double b = i < m_eq ? a.b_eq[i] : a.b_ub[i - m_eq];
        double v = i < m_eq ? a.a_eq[(int64_t)i * n + j] : a.a_ub[(int64_t)(i - m_eq) * n + j];
        T[(int64_t)i * c.ld + j] = b < 0 ? -v : v;
    }
    for (int i = tid; i < c.m; i += nth) {
        const double b = i < m_eq ? a.b_eq[i] : a.b_ub[i - m_eq];
        if (i >= m_eq) T[(int64_t)i * c.ld + n + (i - m_eq)] = b < 0 ? -1.0 : 1.0;
        T[(int64_t)i * c.ld + ncols_rhs_at] = b < 0 ? -b : b;
    }
    (void)with_slack_art;
    (void)n_art_max;
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
    c.prow = sv + kThreads;
    c.scol = c.prow + a.ld;
    c.sratio = c.scol + (c.m + 1);
    int *si = reinterpret_cast<int *>(c.sratio + m1);
    c.nz = si + kThreads;
    c.basis = c.nz + a.ld;
    c.rows = c.basis + m1;
    c.s_int = c.rows + (c.m + 1);
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
        c.T = a.T0;
        c.total = width;
        assemble(c, a, c.T, width, true, 0);
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
                a.T1[(int64_t)assigned[i] * c.ld + j] = ldcg(c.T + (int64_t)i * c.ld + j);
            }
            cluster_sync(c);
            c.T = a.T1;
            for (int i = threadIdx.x; i < m; i += kThreads) c.basis[i] = want[i];
            __syncthreads();
            int infeas = INT_MAX;
            for (int i = threadIdx.x; i < m; i += kThreads)
                if (ldcg(c.T + (int64_t)i * c.ld + width) < -c.tol) infeas = i;
            infeas = block_min_int(infeas, c.s_int);
            if (infeas == INT_MAX) {
                warm = 1;
                // objective row: c, then eliminate the basic columns in basis-row order
                // (basic columns are exact unit vectors here, so each column is independent)
                double *obj = c.T + (int64_t)m * c.ld;
                for (int j = threadIdx.x + c.rank * kThreads; j <= width; j += nth) {
                    double o = j < n ? a.c[j] : 0.0;
                    for (int i = 0; i < m; ++i) {
                        const int bvi = c.basis[i];
                        const double coeff = bvi < n ? a.c[bvi] : 0.0;
                        if (coeff != 0.0) o = __dsub_rn(o, __dmul_rn(coeff, ldcg(c.T + (int64_t)i * c.ld + j)));
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
        c.T = a.T0;
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
        assemble(c, a, c.T, c.total, true, n_art);
        const int tid = threadIdx.x + c.rank * kThreads, nth = kThreads * c.ncta;
        for (int i = tid; i < m; i += nth)
            if (c.basis[i] >= width) c.T[(int64_t)i * c.ld + c.basis[i]] = 1.0;
        cluster_sync(c);
        if (n_art) {
            // objective: 1 on the artificial columns, minus every artificial row in
            // row order (column-independent sequential subtraction)
            double *obj = c.T + (int64_t)m * c.ld;
            for (int j = tid; j <= c.total; j += nth) {
                double o = (j >= width && j < c.total) ? 1.0 : 0.0;
                for (int i = 0; i < m; ++i)
                    if (c.basis[i] >= width) o = __dsub_rn(o, ldcg(c.T + (int64_t)i * c.ld + j));
                obj[j] = o;
            }
            cluster_sync(c);
            p1 = run_phase(c, c.total, c.total + 1, a.max_iter, &status);
            iters += p1;
            if (status == ST_OK && ldcg(obj + c.total) < -1e-7) status = ST_INFEASIBLE;
            if (status == ST_OK) {
                // drive surviving artificials out of the basis where possible
                for (int i = 0; i < m; ++i) {
                    if (c.basis[i] < width) continue;
                    int j0 = INT_MAX;
                    const double *Ti = c.T + (int64_t)i * c.ld;
                    for (int j = threadIdx.x; j < width; j += kThreads)
                        if (fabs(ldcg(Ti + j)) > c.tol) { j0 = j; break; }
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
            double *obj = c.T + (int64_t)m * c.ld;
            for (int j = tid; j <= c.total; j += nth) {
                double o = j < n ? a.c[j] : 0.0;
                for (int i = 0; i < m; ++i) {
                    const int bvi = c.basis[i];
                    const double coeff = bvi < n ? a.c[bvi] : 0.0;
                    if (coeff != 0.0) o = __dsub_rn(o, __dmul_rn(coeff, ldcg(c.T + (int64_t)i * c.ld + j)));
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
            if (bv < width) a.x_full[bv] = ldcg(c.T + (int64_t)i * c.ld + c.total);
            a.basis_out[i] = bv;
        }
        if (threadIdx.x == 0) {
            a.info[0] = iters;
            a.info[1] = status;
            a.info[2] = warm;
            a.info[3] = n_art;
            a.info[4] = p1;
            a.info[5] = p2;
        }
    }
}

static size_t smem_bytes(int64_t ld, int64_t m) {
    // sv/prow doubles, si/nz/basis ints, scratch ints (kWarps + 8 +
    // assigned[m] + want[m] + 1) + argmax scratch (kThreads doubles + ints)
    const size_t m1 = m > 0 ? (size_t)m : 1;
    size_t b = (size_t)(kThreads + ld + (m + 1) + m1) * sizeof(double) + (size_t)(kThreads + ld) * sizeof(int);
    b += (m1 + (size_t)(m + 1)) * sizeof(int) + (size_t)(kWarps + 8 + 2 * m + 2) * sizeof(int);
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
    HEP_CHECK_CUDA(cudaFuncSetAttribute(lp::lp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    lp::Args a;
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
    cfg.dynamicSmemBytes = smem;
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
