/*
 * hep.h — C ABI of the B200-native HarmonyEP token-scheduling MoE path.
 *
 * Plain C types only (pointers, sizes, int status codes); no torch types.
 * Every pointer named d_* is a DEVICE pointer (cudaMalloc / torch CUDA
 * tensor storage); every other pointer is host memory.  `stream` is a
 * cudaStream_t passed as void*.  Nothing in this ABI allocates or
 * synchronizes inside a hot call (hep_sched_solve, hep_moe_*): buffers are
 * caller-owned, and the handle owns only its placement tables.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/harmonyep/).
 *
 * Status codes mirror the reference error classes (core.py:36-84):
 */
#ifndef HEP_H_
#define HEP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HEP_OK 0
#define HEP_E_DIMENSION 1  /* core.DimensionError  */
#define HEP_E_PLACEMENT 2  /* core.PlacementError  */
#define HEP_E_CONTRACT 3   /* core.ContractViolation */
#define HEP_E_STALE 4      /* core.StaleStateError */
#define HEP_E_CAPACITY 5   /* core.CapacityError   */
#define HEP_E_INTERNAL 99
#define HEP_E_CUDA 100     /* CUDA runtime / launch failure (message in hep_last_error) */

/* Largest scheduling group the device solver handles (2^G subsets live in
 * registers of one warp).  The reference's own tests use G <= 10. */
#define HEP_MAX_GPUS 10

/* Thread-local message for the last non-zero status returned on this thread. */
const char *hep_last_error(void);
int hep_abi_version(void);
/* Number of SMs of the current device (grid sizing helper for callers). */
int hep_device_sm_count(void);

/*
 * Launch-shape tuning, process-wide and explicit (the library never reads the
 * environment).  The defaults are the measured winners; the A/B tools
 * in tools/ change them through hep_tuning_set.  Values are read when an entry point
 * launches, so a CUDA graph keeps the tuning that was active at capture time.
 * A field set to -1 keeps / restores its default.
 */
typedef struct {
    int st256;              /* 1: 256-bit epilogue stores / pre-activation loads when rows are 32-B aligned */
    int pair_wait_cluster;  /* 1: CTA-pair mbarrier waits with .acquire.cluster (0, measured slower) */
    int ffn_pair;           /* CTA-pair grouped GEMM: -2 auto (>= 512 rows per expert), 0 never, 1 always */
    int ffn_light_rows;     /* light-expert split threshold in rows (default 256; 0 disables) */
    int wgrad_order;        /* 1: weight-gradient tiles visit experts heaviest first */
    int l2_policy;          /* 0: default TMA L2 hints; else (A | B << 2), 1 normal, 2 last, 3 first */
    int light_first;        /* 1: single-m-tile experts load their weights evict-first */
    int raster_gm1;         /* raster band (m-tiles) of the SwiGLU GEMM (16) */
    int raster_gm2;         /* raster band of the down projection (8) */
    int sched_lexmin_warps; /* warps on the scheduler's lex-min arc chain (4) */
    int lsu256;             /* 1: 256-bit LDG/STG permute / combine when 32-B aligned */
    int ffn_clock;          /* 1: diagnostics, CTA 0 of each expert GEMM stamps clock64/globaltimer */
    int router_tile_rows;   /* router GEMM rows per CTA tile, multiple of 16 (0 = 128; shorter tiles measured slower) */
    int pair_wave_sync;     /* > 0: grouped CTA-pair GEMMs with >= this many 64-deep k-blocks per tile start
                               each wave of tiles together (TMA producers meet at a grid-wide counter) */
    int lp_dsm;             /* 1: comm-aware LP tableau in the cluster's distributed shared memory when it fits */
    int light_wave_sync;    /* 1: the 1-CTA grouped GEMMs (light experts) also start waves together (same threshold;
                               0 by default: DSv3 light GEMMs already read only their algorithmic bytes,
                               profiles/r02/wave_ab_r02h.txt) */
    int router_mc;          /* router GEMM: thread-block cluster size sharing each Wg tile by TMA multicast
                               (0 auto, 1 off, 2 or 4) */
    int router_pair;        /* router GEMM on CTA pairs (cta_group::2, half the Wg tile per CTA): 0 auto (E_pad > 128),
                               1 off, 2 on (E_pad > 64) */
    int wgrad_wave_sync;    /* 1: the weight-gradient CTA-pair GEMMs start each wave of tiles together */
    int wgrad_raster;       /* 1: weight-gradient tiles walk the shorter tile dimension fastest */
    int sched_route_serial; /* 1: scheduler routing (Algorithm 1) always as per-thread merges; 0: one lane
                               per (expert, source) with warp-shuffle prefixes while E <= 32 (G <= 8) */
    int reserved[1];
} hep_tuning;
int hep_tuning_get(hep_tuning *out);
int hep_tuning_set(const hep_tuning *in);

/* ======================================================================
 * Scheduler: exact min-max replica loads + canonical lex-min plan,
 * integerization, locality-first routing, transfer volumes.
 * ====================================================================== */
typedef struct hep_sched *hep_sched_t;

/*
 * Build the device placement tables (the `_BalanceNetwork` analogue,
 * scheduler.py:181-207, built once per placement and owned by the handle —
 * the SolverState of scheduler.py:151-170).
 *   grp_off[E+1], grp_gpu[grp_off[E]] : EDP groups in LIST order (core.py:164-226)
 *   slots[E]                           : local slot per expert (may be NULL)
 *   gpus_per_node                      : 0 = single node (core.py:99)
 * Replaces: SolverState(placement, options) / Placement validation (core.py:180-185).
 */
int hep_sched_create(int num_gpus, int num_experts, const int32_t *grp_off, const int32_t *grp_gpu,
                     const int32_t *slots, int gpus_per_node, hep_sched_t *out);
int hep_sched_destroy(hep_sched_t h);
/* nnz = number of (expert, gpu) replicas; max_ranges = routing-table capacity;
 * Q = lcm(1..G) (scheduler.py:184); transfer_len = G*G + 8*G + 2. */
int hep_sched_sizes(hep_sched_t h, int64_t *nnz, int64_t *max_ranges, int64_t *Q, int64_t *transfer_len);

/* Stage flags for hep_sched_solve */
#define HEP_SCHED_SOLVE 1      /* m + lex-min plan      (scheduler.py:337-402)          */
#define HEP_SCHED_INTEGERIZE 2 /* largest remainder     (scheduler.py:697-735)          */
#define HEP_SCHED_ROUTE 4      /* Algorithm 1 ranges    (router.py:114-163)             */
#define HEP_SCHED_TRANSFER 8   /* pair/send/recv/local  (router.py:178-226)             */
#define HEP_SCHED_TOPO 16      /* route_topology_aware  (router.py:166-175) instead of route_tokens */
#define HEP_SCHED_ALL 15
#define HEP_SCHED_PROFILE 32   /* diagnostics: record per-phase clock64 stamps (hep_sched_debug_timing) */

/* Device output buffers, caller-allocated (sizes from hep_sched_sizes). */
typedef struct {
    int64_t *d_m;          /* [4]  m numerator, m denominator, Q, integerized objective */
    int64_t *d_xq;         /* [nnz] replica loads x*Q, EDP-list order (ReplicaLoadPlan.entries) */
    int64_t *d_xi;         /* [nnz] integerized replica loads */
    int64_t *d_gpu_load;   /* [G]   integerized per-GPU load (ReplicaLoadPlan.gpu_loads) */
    int64_t *d_ranges;     /* [max_ranges*4] (expert, src, dst, count) — RoutingTable.ranges */
    int64_t *d_n_ranges;   /* [1] */
    int64_t *d_transfer;   /* [G*G+8G+2] pair, send, recv, local, send_intra, recv_intra,
                              send_inter, recv_inter, intra_volume, inter_volume (TransferPlan) */
    int32_t *d_status;     /* [1] device-detected error (HEP_E_PLACEMENT, HEP_E_CAPACITY, ...) */
} hep_sched_out;

/*
 * One micro-batch: loads -> m, plan, integerized plan, routing table, transfer plan,
 * in ONE single-CTA kernel launch on `stream` (no host sync).
 *   d_loads : int64 load matrix input_e^g, element (e,g) at d_loads[e*stride_e + g*stride_g]
 *             ([E][G] expert-major: stride_e=G, stride_g=1; the all-gathered [G][E]
 *             histogram: stride_e=1, stride_g=E)
 *   d_base  : int64 [G] gpu_base (pipelined share, scheduler.py:405-433) or NULL
 * Replaces: solve_replica_loads (scheduler.py:405-433), warm_solve (:436-461),
 *           integerize_plan (:697-735), route_tokens (router.py:161-163),
 *           route_topology_aware (:166-175), build_transfer_plan (:178-226).
 * Canonical result: the unique lex-min optimal plan (scheduler.py:19-26), so the
 * output is a pure function of (placement, loads): warm == cold, bit-identical
 * on every rank.
 */
int hep_sched_solve(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                    const int64_t *d_base, int flags, const hep_sched_out *out, void *stream);

/*
 * Integerize an arbitrary rational plan x = d_xnum / den (common denominator)
 * on the device.  Replaces integerize_plan (scheduler.py:697-735) for plans not
 * produced by hep_sched_solve.  Non-integer expert totals -> d_status = HEP_E_CONTRACT.
 */
int hep_sched_integerize(hep_sched_t h, const int64_t *d_xnum, int64_t den, const hep_sched_out *out,
                         void *stream);
/*
 * Route a caller-provided integral plan d_xi (EDP-list order) against d_loads.
 * Replaces route_tokens / route_topology_aware (router.py:114-175) incl. the
 * _check_plan contract (router.py:97-111) -> d_status = HEP_E_CONTRACT.
 */
int hep_sched_route(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g,
                    const int64_t *d_xi, int flags, const hep_sched_out *out, void *stream);
/*
 * Pipelined split (the reference's harmony_pipelined strategy, simulator.py:420-435):
 *   former = floor(loads * share_num / share_den), latter = loads - former   (_split_loads :291-298)
 *   static phase:    even split of each expert's former total over its replicas
 *                    (_even_split_plan :301-322), integerized, routed, transfer plan -> *former
 *   scheduled phase: exact solve of latter with gpu_base = the static phase's integerized
 *                    GPU loads, integerize, route, transfer                          -> *latter
 * share = 1 - pipeline_ratio (:375).  d_split: caller buffer int64 [2*E*G + G]: former and
 * latter loads ([E][G] each, expert-major; the route stages read them) and the static phase's
 * integerized GPU loads [G] (= the scheduled phase's gpu_base, computed by the split kernel).
 * stream_static (a cudaStream_t, or NULL = `stream`): the static phase's integerize / route /
 * transfer run there, forked after the split, concurrently with the scheduled phase's solve
 * on `stream`; its assignment and dispatch can follow on stream_static (simulator.py:451-453)
 * and the caller joins it back before the expert GEMMs.  The phases need distinct d_status
 * words.  flags: TRANSFER / TOPO as for hep_sched_solve.
 */
int hep_sched_pipelined(hep_sched_t h, const int64_t *d_loads, int64_t stride_e, int64_t stride_g, int64_t share_num,
                        int64_t share_den, int flags, int64_t *d_split, const hep_sched_out *former,
                        const hep_sched_out *latter, void *stream, void *stream_static);
/* Diagnostics: per-phase SM clock stamps of the last HEP_SCHED_PROFILE launch (n <= 16). */
int hep_sched_debug_timing(int64_t *host_out, int n);
/* Dense two-phase primal simplex with Bland's rule on one thread-block cluster (csrc/lp.cu).
 * Replaces simplex_solve (simplex.py:99-192), the solver of solve_comm_aware
 * (scheduler.py:622-689) on the _comm_aware_lp (:480-547) / _topology_aware_lp (:550-619)
 * programs:  min c.x  s.t.  a_eq x = b_eq,  a_ub x <= b_ub,  x >= 0.  All matrices dense
 * row-major fp64 in device memory (a_eq [m_eq][n], a_ub [m_ub][n]).  d_basis_in: the
 * previous optimal basis [m_eq+m_ub] (warm start, simplex.py:127-144) or NULL.  Outputs:
 * d_x_full [n+m_ub] (structural values first; the caller clips [:n] at 0), d_basis_out
 * [m_eq+m_ub], d_info [8] = {pivots, status (0 ok, 1 infeasible, 2 unbounded, 3 pivot
 * limit), warm start used, artificials, phase-1 pivots, phase-2 pivots, cluster size when the
 * tableau sat in distributed shared memory (0: global memory)}.  A cold solve
 * is bit-identical to the reference (same pivots, same fp64 roundings).  d_work: caller-
 * owned, hep_lp_workspace() bytes.  Asynchronous on `stream`. */
size_t hep_lp_workspace(int64_t n, int64_t m_eq, int64_t m_ub);
int hep_lp_solve(const double *d_c, const double *d_a_eq, const double *d_b_eq, const double *d_a_ub,
                 const double *d_b_ub, int64_t n, int64_t m_eq, int64_t m_ub, const int64_t *d_basis_in,
                 double tol, int64_t max_iter, void *d_work, size_t work_bytes, double *d_x_full,
                 int64_t *d_basis_out, int64_t *d_info, void *stream);

/* Aggregate an arbitrary routing table. Replaces build_transfer_plan (router.py:178-226). */
int hep_transfer_plan(int num_gpus, int gpus_per_node, const int64_t *d_ranges, int64_t n_ranges,
                      int64_t *d_transfer, int32_t *d_status, void *stream);

/* ======================================================================
 * MoE layer data path (builder-defined semantics; the reference models it only
 * as a cost, simulator.py:439-476).  bf16 activations / weights, fp32 accumulate.
 * ====================================================================== */

/*
 * K1 gate epilogue: top-K over fp32 router logits (+ optional per-expert
 * selection bias), weights = softmax over the K selected logits, and the
 * per-(source, expert) histogram (the load matrix column of source g,
 * LoadMatrix core.py:229-268).  Tokens [t0, t0+tokens_per_src) belong to
 * source (t / tokens_per_src).  Ties -> lower expert id.
 *   d_logits [T][ld_logits] fp32 (first E columns used), d_bias [E] or NULL,
 *   d_topk_idx [T][K] int32, d_topk_w [T][K] fp32, d_hist [n_src][E] int64 (zeroed here)
 */
int hep_gate_topk(const float *d_logits, int64_t ld_logits, const float *d_bias, int64_t T, int E, int K,
                  int64_t tokens_per_src, int n_src, int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist,
                  void *stream);

/*
 * K1 fused: router GEMM logits = x . Wg^T (tcgen05, fp32 accumulators in TMEM) with the
 * gate in its epilogue — one TMEM lane holds one token's whole logit row, so top-K,
 * the top-K softmax and the histogram (exactly hep_gate_topk's semantics, bit for bit)
 * are computed without the logits leaving the SM.
 *   d_x [T][d_model] bf16, d_wg [e_pad][d_model] bf16 (rows >= E zero), e_pad % 16 == 0
 *   d_logits [T][e_pad] fp32 or NULL (written when given; required when e_pad > 256 or
 *   K > 8, which take the unfused hep_gemm_bf16 + hep_gate_topk path)
 *   d_chunk_cnt: NULL, or the per-64-token-chunk expert counts hep_moe_assign_precounted
 *   consumes ([n_src][ceil(tps/64)][E] int32 at hep_moe_assign_chunk_offset of its
 *   workspace); fused into the epilogue when tokens_per_src % 64 == 0
 * Replaces: the LoadMatrix producer (core.py:229-268; the reference never models the gate).
 */
int hep_router_topk(const void *d_x, const void *d_wg, int64_t T, int64_t d_model, int E, int e_pad,
                    const float *d_bias, int K, int64_t tokens_per_src, int n_src, float *d_logits,
                    int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist, int32_t *d_chunk_cnt, void *stream);
/*
 * hep_router_topk without the separate zeroing launch of d_hist: the fused kernel's CTA 0
 * zeroes it and the other CTAs add their counts once it is done, synchronised through
 * d_sync (hep_router_sync_bytes() bytes, zeroed once by the caller; the kernel leaves them
 * zero again, so the call can be captured in a CUDA graph and replayed).  One d_sync per
 * concurrently running call (per layer / stream).  The unfused path ignores d_sync.
 */
int hep_router_topk_ws(const void *d_x, const void *d_wg, int64_t T, int64_t d_model, int E, int e_pad,
                       const float *d_bias, int K, int64_t tokens_per_src, int n_src, float *d_logits,
                       int32_t *d_topk_idx, float *d_topk_w, int64_t *d_hist, int32_t *d_chunk_cnt,
                       unsigned int *d_sync, void *stream);
size_t hep_router_sync_bytes(void);
/* Per-64-token-chunk expert counts of a top-K assignment (the unfused producer of d_chunk_cnt). */
int hep_gate_chunk_counts(const int32_t *d_topk_idx, int64_t T, int K, int E, int64_t tokens_per_src, int n_src,
                          int32_t *d_chunk_cnt, void *stream);

/*
 * Dense bf16 GEMM on tcgen05/TMEM/TMA (sm_100a): D[M][N] = A[M][K] . B[N][K]^T,
 * fp32 accumulate, fp32 or bf16 output.  Used for the router logits (K1).
 * Requires K % 64 == 0, N % 16 == 0, N <= 256 or N % 256 == 0.
 */
#define HEP_OUT_F32 0
#define HEP_OUT_BF16 1
int hep_gemm_bf16(const void *d_A, const void *d_B, void *d_D, int64_t M, int64_t N, int64_t K, int out_kind,
                  void *stream);

/*
 * K4: per-assignment destination rows from the routing table (RoutingTable
 * "ranges partition that source's tokens in sequence order", router.py:38-46).
 * Receive layout ("rows"): [expert ascending][dst GPU ascending][src GPU ascending][rank]
 * (each expert's rows contiguous: one grouped-GEMM segment per expert).
 * Outputs:
 *   d_tok_row [T][K] int32  row of assignment (t,k)
 *   d_row_tok [R]    int32  token of each row (R = total assignments)
 *   d_seg      [nnz][4] int32 (row_start, rows, expert, dst) per replica, in row order
 *   d_expert_rows [E+1] int64 first row of each expert's contiguous block
 * Needs the hep_sched_out of the same micro-batch (ranges + xi).  row_align: every
 * expert block starts on a multiple of row_align rows (1 = dense; 64 for training, so the
 * weight-gradient GEMMs contract over whole 64-row blocks; padding rows are never written).
 */
int hep_moe_assign(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K,
                   int64_t tokens_per_src, int row_align, int32_t *d_tok_row, int32_t *d_row_tok, int32_t *d_seg,
                   int64_t *d_expert_rows, void *workspace, size_t workspace_bytes, void *stream);
size_t hep_moe_assign_workspace(hep_sched_t h, int64_t T, int K);
/* hep_moe_assign with the chunk counts already in the workspace (written by
 * hep_router_topk's epilogue at byte offset hep_moe_assign_chunk_offset); the counts
 * are left intact, so the call is repeatable on the same micro-batch. */
int hep_moe_assign_precounted(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K,
                              int64_t tokens_per_src, int row_align, int32_t *d_tok_row, int32_t *d_row_tok,
                              int32_t *d_seg, int64_t *d_expert_rows, void *workspace, size_t workspace_bytes,
                              void *stream);
size_t hep_moe_assign_chunk_offset(hep_sched_t h, int64_t T, int K);
/*
 * K4 for one phase (0 static, 1 scheduled) of the pipelined split (hep_sched_pipelined,
 * d_split = its [2][E][G] split): the assignments of (expert e, source src) whose rank q
 * (sequence order) lies in this phase's window -- [0, former[e][src]) for phase 0,
 * [former[e][src], former + latter) for phase 1 -- get rows; the others are left untouched in
 * d_tok_row and set to -1 in d_tok_row_phase (optional [T][K]: this phase's own row map, the
 * input of its hep_moe_permute, which skips negative rows).  Receive layout
 * [expert][phase][dst][src][rank]: expert e's block starts at the prefix of the experts' total
 * loads (known from d_split before the scheduled phase is solved) and holds the static rows
 * first, so each expert stays one contiguous grouped-GEMM run and the two phases write
 * disjoint rows: they may run concurrently on two streams, each with ITS OWN workspace.
 * d_seg gets this phase's nnz segments; row_align = 1.
 */
int hep_moe_assign_phase(hep_sched_t h, const hep_sched_out *sched, const int64_t *d_split, int phase,
                         const int32_t *d_topk_idx, int64_t T, int K, int64_t tokens_per_src, int32_t *d_tok_row,
                         int32_t *d_tok_row_phase, int32_t *d_row_tok, int32_t *d_seg, int64_t *d_expert_rows,
                         void *workspace, size_t workspace_bytes, void *stream);

/*
 * K4 for one rank of a real EP group (one process per GPU, rank r = source r
 * of its own T tokens and destination r of its replicas).  Outputs:
 *   d_tok_row [T][K] int32  position of assignment (t,k) in the send buffer
 *                           [dst][expert asc][rank]; after the dispatch and the
 *                           reverse (combine) all-to-all the expert outputs come
 *                           back at the same positions
 *   d_seg     [G*n_hosted][4] int32 receive-buffer segments ([src][hosted expert
 *                           asc]): (row_start, rows, local weight slot, src)
 *   d_counts  [2G] int64    rows sent to each dst, rows received from each src
 *                           (the all-to-all-v split sizes)
 * recv_capacity > 0: rows a rank's fixed receive buffer holds (the NVLink path).  If the
 * schedule sends more rows than that to ANY rank (every rank checks every destination on
 * the identical plan, so all agree), sched->d_status = HEP_E_CAPACITY and the exchange is
 * empty (zero counts and segments).  0 = unbounded (NCCL path, buffers sized per call).
 * On a scheduler error (d_status set) the send positions are the identity t*K + k and
 * the exchange is empty; the layer raises the status.
 */
int hep_moe_assign_ep(hep_sched_t h, const hep_sched_out *sched, const int32_t *d_topk_idx, int64_t T, int K, int rank,
                      int64_t recv_capacity, int32_t *d_tok_row, int32_t *d_seg, int64_t *d_counts, void *workspace,
                      size_t workspace_bytes, void *stream);
size_t hep_moe_assign_ep_workspace(hep_sched_t h, int64_t T, int K);
/*
 * hep_moe_assign_ep for one phase of the pipelined split (simulator.py:420-435) in the EP
 * layer: sched = that phase's plan (hep_sched_pipelined: former = phase 0, the static share;
 * latter = phase 1), d_split its [2][E][G] split.  Phase p owns the ranks [lo, lo + share)
 * of every (expert, this source) token sequence (lo = 0, or the static share for phase 1);
 * its assignments get send positions from send_row_offset on (the phases share one send
 * buffer), the others are left untouched in d_tok_row and -1 in d_tok_row_phase (the input
 * of this phase's hep_moe_permute).  d_seg / d_counts: this phase's receive segments and
 * split sizes.  The two phases may run concurrently on two streams, each with its own
 * workspace: the static share's exchange then overlaps the scheduled share's solve.
 */
int hep_moe_assign_ep_phase(hep_sched_t h, const hep_sched_out *sched, const int64_t *d_split, int phase,
                            const int32_t *d_topk_idx, int64_t T, int K, int rank, int64_t send_row_offset,
                            int32_t *d_tok_row, int32_t *d_tok_row_phase, int32_t *d_seg, int64_t *d_counts,
                            void *workspace, size_t workspace_bytes, void *stream);
/*
 * EP training layout: map the receive buffer ([src][hosted expert], d_seg from
 * hep_moe_assign_ep) onto a [local slot][src] layout where every slot's rows form one
 * block starting on a multiple of row_align (the weight-gradient GEMMs contract over
 * whole 64-row blocks).  Outputs: d_row_map [R_recv] aligned row of each received row,
 * d_seg_out [n_slots][4] (row_start, rows, slot, 0) and d_slot_rows [n_slots+1] (block
 * starts; the last entry = rows of the aligned buffer), the d_seg / d_expert_rows
 * arguments of hep_moe_expert_ffn_train / hep_moe_expert_ffn_bwd with n_experts = n_slots.
 * row_map_len > 0: entries [R_recv, row_map_len) are set to -1 (the NVLink path's fixed-size
 * receive buffer, R_recv known only on the device; hep_moe_permute skips them).
 * G = the number of [src] blocks in d_seg (up to 2 * HEP_MAX_GPUS: the pipelined split's
 * two phases).  With row_align = 1 it is also the inference regrouping of the NCCL path
 * (one contiguous run per local slot instead of one per (source, slot)).
 */
int hep_moe_ep_train_layout(const int32_t *d_seg, int n_hosted, int G, int n_slots, int row_align, int32_t *d_row_map,
                            int64_t row_map_len, int32_t *d_seg_out, int64_t *d_slot_rows, void *stream);
/* experts hosted by `rank` and the number of local weight slots it needs */
int hep_sched_hosted(hep_sched_t h, int rank, int *n_hosted, int *n_slots);

/*
 * EP exchange over NVLink peer memory (one kernel per direction, no NCCL on the data
 * path; every rank derives all offsets from the identical transfer plan):
 *   d_pair         = hep_sched_out.d_transfer (pair[s][d] first, G*G int64)
 *   d_peer_recv[d] = address of rank d's receive buffer ([src][hosted expert] rows)
 *   d_peer_back[s] = address of rank s's return buffer ([dst][expert][rank] = send layout)
 * hep_moe_dispatch_p2p: K5 fused with the dispatch all-to-all — x[t] of every
 *   assignment (send position tok_row[t][k] from hep_moe_assign_ep) is stored straight
 *   into its destination rank's receive buffer.
 * hep_moe_return_addr: per received row, the address of its slot in the source rank's
 *   return buffer (capacity rows at most); hep_moe_expert_ffn_p2p stores the
 *   down-projection output rows there from the GEMM epilogue (combine all-to-all fused
 *   into the GEMM), after which hep_moe_combine runs on the source as usual.  R = capacity
 *   of the receive buffer (rows actually present come from d_seg on the device);
 *   rows_hint = expected rows (picks the 1-CTA / CTA-pair tile shape like R does for
 *   hep_moe_expert_ffn).
 * The caller orders the exchanges across ranks (stream sync + a barrier): a rank's
 * receive buffer is complete once every source's dispatch kernel has finished.
 * hep_moe_dispatch_p2p stores nothing when d_status (the scheduler's, may be NULL) is
 * set or when any rank's receive total exceeds recv_capacity rows (0 = unchecked).
 */
int hep_moe_dispatch_p2p(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model, int rank,
                         int num_gpus, const int64_t *d_pair, const uint64_t *d_peer_recv, int64_t recv_capacity,
                         const int32_t *d_status, void *stream);
int hep_moe_return_addr(const int64_t *d_pair, int rank, int num_gpus, const uint64_t *d_peer_back, int64_t row_bytes,
                        int64_t capacity, uint64_t *d_addr, void *stream);
/* hep_moe_return_addr for received rows regrouped per weight slot: receive row i's return
 * address goes to d_addr[d_row_map[i]] (d_row_map from hep_moe_ep_train_layout), so the
 * FFN on the regrouped rows stores every output row straight to its source. */
int hep_moe_return_addr_map(const int64_t *d_pair, int rank, int num_gpus, const uint64_t *d_peer_back,
                            int64_t row_bytes, int64_t capacity, const int32_t *d_row_map, uint64_t *d_addr,
                            void *stream);
/* Received rows back to their sources (the NVLink return of the training path): row
 * d_src[d_row_map ? d_row_map[i] : i] -> d_addr[i] (hep_moe_return_addr's table), for i below
 * this rank's received count (sum_s pair[s][rank], at most capacity); nothing when d_status is
 * set. */
int hep_moe_rows_to_addr(const void *d_src, const int32_t *d_row_map, const int64_t *d_pair, int rank, int num_gpus,
                         int64_t capacity, int64_t d_model, const uint64_t *d_addr, const int32_t *d_status,
                         void *stream);
int hep_moe_expert_ffn_p2p(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg, int n_seg,
                           int64_t R, int64_t rows_hint, int64_t d_model, int64_t ffn, int n_experts, void *d_h,
                           const uint64_t *d_y_addr, void *d_workspace, size_t workspace_bytes, int32_t *d_status,
                           void *stream);
/*
 * Device-side group barrier over peer memory (no host synchronisation; graph-capturable).
 * d_my_flags: this rank's uint32 [world + 2], zero-initialised, mapped by every peer
 * (slot world + 1 becomes 1 if a wait gave up after ~10 s: a peer never arrived);
 * d_peer_flags[i] = rank i's flags array.  Each call arrives (release, system scope) in
 * slot `rank` of every peer and waits (acquire) until every peer arrived with the same
 * epoch.  hep_p2p_allgather first stores this rank's `bytes` (multiple of 16) of d_src
 * at d_peer_dst[i] + rank * bytes of every rank i, then runs the barrier.
 * Replaces: the dist.barrier / all_gather of the modelled all-to-all (simulator.py:457-463).
 */
int hep_p2p_barrier(const uint64_t *d_peer_flags, uint32_t *d_my_flags, int rank, int world, void *stream);
int hep_p2p_allgather(const void *d_src, int64_t bytes, const uint64_t *d_peer_dst, const uint64_t *d_peer_flags,
                      uint32_t *d_my_flags, int rank, int world, void *stream);
/* CUDA IPC plumbing for the peer buffers: 64-byte handle of the allocation holding d_ptr
 * plus d_ptr's byte offset in it (exchanged by the host); open maps the allocation base. */
int hep_ipc_handle(const void *d_ptr, void *handle_out, int64_t *offset_out);
int hep_ipc_open(const void *handle, void **d_ptr);
int hep_ipc_close(void *d_ptr);

/* K5 permute/dispatch: rows[tok_row[t][k]] = x[t]  (bf16, 128/256-bit vectorised scatter);
 * negative rows are skipped, and a token with no non-negative row is not read. */
int hep_moe_permute(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model, void *d_rows,
                    void *stream);
/* hep_moe_permute with at most blocks_per_sm (1..8) resident 256-thread blocks per SM (8 fills
 * every SM): the pipelined split's static-phase permute leaves room for the scheduled phase's
 * solve / assignment kernels on the other stream. */
int hep_moe_permute_ex(const void *d_x, const int32_t *d_tok_row, int64_t T, int K, int64_t d_model, void *d_rows,
                       int blocks_per_sm, void *stream);

/*
 * K6 expert FFN as grouped GEMM (tcgen05/TMEM/TMA, SwiGLU fused in the first
 * GEMM's epilogue):  per segment s with expert e:
 *   H[r] = silu(X[r] W1_e^T) * (X[r] W3_e^T),  Y[r] = H[r] W2_e^T
 *   d_w13 [E][2F][d]  rows interleaved in blocks of 128 (W1 block j, then W3 block j)
 *   d_w2  [E][d][F]
 *   d_h   [R][F] scratch, d_y [R][d] output (bf16)
 * Segments/rows are read on the device (no host sync): d_seg as from hep_moe_assign
 * (n_seg entries, R = capacity of d_rows / d_h / d_y in rows).
 */
int hep_moe_expert_ffn(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg,
                       int n_seg, int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h, void *d_y,
                       void *d_workspace, size_t workspace_bytes, int32_t *d_status, void *stream);
/*
 * hep_moe_expert_ffn with the permute (K5) fused into the first GEMM: its A operand is
 * gathered straight from the token activations d_x [T][d_model] by TMA tile::gather4,
 * receive row r being token d_row_tok[r] (hep_moe_assign's row_tok), so the permuted
 * rows buffer is never written or read.  Bit-identical to hep_moe_permute followed by
 * hep_moe_expert_ffn.  Forward (inference) only; training keeps the rows buffer for the
 * weight gradients.
 */
/* Diagnostics: with HEP_FFN_CLOCK=1 in the environment, CTA 0 of each expert GEMM records
 * (clock64, globaltimer ns) at entry and exit; out[8] = GEMM1 {c0, t0, c1, t1}, GEMM2 {...}
 * of the last such launch, i.e. the SM clock the tensor cores ran at. */
int hep_ffn_debug_clock(int64_t *host_out8);
int hep_moe_expert_ffn_gather(const void *d_x, int64_t T, const int32_t *d_row_tok, const void *d_w13,
                              const void *d_w2, const int32_t *d_seg, int n_seg, int64_t R, int64_t d_model,
                              int64_t ffn, int n_experts, void *d_h, void *d_y, void *d_workspace,
                              size_t workspace_bytes, int32_t *d_status, void *stream);
/* workspace for hep_moe_expert_ffn's device-built m-tile list */
size_t hep_moe_ffn_workspace(int n_seg, int64_t R, int n_experts);
/* Kernel launches one expert-FFN forward issues for R rows over n_experts (4: two
 * tile-list kernels + two GEMMs; 8 when the light experts run as a second 1-CTA
 * GEMM pair).  gather != 0: the fused-permute variant. */
int hep_moe_ffn_launches(int64_t R, int n_experts, int gather);
/* Kernel launches one hep_moe_expert_ffn_bwd issues (9, or 13 with the light split;
 * one fewer each with HEP_WGRAD_ORDER=0). */
int hep_moe_ffn_bwd_launches(int64_t Rcap, int n_experts);

/* K7 combine/un-permute: out[t] = sum_k w[t][k] * y[tok_row[t][k]] (fp32 accumulate in k order). */
int hep_moe_combine(const void *d_y, const int32_t *d_tok_row, const float *d_topk_w, int64_t T, int K,
                    int64_t d_model, void *d_out, void *stream);

/* K7 with unit weights and an optional addend: out[t] = add[t] + sum_k w[t][k] y[row(t,k)]
 * (d_topk_w may be NULL = all ones; d_add may be NULL).  The permute's transpose. */
int hep_moe_gather_sum(const void *d_y, const int32_t *d_tok_row, const float *d_topk_w, const void *d_add, int64_t T,
                       int K, int64_t d_model, void *d_out, void *stream);

/* ======================================================================
 * Backward (training).  Gradients of the layer above, all on the device.
 * ====================================================================== */
/* K7^T: dY[row(t,k)] = w[t][k] dout[t] (bf16), dw[t][k] = <dout[t], Y[row(t,k)]> (fp32) */
int hep_moe_combine_bwd(const void *d_dout, const void *d_y, const int32_t *d_tok_row, const float *d_topk_w,
                        int64_t T, int K, int64_t d_model, void *d_dy, float *d_dw, void *stream);
/* zero the alignment padding rows of every expert block of a [rows][width] bf16 buffer */
int hep_moe_zero_padding(const int64_t *d_expert_rows, const int32_t *d_seg, int n_seg, int E, void *d_buf,
                         int64_t width, void *stream);
/*
 * K6^T: expert FFN backward.  Inputs: receive rows X, pre-activations A13 [R][2F]
 * (stored by the forward when hep_moe_expert_ffn_train is used), H, dY (padding rows
 * are zeroed here), weights.  Outputs: dA13 scratch, dX rows (bf16), dW13 / dW2 (fp32,
 * [E][2F][d] W13 interleave, [E][d][F]).  Requires d % 256 == 0, F % 256 == 0.
 */
int hep_moe_expert_ffn_bwd(const void *d_rows, const void *d_pre, const void *d_h, void *d_dy, const void *d_w13,
                           const void *d_w2, const int32_t *d_seg, int n_seg, const int64_t *d_expert_rows,
                           int64_t Rcap, int64_t d_model, int64_t ffn, int n_experts, void *d_da13, void *d_dx_rows,
                           float *d_dw13, float *d_dw2, void *d_workspace, size_t workspace_bytes, int32_t *d_status,
                           void *stream);
/* forward FFN that also stores the pre-activations A13 for the backward */
int hep_moe_expert_ffn_train(const void *d_rows, const void *d_w13, const void *d_w2, const int32_t *d_seg, int n_seg,
                             int64_t R, int64_t d_model, int64_t ffn, int n_experts, void *d_h, void *d_y,
                             void *d_pre, void *d_workspace, size_t workspace_bytes, int32_t *d_status, void *stream);
/* router backward: dlogit = w (dw - sum w dw) on the selected experts, bf16 [T][ld] */
int hep_gate_bwd(const int32_t *d_topk_idx, const float *d_topk_w, const float *d_dw, int64_t T, int K, int64_t ld,
                 void *d_dlogits, void *stream);
/* dWg = dlogits^T x (fp32 [E64][d]), dx_gate = dlogits Wg (bf16 [T][d]) */
int hep_router_bwd(const void *d_x, const void *d_wg, const void *d_dlogits, int64_t T, int64_t d_model, int E64,
                   float *d_dwg, void *d_dxg, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HEP_H_ */
