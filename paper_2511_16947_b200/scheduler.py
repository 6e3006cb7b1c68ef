"""Per-micro-batch replica-load scheduling on the GPU (drop-in API).

Same public surface as the reference ``harmonyep.scheduler``
(``/root/reference/pkg/src/harmonyep/scheduler.py``):

  SolveOptions          :67-94
  CommPlanStats         :97-135
  solve_comm_aware      :622-689  (LP on the device: simplex.py / csrc/lp.cu)
  SolveStats            :138-148
  SolverState           :151-170  (here: owns the device placement tables + output buffers)
  solve_replica_loads   :405-433
  warm_solve            :436-461
  integerize_plan       :697-735

Every solve is ONE launch of the single-CTA sm_100a scheduler kernel
(``csrc/sched.cu``) through the C ABI ``hep_sched_solve`` (include/hep.h).
The host only uploads the load matrix and, for this inspection API, reads the
result back to build the reference's immutable plan objects; the MoE layer
(``layer.py``) keeps everything on the device.

The result is the unique lexicographically-minimal optimal plan, so it is a
pure function of (placement, loads): warm and cold solves are bit-identical
and independent replicas agree (scheduler.py:19-26).
"""

from __future__ import annotations

import ctypes
import math
from collections import OrderedDict
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from .core import (
    CapacityError,
    ContractViolation,
    DimensionError,
    LoadMatrix,
    Placement,
    PlacementError,
    ReplicaLoadPlan,
    StaleStateError,
    Topology,
)

BALANCE_ONLY = "balance_only"
COMM_AWARE = "comm_aware"
TOPOLOGY_AWARE = "topology_aware"
_MODES = (BALANCE_ONLY, COMM_AWARE, TOPOLOGY_AWARE)

HEP_SCHED_SOLVE = 1
HEP_SCHED_INTEGERIZE = 2
HEP_SCHED_ROUTE = 4
HEP_SCHED_TRANSFER = 8
HEP_SCHED_TOPO = 16
HEP_SCHED_ALL = 15
MAX_GPUS = 10  # HEP_MAX_GPUS


@dataclass(frozen=True)
class SolveOptions:
    """Solver configuration (reference scheduler.py:67-94, same validation)."""

    mode: str = BALANCE_ONLY
    alpha: float = 1.0
    alpha_intra: float = 0.1
    alpha_inter: float = 1.0
    tolerance: float = 1e-9
    warm_state: "SolverState | None" = None

    def __post_init__(self):
        if self.mode not in _MODES:
            raise ContractViolation(f"unknown mode {self.mode!r}; expected one of {_MODES}")
        if min(self.alpha, self.alpha_intra, self.alpha_inter) < 0:
            raise ContractViolation("communication weights must be >= 0")
        if self.alpha_intra > self.alpha_inter:
            raise ContractViolation("alpha_intra must not exceed alpha_inter (intra-node links are cheaper)")
        if self.tolerance < 0:
            raise ContractViolation("tolerance must be >= 0")


@dataclass
class SolveStats:
    """Counters (reference :138-148), restated for the device solver.  It has no probe
    loop and no augmenting paths: one exact density evaluation over the 2^G GPU subsets
    gives m (counted as one probe) and the lex-min sweep fixes one (expert, GPU) arc per
    step (each step is the reference's reroute max-flow of ``lex_min_plan``, counted in
    ``bfs_phases``).  A cold solve (fresh ``SolverState``) also builds the flow network --
    the placement tables the reference keeps in ``SolverState._flow`` -- counted in
    ``network_builds``; a warm solve reuses them, which is all a warm start saves here
    (the plan is the same canonical lex-min plan either way, reference test C7).
    ``iterations_last`` = the last solve's network build + probe + arc steps;
    ``device_us_last`` = its scheduler kernel time (CUDA events)."""

    solves: int = 0
    probes: int = 0
    bfs_phases: int = 0
    pivots: int = 0
    iterations_last: int = 0
    network_builds: int = 0
    device_us_last: float = 0.0
    device_us_total: float = 0.0

    @property
    def iterations_total(self) -> int:
        return self.probes + self.bfs_phases + self.pivots


class DeviceScheduler:
    """Owns one ``hep_sched_t`` (device placement tables) plus the device output
    buffers of one micro-batch (``hep_sched_out``)."""

    def __init__(self, placement: Placement, gpus_per_node: int = 0, device=None):
        torch = _lib.require_cuda()
        self.placement = placement
        self.G = placement.num_gpus
        self.E = placement.num_experts
        if self.G > MAX_GPUS:
            raise CapacityError(f"device scheduler handles up to {MAX_GPUS} GPUs per scheduling group, got {self.G}")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        off, gpu = placement.csr()
        slots = np.asarray(placement.slots, dtype=np.int32)
        h = ctypes.c_void_p()
        L = _lib.lib()
        _lib.check(
            L.hep_sched_create(
                self.G, self.E,
                off.ctypes.data_as(_lib.c_i32p),
                gpu.ctypes.data_as(_lib.c_i32p) if gpu.size else None,
                slots.ctypes.data_as(_lib.c_i32p) if slots.size else None,
                int(gpus_per_node),
                ctypes.byref(h),
            ),
            "hep_sched_create",
        )
        self._h = h
        self.off = off
        nnz, max_ranges, Q, tlen = (ctypes.c_int64() for _ in range(4))
        _lib.check(L.hep_sched_sizes(h, ctypes.byref(nnz), ctypes.byref(max_ranges), ctypes.byref(Q), ctypes.byref(tlen)),
                   "hep_sched_sizes")
        self.nnz, self.max_ranges, self.Q, self.tlen = nnz.value, max_ranges.value, Q.value, tlen.value
        i64 = dict(dtype=torch.int64, device=self.device)
        self.m = torch.zeros(4, **i64)
        self.xq = torch.zeros(max(self.nnz, 1), **i64)
        self.xi = torch.zeros(max(self.nnz, 1), **i64)
        self.gpu_load = torch.zeros(self.G, **i64)
        self.ranges = torch.zeros(4 * self.max_ranges, **i64)
        self.n_ranges = torch.zeros(1, **i64)
        self.transfer = torch.zeros(self.tlen, **i64)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.out = _lib.HepSchedOut(
            self.m.data_ptr(), self.xq.data_ptr(), self.xi.data_ptr(), self.gpu_load.data_ptr(),
            self.ranges.data_ptr(), self.n_ranges.data_ptr(), self.transfer.data_ptr(), self.status.data_ptr(),
        )
        self.former: SchedBuffers | None = None  # static phase of the pipelined split

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._LIB is not None:
            _lib._LIB.hep_sched_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    # -- launches (asynchronous on `stream`) ------------------------------
    def launch_solve(self, d_loads, stride_e: int, stride_g: int, d_base=None, flags: int = HEP_SCHED_ALL, stream=None):
        _lib.check(
            _lib.lib().hep_sched_solve(
                self._h, d_loads.data_ptr(), stride_e, stride_g, _lib.ptr(d_base), flags,
                ctypes.byref(self.out), _lib.stream_handle(stream),
            ),
            "hep_sched_solve",
        )

    def launch_integerize(self, den: int, stream=None):
        _lib.check(
            _lib.lib().hep_sched_integerize(self._h, self.xq.data_ptr(), int(den), ctypes.byref(self.out),
                                            _lib.stream_handle(stream)),
            "hep_sched_integerize",
        )

    def launch_route(self, d_loads, stride_e, stride_g, d_xi, flags=0, stream=None):
        _lib.check(
            _lib.lib().hep_sched_route(self._h, d_loads.data_ptr(), stride_e, stride_g, d_xi.data_ptr(), flags,
                                       ctypes.byref(self.out), _lib.stream_handle(stream)),
            "hep_sched_route",
        )

    def launch_pipelined(self, d_loads, stride_e: int, stride_g: int, share, flags: int = HEP_SCHED_ALL, stream=None,
                         stream_static=None):
        """Pipelined split (``simulator.py:420-435``): the static share's phase goes to
        ``self.former`` (a ``SchedBuffers``), the scheduled share's to this object.
        ``share`` = static share as a Fraction (1 - pipeline_ratio).  ``stream_static``: the
        static phase runs there, concurrently with the scheduled phase's solve (the caller
        joins it back)."""
        share = Fraction(share)
        if self.former is None:
            self.former = SchedBuffers(self)
            # [former E*G | latter E*G | static phase's integerized GPU loads G]
            self.split = _lib.require_cuda().zeros(2 * max(self.E * self.G, 1) + self.G,
                                                   dtype=_lib.require_cuda().int64, device=self.device)
        _lib.check(
            _lib.lib().hep_sched_pipelined(
                self._h, d_loads.data_ptr(), stride_e, stride_g, share.numerator, share.denominator, flags,
                self.split.data_ptr(), ctypes.byref(self.former.out), ctypes.byref(self.out),
                _lib.stream_handle(stream), None if stream_static is None else stream_static.cuda_stream,
            ),
            "hep_sched_pipelined",
        )

    def check_status(self, where: str):
        _lib.raise_status(int(self.status.item()), where)
        if self.former is not None:
            _lib.raise_status(int(self.former.status.item()), where + " (static phase)")

    # -- host views (synchronising; inspection / parity API only) ---------
    def rows(self, t) -> list[list[int]]:
        flat = t[: self.nnz].cpu().tolist() if self.nnz else []
        return [flat[self.off[e]: self.off[e + 1]] for e in range(self.E)]

    def host_ranges(self) -> tuple[tuple[int, int, int, int], ...]:
        n = int(self.n_ranges.item())
        if n == 0:
            return ()
        arr = self.ranges[: 4 * n].view(n, 4).cpu().tolist()
        return tuple(tuple(r) for r in arr)


class SchedBuffers:
    """A second set of ``hep_sched_out`` buffers on the same placement (the
    static phase of the pipelined split); same field names and host views as
    ``DeviceScheduler``."""

    def __init__(self, ds: DeviceScheduler):
        torch = _lib.require_cuda()
        self.E, self.G, self.nnz, self.off = ds.E, ds.G, ds.nnz, ds.off
        i64 = dict(dtype=torch.int64, device=ds.device)
        self.m = torch.zeros(4, **i64)
        self.xq = torch.zeros(max(ds.nnz, 1), **i64)
        self.xi = torch.zeros(max(ds.nnz, 1), **i64)
        self.gpu_load = torch.zeros(ds.G, **i64)
        self.ranges = torch.zeros(4 * ds.max_ranges, **i64)
        self.n_ranges = torch.zeros(1, **i64)
        self.transfer = torch.zeros(ds.tlen, **i64)
        self.status = torch.zeros(1, dtype=torch.int32, device=ds.device)
        self.out = _lib.HepSchedOut(
            self.m.data_ptr(), self.xq.data_ptr(), self.xi.data_ptr(), self.gpu_load.data_ptr(),
            self.ranges.data_ptr(), self.n_ranges.data_ptr(), self.transfer.data_ptr(), self.status.data_ptr(),
        )

    rows = DeviceScheduler.rows
    host_ranges = DeviceScheduler.host_ranges


_HANDLE_CACHE: "OrderedDict[tuple, DeviceScheduler]" = OrderedDict()


def device_scheduler(placement: Placement, gpus_per_node: int = 0) -> DeviceScheduler:
    """LRU cache of device schedulers keyed by placement (init-time objects)."""
    torch = _lib.require_cuda()
    key = (placement.num_gpus, placement.edp_groups, placement.slots, gpus_per_node, torch.cuda.current_device())
    ds = _HANDLE_CACHE.get(key)
    if ds is None:
        ds = DeviceScheduler(placement, gpus_per_node)
        _HANDLE_CACHE[key] = ds
        while len(_HANDLE_CACHE) > 64:
            _HANDLE_CACHE.popitem(last=False)
    else:
        _HANDLE_CACHE.move_to_end(key)
    return ds


class SolverState:
    """Warm-start state (reference :151-170), reusable across micro-batches on
    one placement.  Holds the device scheduler (placement tables already on
    the GPU), so warm solves skip the placement upload."""

    def __init__(self, placement: Placement, options: SolveOptions, topology: Topology | None = None):
        self.placement = placement
        self.options = options
        self.topology = topology
        self.stats = SolveStats()
        self.last_objective = None
        self._dev: DeviceScheduler | None = None
        self._basis = None  # device simplex basis of the comm-aware modes (warm start)

    def _check_loads(self, loads: LoadMatrix) -> None:
        if (loads.num_experts, loads.num_gpus) != (self.placement.num_experts, self.placement.num_gpus):
            raise StaleStateError(
                f"state placement is {self.placement.num_experts}x{self.placement.num_gpus}, "
                f"loads are {loads.num_experts}x{loads.num_gpus}"
            )


def _check_dims(placement: Placement, loads: LoadMatrix) -> None:
    if loads.num_experts != placement.num_experts:
        raise DimensionError(f"loads cover {loads.num_experts} experts, placement {placement.num_experts}")
    if loads.num_gpus != placement.num_gpus:
        raise DimensionError(f"loads cover {loads.num_gpus} GPUs, placement {placement.num_gpus}")


def _device_solve(state: SolverState, loads: LoadMatrix, gpu_base) -> ReplicaLoadPlan:
    import torch

    placement = state.placement
    if state._dev is None:
        state._dev = device_scheduler(placement)
    dev = state._dev
    G = placement.num_gpus
    d_loads = torch.as_tensor(loads.as_array(), dtype=torch.int64).to(dev.device)
    d_base = None
    if gpu_base is not None:
        if len(gpu_base) != G:
            raise DimensionError(f"gpu_base has {len(gpu_base)} entries for {G} GPUs")
        d_base = torch.as_tensor(np.asarray(gpu_base, dtype=np.int64)).to(dev.device)
    st = torch.cuda.current_stream(dev.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    dev.launch_solve(d_loads, G, 1, d_base, flags=HEP_SCHED_SOLVE, stream=st)
    e1.record(st)
    dev.check_status("solve_replica_loads")
    m_num, m_den, Q, _ = dev.m.cpu().tolist()
    xq = dev.rows(dev.xq)
    entries = tuple(tuple(Fraction(v, Q) for v in row) for row in xq)
    objective = Fraction(m_num, m_den)
    cold = state.stats.solves == 0  # a fresh state builds (or fetches) the placement tables
    steps = dev.nnz  # lex-min arc steps
    state.stats.solves += 1
    state.stats.probes += 1
    state.stats.bfs_phases += steps
    state.stats.network_builds += int(cold)
    state.stats.iterations_last = int(cold) + 1 + steps
    us = 1e3 * e0.elapsed_time(e1)
    state.stats.device_us_last = us
    state.stats.device_us_total += us
    state.last_objective = objective
    return ReplicaLoadPlan(num_gpus=G, groups=placement.edp_groups, entries=entries, objective=objective)


def solve_replica_loads(placement: Placement, loads: LoadMatrix, options: SolveOptions | None = None, *,
                        gpu_base: tuple[int, ...] | None = None) -> tuple[ReplicaLoadPlan, SolverState]:
    """Exact min-max replica loads, canonical lex-min plan (reference :405-433)."""
    options = options or SolveOptions()
    if options.mode != BALANCE_ONLY:
        raise ContractViolation(f"solve_replica_loads requires mode={BALANCE_ONLY!r}; use solve_comm_aware")
    if options.warm_state is not None:
        return warm_solve(options.warm_state, loads, gpu_base=gpu_base)
    _check_dims(placement, loads)
    state = SolverState(placement, options)
    plan = _device_solve(state, loads, gpu_base)
    return plan, state


def warm_solve(prev_state: SolverState, new_loads: LoadMatrix, *,
               gpu_base: tuple[int, ...] | None = None) -> tuple[ReplicaLoadPlan, SolverState]:
    """Re-solve on the same placement (reference :436-461); identical to cold."""
    if not isinstance(prev_state, SolverState):
        raise StaleStateError("warm state is not a SolverState")
    prev_state._check_loads(new_loads)
    if prev_state.options.mode != BALANCE_ONLY:
        if prev_state.topology is None:
            raise StaleStateError("comm-mode state lost its topology")
        plan, _stats, state = solve_comm_aware(prev_state.placement, new_loads, prev_state.topology,
                                               prev_state.options, _state=prev_state)
        return plan, state
    plan = _device_solve(prev_state, new_loads, gpu_base)
    return plan, prev_state


def integerize_plan(plan: ReplicaLoadPlan) -> ReplicaLoadPlan:
    """Largest-remainder rounding on the device (reference :697-735): per
    expert, +1 to the largest fractional parts, ties to the lowest GPU id."""
    import torch

    exact = [[Fraction(v) for v in row] for row in plan.entries]
    width = max(1, max((len(r) for r in exact), default=1))
    den = 1
    for row in exact:
        for v in row:
            den = math.lcm(den, v.denominator)
    nums = [[int(v * den) for v in row] for row in exact]
    biggest = max((abs(x) for row in nums for x in row), default=0)
    if biggest * width >= (1 << 62):
        # The common denominator of arbitrary (e.g. float) entries overflows int64.  The
        # rounding depends only on each entry's floor, the order of the fractional parts
        # within an expert and the expert total (integral within 1e-6, reference :707-713,
        # the same tolerance the device applies), so use the finest binary fixed point
        # that fits: den = 2^k, entries rounded to nearest.  Exact for the scheduler's own
        # plans (denominator Q); a float plan differs from the reference only if two
        # fractional parts of one expert agree to within 2^-k.
        top = max((abs(v) for row in exact for v in row), default=Fraction(0))
        k = 61 - (int(top) + 1).bit_length() - width.bit_length()
        if k < 20:
            raise CapacityError("plan entries too large for int64 integerization")
        den = 1 << k
        nums = [[round(v * den) for v in row] for row in exact]
    placement = Placement(plan.num_gpus, plan.groups, tuple(range(len(plan.groups))))
    dev = device_scheduler(placement)
    flat = [x for row in nums for x in row]
    if flat:
        dev.xq[: len(flat)].copy_(torch.tensor(flat, dtype=torch.int64))
    dev.launch_integerize(den)
    dev.check_status("integerize_plan")
    xi = dev.rows(dev.xi)
    objective = int(dev.m[3].item()) if plan.num_gpus else 0
    return ReplicaLoadPlan(num_gpus=plan.num_gpus, groups=plan.groups, entries=tuple(tuple(r) for r in xi),
                           objective=objective)


@dataclass(frozen=True)
class CommPlanStats:
    """Per-GPU all-to-all volumes implied by a plan (reference scheduler.py:97-135):
    ``local[g]`` = tokens kept on their source GPU, ``send[g]`` = tokens leaving g
    (including tokens of experts g does not host), ``recv[g]`` = tokens arriving,
    ``comp`` = max GPU load, ``comm`` = max over GPUs of max(send, recv)."""

    send: tuple
    recv: tuple
    local: tuple
    comp: object
    comm: object

    @classmethod
    def from_plan(cls, placement: Placement, loads: LoadMatrix, plan: ReplicaLoadPlan) -> "CommPlanStats":
        G = placement.num_gpus
        inp = loads.entries
        local = [0] * G
        recv = [0] * G
        gpu = [0] * G
        for e, grp in enumerate(placement.edp_groups):
            for g, x in zip(grp, plan.entries[e]):
                kept = min(x, inp[e][g])
                local[g] += kept
                recv[g] += x - kept
                gpu[g] += x
        send = [sum(inp[e][g] for e in range(loads.num_experts)) - local[g] for g in range(G)]
        comp = max(gpu) if gpu else 0
        comm = max((max(a, b) for a, b in zip(send, recv)), default=0)
        return cls(tuple(send), tuple(recv), tuple(local), comp, comm)


def _comm_aware_lp(placement: Placement, loads: LoadMatrix, alpha: float):
    """min comp + alpha*comm over replica loads x and kept-local volumes l
    (reference scheduler.py:480-547; same variable and row order, so the device
    simplex walks the same pivots).  Columns: x[arcs] | l[arcs] | comp | comm, arcs =
    (expert, GPU) in EDP-list order.  Rows: per-expert conservation (eq); then
    comp >= load(g); l <= x and l <= input per arc; send(g) <= comm, recv(g) <= comm."""
    from .simplex import LinearProgram

    E, G = placement.num_experts, placement.num_gpus
    ae = np.array([e for e, grp in enumerate(placement.edp_groups) for _ in grp], dtype=np.int64)
    ag = np.array([g for grp in placement.edp_groups for g in grp], dtype=np.int64)
    na = ae.size
    n = 2 * na + 2
    i_comp, i_comm = 2 * na, 2 * na + 1
    inp = loads.as_array().astype(np.float64)  # [E][G]
    arange = np.arange(na)
    c = np.zeros(n)
    c[i_comp], c[i_comm] = 1.0, alpha
    a_eq = np.zeros((E, n))
    a_eq[ae, arange] = 1.0
    b_eq = np.asarray(loads.expert_totals(), dtype=np.float64)
    # inequality rows: [G comp] [2 per arc] [2 per GPU: send, recv]
    m_ub = G + 2 * na + 2 * G
    a_ub = np.zeros((m_ub, n))
    b_ub = np.zeros(m_ub)
    a_ub[ag, arange] = 1.0
    a_ub[:G, i_comp] = -1.0
    r_lx = G + 2 * arange  # l - x <= 0
    a_ub[r_lx, na + arange] = 1.0
    a_ub[r_lx, arange] = -1.0
    r_li = r_lx + 1  # l <= input
    a_ub[r_li, na + arange] = 1.0
    b_ub[r_li] = inp[ae, ag]
    r_send = G + 2 * na + 2 * np.arange(G)
    r_recv = r_send + 1
    a_ub[r_send[ag], na + arange] = -1.0
    a_ub[r_recv[ag], arange] = 1.0
    a_ub[r_recv[ag], na + arange] = -1.0
    a_ub[r_send, i_comm] = -1.0
    a_ub[r_recv, i_comm] = -1.0
    b_ub[r_send] = -inp.sum(axis=0)
    arcs = list(zip(ae.tolist(), ag.tolist()))
    return LinearProgram(c=c, a_eq=a_eq, b_eq=b_eq, a_ub=a_ub, b_ub=b_ub), arcs


def _topology_aware_lp(placement: Placement, loads: LoadMatrix, topology: Topology, alpha_intra: float,
                       alpha_inter: float):
    """min comp + a1*comm_intra + a2*comm_inter over explicit token flows
    f[(e, src, dst)] (reference scheduler.py:550-619; same column and row order).
    Columns: flows (expert, source GPU, replica GPU in EDP-list order) | comp | ci | cx.
    Rows: per-(expert, source) conservation for experts with replicas (eq); then
    comp >= load(dst); then per GPU the non-empty rows of intra send / intra recv /
    inter send / inter recv <= ci / ci / cx / cx."""
    from .simplex import LinearProgram

    G = placement.num_gpus
    fe, fs, fd = [], [], []
    for e, grp in enumerate(placement.edp_groups):
        for src in range(G):
            for dst in grp:
                fe.append(e)
                fs.append(src)
                fd.append(dst)
    fe, fs, fd = (np.array(v, dtype=np.int64) for v in (fe, fs, fd))
    nf = fe.size
    n = nf + 3
    i_comp, i_ci, i_cx = nf, nf + 1, nf + 2
    c = np.zeros(n)
    c[i_comp], c[i_ci], c[i_cx] = 1.0, alpha_intra, alpha_inter
    hosted = [e for e, grp in enumerate(placement.edp_groups) if grp]
    eq_row = {e: i for i, e in enumerate(hosted)}  # row of (e, src) = eq_row[e] * G + src
    inp = loads.as_array().astype(np.float64)
    a_eq = np.zeros((len(hosted) * G, n))
    fidx = np.arange(nf)
    if nf:
        rows = np.array([eq_row[e] for e in fe.tolist()], dtype=np.int64) * G + fs
        a_eq[rows, fidx] = 1.0
    b_eq = inp[np.repeat(np.array(hosted, dtype=np.int64), G), np.tile(np.arange(G), len(hosted))] \
        if hosted else np.zeros(0)
    node = np.array([topology.node_of(g) for g in range(G)], dtype=np.int64)
    comp = np.zeros((G, n))
    comp[fd, fidx] = 1.0
    comp[:, i_comp] = -1.0
    cross = fs != fd
    same = node[fs] == node[fd]
    si, ri, sx, rx = (np.zeros((G, n)) for _ in range(4))
    m_i = cross & same
    m_x = cross & ~same
    si[fs[m_i], fidx[m_i]] = 1.0
    ri[fd[m_i], fidx[m_i]] = 1.0
    sx[fs[m_x], fidx[m_x]] = 1.0
    rx[fd[m_x], fidx[m_x]] = 1.0
    ub = [comp[g] for g in range(G)]
    for g in range(G):
        for mat, iv in ((si, i_ci), (ri, i_ci), (sx, i_cx), (rx, i_cx)):
            row = mat[g]
            if row.any():
                row[iv] = -1.0
                ub.append(row)
    a_ub = np.array(ub)
    b_ub = np.zeros(len(ub))
    flows = list(zip(fe.tolist(), fs.tolist(), fd.tolist()))
    return LinearProgram(c=c, a_eq=a_eq, b_eq=b_eq, a_ub=a_ub, b_ub=b_ub), flows


def solve_comm_aware(placement: Placement, loads: LoadMatrix, topology: Topology, options: SolveOptions, *,
                     _state: SolverState | None = None):
    """Minimise comp + alpha*comm (``comm_aware``) or comp + alpha_intra*intra +
    alpha_inter*inter (``topology_aware``) -- reference scheduler.py:622-689.  The LP is
    built on the host and solved by the device simplex (``simplex.simplex_solve`` ->
    ``hep_lp_solve``), warm-started from the state's previous basis.  Returns
    (float plan, CommPlanStats recomputed from the plan, state)."""
    from .simplex import simplex_solve

    if options.mode not in (COMM_AWARE, TOPOLOGY_AWARE):
        raise ContractViolation(
            f"solve_comm_aware requires mode in {{{COMM_AWARE}, {TOPOLOGY_AWARE}}}, got {options.mode!r}")
    if _state is None and options.warm_state is not None:
        _state = options.warm_state
    _check_dims(placement, loads)
    if topology.num_gpus != placement.num_gpus:
        raise DimensionError("topology does not match placement")
    for e, (load, grp) in enumerate(zip(loads.expert_totals(), placement.edp_groups)):
        if load > 0 and not grp:
            raise PlacementError(f"expert {e} has load {load} but an empty EDP group")
    state = _state or SolverState(placement, options, topology)
    state._check_loads(loads)
    if options.mode == COMM_AWARE:
        lp, keys = _comm_aware_lp(placement, loads, options.alpha)
    else:
        lp, keys = _topology_aware_lp(placement, loads, topology, options.alpha_intra, options.alpha_inter)
    res = simplex_solve(lp, basis=state._basis)
    state._basis = res.basis
    state.stats.pivots += res.iterations
    state.stats.iterations_last = res.iterations
    state.stats.solves += 1
    state.stats.device_us_last = res.device_us
    state.stats.device_us_total += res.device_us
    E, G = placement.num_experts, placement.num_gpus
    x = [[0.0] * G for _ in range(E)]
    if options.mode == COMM_AWARE:
        for k, (e, g) in enumerate(keys):
            x[e][g] = float(res.x[k])
    else:
        for k, (e, _src, dst) in enumerate(keys):
            x[e][dst] += float(res.x[k])  # flow order, as the reference accumulates
    entries = tuple(tuple(x[e][g] for g in grp) for e, grp in enumerate(placement.edp_groups))
    loads_g = [0.0] * G
    for e, grp in enumerate(placement.edp_groups):
        for g, v in zip(grp, entries[e]):
            loads_g[g] += v
    plan = ReplicaLoadPlan(num_gpus=G, groups=placement.edp_groups, entries=entries,
                           objective=max(loads_g) if loads_g else 0.0)
    stats = CommPlanStats.from_plan(placement, loads, plan)
    state.last_objective = res.objective
    return plan, stats, state
