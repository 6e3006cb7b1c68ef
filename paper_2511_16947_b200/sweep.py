"""Counts-mode driver: the reference simulator's per-micro-batch schedule loop
with every schedule computed by the device scheduler.

Mirrors ``run_strategy`` / ``run_skew_sweep`` / ``SweepResult``
(reference ``simulator.py:346-600``) for the strategies on this path —
``harmony``, ``harmony_pipelined``, ``merged_ep`` (harmony on the identical
placement) and the ``vanilla_ep`` baseline — and emits the reference's
``metrics.csv`` / ``summary.json`` schema.  ``max_load``, ``balance_ratio``,
the all-to-all volumes and ``local`` come from the device's integerized plans
and transfer plans (bit-exact with the reference); ``layer_time`` is the
reference's abstract cost model evaluated on them (same float operations, so
the CSV is byte-identical); the measured device time of each micro-batch's
scheduler launches is reported beside it (``RunResult.sched_us``), not in the
CSV.  ``harmony_comm_aware`` (a float simplex, out of scope) raises.
"""

from __future__ import annotations

import io
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib
from .adaptive import LoadHistory, ReplacementPolicy, evaluate_and_maybe_replace
from .core import (
    ClusterShape,
    ConfigError,
    ContractViolation,
    Placement,
    Topology,
    aggregate_expert_loads,
    gpu_load_balance_ratio,
)
from .placement import identical_placement
from .router import RoutingTable, TransferPlan
from .scheduler import (
    COMM_AWARE,
    HEP_SCHED_ALL,
    HEP_SCHED_ROUTE,
    HEP_SCHED_TOPO,
    HEP_SCHED_TRANSFER,
    TOPOLOGY_AWARE,
    DeviceScheduler,
    SolveOptions,
    integerize_plan,
    solve_comm_aware,
    warm_solve,
)
from .workload import Workload, gen_zipf_workload

STRATEGIES = ("vanilla_ep", "merged_ep", "harmony", "harmony_comm_aware", "harmony_pipelined")
DEVICE_STRATEGIES = ("vanilla_ep", "merged_ep", "harmony", "harmony_pipelined")

METRICS_CSV_HEADER = (
    "strategy,s,seed,microbatch,max_load,balance_ratio,a2a_intra,a2a_inter,local,layer_time"
)


@dataclass(frozen=True)
class CostModel:
    """The reference's abstract per-token cost model (``simulator.py:97-118``)."""

    t_token: float = 1.0
    alpha_intra: float = 0.1
    alpha_inter: float = 1.0
    t_schedule: float = 100.0
    overlap_schedule: bool = False
    pipeline_ratio: float = 1.0

    def __post_init__(self):
        if min(self.t_token, self.alpha_intra, self.alpha_inter, self.t_schedule) < 0:
            raise ContractViolation("cost model times must be >= 0")
        if not (0.0 < self.pipeline_ratio <= 1.0):
            raise ContractViolation("pipeline_ratio must be in (0, 1]")


@dataclass(frozen=True)
class MicrobatchMetrics:
    index: int
    max_gpu_load: int
    balance_ratio: float
    a2a_intra: int
    a2a_inter: int
    local_volume: int
    layer_time: float
    schedule_time_hidden: bool
    breakdown: dict = field(compare=False)


@dataclass
class RunResult:
    strategy: str
    metrics: list
    events: list
    lp_solves: int
    tables: list | None = None
    sched_us: list = field(default_factory=list)  # measured device time of the schedule launches

    def mean_balance_ratio(self) -> float:
        return sum(m.balance_ratio for m in self.metrics) / max(len(self.metrics), 1)

    def max_balance_ratio(self) -> float:
        return max((m.balance_ratio for m in self.metrics), default=1.0)

    def mean_layer_time(self) -> float:
        return sum(m.layer_time for m in self.metrics) / max(len(self.metrics), 1)


@dataclass
class _Phase:
    ranges: tuple
    transfer: TransferPlan
    gpu_loads: tuple


def _vanilla_xi(shape: ClusterShape, placement: Placement, loads) -> list[list[int]]:
    """``_vanilla_plan`` (simulator.py:260-280): replica k of an expert takes the
    tokens of EP group k's sources."""
    ep = shape.ep_degree
    return [[sum(loads.entries[e][src] for src in range(k * ep, (k + 1) * ep)) for k in range(len(group))]
            for e, group in enumerate(placement.edp_groups)]


def _require_identical(shape: ClusterShape, placement: Placement, strategy: str) -> None:
    if placement.edp_groups != identical_placement(shape).edp_groups:
        raise ConfigError([f"{strategy} requires the identical per-EP-group placement for this shape"])


class _Runner:
    """Device scheduler handles per placement + reusable device load buffer."""

    def __init__(self, shape: ClusterShape, device):
        self.torch = _lib.require_cuda()
        self.shape = shape
        self.device = device
        self._ds: dict = {}
        t = self.torch
        self.loads = t.zeros(shape.num_experts, shape.num_gpus, dtype=t.int64, device=device)
        self.ev = (t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True))

    def ds(self, placement: Placement) -> DeviceScheduler:
        key = (placement.edp_groups, placement.slots)
        d = self._ds.get(key)
        if d is None:
            d = self._ds[key] = DeviceScheduler(placement, gpus_per_node=self.shape.gpus_per_node, device=self.device)
        return d

    def phase_of(self, ds, bufs, gpu_loads=None) -> _Phase:
        G = self.shape.num_gpus
        tp = TransferPlan.from_flat(G, bufs.transfer.cpu().tolist())
        gl = tuple(bufs.gpu_load.cpu().tolist()) if gpu_loads is None else tuple(gpu_loads)
        return _Phase(bufs.host_ranges(), tp, gl)

    def run_comm_aware(self, placement: Placement, loads, cost: "CostModel", state):
        """``harmony_comm_aware`` (simulator.py:406-419): the device simplex solves
        comp + alpha*comm (topology-aware when the shape has several nodes), cold on the
        first micro-batch of a placement and warm from the previous basis after; the
        integerized plan is routed topology-aware on the device.  Returns (phases,
        device µs = LP solve + routing, state)."""
        t = self.torch
        G = self.shape.num_gpus
        topology = Topology.from_shape(self.shape)
        if state is None:
            mode = TOPOLOGY_AWARE if topology.num_nodes > 1 else COMM_AWARE
            opts = SolveOptions(mode=mode, alpha=cost.alpha_inter, alpha_intra=cost.alpha_intra,
                                alpha_inter=cost.alpha_inter)
            plan, _stats, state = solve_comm_aware(placement, loads, topology, opts)
        else:
            plan, state = warm_solve(state, loads)
        lp_us = state.stats.device_us_last
        ip = integerize_plan(plan)
        self.loads.copy_(t.as_tensor(np.asarray(loads.as_array(), dtype=np.int64)))
        ds = self.ds(placement)
        flat = [v for row in ip.entries for v in row]
        d_xi = t.tensor(flat or [0], dtype=t.int64, device=self.device)
        s0, s1 = self.ev
        s0.record()
        ds.launch_route(self.loads, G, 1, d_xi, HEP_SCHED_ROUTE | HEP_SCHED_TRANSFER | HEP_SCHED_TOPO)
        s1.record()
        t.cuda.synchronize(self.device)
        ds.check_status("harmony_comm_aware")
        gl = [0] * G
        for group, row in zip(placement.edp_groups, ip.entries):
            for g, v in zip(group, row):
                gl[g] += v
        return [self.phase_of(ds, ds, gl)], lp_us + 1e3 * s0.elapsed_time(s1), state

    def run_mb(self, strategy: str, placement: Placement, loads, static_share: Fraction):
        t = self.torch
        G = self.shape.num_gpus
        self.loads.copy_(t.as_tensor(np.asarray(loads.as_array(), dtype=np.int64)))
        ds = self.ds(placement)
        s0, s1 = self.ev
        s0.record()
        if strategy in ("harmony", "merged_ep"):
            ds.launch_solve(self.loads, G, 1, None, HEP_SCHED_ALL)
        elif strategy == "harmony_pipelined":
            ds.launch_pipelined(self.loads, G, 1, static_share, HEP_SCHED_ALL)
        else:  # vanilla_ep: fixed plan, routed on the device
            xi = _vanilla_xi(self.shape, placement, loads)
            flat = [v for row in xi for v in row]
            d_xi = t.tensor(flat or [0], dtype=t.int64, device=self.device)
            ds.launch_route(self.loads, G, 1, d_xi, HEP_SCHED_ROUTE | HEP_SCHED_TRANSFER)
        s1.record()
        t.cuda.synchronize(self.device)
        us = 1e3 * s0.elapsed_time(s1)
        ds.check_status(strategy)
        if strategy == "harmony_pipelined":
            phases = [self.phase_of(ds, ds.former), self.phase_of(ds, ds)]
        elif strategy == "vanilla_ep":
            gl = [0] * G
            for group, row in zip(placement.edp_groups, xi):
                for g, v in zip(group, row):
                    gl[g] += v
            phases = [self.phase_of(ds, ds, gl)]
        else:
            phases = [self.phase_of(ds, ds)]
        return phases, us


def _comm_times(cost: CostModel, transfers) -> tuple[float, float]:
    intra = sum(cost.alpha_intra * t.max_intra() for t in transfers)
    inter = sum(cost.alpha_inter * t.max_inter() for t in transfers)
    return intra, inter


def run_strategy(workload: Workload, strategy: str, placement: Placement | None, cost: CostModel,
                 policy: ReplacementPolicy | None = None, *, seed: int = 0, keep_tables: bool = False,
                 device=None, _runner: _Runner | None = None) -> RunResult:
    """Reference ``run_strategy`` (simulator.py:346-483) on the device scheduler."""
    if strategy not in STRATEGIES:
        raise ConfigError([f"unknown strategy {strategy!r}; expected one of {STRATEGIES}"])
    shape = workload.shape
    if strategy in ("vanilla_ep", "merged_ep"):
        placement = placement if placement is not None else identical_placement(shape)
        _require_identical(shape, placement, strategy)
    elif placement is None:
        raise ConfigError([f"{strategy} requires an explicit placement"])
    if placement.num_gpus != shape.num_gpus or placement.num_experts != shape.num_experts:
        raise ConfigError(["placement does not match the workload shape"])
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    runner = _runner or _Runner(shape, dev)

    metrics, events, sched_us = [], [], []
    tables = [] if keep_tables else None
    lp_solves = 0
    history = LoadHistory(policy.window) if policy else None
    current = placement
    schedules = strategy != "vanilla_ep"
    static_share = Fraction(1) - Fraction(cost.pipeline_ratio)
    comm_state = None  # warm-start state of harmony_comm_aware, reset on replacement
    for i, loads in enumerate(workload.micro_batches):
        migration = 0.0
        if (policy is not None and schedules and strategy != "merged_ep" and i > 0
                and i % policy.check_interval == 0 and len(history) > 0):
            decision = evaluate_and_maybe_replace(current, history, policy, shape, seed)
            if decision.replaced:
                current = decision.placement
                comm_state = None
                migration = decision.migration_cost_total
                events.append(decision.to_event(i))
        if strategy == "harmony_comm_aware":
            phases, us, comm_state = runner.run_comm_aware(current, loads, cost, comm_state)
        else:
            phases, us = runner.run_mb(strategy, current, loads, static_share)
        sched_us.append(us)
        if schedules:
            lp_solves += 1
        comm_former_time = 0.0
        if strategy == "harmony_pipelined":
            fi, fe = _comm_times(cost, [phases[0].transfer])
            comm_former_time = fi + fe
        gpu_loads = [0] * shape.num_gpus
        for ph in phases:
            for g, v in enumerate(ph.gpu_loads):
                gpu_loads[g] += v
        max_load = max(gpu_loads)
        intra_time, inter_time = _comm_times(cost, [ph.transfer for ph in phases])
        if not schedules:
            schedule_visible, hidden = 0.0, False
        elif cost.overlap_schedule:
            schedule_visible, hidden = 0.0, True
        elif strategy == "harmony_pipelined":
            schedule_visible = max(0.0, cost.t_schedule - comm_former_time)
            hidden = schedule_visible == 0.0
        else:
            schedule_visible, hidden = cost.t_schedule, False
        breakdown = {
            "compute": cost.t_token * max_load,
            "comm_intra": intra_time,
            "comm_inter": inter_time,
            "schedule": schedule_visible,
            "migration": migration,
        }
        metrics.append(MicrobatchMetrics(
            index=i, max_gpu_load=max_load, balance_ratio=gpu_load_balance_ratio(gpu_loads),
            a2a_intra=sum(ph.transfer.intra_volume for ph in phases),
            a2a_inter=sum(ph.transfer.inter_volume for ph in phases),
            local_volume=sum(ph.transfer.local_volume for ph in phases),
            layer_time=sum(breakdown.values()), schedule_time_hidden=hidden, breakdown=breakdown))
        if tables is not None:
            tables.append(RoutingTable(tuple(r for ph in phases for r in ph.ranges)))
        if history is not None:
            history.push(aggregate_expert_loads(loads))
    return RunResult(strategy, metrics, events, lp_solves, tables, sched_us)


@dataclass
class SweepRow:
    strategy: str
    s: float
    seed: int
    microbatch: int
    max_load: int
    balance_ratio: float
    a2a_intra: int
    a2a_inter: int
    local: int
    layer_time: float


@dataclass
class SweepResult:
    rows: list
    lp_solves: dict
    events: list
    sched_us: dict = field(default_factory=dict)  # strategy -> measured µs per micro-batch

    def to_csv(self) -> str:
        """The reference's metrics.csv (``simulator.py:526-536``)."""
        buf = io.StringIO()
        buf.write(METRICS_CSV_HEADER + "\n")
        for r in self.rows:
            buf.write(f"{r.strategy},{r.s:.6f},{r.seed},{r.microbatch},{r.max_load},"
                      f"{r.balance_ratio:.6f},{r.a2a_intra},{r.a2a_inter},{r.local},"
                      f"{r.layer_time:.6f}\n")
        return buf.getvalue()

    def summary(self) -> dict:
        """The reference's summary.json body (``simulator.py:538-556``)."""
        groups: dict = {}
        for r in self.rows:
            groups.setdefault((r.strategy, r.s), []).append(r)
        out: dict = {}
        for (strategy, s), rows in sorted(groups.items()):
            ratios = sorted(r.balance_ratio for r in rows)
            p99 = ratios[min(len(ratios) - 1, int(0.99 * len(ratios)))]
            out.setdefault(strategy, {})[f"{s:.6f}"] = {
                "mean_balance_ratio": round(sum(ratios) / len(ratios), 6),
                "max_balance_ratio": round(ratios[-1], 6),
                "p99_balance_ratio": round(p99, 6),
                "mean_layer_time": round(sum(r.layer_time for r in rows) / len(rows), 6),
            }
        return out


def run_skew_sweep(shape: ClusterShape, s_values, strategies, seeds, *, placement: Placement | None = None,
                   tokens_per_gpu: int = 2048, n_microbatches: int = 50, cost: CostModel | None = None,
                   policy: ReplacementPolicy | None = None, workers: int | None = None, device=None) -> SweepResult:
    """Reference ``run_skew_sweep`` (simulator.py:566-640): the same task order and
    merged rows; every micro-batch scheduled on the device (one GPU, so
    ``workers`` is accepted for signature compatibility and ignored)."""
    cost = cost or CostModel()
    for st in strategies:
        if st not in STRATEGIES:
            raise ConfigError([f"unknown strategy {st!r}"])
    torch = _lib.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    runner = _Runner(shape, dev)
    tasks = [(strategy, float(s), int(seed)) for strategy in strategies for s in s_values for seed in seeds]
    rows, lp_solves, events, us = [], {}, [], {}
    for strategy, s, seed in tasks:
        workload = gen_zipf_workload(shape, s, tokens_per_gpu, n_microbatches, seed)
        pl = identical_placement(shape) if strategy in ("vanilla_ep", "merged_ep") else placement
        res = run_strategy(workload, strategy, pl, cost, policy, seed=seed, device=dev, _runner=runner)
        lp_solves[strategy] = lp_solves.get(strategy, 0) + res.lp_solves
        us.setdefault(strategy, []).extend(res.sched_us)
        for ev in res.events:
            events.append({"strategy": strategy, "s": s, "seed": seed, **ev})
        for m in res.metrics:
            rows.append(SweepRow(strategy=strategy, s=s, seed=seed, microbatch=m.index, max_load=m.max_gpu_load,
                                 balance_ratio=m.balance_ratio, a2a_intra=m.a2a_intra, a2a_inter=m.a2a_inter,
                                 local=m.local_volume, layer_time=m.layer_time))
    return SweepResult(rows, lp_solves, events, us)
