"""B200-native HarmonyEP token-scheduling MoE path.

Drop-in for the reference ``harmonyep`` scheduler/router/config API
(``/root/reference/pkg/src/harmonyep/__init__.py:11-82``, the names on the
hot path), backed by hand-written sm_100a kernels behind the C ABI in
``include/hep.h`` (``libhep.so``), plus the device MoE layer
(``MoELayer``) that runs gate -> histogram -> scheduler -> permute ->
grouped GEMM -> combine entirely on the GPU.
"""

from .core import (
    CapacityError,
    ClusterShape,
    ConfigError,
    ConstructionError,
    ContractViolation,
    DimensionError,
    HarmonyError,
    LoadMatrix,
    Placement,
    PlacementError,
    ReplicaLoadPlan,
    StaleStateError,
    Topology,
    TraceParseError,
    UndefinedMetricError,
    aggregate_expert_loads,
    balance_ratio,
    gpu_load_balance_ratio,
)
from .placement import (
    DensityReport,
    PlacementGraph,
    cayley_symmetric,
    density_oracle,
    greedy_replica_counts,
    identical_placement,
    monte_carlo_placement,
    random_placement,
    symmetric_placement,
    validate_placement,
)
from .adaptive import (
    LoadHistory,
    ReplacementDecision,
    ReplacementPolicy,
    evaluate_and_maybe_replace,
    predict_loads,
)
from .router import (
    RoutingTable,
    TransferPlan,
    build_transfer_plan,
    route_tokens,
    route_topology_aware,
)
from .scheduler import (
    BALANCE_ONLY,
    COMM_AWARE,
    TOPOLOGY_AWARE,
    CommPlanStats,
    SolveOptions,
    SolverState,
    SolveStats,
    integerize_plan,
    solve_comm_aware,
    solve_replica_loads,
    warm_solve,
)
from .simplex import LinearProgram, SimplexError, SimplexResult, simplex_solve
from .workload import Workload, gen_zipf_workload, load_trace, save_trace, zipf_gate_bias
from .sweep import STRATEGIES, CostModel, MicrobatchMetrics, RunResult, SweepResult, run_skew_sweep, run_strategy
from .layer import MoELayer

__all__ = [n for n in dir() if not n.startswith("_")]
