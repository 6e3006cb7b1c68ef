"""CPU tests of the host-side pieces: domain types, placement constructors,
workload generator, C-ABI symbol table.  No compute calls (no GPU here)."""

import ctypes
import json
import os
import re
from fractions import Fraction

import pytest

from conftest import ROOT, load_golden
from paper_2511_16947_b200 import (
    ClusterShape,
    ContractViolation,
    DimensionError,
    LoadMatrix,
    Placement,
    PlacementError,
    ReplicaLoadPlan,
    UndefinedMetricError,
    balance_ratio,
    cayley_symmetric,
    gen_zipf_workload,
    identical_placement,
    validate_placement,
)
from paper_2511_16947_b200.core import gpu_load_balance_ratio


def test_cluster_shape_validation():
    with pytest.raises(DimensionError):
        ClusterShape(4, 8, 1)
    with pytest.raises(DimensionError):
        ClusterShape(4, 8, 5)
    with pytest.raises(DimensionError):
        ClusterShape(6, 8, 2, gpus_per_node=4)
    s = ClusterShape(8, 16, 2)
    assert s.gpus_per_node == 8 and s.num_nodes == 1 and s.ep_degree == 4
    with pytest.raises(DimensionError):
        _ = ClusterShape(6, 8, 4).ep_degree


def test_placement_validation_and_json():
    with pytest.raises(PlacementError):
        Placement(2, ((0, 2),), (0,))
    with pytest.raises(PlacementError):
        Placement(2, ((1, 1),), (0,))
    with pytest.raises(DimensionError):
        Placement(2, ((0, 1),), (0, 1))
    pl = Placement(4, ((0, 3), (0, 1), (1, 2), (2, 3)), (0, 0, 1, 1))
    assert pl.hosted == ((0, 1), (1, 2), (2, 3), (0, 3))
    assert Placement.from_json_dict(json.loads(json.dumps(pl.to_json_dict()))) == pl
    with pytest.raises(ContractViolation):
        Placement.from_json_dict({"num_gpus": 2})
    off, gpu = pl.csr()
    assert off.tolist() == [0, 2, 4, 6, 8] and gpu.tolist() == [0, 3, 0, 1, 1, 2, 2, 3]


def test_load_matrix():
    lm = LoadMatrix(((1, 2), (3, 4)))
    assert lm.expert_totals() == (3, 7) and lm.total() == 10 and lm.num_gpus == 2
    assert lm.scaled(3).entries == ((3, 6), (9, 12))
    with pytest.raises(ContractViolation):
        LoadMatrix(((1, -1),))
    with pytest.raises(DimensionError):
        LoadMatrix(((1, 2), (3,)))


def test_balance_ratio():
    plan = ReplicaLoadPlan(2, ((0, 1),), ((5, 3),), 5)
    assert balance_ratio(plan, ClusterShape(2, 1, 2)) == Fraction(5, 4)
    with pytest.raises(UndefinedMetricError):
        balance_ratio(ReplicaLoadPlan(2, ((0, 1),), ((0, 0),), 0), ClusterShape(2, 1, 2))
    assert gpu_load_balance_ratio([20, 4, 4, 4]) == 2.5
    assert gpu_load_balance_ratio([0, 0]) == 1.0


def test_plan_integrality():
    assert ReplicaLoadPlan(2, ((0, 1),), ((Fraction(4, 2), 3),), 3).is_integral()
    assert not ReplicaLoadPlan(2, ((0, 1),), ((2.5, 3),), 3).is_integral()


def test_cayley_matches_reference_goldens():
    """Reference goldens (tests/golden/cayley_*.json, acceptance C6) re-exported
    in tests/golden/placements.json, incl. the DSv3 (8x256) and Qwen3 (8x128) shapes."""
    gold = load_golden("placements.json")
    n = 0
    for key, want in gold.items():
        if key.startswith("identical_"):
            G, E = (int(x[1:]) for x in key.split("_")[1:])
            got = identical_placement(ClusterShape(G, E, 2))
        else:
            G, E = (int(x[1:]) for x in key.split("_"))
            got = cayley_symmetric(ClusterShape(G, E, 2))
        assert got.to_json_dict() == want, key
        assert validate_placement(got, ClusterShape(G, E, 2), uniform=not key.startswith("identical_")) == []
        n += 1
    assert n >= 12


def test_zipf_generator_matches_reference():
    for rec in load_golden("zipf_counts.json.gz"):
        wl = gen_zipf_workload(ClusterShape(rec["G"], rec["E"], 2), rec["s"], rec["T"], len(rec["mbs"]), rec["seed"])
        assert [list(map(list, mb.entries)) for mb in wl.micro_batches] == rec["mbs"]


def _header_symbols():
    hdr = open(os.path.join(ROOT, "include", "hep.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(hep_[a-z0-9_]+)\s*\(", hdr)))


def test_capi_library_exports_every_header_symbol():
    from paper_2511_16947_b200 import _lib

    path = _lib.LIB_PATH
    if not os.path.exists(path):
        from paper_2511_16947_b200.build import build

        build()
    L = ctypes.CDLL(path)  # loads without a GPU: no CUDA calls at load time
    syms = _header_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert L.hep_abi_version() == 1


def test_product_path_has_no_cpu_fallback():
    """Compute entry points must fail loudly without a CUDA device."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2511_16947_b200 import solve_replica_loads

    pl = Placement(2, ((0, 1),), (0,))
    with pytest.raises(RuntimeError, match="CUDA"):
        solve_replica_loads(pl, LoadMatrix(((1, 1),)))


def test_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_16947_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "hep_oracle", "libhep_oracle"):
                    assert bad not in src, (f, bad)


REFERENCE_NAMES = (  # harmonyep/__init__.py:11-82 minus the comm-aware LP statistics type
    "CapacityError ClusterShape ConfigError ConstructionError ContractViolation DimensionError HarmonyError "
    "LoadMatrix Placement PlacementError ReplicaLoadPlan StaleStateError Topology TraceParseError "
    "UndefinedMetricError aggregate_expert_loads balance_ratio BALANCE_ONLY COMM_AWARE TOPOLOGY_AWARE SolveOptions "
    "SolverState integerize_plan solve_comm_aware solve_replica_loads warm_solve RoutingTable TransferPlan "
    "build_transfer_plan route_tokens route_topology_aware DensityReport PlacementGraph cayley_symmetric "
    "density_oracle greedy_replica_counts identical_placement monte_carlo_placement random_placement "
    "symmetric_placement validate_placement LoadHistory ReplacementDecision ReplacementPolicy "
    "evaluate_and_maybe_replace predict_loads STRATEGIES CostModel MicrobatchMetrics RunResult SweepResult Workload "
    "gen_zipf_workload load_trace run_skew_sweep run_strategy save_trace"
).split()


def test_reference_api_surface_is_exported():
    import paper_2511_16947_b200 as P

    missing = [n for n in REFERENCE_NAMES if not hasattr(P, n)]
    assert not missing, missing


def test_trace_roundtrip_and_errors(tmp_path):
    import paper_2511_16947_b200 as P

    shape = P.ClusterShape(4, 8, 2)
    wl = P.gen_zipf_workload(shape, 1.2, 300, 4, 5)
    path = tmp_path / "t.csv"
    P.save_trace(wl, str(path))
    back = P.load_trace(str(path), shape)
    assert back.micro_batches == wl.micro_batches
    bad = tmp_path / "bad.csv"
    bad.write_text("microbatch,expert,gpu,tokens\n0,1,2,3\n0,9,0,1\n")
    with pytest.raises(P.TraceParseError) as ei:
        P.load_trace(str(bad), shape)
    assert ei.value.line_no == 3 and "expert 9 out of range 0..7" in str(ei.value)
    bad.write_text("mb,expert,gpu,tokens\n")
    with pytest.raises(P.TraceParseError):
        P.load_trace(str(bad), shape)
    # repeated rows add up; gaps are empty micro-batches
    ok = tmp_path / "ok.csv"
    ok.write_text("microbatch,expert,gpu,tokens\n2,0,0,5\n2,0,0,6\n")
    w = P.load_trace(str(ok), shape)
    assert len(w.micro_batches) == 3 and w.micro_batches[2].entries[0][0] == 11 and w.micro_batches[0].total() == 0


def test_tuning_struct_matches_header():
    """hep_tuning (include/hep.h) and its ctypes mirror (_lib.HepTuning) list the same int
    fields in the same order, reserved tail included: a mismatch would silently shift every
    tuning knob after it.  The library's defaults round-trip through hep_tuning_get / set."""
    import re

    from paper_2511_16947_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "hep.h")).read()
    body = re.search(r"typedef struct \{(.*?)\} hep_tuning;", hdr, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"int\s+(\w+)\s*(?:\[(\d+)\])?\s*;", body)
    names = [f for f, n in fields if not n]
    reserved = [int(n) for f, n in fields if n]
    assert tuple(names) == _lib.TUNING_FIELDS
    assert reserved == [dict(_lib.HepTuning._fields_)["reserved"]._length_]
    t = _lib.get_tuning()
    assert set(t) == set(_lib.TUNING_FIELDS)


def test_capi_argument_validation_without_a_device():
    """Entry points validate their arguments before touching the device: bad shapes and
    contract violations come back as the reference's error classes (status codes 1 / 3),
    on a machine without a GPU too."""
    import ctypes

    from paper_2511_16947_b200 import _lib
    from paper_2511_16947_b200.core import ContractViolation, DimensionError

    L = _lib.lib()
    fake = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    # hep_moe_permute_ex: blocks_per_sm outside 1..8
    with pytest.raises(ContractViolation):
        _lib.check(L.hep_moe_permute_ex(fake, fake, 16, 2, 64, fake, 9, None), "hep_moe_permute_ex")
    with pytest.raises(DimensionError):  # d_model % 8
        _lib.check(L.hep_moe_permute_ex(fake, fake, 16, 2, 60, fake, 8, None), "hep_moe_permute_ex")
    # hep_router_topk_ws: K > E, e_pad not a multiple of 16
    with pytest.raises(DimensionError):
        _lib.check(L.hep_router_topk_ws(fake, fake, 128, 256, 4, 16, None, 8, 128, 1, None, fake, fake, fake, None,
                                        None, None), "hep_router_topk_ws")
    with pytest.raises(DimensionError):
        _lib.check(L.hep_router_topk_ws(fake, fake, 128, 256, 8, 12, None, 2, 128, 1, None, fake, fake, fake, None,
                                        None, None), "hep_router_topk_ws")
    # hep_moe_assign_ep_phase: phase must be 0 or 1
    out = _lib.HepSchedOut()
    with pytest.raises(ContractViolation):
        _lib.check(L.hep_moe_assign_ep_phase(fake, ctypes.byref(out), fake, 2, fake, 16, 2, 0, 0, fake, fake, fake,
                                             fake, fake, 1 << 20, None), "hep_moe_assign_ep_phase")
