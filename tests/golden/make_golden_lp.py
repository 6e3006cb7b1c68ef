"""Generate the golden fixtures that pin the device simplex (``csrc/lp.cu``) and the
communication-aware scheduling modes to the reference.

Runs ONLY in the build container, where the reference package can be imported
read-only from ``/root/reference/pkg/src``.  The GPU box sees only the committed
output ``tests/golden/lp_cases.json.gz``.

    python tests/golden/make_golden_lp.py

Recorded from the reference's own code:

* ``_comm_aware_lp`` / ``_topology_aware_lp`` (scheduler.py:480-619): a SHA-256 of the
  LP matrices, so the host builders are checked byte for byte on CPU;
* ``simplex_solve`` (simplex.py:99-192) through ``solve_comm_aware`` (:622-689): x (as
  float.hex), basis, pivot count, objective, the float plan, CommPlanStats and the
  integerized plan;
* ``warm_solve`` (:436-461) sequences on one state (warm-started simplex);
* acceptance C9 (test_acceptance.py:236-262): the 100 topology-aware instances with the
  balance-only and topology-aware inter-node volumes;
* ``run_skew_sweep`` with ``harmony_comm_aware`` (simulator.py:406-419): metrics.csv.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _h():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import harmonyep

    return harmonyep


def lp_sha(lp) -> str:
    h = hashlib.sha256()
    for a in (lp.c, lp.a_eq, lp.b_eq, lp.a_ub, lp.b_ub):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def hexl(v):
    return [float(x).hex() for x in v]


def record(h, placement, loads, topology, options, state=None):
    from harmonyep import scheduler as S
    from harmonyep.simplex import simplex_solve

    if options.mode == S.COMM_AWARE:
        lp, _keys = S._comm_aware_lp(placement, loads, options.alpha)
    else:
        lp, _keys = S._topology_aware_lp(placement, loads, topology, options.alpha_intra, options.alpha_inter)
    basis_in = None if state is None else (None if state._basis is None else list(map(int, state._basis)))
    t0 = time.perf_counter()
    res = simplex_solve(lp, basis=None if state is None else state._basis)
    ref_ms = 1e3 * (time.perf_counter() - t0)
    if state is None:
        plan, stats, st = h.solve_comm_aware(placement, loads, topology, options)
    else:
        plan, stats, st = h.solve_comm_aware(placement, loads, topology, options, _state=state)
    ip = h.integerize_plan(plan)
    rec = {
        "G": placement.num_gpus,
        "E": placement.num_experts,
        "gpn": topology.gpus_per_node,
        "groups": [list(g) for g in placement.edp_groups],
        "slots": list(placement.slots),
        "loads": [list(r) for r in loads.entries],
        "mode": options.mode,
        "alpha": options.alpha,
        "alpha_intra": options.alpha_intra,
        "alpha_inter": options.alpha_inter,
        "lp_shape": [int(lp.c.size), int(lp.b_eq.size), int(lp.b_ub.size)],
        "lp_sha": lp_sha(lp),
        "basis_in": basis_in,
        "x": hexl(res.x),
        "basis": [int(b) for b in res.basis],
        "iterations": int(res.iterations),
        "objective": float(res.objective).hex(),
        "plan": [hexl(r) for r in plan.entries],
        "plan_objective": float(plan.objective).hex(),
        "stats": {k: [float(v).hex() for v in getattr(stats, k)] for k in ("send", "recv", "local")}
        | {"comp": float(stats.comp).hex(), "comm": float(stats.comm).hex()},
        "int_plan": [list(map(int, r)) for r in ip.entries],
        "ref_ms": ref_ms,
    }
    return rec, st


def main():
    h = _h()
    from harmonyep.scheduler import COMM_AWARE, TOPOLOGY_AWARE

    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_instance  # the reference's own property-test generator

    cases = []
    # known answers of the reference tests (test_scheduler.py:240-294)
    pl = h.Placement(2, ((0, 1),), (0,))
    for alpha in (1.5, 2.0, 10.0):
        cases.append(record(h, pl, h.LoadMatrix(((4, 0),)), h.Topology(2, 2),
                            h.SolveOptions(mode=COMM_AWARE, alpha=alpha))[0] | {"family": "all_local"})
    pl = h.Placement(2, ((0, 1), (0, 1)), (0, 1))
    cases.append(record(h, pl, h.LoadMatrix(((4, 0), (4, 0))), h.Topology(2, 2),
                        h.SolveOptions(mode=COMM_AWARE, alpha=0.1))[0] | {"family": "two_expert_split"})
    ring4 = h.Placement(4, ((0, 3), (0, 1), (1, 2), (2, 3)), (0, 0, 1, 1))
    ring4_loads = h.LoadMatrix(((4, 0, 0, 0), (0, 6, 0, 0), (0, 0, 14, 0), (0, 0, 0, 8)))
    cases.append(record(h, ring4, ring4_loads, h.Topology(4, 4),
                        h.SolveOptions(mode=COMM_AWARE, alpha=1e6))[0] | {"family": "ring4_large_alpha"})
    # property suites (alpha = 0 == balance, stats identity)
    for seed, alpha, n in ((7, 0.0, 15), (13, 0.3, 10), (21, 1.0, 10)):
        rng = np.random.default_rng(seed)
        for _ in range(n):
            _shape, placement, loads = random_instance(rng, max_gpus=7, max_experts=10, d_choices=(2,))
            topo = h.Topology(placement.num_gpus, placement.num_gpus)
            bal = h.solve_replica_loads(placement, loads)[0]
            r = record(h, placement, loads, topo, h.SolveOptions(mode=COMM_AWARE, alpha=alpha))[0]
            r["family"] = f"random_comm_a{alpha}"
            r["balance_objective"] = float(bal.objective).hex()
            cases.append(r)
    rng = np.random.default_rng(9)
    for _ in range(8):
        E = int(rng.integers(4, 10))
        shape = h.ClusterShape(8, E, 2, gpus_per_node=4)
        placement = h.random_placement(shape, int(rng.integers(0, 10**6)))
        loads = h.LoadMatrix.from_array(rng.integers(0, 50, size=(E, 8)))
        bal = h.solve_replica_loads(placement, loads)[0]
        r = record(h, placement, loads, h.Topology(8, 4),
                   h.SolveOptions(mode=TOPOLOGY_AWARE, alpha_intra=0.0, alpha_inter=0.0))[0]
        r["family"] = "topo_alpha0"
        r["balance_objective"] = float(bal.objective).hex()
        cases.append(r)
    # acceptance C9 (test_acceptance.py:236-262)
    shape = h.ClusterShape(8, 12, 2, gpus_per_node=4)
    topology = h.Topology(8, 4)
    rng = np.random.default_rng(42)
    for _ in range(100):
        placement = h.random_placement(shape, int(rng.integers(0, 10**6)))
        loads = h.LoadMatrix.from_array(rng.integers(0, 101, size=(12, 8)))
        bal_plan = h.integerize_plan(h.solve_replica_loads(placement, loads)[0])
        bal_tp = h.build_transfer_plan(h.route_topology_aware(placement, loads, bal_plan, topology), topology)
        r, _ = record(h, placement, loads, topology,
                      h.SolveOptions(mode=TOPOLOGY_AWARE, alpha_intra=0.1, alpha_inter=1.0))
        ip = h.integerize_plan(h.solve_comm_aware(placement, loads, topology, h.SolveOptions(
            mode=TOPOLOGY_AWARE, alpha_intra=0.1, alpha_inter=1.0))[0])
        topo_tp = h.build_transfer_plan(h.route_topology_aware(placement, loads, ip, topology), topology)
        r["family"] = "c9"
        r["balance_inter"] = int(bal_tp.inter_volume)
        r["topo_inter"] = int(topo_tp.inter_volume)
        cases.append(r)
    # broad random family: the reference's property-test generator, G 4..10, E 4..20,
    # d 2..3, both modes, several alphas / node sizes
    rng = np.random.default_rng(20251017)
    for i in range(300):
        _shape, placement, loads = random_instance(rng)
        G = placement.num_gpus
        if i % 2 == 0:
            alpha = float(rng.choice([0.05, 0.1, 0.5, 1.0, 2.0]))
            opts = h.SolveOptions(mode=COMM_AWARE, alpha=alpha)
            topo = h.Topology(G, G)
        else:
            gpn = int(rng.choice([g for g in (1, 2, 3, 4, 5) if G % g == 0 and g < G] or [G]))
            ai = float(rng.choice([0.0, 0.1, 0.3]))
            opts = h.SolveOptions(mode=TOPOLOGY_AWARE, alpha_intra=ai, alpha_inter=max(ai, float(rng.choice([0.5, 1.0]))))
            topo = h.Topology(G, gpn)
        r = record(h, placement, loads, topo, opts)[0]
        r["family"] = "random300"
        cases.append(r)
    # larger comm-aware LPs (Cayley placements at BASELINE-like expert counts, one node)
    for E in (32, 64):
        shape = h.ClusterShape(8, E, 2)
        placement = h.cayley_symmetric(shape)
        wl = h.gen_zipf_workload(shape, 1.0, 4096, 1, 3)
        r = record(h, placement, wl.micro_batches[0], h.Topology(8, 8),
                   h.SolveOptions(mode=COMM_AWARE, alpha=0.1))[0]
        r["family"] = f"cayley_E{E}"
        cases.append(r)

    # warm sequences (warm_solve on one state)
    warm = []
    for E, gpn, mode, n_mb in ((16, 8, COMM_AWARE, 8), (16, 4, TOPOLOGY_AWARE, 8), (8, 8, COMM_AWARE, 30)):
        shape = h.ClusterShape(8, E, 2, gpus_per_node=gpn)
        placement = h.cayley_symmetric(shape)
        topo = h.Topology(8, gpn)
        wl = h.gen_zipf_workload(shape, 1.0, 1024, n_mb, 5)
        opts = h.SolveOptions(mode=mode, alpha=1.0, alpha_intra=0.1, alpha_inter=1.0)
        state = None
        seq = []
        for loads in wl.micro_batches:
            r, state = record(h, placement, loads, topo, opts, state)
            seq.append(r)
        warm.append(seq)

    # the sweep strategy (metrics.csv, simulator.py:406-419)
    sweep = []
    for G, E, gpn in ((8, 16, 8), (8, 16, 4)):
        shape = h.ClusterShape(G, E, 2, gpus_per_node=gpn)
        placement = h.cayley_symmetric(shape)
        res = h.run_skew_sweep(shape, (0.5, 1.5), ("harmony_comm_aware",), (0, 1), placement=placement,
                               tokens_per_gpu=512, n_microbatches=6, cost=h.CostModel())
        sweep.append({"G": G, "E": E, "gpn": gpn, "groups": [list(g) for g in placement.edp_groups],
                      "slots": list(placement.slots), "csv": res.to_csv(), "summary": res.summary(),
                      "lp_solves": res.lp_solves})

    out = {"cases": cases, "warm": warm, "sweep": sweep}
    path = os.path.join(HERE, "lp_cases.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, sort_keys=True)
    print(path, len(cases), "cases,", sum(len(s) for s in warm), "warm solves,", len(sweep), "sweeps")


if __name__ == "__main__":
    main()
