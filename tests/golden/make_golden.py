"""Generate the golden fixtures that pin the oracle and the CUDA scheduler.

Runs ONLY in the build container, where the reference package can be
imported read-only from ``/root/reference/pkg/src`` (pure Python, numpy).
The GPU box never sees the reference; it only sees the committed outputs
of this script (``tests/golden/*.json.gz``).

    python tests/golden/make_golden.py

Every fixture records the reference's own outputs for the hot path:

* ``solve_replica_loads``  (reference ``scheduler.py:405-433``)  -> m, x*Q
* ``integerize_plan``      (``scheduler.py:697-735``)            -> x_int
* ``route_tokens``         (``router.py:161-163``)               -> ranges
* ``route_topology_aware`` (``router.py:166-175``)               -> ranges
* ``build_transfer_plan``  (``router.py:178-226``)               -> pair/send/recv/local/intra/inter

Instance families:
  known      hand-derived known answers of the reference tests (ring4 ...)
  random500  acceptance criterion C1/C5 suite (``test_acceptance.py:55-69``, seed 20240809)
  baseline   Cayley placements for every BASELINE shape x G in {2,4,8} x zipf s in {0,.5,1,1.5,2}
             with the exact ``gen_zipf_workload`` load matrices stored (numpy stream not pinned)
  warm100    100 micro-batches on one placement (``test_scheduler.py:188-201``)
  base       pipelined solves with ``gpu_base`` (``simulator.py:420-435``)
  asym       adaptive asymmetric placements (greedy counts + Monte-Carlo, ``placement.py:377-450``)
  pipelined  both phases of the pipelined split (static even share + gpu_base solve)
"""

from __future__ import annotations

import gzip
import json
import math
import os
import sys
from fractions import Fraction

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import harmonyep  # noqa: F401

    return harmonyep


def record(h, placement, loads, base=None, gpn=0, solve=True):
    """Run the reference hot path on one instance and capture every output."""
    G = placement.num_gpus
    Q = math.lcm(*range(1, G + 1))
    rec = {
        "G": G,
        "E": placement.num_experts,
        "groups": [list(g) for g in placement.edp_groups],
        "slots": list(placement.slots),
        "loads": [list(r) for r in loads.entries],
        "base": list(base) if base is not None else None,
        "gpn": gpn or G,
        "Q": Q,
    }
    plan, state = h.solve_replica_loads(placement, loads, gpu_base=base)
    m = Fraction(plan.objective)
    rec["m"] = [m.numerator, m.denominator]
    xq = []
    for row in plan.entries:
        out = []
        for v in row:
            v = Fraction(v)
            assert (v * Q).denominator == 1
            out.append(int(v * Q))
        xq.append(out)
    rec["xq"] = xq
    ip = h.integerize_plan(plan)
    rec["xi"] = [[int(v) for v in row] for row in ip.entries]
    rec["obj_int"] = int(ip.objective)
    table = h.route_tokens(placement, loads, ip)
    rec["ranges"] = [list(r) for r in table.ranges]
    topo = h.Topology(G, gpn or G)
    if gpn and gpn < G:
        ttab = h.route_topology_aware(placement, loads, ip, topo)
        rec["ranges_topo"] = [list(r) for r in ttab.ranges]
    tp = h.build_transfer_plan(table, topo)
    rec["pair"] = [list(r) for r in tp.pair_counts]
    rec["send"] = list(tp.send)
    rec["recv"] = list(tp.recv)
    rec["local"] = list(tp.local)
    rec["intra"] = tp.intra_volume
    rec["inter"] = tp.inter_volume
    rec["iters"] = state.stats.iterations_last
    return rec


def fam_known(h):
    P, L = h.Placement, h.LoadMatrix
    out = []
    ring4 = P(4, ((0, 3), (0, 1), (1, 2), (2, 3)), (0, 0, 1, 1))
    ring4_loads = L(((4, 0, 0, 0), (0, 6, 0, 0), (0, 0, 14, 0), (0, 0, 0, 8)))
    out.append(dict(name="ring4", **record(h, ring4, ring4_loads)))
    ident4 = P(4, ((0, 2), (0, 2), (1, 3), (1, 3)), (0, 1, 0, 1))
    out.append(dict(name="identical4", **record(h, ident4, ring4_loads)))
    cyc = P(8, tuple((v, (v + 1) % 8) for v in range(8)), tuple(e % 2 for e in range(8)))
    cyc_loads = L(tuple(tuple(7 if g == e else 0 for g in range(8)) for e in range(8)))
    out.append(dict(name="cycle8_uniform", **record(h, cyc, cyc_loads)))
    out.append(dict(name="ring4_zero", **record(h, ring4, L(((0,) * 4,) * 4))))
    empty_ok = P(2, ((), (0, 1)), (0, 0))
    out.append(dict(name="empty_group_zero_load", **record(h, empty_ok, L(((0, 0), (1, 1))))))
    unsorted = P(4, ((2, 0, 3),), (0,))
    out.append(dict(name="unsorted_group", **record(h, unsorted, L(((0, 0, 9, 0),)))))
    two = P(3, ((0, 1),), (0,))
    out.append(dict(name="remote_split", **record(h, two, L(((0, 0, 4),)))))
    node = P(4, ((1, 2),), (0,))
    out.append(dict(name="same_node_first", **record(h, node, L(((4, 0, 0, 0),)), gpn=2)))
    return out


def fam_random500(h):
    rng = np.random.default_rng(20240809)
    out = []
    for _ in range(500):
        num_gpus = int(rng.integers(4, 11))
        num_experts = int(rng.integers(4, 21))
        d = int(rng.choice((2, 3)))
        shape = h.ClusterShape(num_gpus, num_experts, d)
        placement = h.random_placement(shape, int(rng.integers(0, 10**6)))
        loads = h.LoadMatrix.from_array(rng.integers(0, 101, size=(num_experts, num_gpus)))
        gpn = num_gpus // 2 if num_gpus % 2 == 0 else 0
        out.append(record(h, placement, loads, gpn=gpn))
    return out


# BASELINE.json configs: (name, E, K, tokens per source GPU)
SHAPES = [
    ("tiny", 8, 2, 1024),
    ("mixtral", 8, 2, 16384),
    ("qwen3", 128, 8, 32768),
    ("dsv3", 256, 8, 16384),
]


def fam_baseline(h):
    out = []
    for name, E, K, T in SHAPES:
        for G in (2, 4, 8):
            shape = h.ClusterShape(G, E, 2)
            placement = h.cayley_symmetric(shape)
            for s in (0.0, 0.5, 1.0, 1.5, 2.0):
                n_mb = 2 if E >= 128 else 3
                wl = h.gen_zipf_workload(shape, s, T * K, n_mb, seed=0)
                for i, loads in enumerate(wl.micro_batches):
                    rec = record(h, placement, loads)
                    rec.update(shape_name=name, s=s, mb=i, K=K, T=T)
                    out.append(rec)
    return out


def fam_warm100(h):
    rng = np.random.default_rng(17)
    shape = h.ClusterShape(6, 10, 2)
    placement = h.random_placement(shape, 3)
    out = []
    for _ in range(100):
        loads = h.LoadMatrix.from_array(rng.integers(0, 60, size=(10, 6)))
        out.append(record(h, placement, loads))
    return out


def fam_base(h):
    """Pipelined share: static even split routed first, then a gpu_base solve
    (``simulator.py:420-435``, ``_split_loads`` ``:283-291``)."""
    from harmonyep.simulator import _even_split_plan, _split_loads

    out = []
    rng = np.random.default_rng(99)
    for G, E in ((4, 8), (8, 32), (8, 128)):
        shape = h.ClusterShape(G, E, 2)
        placement = h.cayley_symmetric(shape) if E >= G else h.random_placement(shape, 1)
        wl = h.gen_zipf_workload(shape, float(rng.choice([0.5, 1.0, 1.5])), 512, 3, seed=int(rng.integers(0, 1000)))
        for loads in wl.micro_batches:
            former, latter = _split_loads(loads, Fraction(1, 2))
            fplan = h.integerize_plan(_even_split_plan(placement, former))
            base = tuple(int(v) for v in fplan.gpu_loads())
            out.append(record(h, placement, latter, base=base))
    return out


def fam_pipelined(h):
    """Both phases of ``harmony_pipelined`` (``simulator.py:420-435``): split by the
    static share (``_split_loads`` :291-298, share = 1 - pipeline_ratio :375), the
    static share's even plan (``_even_split_plan`` :301-322) integerized and routed,
    then the scheduled share solved with the static phase's GPU loads as gpu_base."""
    from harmonyep.simulator import _even_split_plan, _split_loads

    out = []
    rng = np.random.default_rng(2025)
    cases = [(4, 8, "cayley"), (8, 8, "cayley"), (8, 32, "cayley"), (8, 128, "cayley"), (8, 16, "asym"), (6, 12, "random")]
    ratios = [0.5, 0.3, 0.75, 1.0, 0.1]
    for ci, (G, E, kind) in enumerate(cases):
        shape = h.ClusterShape(G, E, 2)
        s = float(rng.choice([0.5, 1.0, 1.5, 2.0]))
        wl = h.gen_zipf_workload(shape, s, 1024 if E <= 32 else 8192, 2, seed=int(rng.integers(0, 1000)))
        if kind == "cayley":
            placement = h.cayley_symmetric(shape)
        elif kind == "asym":
            totals = wl.micro_batches[0].expert_totals()
            placement = h.monte_carlo_placement(totals, h.greedy_replica_counts(totals, 2 * E, max_count=G), shape, 10, ci)
        else:
            placement = h.random_placement(shape, ci)
        for mi, loads in enumerate(wl.micro_batches):
            ratio = ratios[(ci + mi) % len(ratios)]
            share = Fraction(1) - Fraction(ratio)
            former, latter = _split_loads(loads, share)
            fplan = h.integerize_plan(_even_split_plan(placement, former))
            ftab = h.route_tokens(placement, former, fplan)
            ftp = h.build_transfer_plan(ftab, h.Topology(G, G))
            base = tuple(int(v) for v in fplan.gpu_loads())
            lat = record(h, placement, latter, base=base)
            out.append(dict(
                G=G, E=E, groups=[list(g) for g in placement.edp_groups], slots=list(placement.slots),
                loads=[list(r) for r in loads.entries], ratio=ratio, share=[share.numerator, share.denominator],
                former=dict(loads=[list(r) for r in former.entries], xi=[[int(v) for v in r] for r in fplan.entries],
                            gpu_load=list(base), ranges=[list(r) for r in ftab.ranges],
                            pair=[list(r) for r in ftp.pair_counts], send=list(ftp.send), recv=list(ftp.recv),
                            local=list(ftp.local)),
                latter=lat))
    return out


def fam_sweep(h):
    """``run_skew_sweep`` metrics.csv / summary.json / replacement events
    (simulator.py:566-640) for the device-scheduled strategies."""
    from harmonyep.simulator import CostModel, run_skew_sweep

    out = []
    cases = [
        (4, 8, 2, ("vanilla_ep", "merged_ep", "harmony", "harmony_pipelined"), 0.5, None),
        (8, 32, 8, ("harmony", "harmony_pipelined", "merged_ep"), 0.7, dict(check_interval=4, mc_samples=10)),
        (8, 16, 4, ("harmony", "vanilla_ep"), 1.0, dict(check_interval=3, mc_samples=8, threshold=1.05)),
    ]
    for G, E, gpn, strategies, ratio, pol in cases:
        shape = h.ClusterShape(G, E, 2, gpus_per_node=gpn)
        placement = h.cayley_symmetric(shape)
        cost = CostModel(pipeline_ratio=ratio)
        policy = h.ReplacementPolicy(**pol) if pol else None
        res = run_skew_sweep(shape, (0.5, 1.5), strategies, (0, 1), placement=placement, tokens_per_gpu=512,
                             n_microbatches=10, cost=cost, policy=policy, workers=1)
        out.append(dict(G=G, E=E, gpn=gpn, strategies=list(strategies), ratio=ratio, policy=pol,
                        groups=[list(g) for g in placement.edp_groups], slots=list(placement.slots),
                        csv=res.to_csv(), summary=res.summary(), events=res.events, lp_solves=res.lp_solves))
    return out


def fam_asym(h):
    """Asymmetric placements as the adaptive replacement would build them."""
    out = []
    for E, G, s, seed in ((8, 8, 1.5, 0), (8, 8, 2.0, 1), (32, 8, 1.25, 2), (16, 4, 2.0, 3), (128, 8, 2.0, 4)):
        shape = h.ClusterShape(G, E, 2)
        wl = h.gen_zipf_workload(shape, s, 2048, 3, seed=seed)
        totals = wl.micro_batches[0].expert_totals()
        counts = h.greedy_replica_counts(totals, E * 2, max_count=G)
        placement = h.monte_carlo_placement(totals, counts, shape, 20, seed)
        for loads in wl.micro_batches:
            rec = record(h, placement, loads)
            rec.update(s=s)
            out.append(rec)
    return out


def fam_placements(h):
    """Cayley catalogue placements the layer consumes at init (``placement.py:207-301``)."""
    out = {}
    for G in (2, 4, 8):
        for E in (8, 16, 32, 128, 256):
            try:
                pl = h.cayley_symmetric(h.ClusterShape(G, E, 2))
            except h.ConstructionError:
                continue
            out[f"G{G}_E{E}"] = pl.to_json_dict()
    for G, E in ((4, 8), (8, 8), (8, 32)):
        out[f"identical_G{G}_E{E}"] = h.identical_placement(h.ClusterShape(G, E, 2)).to_json_dict()
    return out


def fam_zipf(h):
    """gen_zipf_workload counts (``simulator.py:163-195``) for the workload generator port."""
    out = []
    for G, E, T, s, seed in ((4, 8, 2048, 1.0, 0), (8, 128, 4096, 1.5, 3), (8, 256, 1000, 0.0, 7), (2, 8, 333, 2.0, 11)):
        wl = h.gen_zipf_workload(h.ClusterShape(G, E, 2), s, T, 3, seed)
        out.append(dict(G=G, E=E, T=T, s=s, seed=seed, mbs=[[list(r) for r in mb.entries] for mb in wl.micro_batches]))
    return out


def fam_adaptive(h):
    """evaluate_and_maybe_replace decisions (adaptive.py:119-166) on zipf histories."""
    from fractions import Fraction

    out = []
    for G, E, s, seed in ((8, 8, 1.5, 0), (8, 32, 1.25, 1), (4, 16, 2.0, 2), (8, 32, 0.2, 3), (8, 128, 2.0, 4)):
        shape = h.ClusterShape(G, E, 2)
        cur = h.cayley_symmetric(shape)
        wl = h.gen_zipf_workload(shape, s, 1024, 6, seed=seed)
        hist = h.LoadHistory(4)
        for mb in wl.micro_batches:
            hist.push(h.aggregate_expert_loads(mb))
        pol = h.ReplacementPolicy(mc_samples=25)
        dec = h.evaluate_and_maybe_replace(cur, hist, pol, shape, seed)
        out.append(dict(G=G, E=E, s=s, seed=seed, history=[list(r) for r in hist.entries],
                        replaced=dec.replaced, groups=[list(g) for g in dec.placement.edp_groups],
                        slots=list(dec.placement.slots), ratio=dec.predicted_ratio,
                        old_m=[Fraction(dec.old_m).numerator, Fraction(dec.old_m).denominator],
                        new_m=None if dec.new_m is None else [Fraction(dec.new_m).numerator, Fraction(dec.new_m).denominator],
                        changed=dec.changed_slots, cost=dec.migration_cost_total))
    return out


def dump(name, obj):
    path = os.path.join(HERE, name)
    data = json.dumps(obj, separators=(",", ":")).encode()
    if name.endswith(".gz"):
        with gzip.GzipFile(path, "wb", mtime=0) as f:
            f.write(data)
    else:
        with open(path, "wb") as f:
            f.write(data)
    print(f"{name}: {len(data) / 1e3:.1f} kB raw")


def main():
    h = _import_reference()
    dump("sched_known.json", fam_known(h))
    dump("sched_random500.json.gz", fam_random500(h))
    dump("sched_baseline.json.gz", fam_baseline(h))
    dump("sched_warm100.json.gz", fam_warm100(h))
    dump("sched_base.json.gz", fam_base(h))
    dump("sched_asym.json.gz", fam_asym(h))
    dump("sched_pipelined.json.gz", fam_pipelined(h))
    dump("sweep_metrics.json.gz", fam_sweep(h))
    dump("placements.json", fam_placements(h))
    dump("zipf_counts.json.gz", fam_zipf(h))
    dump("adaptive.json", fam_adaptive(h))


if __name__ == "__main__":
    main()
