"""Pin the CPU oracle (oracle/hep_oracle.c) against the reference's own outputs.

The fixtures were produced by importing the reference package
(tests/golden/make_golden.py).  The oracle restates the reference algorithm
(Dinic + min-cut probing + lex-min reroute), so beyond the outputs it must
also reproduce the reference's solver iteration counter (probes + BFS phases,
scheduler.py:383-386) — a check that the traversal order itself is restated.
"""

import pytest

from conftest import SCHED_FAMILIES, load_golden


def _compare(out, rec):
    assert list(out["m"]) == rec["m"]
    assert out["Q"] == rec["Q"]
    assert out["xq"] == rec["xq"]
    assert out["xi"] == rec["xi"]
    assert out["obj_int"] == rec["obj_int"]
    assert [list(r) for r in out["ranges"]] == rec["ranges"]
    if "ranges_topo" in rec:
        assert [list(r) for r in out["ranges_topo"]] == rec["ranges_topo"]
    for k in ("pair", "send", "recv", "local", "intra", "inter"):
        assert out[k] == rec[k], k


@pytest.mark.parametrize("family", SCHED_FAMILIES)
def test_oracle_matches_reference_fixtures(oracle_lib, family):
    recs = load_golden(family)
    assert recs
    for rec in recs:
        out = oracle_lib.full_path(rec["G"], rec["groups"], rec["loads"], rec["base"], rec["gpn"])
        _compare(out, rec)
        assert out["iters"] == rec["iters"], "Dinic traversal order diverged from the reference"


def test_oracle_pipelined_matches_reference(oracle_lib):
    """harmony_pipelined (simulator.py:420-435): the static phase's split loads,
    even-split integerized plan, GPU loads, routing and transfer, and the
    scheduled phase's gpu_base solve — all bit-exact."""
    recs = load_golden("sched_pipelined.json.gz")
    assert len(recs) >= 10
    for rec in recs:
        num, den = rec["share"]
        f, lat = oracle_lib.pipelined_path(rec["G"], rec["groups"], rec["loads"], num, den)
        ref_f = rec["former"]
        assert f["loads"] == ref_f["loads"]
        assert lat["loads"] == rec["latter"]["loads"]
        assert f["xi"] == ref_f["xi"] and f["gpu_load"] == ref_f["gpu_load"]
        assert [list(r) for r in f["ranges"]] == ref_f["ranges"]
        for k in ("pair", "send", "recv", "local"):
            assert f[k] == ref_f[k], k
        _compare(lat, rec["latter"])
        assert lat["iters"] == rec["latter"]["iters"]


def test_known_answers(oracle_lib):
    """Hand-derived answers of the reference tests (test_scheduler.py:33-69,
    test_router.py:32-151)."""
    known = {r["name"]: r for r in load_golden("sched_known.json")}
    ring4 = known["ring4"]
    out = oracle_lib.full_path(ring4["G"], ring4["groups"], ring4["loads"])
    assert out["m"] == (8, 1)
    assert out["xq"] == [[2 * 12, 2 * 12], [6 * 12, 0], [8 * 12, 6 * 12], [2 * 12, 6 * 12]]  # Q = 12
    assert out["gpu_load"] == [8, 8, 8, 8]
    ident = known["identical4"]
    assert oracle_lib.full_path(ident["G"], ident["groups"], ident["loads"])["m"] == (11, 1)
    uns = known["unsorted_group"]
    r = oracle_lib.route(uns["G"], uns["groups"], uns["loads"], [[3, 4, 2]])
    assert r == [(0, 2, 2, 3), (0, 2, 0, 4), (0, 2, 3, 2)]
    rs = known["remote_split"]
    assert oracle_lib.route(rs["G"], rs["groups"], rs["loads"], [[3, 1]]) == [(0, 2, 0, 3), (0, 2, 1, 1)]
    sn = known["same_node_first"]
    assert oracle_lib.route(sn["G"], sn["groups"], sn["loads"], [[2, 2]], gpn=2) == [(0, 0, 1, 2), (0, 0, 2, 2)]


def test_integerize_known(oracle_lib):
    """test_scheduler.py:210-227: (5/2,5/2)->(3,2); (1.2,1.2,1.6)->(1,1,2); bad totals."""
    xi, _, _ = oracle_lib.integerize(2, [(0, 1)], [[5, 5]], 2)
    assert xi == [[3, 2]]
    xi, _, _ = oracle_lib.integerize(3, [(0, 1, 2)], [[12, 12, 16]], 10)
    assert xi == [[1, 1, 2]]
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.integerize(2, [(0, 1)], [[2, 1]], 4)  # 0.5 + 0.25


def test_placement_error(oracle_lib):
    st = oracle_lib.OracleState(2, [(), (0, 1)])
    with pytest.raises(oracle_lib.OracleError) as ei:
        st.solve([[3, 0], [1, 1]])
    assert ei.value.kind == "PlacementError"
    st2 = oracle_lib.OracleState(2, [(), (0, 1)])
    assert st2.solve([[0, 0], [1, 1]])["m"] == (1, 1)


def test_warm_equals_cold_and_is_cheaper(oracle_lib):
    """Reference test_scheduler.py:188-201 and acceptance C7 (:202-219): warm
    solves reuse the flow and critical subsets, give identical plans and need
    fewer solver iterations."""
    recs = load_golden("sched_warm100.json.gz")
    st = oracle_lib.OracleState(recs[0]["G"], recs[0]["groups"])
    warm_iters = cold_iters = 0
    for rec in recs:
        warm = st.solve(rec["loads"])
        cold = oracle_lib.OracleState(rec["G"], rec["groups"]).solve(rec["loads"])
        assert warm["xq"] == cold["xq"] == rec["xq"]
        assert list(warm["m"]) == rec["m"]
        warm_iters += warm["iters"]
        cold_iters += cold["iters"]
    assert warm_iters < cold_iters
