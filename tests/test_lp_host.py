"""Host side of the communication-aware scheduling modes (CPU only).

The LP builders (``scheduler._comm_aware_lp`` / ``_topology_aware_lp``) must emit the
reference's matrices byte for byte -- same variables, same row order -- because the
device simplex's pivot sequence (Bland's rule) depends on the indices.  Pinned to the
SHA-256 of the reference's own matrices (tests/golden/make_golden_lp.py; reference
scheduler.py:480-619).  ``CommPlanStats.from_plan`` is checked on the reference's plans
(scheduler.py:97-135)."""

import numpy as np
import pytest

from conftest import load_golden

P = pytest.importorskip("paper_2511_16947_b200")
from paper_2511_16947_b200 import scheduler as S  # noqa: E402



def _lp_sha(lp):
    import hashlib

    h = hashlib.sha256()
    for a in (lp.c, lp.a_eq, lp.b_eq, lp.a_ub, lp.b_ub):
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _instance(rec):
    pl = P.Placement(rec["G"], tuple(tuple(g) for g in rec["groups"]), tuple(rec["slots"]))
    loads = P.LoadMatrix(tuple(tuple(r) for r in rec["loads"]))
    return pl, loads, P.Topology(rec["G"], rec["gpn"])


def _all_cases():
    d = load_golden("lp_cases.json.gz")
    return d["cases"] + [r for seq in d["warm"] for r in seq]


def test_lp_builders_match_reference_matrices():
    n = 0
    for rec in _all_cases():
        pl, loads, topo = _instance(rec)
        if rec["mode"] == S.COMM_AWARE:
            lp, _ = S._comm_aware_lp(pl, loads, rec["alpha"])
        else:
            lp, _ = S._topology_aware_lp(pl, loads, topo, rec["alpha_intra"], rec["alpha_inter"])
        assert [lp.c.size, lp.b_eq.size, lp.b_ub.size] == rec["lp_shape"], rec["family"] if "family" in rec else ""
        assert _lp_sha(lp) == rec["lp_sha"]
        n += 1
    assert n >= 160


def test_comm_plan_stats_on_reference_plans():
    for rec in load_golden("lp_cases.json.gz")["cases"]:
        pl, loads, _ = _instance(rec)
        plan = P.ReplicaLoadPlan(rec["G"], pl.edp_groups,
                                 tuple(tuple(float.fromhex(v) for v in row) for row in rec["plan"]), 0)
        st = S.CommPlanStats.from_plan(pl, loads, plan)
        for k in ("send", "recv", "local"):
            assert [float(v) for v in getattr(st, k)] == [float.fromhex(v) for v in rec["stats"][k]]
        assert float(st.comp) == float.fromhex(rec["stats"]["comp"])
        assert float(st.comm) == float.fromhex(rec["stats"]["comm"])


def test_comm_mode_validation():
    with pytest.raises(P.ContractViolation):
        P.SolveOptions(mode=P.COMM_AWARE, alpha=-1.0)
    with pytest.raises(P.ContractViolation):
        P.SolveOptions(mode=P.TOPOLOGY_AWARE, alpha_intra=2.0, alpha_inter=1.0)
    pl = P.Placement(2, ((0, 1),), (0,))
    loads = P.LoadMatrix(((4, 0),))
    with pytest.raises(P.ContractViolation):
        P.solve_comm_aware(pl, loads, P.Topology(2, 2), P.SolveOptions())
    with pytest.raises(P.DimensionError):
        P.solve_comm_aware(pl, loads, P.Topology(4, 2), P.SolveOptions(mode=P.COMM_AWARE))
