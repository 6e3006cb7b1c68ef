"""Solve one C9 golden LP a few times (for ncu captures of the device simplex)."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2511_16947_b200 as P  # noqa: E402
from conftest import load_golden  # noqa: E402

rec = [c for c in load_golden("lp_cases.json.gz")["cases"] if c["family"] == "c9"][0]
pl = P.Placement(8, tuple(tuple(g) for g in rec["groups"]), tuple(rec["slots"]))
loads = P.LoadMatrix(tuple(tuple(r) for r in rec["loads"]))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    _p, _s, st = P.solve_comm_aware(pl, loads, P.Topology(8, 4), P.SolveOptions(
        mode=P.TOPOLOGY_AWARE, alpha_intra=0.1, alpha_inter=1.0))
    print(st.stats.iterations_last, round(st.stats.device_us_last, 1))
