"""Device simplex timing (hep_lp_solve) vs the reference's simplex_solve wall time.

Cold and warm solves of the comm-aware LP on Cayley placements (G = 8, one node) at
E = 32 / 64 (the golden cases, whose reference times were taken in the build
container) and E = 128 / 256 (device only), plus the 100 C9 topology-aware instances.
Prints one JSON line per configuration: pivots, device µs per solve (CUDA events), µs
per pivot, and the reference ms where known."""

import json
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")

import numpy as np  # noqa: E402

import paper_2511_16947_b200 as P  # noqa: E402
from conftest import load_golden  # noqa: E402


def main():
    from paper_2511_16947_b200 import _lib

    if len(sys.argv) > 1:  # e.g. "lp_dsm=0"
        k, v = sys.argv[1].split("=")
        _lib.set_tuning(**{k: int(v)})
        print(json.dumps({"tuning": {k: int(v)}}))
    G = load_golden("lp_cases.json.gz")
    ref_ms = {c["family"]: c["ref_ms"] for c in G["cases"] if c["family"].startswith("cayley")}
    c9 = [c for c in G["cases"] if c["family"] == "c9"]
    out = []
    for E in (32, 64, 128, 256):
        shape = P.ClusterShape(8, E, 2)
        pl = P.cayley_symmetric(shape)
        wl = P.gen_zipf_workload(shape, 1.0, 4096, 6, 3)
        topo = P.Topology(8, 8)
        opts = P.SolveOptions(mode=P.COMM_AWARE, alpha=0.1)
        rows = []
        state = None
        for i, loads in enumerate(wl.micro_batches):
            if state is None:
                _plan, _s, state = P.solve_comm_aware(pl, loads, topo, opts)
            else:
                _plan, state = P.warm_solve(state, loads)
            rows.append((state.stats.iterations_last, state.stats.device_us_last))
        # repeat the first (cold) solve to take it warm-GPU
        _plan, _s, st2 = P.solve_comm_aware(pl, wl.micro_batches[0], topo, opts)
        cold = (st2.stats.iterations_last, st2.stats.device_us_last)
        warm = rows[1:]
        rec = {"E": E, "lp": "comm_aware G=8 alpha=0.1", "cold_pivots": cold[0], "cold_us": round(cold[1], 1),
               "cold_us_per_pivot": round(cold[1] / max(cold[0], 1), 2),
               "warm_pivots_median": int(np.median([r[0] for r in warm])),
               "warm_us_median": round(float(np.median([r[1] for r in warm])), 1),
               "ref_ms_cold": round(ref_ms.get(f"cayley_E{E}", float("nan")), 1)}
        out.append(rec)
        print(json.dumps(rec), flush=True)
    us, piv = [], []
    for rec in c9:
        pl = P.Placement(8, tuple(tuple(g) for g in rec["groups"]), tuple(rec["slots"]))
        loads = P.LoadMatrix(tuple(tuple(r) for r in rec["loads"]))
        _p, _s, st = P.solve_comm_aware(pl, loads, P.Topology(8, 4), P.SolveOptions(
            mode=P.TOPOLOGY_AWARE, alpha_intra=0.1, alpha_inter=1.0))
        us.append(st.stats.device_us_last)
        piv.append(st.stats.iterations_last)
    rec = {"lp": "C9 topology_aware G=8 E=12 gpn=4", "n": len(us), "pivots_median": int(np.median(piv)),
           "device_us_median": round(float(np.median(us)), 1),
           "ref_ms_median": round(float(np.median([c["ref_ms"] for c in c9])), 1)}
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
