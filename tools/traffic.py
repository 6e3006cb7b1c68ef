"""Per-launch DRAM traffic of the hot kernels from ncu launch lists.

    python tools/traffic.py profiles/r01/launches_<cfg>_<round>.csv ... > profiles/traffic.json

Each CSV is one `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` run of `bench.py --config <cfg> --profile`.  The
expert FFN (`hep_moe_expert_ffn` = two tile-list kernels + two grouped GEMMs) is
summed over its four launches; permute and combine are single launches.
bench.py reads the resulting JSON to fill `roofline.traffic`."""
import csv
import json
import os
import re
import sys


def launches(path):
    rows = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        d = rows.setdefault(int(r["ID"]), {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return [rows[k] for k in sorted(rows)]


def summarise(path):
    ks = launches(path)
    out = {"source": os.path.relpath(path)}
    for i, k in enumerate(ks):
        if "tile_count_kernel" in k["name"] and i + 3 < len(ks):
            trio = ks[i:i + 4]  # tile count, tile list, SwiGLU GEMM, down-projection GEMM
            out["ffn"] = {
                "bytes": sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in trio),
                "read": sum(x.get("dram__bytes_read.sum", 0) for x in trio),
                "write": sum(x.get("dram__bytes_write.sum", 0) for x in trio),
                "ns": sum(x.get("gpu__time_duration.sum", 0) for x in trio),
                "kernels": [re.sub(r"\(.*", "", x["name"]) for x in trio],
            }
            break
    for key, pat in (("permute", r"permute(_v8)?_kernel"), ("combine", r"combine(_v8)?_kernel"), ("sched", "sched_kernel"),
                     ("router_gate", r"gemm_kernel<\d+, \d+, 4,")):
        for k in ks:
            if re.search(pat, k["name"]):
                out[key] = {"bytes": k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0),
                            "ns": k.get("gpu__time_duration.sum", 0)}
                break
    return out


if __name__ == "__main__":
    res = {}
    for p in sys.argv[1:]:
        m = re.search(r"launches_([a-z0-9]+)_", os.path.basename(p))
        res[m.group(1) if m else p] = summarise(p)
    print(json.dumps(res, indent=1))
