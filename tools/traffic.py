"""Per-launch DRAM traffic of the hot kernels from ncu launch lists.

    python tools/traffic.py [--tracked=profiles/<round>] launches_<cfg>_<round>.csv ... > profiles/traffic.json

Each CSV is one `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` run of `bench.py --config <cfg> --profile`.  The
expert FFN (`hep_moe_expert_ffn` = its tile-list kernels + grouped GEMMs: 4 launches, 8
with the light-expert split) is summed from the first tile-list kernel up to the combine; permute and combine are single launches.
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


def summarise(path, tracked_dir=None):
    ks = launches(path)
    # the launch lists are copied into profiles/<round>/ (tracked); record that path
    out = {"source": os.path.join(tracked_dir, os.path.basename(path)) if tracked_dir else os.path.relpath(path)}
    for i, k in enumerate(ks):
        if "tile_count_kernel" in k["name"]:
            # hep_moe_expert_ffn: its tile-list kernels and grouped GEMMs (two, or four with the
            # light-expert 1-CTA pair), up to the combine that follows
            grp = []
            for x in ks[i:]:
                if re.search(r"combine", x["name"]):
                    break
                grp.append(x)
            if not any(re.search(r"gemm(2sm)?_kernel", x["name"]) for x in grp) or not re.search(
                    r"combine", " ".join(x["name"] for x in ks[i + len(grp):i + len(grp) + 1])):
                break  # launch list cut before the FFN ended: no FFN entry
            out["ffn"] = {
                "bytes": sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in grp),
                "read": sum(x.get("dram__bytes_read.sum", 0) for x in grp),
                "write": sum(x.get("dram__bytes_write.sum", 0) for x in grp),
                "ns": sum(x.get("gpu__time_duration.sum", 0) for x in grp),
                "kernels": [re.sub(r"\(.*", "", x["name"]) for x in grp],
            }
            break
    for key, pat in (("permute", r"permute(_v8)?_kernel"), ("combine", r"combine(_v8)?_kernel"), ("sched", "sched_kernel"),
                     ("router_gate", r"gemm_kernel<\d+, \d+, 4,|gemm2sm_kernel<\d+, 4,")):
        for k in ks:
            if re.search(pat, k["name"]):
                out[key] = {"bytes": k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0),
                            "ns": k.get("gpu__time_duration.sum", 0)}
                break
    return out


if __name__ == "__main__":
    res = {}
    args = sys.argv[1:]
    tracked = None
    if args and args[0].startswith("--tracked="):
        tracked = args.pop(0).split("=", 1)[1]
    for p in args:
        m = re.search(r"launches_([a-z0-9]+)_", os.path.basename(p))
        res[m.group(1) if m else p] = summarise(p, tracked)
    print(json.dumps(res, indent=1))
