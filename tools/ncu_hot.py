"""Top stall-sampled SASS instructions of one kernel in an .ncu-rep
(needs -lineinfo + --import-source at capture).  Usage:
    python tools/ncu_hot.py rep.ncu-rep <kernel-regex> [N] [skip]   (skip: matching launches to skip)"""
import csv
import io
import subprocess
import sys


def main(rep, kern, n=30, skip=0):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--launch-skip", str(skip), "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[1]
    si = h.index("Warp Stall Sampling (All Samples)")
    ei = h.index("Instructions Executed")
    data = []
    for r in rows[2:]:
        try:
            data.append((float(r[si]), int(float(r[ei] or 0)), r[0], r[1].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"total samples {tot:.0f}, instructions {len(data)}")
    for s, ex, addr, src in sorted(data, reverse=True)[:n]:
        print(f"{s:7.0f} {100 * s / tot:5.1f}%  exec={ex:8d}  {addr[-5:]}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30, int(sys.argv[4]) if len(sys.argv) > 4 else 0)
