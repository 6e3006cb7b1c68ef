"""Summarise an .ncu-rep (read here, on the CPU box) into a markdown table:
per kernel launch: duration, DRAM bytes, DRAM/tensor/SM utilisation."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor_hmma%"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "pipe_tc_inst%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    cols = {}
    for k, nm in KEYS:
        cands = [i for i, c in enumerate(h) if c == k or c.endswith("." + k) or c.endswith(k)]
        if cands:
            cols[nm] = cands[0]
    ki = h.index("Kernel Name")
    out = ["| kernel | " + " | ".join(cols) + " |", "|---" * (len(cols) + 1) + "|"]
    for r in rows[2:]:
        out.append("| " + r[ki][:70] + " | " + " | ".join(f"{r[i]} {units[i]}".strip() for i in cols.values()) + " |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
