#!/usr/bin/env python
"""Summarise ncu --set full reports (one launch each) into a markdown table.

    python scripts/ncu_summary.py gpurun_out/prof2/*.ncu-rep > profiles/r01/kernels_ncu.md
    python scripts/ncu_summary.py gpurun_out/prof2/*_raw.csv    # `--page raw --csv` exports
"""
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("time_ms", "gpu__time_duration.sum", 1e-6, "ns"),
    ("dram_read_GB", "dram__bytes_read.sum", None, None),
    ("dram_write_GB", "dram__bytes_write.sum", None, None),
    ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1, None),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1, None),
    ("fma_pipe_%", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1, None),
    ("fp64_pipe_%", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1, None),
    ("alu_pipe_%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1, None),
    ("xu_pipe_%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1, None),
    ("lsu_pipe_%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1, None),
    ("l1_hit_%", "l1tex__t_sector_hit_rate.pct", 1, None),
    ("l2_hit_%", "lts__t_sector_hit_rate.pct", 1, None),
    ("regs", "launch__registers_per_thread", 1, None),
    ("warps_active_%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1, None),
]


def to_gb(val, unit):
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
    return val * scale.get(unit, 1e-9)


def main():
    rows = []
    for path in sys.argv[1:]:
        if path.endswith(".csv"):
            out = open(path).read()
        else:
            out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                                 capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(out)))
        if len(r) < 3:
            continue
        hdr, units, vals = r[0], r[1], r[2]
        d = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        name = os.path.basename(path).replace(".ncu-rep", "").replace("_raw.csv", "")
        kern = d.get("Kernel Name", ("", "?"))[1][:60]
        row = {"case": name, "kernel": kern}
        for label, key, mult, _ in METRICS:
            if key not in d:
                row[label] = "-"
                continue
            u, v = d[key]
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                row[label] = v
                continue
            if label == "time_ms":
                x = x * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                         "nsecond": 1e-6}.get(u, 1.0)
            elif label.endswith("_GB"):
                x = to_gb(x, u)
            row[label] = f"{x:.4g}"
        rows.append(row)
    cols = ["case", "kernel"] + [m[0] for m in METRICS]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for row in rows:
        print("| " + " | ".join(str(row.get(c, "")) for c in cols) + " |")


if __name__ == "__main__":
    main()
