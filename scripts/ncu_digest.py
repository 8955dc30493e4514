#!/usr/bin/env python
"""Digest of one ncu report: headline metrics, stall shares, SASS opcode mix.

    python scripts/ncu_digest.py report.ncu-rep [per_unit_divisor]
"""
import collections
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def page(rep, name, extra=()):
    out = subprocess.run([NCU, "-i", rep, "--page", name, "--csv", *extra], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
    r = page(rep, "raw")
    d = dict(zip(r[0], r[2]))
    print("kernel:", d.get("Kernel Name", "")[:100])
    for k in ("gpu__time_duration.sum", "launch__registers_per_thread",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "smsp__inst_executed.sum"):
        print(f"  {k} = {d.get(k)}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st.append((float(v), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1.0
    print("  stalls %:", ", ".join(f"{k} {100 * x / tot:.1f}" for x, k in sorted(st, reverse=True)[:9]))
    s = page(rep, "source", ["--print-source", "sass"])
    h = s[1]
    iE, iS = h.index("Instructions Executed"), h.index("Source")
    ops = collections.Counter()
    tot = 0
    for row in s[2:]:
        if len(row) < len(h):
            continue
        n = int(row[iE] or 0)
        tot += n
        t = row[iS].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += n
    print(f"  warp instructions {tot}" + (f", lane-instructions per unit {32 * tot / div:.1f}" if div else ""))
    print("  ", ", ".join(f"{op} {32 * n / div:.1f}" if div else f"{op} {n}"
                          for op, n in ops.most_common(24)))


if __name__ == "__main__":
    main()
