#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration per launch) and an optional
`ncu --set full` report into a markdown file for profiles/.

    python scripts/ncu_summary.py gpurun_out/r01a/launches.csv [gpurun_out/r01a/prof.ncu-rep] > profiles/x.md
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name.replace("void ", ""))
    m = re.search(r"gemm3xtf32_kernel<([^>]*)>", name)
    if m:
        return "gemm3xtf32<" + m.group(1) + ">"
    return name.split("::")[-1][:60]


def launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], float(r["Metric Value"])))
    return rows


def main():
    lpath = sys.argv[1]
    rows = launches(lpath)
    agg = collections.OrderedDict()
    for name, grid, blk, ns in rows:
        a = agg.setdefault(name, [0, 0.0, grid, blk])
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values()) or 1.0
    print(f"## Launch list ({lpath}; {len(rows)} launches, cold-cache serialised — compare shares)\n")
    print("| kernel | launches | total us | mean us | share | grid | block |")
    print("|---|---|---|---|---|---|---|")
    for name, (cnt, ns, grid, blk) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {cnt} | {ns / 1e3:.1f} | {ns / cnt / 1e3:.1f} | {ns / tot:.3f} | {grid} | {blk} |")
    if len(sys.argv) > 2:
        rep = sys.argv[2]
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(out)))
        if len(rr) > 2:
            hdr, units = rr[0], rr[1]
            want = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM rd"),
                    ("dram__bytes_write.sum", "DRAM wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
                    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
                    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
                    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
                    ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
            idx = [(hdr.index(k), lab) for k, lab in want if k in hdr]
            print(f"\n## Full capture ({rep})\n")
            print("| kernel | " + " | ".join(f"{lab} [{units[i]}]" if units[i] else lab for i, lab in idx) + " |")
            print("|---" * (len(idx) + 1) + "|")
            ki = hdr.index("Kernel Name")
            for row in rr[2:]:
                print(f"| {short(row[ki])} | " + " | ".join(row[i] for i, _ in idx) + " |")


if __name__ == "__main__":
    main()
