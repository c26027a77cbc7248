#!/usr/bin/env python3
"""Summarise an ncu report: per kernel duration, DRAM bytes, throughputs,
occupancy and the top stall reasons; and a launch list (--csv log) by kernel.

    python profiles/ncu_summary.py report.ncu-rep [launches.csv]
"""
import collections
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"== {name}")
        for w in WANT:
            if w in hdr:
                print(f"   {w:62s} {r[hdr.index(w)]:>16s} {units[hdr.index(w)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("   top stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print("== launch list (ncu, serialised, cold cache): kernel, launches, mean, share of GPU time")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"   {k:60s} n={len(v):4d} mean={sum(v) / len(v) / 1000:9.2f} us share={sum(v) / tot * 100:5.1f}%")


if __name__ == "__main__":
    report(sys.argv[1])
    if len(sys.argv) > 2:
        launches(sys.argv[2])
