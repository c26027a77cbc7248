#!/usr/bin/env python3
"""Split a kernel's executed instructions AND warp-stall samples by named
source ranges across files (phases of the thread-per-scenario K2).

    ncu -i rep --page source --csv --print-source=cuda,sass > src.csv
    python profiles/ncu_func_split.py src.csv file.cu:name:lo-hi [file2.cuh:name:lo-hi ...]
Lines outside every range are reported per file.
"""
import csv
import sys
from collections import defaultdict


def main(path, specs):
    ranges = []
    for sp in specs:
        f, name, r = sp.split(":")
        lo, hi = r.split("-")
        ranges.append((f, name, int(lo), int(hi)))
    rows = list(csv.reader(open(path, errors="replace")))
    fpath, hdr = None, None
    inst, stall = defaultdict(float), defaultdict(float)
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if r[0] == "Function Name" or r[0] == "" or hdr is None:
            continue
        try:
            line = int(r[0])
            i = float(r[hdr.index("Instructions Executed")])
            s = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except (ValueError, IndexError):
            continue
        key = f"other:{fpath}"
        for f, name, lo, hi in ranges:
            if f == fpath and lo <= line <= hi:
                key = name
                break
        inst[key] += i
        stall[key] += s
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    for k in sorted(inst, key=lambda k: -stall[k]):
        print(f"{k:34s} inst {inst[k] / ti * 100:5.1f}%   stall samples {stall[k] / ts * 100:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
