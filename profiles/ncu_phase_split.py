#!/usr/bin/env python3
"""Split a kernel's executed instructions by source-line ranges (phases).

    ncu -i rep --page source --csv --print-source=cuda,sass -k KERNEL > src.csv
    python profiles/ncu_phase_split.py src.csv file.cu name:lo-hi [name:lo-hi ...]
Lines of other files (headers, intrinsics) are reported as "other:<file>".
"""
import csv
import sys
from collections import defaultdict


def main(path, fname, specs):
    ranges = []
    for sp in specs:
        name, r = sp.split(":")
        lo, hi = r.split("-")
        ranges.append((name, int(lo), int(hi)))
    rows = list(csv.reader(open(path, errors="replace")))
    fpath = None
    hdr = None
    agg = defaultdict(float)
    tot = 0.0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            inst = float(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        tot += inst
        line = int(r[0])
        key = f"other:{(fpath or '?').split('/')[-1]}"
        if fpath and fpath.endswith(fname):
            key = "unassigned"
            for name, lo, hi in ranges:
                if lo <= line <= hi:
                    key = name
                    break
        agg[key] += inst
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{k:28s} {v:12.0f} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
