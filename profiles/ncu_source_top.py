#!/usr/bin/env python3
"""Summarise `ncu --page source --csv --print-source=cuda,sass` output:
top CUDA source lines by instructions executed and by stall samples.

    ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > src.csv
    python profiles/ncu_source_top.py src.csv [kernel-substring] [N]
"""
import csv
import sys
from collections import defaultdict


def main(path, kern="", top=30):
    rows = list(csv.reader(open(path)))
    fpath = func = None
    hdr = None
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1]; continue
        if r[0] == "Function Name":
            func = r[1]; continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr is None or not r[0].isdigit() or (kern and kern not in (func or "")):
            continue
        d = dict(zip(hdr[:2], r[:2]))
        try:
            inst = float(r[hdr.index("Instructions Executed")] or 0)
            stall = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        key = (fpath.split("/")[-1], int(r[0]))
        a = agg[key]
        a[0] += inst; a[1] += stall; a[2] = r[1][:80]
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {ti:.0f}, stall samples {ts:.0f}")
    print("-- by instructions")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{k[0]:22s}{k[1]:5d} inst {v[0]/ti*100:5.1f}% stall {v[1]/ts*100:5.1f}% | {v[2]}")
    print("-- by stall samples")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k[0]:22s}{k[1]:5d} inst {v[0]/ti*100:5.1f}% stall {v[1]/ts*100:5.1f}% | {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 30)
