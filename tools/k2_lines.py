#!/usr/bin/env python3
"""Per-line executed instructions of plan_batch_kernel from an ncu report.

    python tools/k2_lines.py gpurun_out/k2.ncu-rep [lo hi]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 10 ** 9)
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k",
                      "plan_batch_kernel"], capture_output=True, text=True, errors="replace").stdout
src = open("paper_2409_14447_b200/csrc/plan_batch.cu").read().split("\n")
fpath = hdr = None
tot = 0
rows = []
for r in csv.reader(io.StringIO(raw)):
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
    inst = float(d.get("Instructions Executed", "0") or 0)
    tot += inst
    if fpath and fpath.endswith("plan_batch.cu") and lo <= int(r[0]) <= hi and inst > 0:
        rows.append((int(r[0]), inst))
print(f"total {tot:.0f}")
for ln, inst in rows:
    print(f"{ln:5d} {inst:10.0f} {100 * inst / tot:5.1f}%  {src[ln - 1].strip()[:90]}")
