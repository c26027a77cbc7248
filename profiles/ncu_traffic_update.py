#!/usr/bin/env python3
"""Refresh profiles/ncu_traffic.json (read by bench.py for roofline.traffic
and the issue roofline) from `ncu --set full` captures: per kernel,
dram__bytes_read/write.sum and smsp__inst_executed.sum of one launch.

    python profiles/ncu_traffic_update.py TAG rep1.ncu-rep [rep2.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "ncu_traffic.json"
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "": 1}


def kernels(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].split("<")[0].split()[-1].split("::")[-1]
        get = lambda m: float(r[hdr.index(m)].replace(",", "")) * UNITS.get(units[hdr.index(m)], 1)  # noqa: E731
        yield short, {"dram_read": int(get("dram__bytes_read.sum")), "dram_write": int(get("dram__bytes_write.sum")),
                      "warp_inst": int(get("smsp__inst_executed.sum"))}


def main(tag, paths):
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    for p in paths:
        for k, v in kernels(p):
            data[k] = v
    data["source"] = (f"profiles/{tag}_ncu_summary.txt (ncu --set full, one launch each; "
                      "warp_inst = smsp__inst_executed.sum)")
    OUT.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
