#!/bin/bash
# A/B of the device-path K2 kernels (tile vs warp) on the C2 bench batch: bench line + ncu
python bench.py --no-cpu --no-extra --no-sweep --steps 200 --warmup 20 > gpurun_out/ab_tile.json 2>/dev/null
PARVA_K2_DEVICE_WARP=1 python bench.py --no-cpu --no-extra --no-sweep --steps 200 --warmup 20 > gpurun_out/ab_warp.json 2>/dev/null
python - <<'PY'
import json
for m in ("tile", "warp"):
    d = json.load(open(f"gpurun_out/ab_{m}.json"))
    print(m, "value %.3e  kernel %.1f us  parity %s" % (d["value"], d["kernel_ms_per_step"] * 1e3, d["parity_vs_oracle_first_2000"]))
PY
ncu --set full --clock-control none --import-source on -k regex:plan_warp_kernel -c 1 -f -o gpurun_out/k2_warp \
  env PARVA_K2_DEVICE_WARP=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-sweep > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:plan_batch_kernel -c 1 -f -o gpurun_out/k2_tile \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-sweep > /dev/null 2>&1
