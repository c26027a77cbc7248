#!/bin/bash
# quick GPU iteration: parity tests + bench summary (used with gpurun)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4
timeout 500 python bench.py --no-cpu "$@" > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -2 gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print("C2 value %.3e scen/s  step %.1f us  kernel %.1f us  e2e %.3e  clocks %s" % (
    d["value"], d["ms_per_step"] * 1e3, d["kernel_ms_per_step"] * 1e3, d["e2e"]["value"], d["clocks"]))
s = d.get("configurator_sweep")
if s:
    print("C3 sweep %.1f us  frac %.3f  parity %s" % (s["ms_per_launch"] * 1e3, s["roofline"]["frac"],
                                                      s["parity_vs_oracle_first_1000"]))
PY
