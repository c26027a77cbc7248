#!/bin/bash
# KG iteration on the GPU box: general-path parity tests, phase cycles, C5 time
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "alloc or c5 or broad_fuzz or reconfigure or fixture or fuzz_plans or propose or mapped_fuzz" 2>&1 | tail -2
timeout 300 python tools/kg_prof.py run 2>&1 | tail -2
timeout 300 python tools/c5_phases.py 2>&1 | tail -2
