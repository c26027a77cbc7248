#!/bin/bash
# One GPU round: parity tests, smoke, bench lines (driver config + default) and
# the reference arm, launch list, ncu --set full captures of the top kernels.
#   usage: bash tools/gpu_round.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke exit $?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench20.json 2> gpurun_out/${TAG}_bench20.err; echo "bench20 exit $?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2>gpurun_out/${TAG}_bench_ref.err; echo "ref exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu --no-extra --no-gate > gpurun_out/${TAG}_ncu_launch_bench.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'plan_thread_kernel' \
  -c 1 -f -o gpurun_out/${TAG}_full_k2 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-gate --no-sweep > gpurun_out/${TAG}_ncu_full_k2.log 2>&1; echo "ncu k2 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'plan_thread_kernel' -s 1 -c 1 -f \
  -o gpurun_out/${TAG}_full_k2_c4 python tools/c5_c4_prof.py c4 > gpurun_out/${TAG}_ncu_full_k2_c4.log 2>&1; echo "ncu k2 c4 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'plan_warp_kernel' \
  -c 1 -f -o gpurun_out/${TAG}_full_k2s python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-gate --no-sweep > gpurun_out/${TAG}_ncu_full_k2s.log 2>&1; echo "ncu k2s exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'configure_sweep_kernel' \
  -c 1 -f -o gpurun_out/${TAG}_full_k1 python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-gate > gpurun_out/${TAG}_ncu_full_k1.log 2>&1; echo "ncu k1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'plan_general_kernel' -c 1 -f \
  -o gpurun_out/${TAG}_full_kg python tools/c5_c4_prof.py c5 > gpurun_out/${TAG}_ncu_full_kg.log 2>&1; echo "ncu kg exit $?"
ls gpurun_out | grep ${TAG}
