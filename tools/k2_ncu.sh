#!/bin/bash
# ncu --set full of plan_batch_kernel on the C2 bench batch -> gpurun_out/$1.ncu-rep
TAG=${1:-k2}
ncu --set full --clock-control none --import-source on -k regex:plan_thread_kernel -c 1 -f -o gpurun_out/$TAG \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-gate --no-sweep > gpurun_out/$TAG.log 2>&1
tail -1 gpurun_out/$TAG.log
