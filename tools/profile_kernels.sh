#!/bin/bash
# `ncu --set full` of the largest launch of each named kernel in one bench step (1 GPU, gpurun).
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-c5 --no-prof-pass"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
for K in "$@"; do
  read TOP IDX < <(python tools/pick_launch.py gpurun_out/launches.csv "$K")
  ncu --set full --clock-control none --import-source on -k regex:"^$TOP" -s "$IDX" -c 1 -o gpurun_out/prof_$K -f $B > gpurun_out/ncu_$K.log 2>&1
done
ls -la gpurun_out
