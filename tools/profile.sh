#!/bin/bash
# Profiling recipe (run under gpurun, 1 GPU): the launch list of the bench command, then
# `ncu --set full` of the dominant kernel's largest launch plus a few other kernels.
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
read TOP IDX < <(python tools/pick_launch.py gpurun_out/launches.csv)
ncu --set full --clock-control none --import-source on -k regex:"$TOP" -s "$IDX" -c 1 -o gpurun_out/prof_top -f $B > gpurun_out/ncu_top.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_slice_tile|k_slice_ex|k_slice_heavy|k_bool" -s 30 -c 6 -o gpurun_out/prof_full -f $B > gpurun_out/ncu_full_bench.log 2>&1
ls -la gpurun_out
