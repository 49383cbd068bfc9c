#!/bin/bash
# Profiling recipe (run under gpurun): launch list + one `ncu --set full` capture of the top kernels.
set -x
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_slice_tile|k_bool|k_slice_heavy|k_slice_pack" -s 200 -c 8 -o gpurun_out/prof_full -f $B > gpurun_out/ncu_full_bench.log 2>&1
ls -la gpurun_out
