mkdir -p gpurun_out
T=${TAG:-nar}
HEDL_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 2>&1 | grep "hedl slice" > gpurun_out/${T}_slice_c4.log
C5=1 TAG=$T bash tools/ab_env.sh HEDL_NO_NARROW=1
