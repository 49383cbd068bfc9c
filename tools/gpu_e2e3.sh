mkdir -p gpurun_out
T=${TAG:-e2g}
HEDL_TIMING=1 timeout 600 python tools/time_e2e.py --no-latency --no-c5 > gpurun_out/${T}_time.log 2>&1
