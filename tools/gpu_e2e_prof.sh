# e2e step breakdown: synchronised phase times (tools/time_e2e.py, HEDL_TIMING planner phases),
# then an ncu launch list of two e2e iterations (compile + device plan + evaluation kernels).
mkdir -p gpurun_out
T=${TAG:-e2e}
HEDL_TIMING=1 timeout 600 python tools/time_e2e.py --no-latency --no-c5 > gpurun_out/${T}_time.log 2>&1
E2E_ITERS=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/time_e2e.py --no-latency --no-c5 > gpurun_out/${T}_ncu.log 2>&1
