# Where the e2e host stalls come from: per-step times with HEDL_TIMING allocation / pinned
# allocation / blocking-launch notes and Python GC pauses, interleaved in one log.
mkdir -p gpurun_out
T=${TAG:-stall}
HEDL_BENCH_GCLOG=1 HEDL_TIMING=1 timeout 900 python bench.py --no-latency --no-c5 --no-cpu-baseline --no-prof-pass 2>&1 | grep -E "bench gc|cudaMallocHost|dev_malloc +[0-9]+ B +[0-9]*[1-9][0-9]*\.|launch record|^\{" > gpurun_out/${T}_log.txt
