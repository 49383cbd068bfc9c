mkdir -p gpurun_out
B="python bench.py --no-latency --no-c5 --no-cpu-baseline --no-e2e --steps 20"
HEDL_TIMING=1 timeout 300 python bench.py --no-latency --no-c5 --no-cpu-baseline --no-e2e --steps 1 --warmup 0 --no-prof-pass 2>&1 | grep "hedl plan" > gpurun_out/ab_plan.log
for r in 1 2; do for f in 0 8 16 24; do timeout 300 $B --eval-flags $f 2>/dev/null | tail -1 > gpurun_out/ab_f${f}_r${r}.json; done; done
