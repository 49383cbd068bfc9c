mkdir -p gpurun_out
B="python bench.py --no-latency --no-c5 --no-cpu-baseline --steps 20"
for r in 1 2; do
  timeout 300 $B > gpurun_out/abg_on_$r.log 2>&1
  HEDL_NO_GRAPH=1 timeout 300 $B > gpurun_out/abg_off_$r.log 2>&1
done
