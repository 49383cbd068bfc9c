mkdir -p gpurun_out
T=${TAG:-gcf}
for r in 1 2; do
HEDL_BENCH_GCLOG=1 timeout 900 python bench.py --no-latency --no-c5 --no-cpu-baseline --no-prof-pass > gpurun_out/${T}_bench_$r.log 2> gpurun_out/${T}_err_$r.log
done
