# Evidence pass at HEAD (1 GPU): per-class DRAM traffic of one C4 and one C5 step (every launch),
# the operator micro-benchmarks (NEXT-1), then compute-sanitizer over every kernel family.
mkdir -p gpurun_out
T=${TAG:-ev}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > gpurun_out/${T}_traffic_c4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c5.csv python bench.py --workload c5 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_traffic_c5.log 2>&1
timeout 1200 python tools/opbench.py gpurun_out/${T}_opbench.json > gpurun_out/${T}_opbench.md 2> gpurun_out/${T}_opbench.err; echo opbench=$? >> gpurun_out/${T}_opbench.err
export HEDL_ALLOCATOR=cuda
for S in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $S --target-processes all --print-limit 200 \
      --log-file gpurun_out/${T}_san_$S.log python tools/sanitize_cases.py > gpurun_out/${T}_san_${S}_stdout.log 2>&1
  echo "$S exit=$?" >> gpurun_out/${T}_san_exit.log
done
ls -la gpurun_out
