# Same-box A/B of programmatic dependent launch (HEDL_NO_PDL=1 = plain launches), C4 and C5,
# then the gather micro-benchmark (32 B vs 64 B gathers) and the parity suites with PDL on.
mkdir -p gpurun_out
T=${TAG:-pdl}
B="python bench.py --no-latency --no-c5 --no-cpu-baseline --steps 20"
for r in 1 2; do
  timeout 300 $B > gpurun_out/${T}_on_$r.log 2>&1
  HEDL_NO_PDL=1 timeout 300 $B > gpurun_out/${T}_off_$r.log 2>&1
done
timeout 300 python bench.py --workload c5 --no-latency --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/${T}_c5_on.log 2>&1
HEDL_NO_PDL=1 timeout 300 python bench.py --workload c5 --no-latency --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/${T}_c5_off.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_bench tools/gather_bench.cu && timeout 300 /tmp/gather_bench > gpurun_out/${T}_gather.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
