# Same-box A/B of environment switches on one libhedl.so: "base" (no switch) vs each NAME=VALUE
# given, ABAB, C4 kernels-only bench (20 steps); C5=1 adds one C5 run per variant; then the GPU
# suites with the default settings.
mkdir -p gpurun_out
T=${TAG:-abe}
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-c5"
for rep in 1 2; do
  timeout 300 $B > gpurun_out/${T}_base_$rep.json 2>gpurun_out/${T}_base_$rep.err
  for v in "$@"; do n=$(echo $v | tr "=" "_"); env $v timeout 300 $B > gpurun_out/${T}_${n}_$rep.json 2>gpurun_out/${T}_${n}_$rep.err; done
done
if [ -n "$C5" ]; then
  timeout 400 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_c5base_1.json 2>/dev/null
  for v in "$@"; do n=$(echo $v | tr "=" "_"); env $v timeout 400 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_c5${n}_1.json 2>/dev/null; done
fi
if [ -z "$NOTEST" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
fi
