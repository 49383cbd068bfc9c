mkdir -p gpurun_out
T=${TAG:-st}
HEDL_TIMING=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 2>&1 | grep "hedl slice\|hedl plan" > gpurun_out/${T}_slice_c4.log
HEDL_TIMING=1 timeout 600 python bench.py --workload c5 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency 2>&1 | grep "hedl slice\|hedl plan" > gpurun_out/${T}_slice_c5.log
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 1200 python tools/opbench.py gpurun_out/${T}_opbench.json > gpurun_out/${T}_opbench.md 2> gpurun_out/${T}_opbench.err
