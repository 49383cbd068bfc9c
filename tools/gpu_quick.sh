# quick GPU check of a kernel change: the parity suites that exercise lane packs, C4 full size, bench
mkdir -p gpurun_out
T=${TAG:-q}
timeout 1200 python -m pytest tests/test_gpu_slice.py tests/test_gpu_parity.py tests/test_gpu_split.py tests/test_gpu_boundary.py tests/test_gpu_fullsize.py tests/test_gpu_dcompile.py -k "not c5 and not c3" -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --no-latency --no-c5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
HEDL_TIMING=1 timeout 300 python bench.py --no-latency --no-c5 --no-cpu-baseline --no-e2e --steps 1 --warmup 0 --no-prof-pass 2>&1 | grep "hedl plan" > gpurun_out/${T}_plan.log
if [ -n "$TRAFFIC" ]; then
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > /dev/null 2>&1
fi
