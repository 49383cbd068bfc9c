mkdir -p gpurun_out
T=${TAG:-dfs}
timeout 1500 python -m pytest tests/test_gpu_slice.py tests/test_gpu_dcompile.py tests/test_gpu_fullsize.py -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
HEDL_TIMING=1 timeout 600 python tools/time_e2e.py --no-latency --no-c5 2>&1 | grep -v dev_malloc > gpurun_out/${T}_time.log
timeout 900 python bench.py --no-latency --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
