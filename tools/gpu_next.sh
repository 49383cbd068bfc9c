mkdir -p gpurun_out
T=${TAG:-nx}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
NOTEST=1 C5=1 TAG=${T}ab bash tools/ab_env.sh HEDL_NO_DRANGE_MULTI=1
HEDL_TIMING=1 timeout 600 python tools/time_e2e.py --no-latency --no-c5 2>&1 | grep -v dev_malloc > gpurun_out/${T}_time.log
timeout 900 python bench.py --no-latency --no-cpu-baseline --no-c5 > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
