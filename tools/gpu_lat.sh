mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dcompile.py -q -k "latency or c2 or golden or c1 or tail or random_tiny" > gpurun_out/lat_pytest.log 2>&1; echo pytest=$? >> gpurun_out/lat_pytest.log
python tools/dbg_lat.py > gpurun_out/lat_dbg.log 2>&1
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench, paper_2412_00802_b200 as hedl
print(json.dumps(bench.c2_latency(hedl, 0)))" > gpurun_out/lat_c2.log 2>&1
