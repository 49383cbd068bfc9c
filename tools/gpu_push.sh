mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "push or c3 or latency or golden or c1" -q -rf > gpurun_out/push_pytest.log 2>&1; echo pytest=$? >> gpurun_out/push_pytest.log
python tools/dbg_push.py > gpurun_out/push_dbg.log 2>&1
timeout 600 python - > gpurun_out/push_c3.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench, paper_2412_00802_b200 as hedl
print(json.dumps(bench.c3_latency(hedl, 0, '/tmp/hedl_cache')))
PY
timeout 600 python tools/dbg_c3.py > gpurun_out/push_c3_classes.log 2>&1
