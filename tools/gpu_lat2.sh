# Latency path A/B: polled completion (default) vs stream synchronisation (HEDL_LAT_SYNC=1).
mkdir -p gpurun_out
T=${TAG:-lat2}
for r in 1 2; do
  timeout 300 python tools/dbg_lat.py > gpurun_out/${T}_poll_$r.log 2>&1
  HEDL_LAT_SYNC=1 timeout 300 python tools/dbg_lat.py > gpurun_out/${T}_sync_$r.log 2>&1
done
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-c5 --steps 3 --warmup 3 --no-prof-pass > gpurun_out/${T}_bench.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "eval_one or latency or interp or c3 or c2 or smoke or opbench" > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_op_exists_unique.csv python tools/op_one.py exists unique 10000000 5 > gpurun_out/${T}_op1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_op_min_single.csv python tools/op_one.py min single 10000000 5 > gpurun_out/${T}_op2.log 2>&1
