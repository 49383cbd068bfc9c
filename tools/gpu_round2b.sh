mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/r2c_pytest.log 2>&1; echo pytest=$? >> gpurun_out/r2c_pytest.log
timeout 900 python bench.py > gpurun_out/r2c_bench.log 2>&1; echo bench=$? >> gpurun_out/r2c_bench.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/traffic_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > gpurun_out/traffic_c4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/traffic_c5.csv python bench.py --workload c5 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency > gpurun_out/traffic_c5.log 2>&1
ls -la gpurun_out
