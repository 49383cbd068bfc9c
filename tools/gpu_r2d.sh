# Round-2 full GPU pass: diag, all GPU tests, smoke, bench, launch list, ncu full of the top kernel.
mkdir -p gpurun_out
T=${TAG:-r2d}
timeout 300 python tools/diag_split.py > gpurun_out/${T}_diag.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-c5 --no-prof-pass"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
read TOP IDX < <(python tools/pick_launch.py gpurun_out/${T}_launches.csv)
echo "top $TOP $IDX" > gpurun_out/${T}_top.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$TOP" -s "$IDX" -c 1 -o gpurun_out/${T}_prof_top -f $B > gpurun_out/${T}_ncu_top.log 2>&1
ls -la gpurun_out
