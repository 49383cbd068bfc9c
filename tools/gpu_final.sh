# Round-end evidence at HEAD (1 GPU): GPU tests, smoke, the default bench line, per-class DRAM
# traffic of one C4 and one C5 step, the launch list of a C4 step + ncu --set full of the
# dominant kernel, the C3 per-class breakdown, the checked build.
mkdir -p gpurun_out
T=${TAG:-fin}
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > gpurun_out/${T}_traffic_c4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c5.csv python bench.py --workload c5 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_traffic_c5.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-c5 --no-prof-pass"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_slice_tileILb1ELi2E" -s 3 -c 1 -o gpurun_out/${T}_prof_tile -f $B > gpurun_out/${T}_ncu_tile.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_slice_tileILb1ELi1E" -s 3 -c 1 -o gpurun_out/${T}_prof_tile_narrow -f $B > gpurun_out/${T}_ncu_tile_narrow.log 2>&1
timeout 600 python tools/dbg_c3.py > gpurun_out/${T}_c3.log 2>&1
TAG=${T}chk bash tools/checked.sh
