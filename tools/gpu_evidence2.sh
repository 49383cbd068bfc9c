# Evidence pass at HEAD (1 GPU): per-class DRAM traffic of one C4 and one C5 step (every launch),
# the launch list of a C4 bench step, ncu --set full of the dominant kernel's largest launch,
# then the checked build over the kernel families and the GPU parity suites.
mkdir -p gpurun_out
T=${TAG:-ev2}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c4.csv python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > gpurun_out/${T}_traffic_c4.log 2>&1
timeout 900 ncu --metrics $M --clock-control none --cache-control none --csv --log-file gpurun_out/${T}_traffic_c5.csv python bench.py --workload c5 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_traffic_c5.log 2>&1
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-c5 --no-prof-pass"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"k_slice_tileILb1ELi2E" -s 5 -c 1 -o gpurun_out/${T}_prof_top -f $B > gpurun_out/${T}_ncu_top.log 2>&1
TAG=${T}chk bash tools/checked.sh
