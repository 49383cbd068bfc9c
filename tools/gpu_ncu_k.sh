# one ncu --set full capture of named kernels in the C4 step (KERNELS = regex, COUNT = launches)
mkdir -p gpurun_out
T=${TAG:-k}
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:${KERNELS}" -c ${COUNT:-2} -o gpurun_out/${T} -f \
  python bench.py --workload c4 --steps 1 --warmup 0 --no-prof-pass --no-e2e --no-cpu-baseline --no-latency --no-c5 > gpurun_out/${T}_ncu.log 2>&1
echo ncu=$? >> gpurun_out/${T}_ncu.log
