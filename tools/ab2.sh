# Same-box A/B: the in-tree libhedl.so ("new") vs ab/<v>/libhedl.so, ABAB, C4 kernels-only bench
# (20 steps); then the GPU suites on "new"; then (CHECKED=1) the checked build over the cases.
mkdir -p gpurun_out
T=${TAG:-ab2}
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-c5"
LIB=paper_2412_00802_b200/libhedl.so
cp $LIB /tmp/new.so
for rep in 1 2; do
  cp /tmp/new.so $LIB; timeout 300 $B > gpurun_out/${T}_new_$rep.json 2>/dev/null
  for v in "$@"; do cp ab/$v/libhedl.so $LIB; timeout 300 $B > gpurun_out/${T}_${v}_$rep.json 2>/dev/null; done
done
cp /tmp/new.so $LIB
if [ -n "$C5" ]; then
  for v in "$@"; do cp ab/$v/libhedl.so $LIB; timeout 300 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_c5_${v}.json 2>/dev/null; done
  cp /tmp/new.so $LIB; timeout 300 python bench.py --workload c5 --steps 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/${T}_c5_new.json 2>/dev/null
fi
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
if [ -n "$CHECKED" ]; then TAG=${T}chk bash tools/checked.sh; fi
