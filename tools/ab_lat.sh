# Same-box A/B of the latency path (C2/C3 through hedl_eval_one): in-tree lib vs ab/<v>, ABAB,
# then the per-node parity tests on the in-tree lib.
mkdir -p gpurun_out
T=${TAG:-abl}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-c5 --no-cpu-baseline --no-prof-pass"
LIB=paper_2412_00802_b200/libhedl.so
cp $LIB /tmp/new.so
for rep in 1 2; do
  cp /tmp/new.so $LIB; timeout 600 $B > gpurun_out/${T}_new_$rep.json 2>/dev/null
  for v in "$@"; do cp ab/$v/libhedl.so $LIB; timeout 600 $B > gpurun_out/${T}_${v}_$rep.json 2>/dev/null; done
done
cp /tmp/new.so $LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_opbench.py tests/test_gpu_fullsize.py -q -rf -k "not c4 and not c5" > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$? >> gpurun_out/${T}_pytest.log
timeout 900 python tools/opbench.py gpurun_out/${T}_opbench.json > gpurun_out/${T}_opbench.md 2> gpurun_out/${T}_opbench.err
