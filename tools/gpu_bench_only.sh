mkdir -p gpurun_out
T=${TAG:-fb}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo bench=$? >> gpurun_out/${T}_bench.log
