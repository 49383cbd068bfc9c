#!/bin/bash
# Where k_slice_tile's time goes: the bench step with parts of the sweep disabled
# (HEDL_DBG_TILE bits: 1 = no light rows, 2 = no medium rows, 4 = no transpose-back;
# results are wrong with any bit set -- timing only; the switches exist only in a library built
# with NVCC_EXTRA=-DHEDL_DEBUG_TILE), then one `ncu --set full` capture.
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-latency"
for D in 0 1 2 3 4 7; do HEDL_DBG_TILE=$D timeout 300 $B > gpurun_out/dbg$D.json 2>/dev/null; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_slice_tile" -s 10 -c 1 -o gpurun_out/prof_tile -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/ncu_tile.log 2>&1
