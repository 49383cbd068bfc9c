#!/bin/bash
# C2/C3 latency legs: in-tree library vs ab/<name>/libhedl.so (same box)
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
LIB=paper_2412_00802_b200/libhedl.so
cp $LIB /tmp/base.so
timeout 900 $B > gpurun_out/c3_base.json 2>/dev/null
cp ab/$1/libhedl.so $LIB; timeout 900 $B > gpurun_out/c3_$1.json 2>/dev/null
cp /tmp/base.so $LIB
