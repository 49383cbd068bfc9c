#!/bin/bash
# A/B of the bench (kernel + e2e legs) between the in-tree libhedl.so and ab_old/libhedl.so
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-latency"
timeout 400 $B > gpurun_out/ab_new1.json 2>/dev/null
cp paper_2412_00802_b200/libhedl.so /tmp/new.so; cp ab_old/libhedl.so paper_2412_00802_b200/libhedl.so
timeout 400 $B > gpurun_out/ab_old.json 2>/dev/null
cp /tmp/new.so paper_2412_00802_b200/libhedl.so
timeout 400 $B > gpurun_out/ab_new2.json 2>/dev/null
