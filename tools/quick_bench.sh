#!/bin/bash
# kernel-only bench step (5 timed steps) and the per-kernel totals
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/q.json 2>gpurun_out/q.err
