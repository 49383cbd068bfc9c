#!/bin/bash
# compute-sanitizer runs over tools/sanitize_cases.py (every kernel family, results checked
# against the oracle): memcheck, racecheck (shared memory), synccheck, initcheck.
# One GPU, under gpurun; logs in gpurun_out/, summary via tools/sanitize_summary.py.
mkdir -p gpurun_out
export HEDL_ALLOCATOR=cuda     # plain cudaMalloc: the sanitizer tracks allocations itself
for T in memcheck racecheck synccheck initcheck; do
  timeout 2400 compute-sanitizer --tool $T --target-processes all --print-limit 200 \
      --log-file gpurun_out/san_$T.log python tools/sanitize_cases.py > gpurun_out/san_${T}_stdout.log 2>&1
  echo "$T exit=$?" >> gpurun_out/san_exit.log
done
