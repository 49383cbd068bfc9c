#!/bin/bash
# Same-box A/B of libhedl.so variants: ab/<name>/libhedl.so vs the in-tree build, run in
# ABAB order (kernel-only bench, 5 timed steps), then the slice parity tests per variant.
# Usage: bash tools/ab.sh name [name ...]
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-c5"
LIB=paper_2412_00802_b200/libhedl.so
cp $LIB /tmp/base.so
for rep in 1 2; do
  cp /tmp/base.so $LIB; timeout 300 $B > gpurun_out/ab_base_$rep.json 2>/dev/null
  for v in "$@"; do cp ab/$v/libhedl.so $LIB; timeout 300 $B > gpurun_out/ab_${v}_$rep.json 2>/dev/null; done
done
for v in "$@"; do
  cp ab/$v/libhedl.so $LIB
  timeout 600 python -m pytest tests/test_gpu_slice.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q > gpurun_out/ab_${v}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/ab_${v}_pytest.log
done
cp /tmp/base.so $LIB
