#!/bin/bash
# Checked build (stands in for compute-sanitizer, which is closed on the GPU pool): libhedl.so
# compiled with -DHEDL_CHECKED (device bounds traps in the hot kernels, 4 KB guard zones of 0xA5
# around every device block checked at free, fresh blocks filled with 0xA5 instead of zeros),
# then every kernel family on small inputs (tools/sanitize_cases.py) and the GPU parity suites,
# all checked against the oracle.  One GPU, under gpurun; log in gpurun_out/.
mkdir -p gpurun_out
T=${TAG:-chk}
export HEDL_ALLOCATOR=cuda
NVCC_EXTRA="-DHEDL_CHECKED" python -c "import __graft_entry__ as g; g.build(force=True)" > gpurun_out/${T}_build.log 2>&1
echo "build=$?" >> gpurun_out/${T}_build.log
timeout 1200 python tools/sanitize_cases.py > gpurun_out/${T}_cases.log 2>&1; echo "cases exit=$?" >> gpurun_out/${T}_cases.log
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slice.py tests/test_gpu_dcompile.py tests/test_gpu_boundary.py tests/test_gpu_strings.py tests/test_gpu_scores.py tests/test_gpu_split.py -k "not torch_allocator" -q -x -rf > gpurun_out/${T}_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/${T}_pytest.log
