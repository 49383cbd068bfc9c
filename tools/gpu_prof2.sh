# ncu --set full of one launch of each hot kernel instantiation (mangled-name regexes), 1 GPU.
mkdir -p gpurun_out
T=${TAG:-p2}
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-latency --no-c5 --no-prof-pass"
i=0
for K in "k_slice_tileILb1ELi2E" "k_slice_tileILb0ELi2E" "k_slice_heavyILb1ELi2E" "k_slice_pack" "k_bool_warp" "k_slice_exILb1E"; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$K" -s 3 -c 1 -o gpurun_out/${T}_$i -f $B > gpurun_out/${T}_$i.log 2>&1
  i=$((i+1))
done
