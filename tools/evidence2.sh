B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 0 -c 1 -o gpurun_out/r1_stitch_build $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_als_kernel -c 1 -o gpurun_out/r1_leaf $B > gpurun_out/ncu_l.log 2>&1
