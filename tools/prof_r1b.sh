B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --queries 300"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 8 -c 1 -o gpurun_out/prof_stitch_q $B > gpurun_out/ncu_q.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 0 -c 1 -o gpurun_out/prof_stitch_b $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_als_kernel -c 1 -o gpurun_out/prof_leaf2 $B > gpurun_out/ncu_l.log 2>&1
