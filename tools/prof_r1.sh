set -x
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --queries 300"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 8 -c 1 -o gpurun_out/prof_stitch $B > gpurun_out/ncu_stitch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_als_kernel -c 1 -o gpurun_out/prof_leaf $B > gpurun_out/ncu_leaf.log 2>&1
ls -la gpurun_out
