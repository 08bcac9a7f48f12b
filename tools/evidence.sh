# Full bench (with CPU baseline), reference arm, launch list and --set full captures.
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 8 -c 1 -o gpurun_out/r1_stitch_query $B > gpurun_out/ncu_q.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 0 -c 1 -o gpurun_out/r1_stitch_build $B > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_als_kernel -c 1 -o gpurun_out/r1_leaf $B > gpurun_out/ncu_l.log 2>&1
./tools/_bin/fp64_probe > gpurun_out/fp64_probe.txt 2>&1
