B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/$3 $B > gpurun_out/ncu_$3.log 2>&1
