M=gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__occupancy_limit_warps,sm__cycles_active.avg,sm__cycles_elapsed.max,launch__grid_size,launch__waves_per_multiprocessor
for c in c3 c2; do
ncu --metrics $M --clock-control none -k regex:leaf_als -c 1 --csv python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline 2>/dev/null | grep -v "^==" | tail -12 > gpurun_out/occ_$c.csv
done
cat gpurun_out/occ_c3.csv gpurun_out/occ_c2.csv | cut -d, -f12-16
