# round-2 evidence pass: GPU suite, smoke, bench lines (default C3 stream, reference arm, burst configs),
# ncu launch list of the bench + --set full captures of the streamed kernel, a solver kernel and the cluster stitch
T=${TAG:-r2i}; O=gpurun_out/$T; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
for c in c1 c2 c4; do timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1; done
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1
# the build-sized streamed pass (pass 2 of sweep 0 of the warm build: 148 CTAs over 192 leaves)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_ttm_kernel -s 1 -c 1 -o $O/grid_ttm $B > $O/ncu_ttm.log 2>&1
# a mode-1 solve of a streamed leaf (the largest solver kernel) and a [0, T) query stitch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grid_solve_mode_kernel -s 40 -c 1 -o $O/grid_solve $B > $O/ncu_solve.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stitch_wide_kernel -s 12 -c 1 -o $O/stitch_wide $B > $O/ncu_stitch.log 2>&1
for r in grid_ttm grid_solve stitch_wide; do
  [ -f $O/$r.ncu-rep ] && ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  [ -f $O/$r.ncu-rep ] && python tools/ncu_lines.py $O/$r.ncu-rep 15 > $O/${r}_lines.txt 2>&1
done
python tools/ncu_summary.py $T $O/launches.csv "c3_stream/stream_pass_build=$O/grid_ttm.ncu-rep" "c3_stream/leaf_solve_mode=$O/grid_solve.ncu-rep" "c3_stream/stitch=$O/stitch_wide.ncu-rep" > $O/summary.log 2>&1
cp profiles/${T}_ncu_summary.md profiles/traffic.json $O/ 2>/dev/null
rm -f $O/*.ncu-rep
ls -la $O; tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
