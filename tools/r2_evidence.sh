# round-2 evidence pass: GPU suite, smoke, bench lines (default C3 stream, reference arm),
# ncu launch list of the bench + one --set full capture of each cluster kernel
O=gpurun_out/${TAG:-r2f}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -k "not sanitize" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaf_wide_kernel -s 12 -c 1 -o $O/leaf_wide $B > $O/ncu_leaf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stitch_wide_kernel -s 12 -c 1 -o $O/stitch_wide $B > $O/ncu_stitch.log 2>&1
# summaries (the .ncu-rep files are too large to bring back)
for r in leaf_wide stitch_wide; do
  [ -f $O/$r.ncu-rep ] && ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  [ -f $O/$r.ncu-rep ] && python tools/ncu_lines.py $O/$r.ncu-rep 15 > $O/${r}_lines.txt 2>&1
done
python tools/ncu_summary.py ${TAG:-r2f} $O/launches.csv "c3_stream/leaf=$O/leaf_wide.ncu-rep" "c3_stream/stitch=$O/stitch_wide.ncu-rep" > $O/summary.log 2>&1
cp profiles/${TAG:-r2f}_ncu_summary.md profiles/traffic.json $O/ 2>/dev/null
rm -f $O/*.ncu-rep
ls -la $O; tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
