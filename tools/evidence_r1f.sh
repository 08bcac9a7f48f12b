# final round-1 evidence: tests, smoke, bench + reference lines, launch list + query-kernel capture summary, configs, streaming
O=gpurun_out/r1f; mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench_default.log 2>&1
python bench.py --steps 5 --warmup 3 > $O/bench_full.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $B > $O/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 8 -c 1 -o /tmp/r1f_stitch_query $B > $O/ncu_q.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 0 -c 1 -o /tmp/r1f_stitch_build $B > $O/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:leaf_als_kernel -c 1 -o /tmp/r1f_leaf $B > $O/ncu_l.log 2>&1
python tools/ncu_summary.py r1f $O/launches.csv "stitch_als_kernel:query batch=/tmp/r1f_stitch_query.ncu-rep" "stitch_build_level1=/tmp/r1f_stitch_build.ncu-rep" "leaf_als_kernel=/tmp/r1f_leaf.ncu-rep" > $O/summary.log 2>&1
cp profiles/r1f_ncu_summary.md profiles/traffic.json $O/
for c in c1 c4 c3; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.log 2>&1
done
timeout 600 python tools/stream_bench.py c3 > $O/stream_c3.log 2>&1
ls -la $O
