# full capture of one query-batch stitch launch + one level-1 build stitch; exports source/raw pages
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:stitch_als_kernel -s 8 -c 1 -o /tmp/q_cur $B > gpurun_out/ncu_q.log 2>&1
ncu -i /tmp/q_cur.ncu-rep --page source --csv --print-source cuda,sass | gzip > gpurun_out/q_cur_source.csv.gz
ncu -i /tmp/q_cur.ncu-rep --page raw --csv | gzip > gpurun_out/q_cur_raw.csv.gz
cp /tmp/q_cur.ncu-rep gpurun_out/
ls -la gpurun_out | tail -4
