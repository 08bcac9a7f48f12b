# short bench lines for the other BASELINE configs
for c in c1 c4 c3; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | cut -c1-600
done
