# parity + A/B on c2 + short c4/c3 bench lines; usage: tools/run_cfgs.sh <old> <new>
bash tools/check_ab.sh "$@"
for c in c4 c3; do
  timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['append'], d['phases_ms_per_step'], d['e2e']['value'], d['solver_per_step'])"
done
