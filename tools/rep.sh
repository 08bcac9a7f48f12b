B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
for v in 1 2 3; do
  $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['append']['value'], d['phases_ms_per_step'], d['e2e']['value'])"
done
