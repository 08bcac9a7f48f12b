# A/B with full logs: each named .so in _lib_ab, alternating twice
for rep in 1 2; do
for v in "$@"; do
  TT_LIB_PATH=paper_2501_06647_b200/_lib_ab/$v.so python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], 'e2e', d['e2e']['value'], d['e2e']['append_slices_per_s'], d['phases_ms_per_step'])" || tail -5 gpurun_out/ab_$v.log
done
done
