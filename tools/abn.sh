# A/B/..: each named .so in _lib_ab (args), alternating twice
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for rep in 1 2; do
for v in "$@"; do
  export TT_LIB_PATH=paper_2501_06647_b200/_lib_ab/$v.so
  $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], 'e2e', d['e2e']['value'], d['e2e']['append_slices_per_s'], d['phases_ms_per_step'])"
done
done
