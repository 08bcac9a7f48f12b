B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for v in old new old new; do
  if [ $v = old ]; then export TT_LIB_PATH=paper_2501_06647_b200/_lib_ab/old.so; else unset TT_LIB_PATH; fi
  $B 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['phases_ms_per_step'])"
done
