# A/B over variants for c2 and c3 (append phase focus)
for c in c2 c3; do for v in "$@"; do
  TT_LIB_PATH=paper_2501_06647_b200/_lib_ab/$v.so timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_${c}.log 2>&1
  tail -1 gpurun_out/ab_${v}_${c}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', d['value'], d['phases_ms_per_step'])" || tail -3 gpurun_out/ab_${v}_${c}.log
done; done
