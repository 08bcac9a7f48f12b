# grid-wide leaf path check: parity tests (grid, golden), leaf-path A/B timings, the default bench, instrumented phase stats
O=gpurun_out/${TAG:-grid}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_golden.py -x -q > $O/pytest_grid.log 2>&1; echo "rc=$?" >> $O/pytest_grid.log
tail -6 $O/pytest_grid.log
python tools/leaf_stats.py c3 64 2>&1 | tee $O/leaf_stats.log | cut -c1-60
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
python - <<'PY'
import json,sys,os
for f in ("bench.log",):
    try:
        l=[x for x in open(os.path.join("gpurun_out",os.environ.get("TAG","grid"),f)) if x.startswith("{")][-1]
        d=json.loads(l); print(f, d["value"], d["e2e"]["value"], d["build"], d["phases_ms_per_step"], d["gpu_launches"])
    except Exception as e: print(f, "ERR", e)
PY
if [ -f paper_2501_06647_b200/_lib_ab/instr.so ]; then
  TT_LIB_PATH=$PWD/paper_2501_06647_b200/_lib_ab/instr.so python tools/stream_stats.py c3 128 2>&1 | tee $O/stream_stats_instr.log
fi
