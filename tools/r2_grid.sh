# grid-wide leaf path check: its parity tests, leaf-path A/B timings, then the default bench with A/B of TT_GRID
O=gpurun_out/${TAG:-grid}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_grid.py -x -q > $O/pytest_grid.log 2>&1; echo "rc=$?" >> $O/pytest_grid.log
tail -6 $O/pytest_grid.log
python tools/leaf_stats.py c3 64 2>&1 | tee $O/leaf_stats.log | cut -c1-60
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
TT_GRID=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_grid1.log 2>&1
python - <<'PY'
import json,sys,os
for f in ("bench.log","bench_grid1.log"):
    try:
        l=[x for x in open(os.path.join("gpurun_out",os.environ.get("TAG","grid"),f)) if x.startswith("{")][-1]
        d=json.loads(l); print(f, d["value"], d["e2e"]["value"], d["build"], d["phases_ms_per_step"], d["gpu_launches"])
    except Exception as e: print(f, "ERR", e)
PY
