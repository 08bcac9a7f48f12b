# round-2 check: full GPU suite (incl. sanitizers), then the streaming bench line
O=gpurun_out/${TAG:-r2c}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -k "not sanitize" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > $O/bench_c3s.log 2>&1; echo "rc=$?" >> $O/bench_c3s.log
tail -5 $O/pytest_gpu.log; tail -c 2500 $O/bench_c3s.log
