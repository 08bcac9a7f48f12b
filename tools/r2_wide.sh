# round-2 check of the cluster leaf kernel: GPU parity (default dispatch: wide
# for small batches), a narrow-forced subset, then the C3 streaming form.
O=gpurun_out/r2a; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
TT_WIDE=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tree or tucker" > $O/pytest_narrow.log 2>&1; echo "rc=$?" >> $O/pytest_narrow.log
timeout 600 python tools/stream_bench.py c3 1024 > $O/stream_c3.log 2>&1
timeout 600 python tools/stream_bench.py c2 2048 > $O/stream_c2.log 2>&1
tail -3 $O/*.log
