# round-2: streaming C3 bench line (default) + reference arm
O=gpurun_out/r2b; mkdir -p $O
timeout 900 python bench.py --steps 8 --warmup 3 > $O/bench_c3s.log 2>&1; echo "rc=$?" >> $O/bench_c3s.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; echo "rc=$?" >> $O/bench_ref.log
tail -c 3000 $O/*.log
