# run every gpu test in its own process (a CUDA fault is sticky per process)
for t in $(python -m pytest tests/test_gpu_parity.py -m gpu --collect-only -q 2>/dev/null | grep "::"); do
  r=$(timeout 120 python -m pytest "$t" -q -m gpu 2>&1 | tail -1)
  echo "$r  $t"
done
