# Builds an instrumented copy (TT_INSTRUMENT phase timers) into _lib_ab/instr.so
set -e
O=paper_2501_06647_b200/_lib_ab; mkdir -p $O
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -DTT_INSTRUMENT -I include"
for s in tt_leaf tt_stitch tt_host; do
  ext=cu; [ $s = tt_host ] && ext=cpp
  nvcc $F -c paper_2501_06647_b200/csrc/$s.$ext -o $O/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $O/tt_leaf.o $O/tt_stitch.o $O/tt_host.o -o $O/instr.so
