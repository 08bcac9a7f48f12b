# Builds a variant of the engine into paper_2501_06647_b200/_lib_ab/<name>.so with extra
# nvcc flags (A/B runs via TT_LIB_PATH), e.g. tools/build_variant.sh instr "-DTT_INSTRUMENT"
# usage: tools/build_variant.sh <name> "<extra flags>"
set -e
O=paper_2501_06647_b200/_lib_ab/$1; mkdir -p $O
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I include $2"
objs=""
for f in paper_2501_06647_b200/csrc/*.cu paper_2501_06647_b200/csrc/tt_host.cpp; do
  b=$(basename $f); o=$O/${b%.*}.o; objs="$objs $o"
  nvcc $F -c $f -o $o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs -o paper_2501_06647_b200/_lib_ab/$1.so
