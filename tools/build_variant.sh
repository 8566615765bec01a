#!/bin/bash
# Build a tuning variant of the library: tools/build_variant.sh NAME 'sed-expr' [more sed-exprs...]
# (applied to pb_compact.cu), output paper_2311_15061_b200/_lib/variants/libpb200_NAME.so
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2311_15061_b200/csrc
O=$R/paper_2311_15061_b200/_lib
T=$(mktemp -d)
cp $C/*.cu $C/*.cuh $T/
for e in "$@"; do sed -i "$e" $T/pb_compact.cu; done
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr -I$R/include -I$C -c $T/pb_compact.cu -o $T/pb_compact.o 2> $T/ptxas.log
objs=""
for f in pb_patches pb_sweep pb_index pb_live pb_compose_tc pb_nccl pb_capi; do objs="$objs $O/$f.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $O/variants/libpb200_$name.so $objs $T/pb_compact.o -ldl
grep -A4 "k_dict_gramILi8ELi.*ELi8ELi1E" $T/ptxas.log | grep -E "spill|Used" | sed "s/^/$name: /"
rm -rf $T
