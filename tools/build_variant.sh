#!/bin/bash
# Build a tuning variant of the library: tools/build_variant.sh NAME 'sed-expr' [more sed-exprs...]
# (applied to pb_compact.cu), output paper_2311_15061_b200/_lib/variants/libpb200_NAME.so.
# Variants are tuning builds (-DPB_TUNING): the PB_* A/B switches of pb_tuning.cuh are live.
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2311_15061_b200/csrc
O=$R/paper_2311_15061_b200/_lib
T=$(mktemp -d)
cp $C/*.cu $C/*.cuh $T/
for e in "$@"; do sed -i "$e" $T/pb_compact.cu; done
mkdir -p $O/variants
objs=""
for f in pb_patches pb_sweep pb_index pb_compact pb_live pb_select pb_compose_tc pb_nccl pb_entry pb_capi; do
  nvcc -DPB_TUNING -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v \
    --expt-relaxed-constexpr -I$R/include -I$C -c $T/$f.cu -o $T/$f.o 2> $T/$f.ptxas.log &
  objs="$objs $T/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $O/variants/libpb200_$name.so $objs -ldl
grep -A4 "k_dict_gramILi8ELi.*ELi8ELi1E" $T/pb_compact.ptxas.log | grep -E "spill|Used" | sed "s/^/$name: /"
rm -rf $T
