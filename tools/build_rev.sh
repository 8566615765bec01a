#!/bin/bash
# Build the production library of a git revision for same-box A/B runs:
# tools/build_rev.sh REV NAME -> paper_2311_15061_b200/_lib/variants/libpb200_NAME.so
# (select it with PB200_LIB_VARIANT=NAME).
set -e
rev=$1; name=$2
R=$(cd "$(dirname "$0")/.." && pwd)
O=$R/paper_2311_15061_b200/_lib
T=$(mktemp -d)
git -C $R archive $rev paper_2311_15061_b200/csrc include | tar -x -C $T
C=$T/paper_2311_15061_b200/csrc
mkdir -p $O/variants
objs=""
for f in $C/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I$T/include -I$C -c $f -o $T/$b.o &
  objs="$objs $T/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $O/variants/libpb200_$name.so $objs -ldl
rm -rf $T
