# time the library variants in _lib/variants (tools/build_variant.sh) against the in-tree build
for v in base $(ls paper_2311_15061_b200/_lib/variants | sed 's/libpb200_//;s/.so//'); do
  if [ $v = base ]; then unset PB200_LIB_VARIANT; else export PB200_LIB_VARIANT=$v; fi
  echo "== $v"; timeout 200 python tools/quick_timing.py ${VAR_CFGS:-2 3} 2>&1 | grep phases
done
