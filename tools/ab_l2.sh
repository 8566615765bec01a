# A/B of dictionary-step tuning variants (scratch): bash tools/ab_l2.sh
for rep in 1 2; do
for spec in "tune:PB_DICT_FLAGS=0" "tune:PB_DICT_FLAGS=1"; do
  v=${spec%%:*}; e=${spec#*:}
  echo "== $v $e"; env PB200_LIB_VARIANT=$v $e timeout 120 python tools/sweep_timing.py 0 1 2 4 --steps 6 2>&1 | grep cfg
done; done
