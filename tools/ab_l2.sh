# A/B of dictionary-step tuning variants (scratch): bash tools/ab_l2.sh
for spec in "tune:PB_DICT_TILE_COST=3000" "tune:PB_DICT_TILE_COST=0" "tune:PB_DICT_TILE_COST=1000" "tune:PB_DICT_TILE_COST=6000" "tune:PB_DICT_TILE_COST=12000"; do
  v=${spec%%:*}; e=${spec#*:}
  echo "== $v $e"; env PB200_LIB_VARIANT=$v $e timeout 120 python tools/sweep_timing.py 1 2 4 --steps 4 2>&1 | grep cfg
done
