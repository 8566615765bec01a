export PB200_LIB_VARIANT=tune
for e in "" "PB_DICT_W_EVICT=1" "PB_L2_PERSIST_MB=90" "PB_DICT_W_EVICT=1 PB_L2_PERSIST_MB=90" "PB_L2_PERSIST_MB=120 PB_DICT_W_EVICT=1"; do
  echo "== $e"; env $e timeout 120 python tools/sweep_timing.py 1 4 --steps 4 2>&1 | grep cfg
done
