for envs in "" "PB_DICT_VARIANT=1" "PB_DICT_MAX_CTAS=148" "PB_DICT_MAX_CTAS=222" "PB_DICT_MAX_CTAS=260"; do
  echo "== $envs"; env $envs timeout 200 python tools/quick_timing.py ${VAR_CFGS:-2 3} 2>&1 | grep phases
done
