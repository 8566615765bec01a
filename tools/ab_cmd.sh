# A/B of environment switches on the quick timing: AB_ENVS="ENV=1 ENV2=3" VAR_CFGS="2 3"
for envs in "" $AB_ENVS; do
  echo "== ${envs:-default}"; env $envs timeout 200 python tools/quick_timing.py ${VAR_CFGS:-2 3} 2>&1 | grep phases
done
