# bench step breakdown under environment variants: scripts/r02_env_ab.sh "X=1" "ENV=..." ...
set -x
export CATGNN_CACHE=/tmp/catgnn_cache
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for v in "$@"; do
  echo "== $v"
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(f\"ms/step {d['ms_per_step']:.2f} clocks {d['clocks']['sm_mhz']}\")
for k,v in d['step_breakdown'].items(): print(f'   {v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
done
