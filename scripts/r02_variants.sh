# bench step breakdown per library variant (CATGNN_LIB), default build first
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
for lib in default $VARIANTS; do
  if [ "$lib" = default ]; then unset CATGNN_LIB; else export CATGNN_LIB=$PWD/paper_2404_02300_b200/build/variants/$lib/libcatgnn.so; fi
  echo "== $lib"
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(f\"ms/step {d['ms_per_step']:.2f} clocks {d['clocks']['sm_mhz']}\")
for k,v in d['step_breakdown'].items(): print(f'   {v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
done
