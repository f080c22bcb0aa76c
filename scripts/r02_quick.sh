# quick GPU loop: GNN parity tests + bench step breakdown
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_sgc.py -q -x > gpurun_out/q_tests.log 2>&1
tail -5 gpurun_out/q_tests.log
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/q_bench.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d.get('e2e',{}).get('value',0)/1e9, d.get('e2e',{}).get('ms_per_step'), d['clocks'])
for k,v in d['step_breakdown'].items(): print(f'{v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
