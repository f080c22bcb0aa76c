# Round-2 verification batch on the GPU box: full -m gpu suite, smoke, bench, launch list.
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_verify_tests.log 2>&1
tail -30 gpurun_out/r02_verify_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/r02_verify_bench.json 2> gpurun_out/r02_verify_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_verify_bench.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['clocks'])
for k,v in d['step_breakdown'].items(): print(f'{v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
