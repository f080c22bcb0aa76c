set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gputest3.log 2>&1
tail -25 gpurun_out/r02_gputest3.log
timeout 300 python scripts/gemm_micro.py 200000 20 > gpurun_out/r02_gemm_micro2.log 2>&1
python bench.py > gpurun_out/r02_bench2.json 2> gpurun_out/r02_bench2.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench2.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['clocks'])
for k,v in d['step_breakdown'].items(): print(f'{v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
