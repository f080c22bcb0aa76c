set -x
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x -k "e2e or gather" 2>&1 | tail -3
CATGNN_E2E_BREAKDOWN=1 python bench.py --no-cpu-baseline > gpurun_out/r02_bench3.json 2> gpurun_out/r02_bench3.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_bench3.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['clocks'])"
grep "\[e2e\]" gpurun_out/r02_bench3.err | head -30
