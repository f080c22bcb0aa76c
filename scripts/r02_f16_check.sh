# fp16 K2 inputs: parity of the GNN layers (single step, 10 epochs, full size) and the bench step.
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_gemm.py tests/test_gpu_gnn_pinned.py -q -x > gpurun_out/r02_f16_tests.log 2>&1
tail -15 gpurun_out/r02_f16_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -x -s > gpurun_out/r02_f16_full.log 2>&1
tail -25 gpurun_out/r02_f16_full.log
python bench.py --no-cpu-baseline > gpurun_out/r02_f16_bench.json 2> gpurun_out/r02_f16_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_f16_bench.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['clocks'])
for k,v in d['step_breakdown'].items(): print(f'{v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
CATGNN_ACT_F16=0 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02_f32_bench.json 2> /dev/null
tail -c 300 gpurun_out/r02_f32_bench.json
