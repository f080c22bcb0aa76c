# guarded fp16 forward: parity (small graph + full size) and the bench step
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
CATGNN_GUARD_STATS=1 timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x -k "single_step or fp16" -s 2>&1 | grep -E "guard|passed|failed|Error|assert" | sort | uniq -c | sort -rn | head -20
timeout 900 python -m pytest tests/test_gpu_gnn.py tests/test_gpu_sgc.py tests/test_gpu_gemm.py -q -x > gpurun_out/g_tests.log 2>&1
tail -3 gpurun_out/g_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -x -s > gpurun_out/g_full.log 2>&1
grep -E "relative|rel err|passed|failed" gpurun_out/g_full.log
CATGNN_GUARD_STATS=1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --graph 0 2>&1 >/dev/null | grep guard | tail -8
python bench.py --no-cpu-baseline > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/g_bench.json').read().strip().splitlines()[-1])
print(d['value']/1e9, d['ms_per_step'], d['e2e']['value']/1e9, d['e2e']['ms_per_step'], d['clocks'])
for k,v in d['step_breakdown'].items(): print(f'{v[\"ms_per_step\"]:8.3f} {v[\"launches_per_step\"]:6.1f}  {k}')"
