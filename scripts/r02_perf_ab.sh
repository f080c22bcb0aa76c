# Round-2 perf A/B batch (GPU box): parity of the changed kernels, GEMM and K2
# micro-benchmarks, bench variants; the reference full-pass check in the background.
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
python scripts/ref_full_pass.py reddit_gcn 0 41,256 > gpurun_out/ref_full_pass.log 2>&1 &
RF=$!
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gnn.py tests/test_gpu_sgc.py \
  "tests/test_gpu_fullscale.py::test_ten_epochs_match_frozen_oracle" tests/test_gpu_gnn_pinned.py -q -x > gpurun_out/r02_ab_tests.log 2>&1
tail -3 gpurun_out/r02_ab_tests.log
timeout 300 python scripts/gemm_micro.py 200000 20 > gpurun_out/r02_gemm_micro.log 2>&1
cat gpurun_out/r02_gemm_micro.log
for v in "X=1" "CATGNN_AGG_NARROW43=0"; do env $v WIDTHS=48 REPS=20 timeout 300 python scripts/agg_micro.py 2>/dev/null | tail -1 | sed "s/^/$v /"; done > gpurun_out/r02_agg48.log
for v in "X=1" "CATGNN_AGG_SLAB=32" "CATGNN_AGG_SLAB=32 CATGNN_AGG_W128_16=1"; do env $v WIDTHS=256 REPS=10 timeout 300 python scripts/agg_micro.py 2>/dev/null | tail -1 | sed "s/^/$v /"; done > gpurun_out/r02_agg256.log
cat gpurun_out/r02_agg48.log gpurun_out/r02_agg256.log
bash scripts/ab.sh "X=1" "CATGNN_AGG_NARROW43=0" "CATGNN_AGG_SLAB=32" "CATGNN_AGG_SLAB=32 CATGNN_AGG_W128_16=1" "X=1" > gpurun_out/r02_ab_bench.log 2>&1
cat gpurun_out/r02_ab_bench.log
wait $RF
cat gpurun_out/ref_full_pass.log | tail -2
