# Round-2 measurement batch (GPU box): K2 traffic of all passes, ncu --set full of partition 0's
# K2 passes / guard exact fix / first K3 launches, launch list, bench lines (reddit default incl.
# e2e + CPU baseline, reference arm, products_sage, papers_gin_s24).
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0 --lanes 1"
python bench.py $ARGS > /dev/null 2> gpurun_out/prep.err
timeout 900 python scripts/k2_traffic.py reddit_gcn gpurun_out/r02_k2_traffic_reddit_gcn.json > gpurun_out/k2t.log 2>&1
cp gpurun_out/r02_k2_traffic_reddit_gcn.json profiles/
ncu --set full --clock-control none --import-source on -k regex:agg_kernel -s 0 -c 4 \
    -o gpurun_out/r02_k2_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:exact_fix -s 0 -c 1 \
    -o gpurun_out/r02_fix_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 0 -c 5 \
    -o gpurun_out/r02_k3_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py $ARGS > /dev/null 2>&1
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_ref.err
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_full_tests.log 2>&1; tail -2 gpurun_out/r02_full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

python bench.py --workload papers_gin_s24 --no-cpu-baseline > gpurun_out/r02_bench_papers_gin_s24.json 2> /dev/null
tail -c 400 gpurun_out/r02_bench.json gpurun_out/r02_bench_reference_arm.json
