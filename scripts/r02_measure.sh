# Round-2 measurement batch: K2 traffic of every pass (ncu), full --set capture of
# partition 0's four K2 passes and the top GEMM, launch list, then the bench line.
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
python bench.py $ARGS > /dev/null 2> gpurun_out/prep.err
timeout 900 python scripts/k2_traffic.py reddit_gcn gpurun_out/r02_k2_traffic_reddit_gcn.json > gpurun_out/k2t.log 2>&1
tail -c 1500 gpurun_out/k2t.log
ncu --set full --clock-control none --import-source on -k regex:agg_kernel -s 0 -c 4 \
    -o gpurun_out/r02_k2_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 0 -c 5 \
    -o gpurun_out/r02_k3_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py $ARGS > /dev/null 2>&1
cp gpurun_out/r02_k2_traffic_reddit_gcn.json profiles/
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
tail -c 3000 gpurun_out/r02_bench.json
