set -x
mkdir -p gpurun_out
(python tests/golden/make_fullscale_fixture.py reddit_gcn 10 > gpurun_out/fixture.log 2>&1; cp tests/golden/fullscale_reddit_gcn.json gpurun_out/ ) &
FIX=$!
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_fullscale.py::test_ten_epochs_match_frozen_oracle > gpurun_out/r02_gputest2.log 2>&1
tail -30 gpurun_out/r02_gputest2.log
timeout 600 python scripts/k2_traffic.py reddit_gcn gpurun_out/r02_k2_traffic_reddit_gcn.json > gpurun_out/k2t.log 2>&1
cp gpurun_out/r02_k2_traffic_reddit_gcn.json profiles/ 2>/dev/null
wait $FIX
tail -2 gpurun_out/fixture.log
python bench.py > gpurun_out/r02_bench1.json 2> gpurun_out/r02_bench1.err
tail -c 600 gpurun_out/r02_bench1.json
