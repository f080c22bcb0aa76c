set -x
export CATGNN_CACHE=/tmp/catgnn_cache
timeout 1200 python -m pytest tests/test_gpu_sgc.py tests/test_gpu_completion.py tests/test_gpu_gnn.py tests/test_gpu_fullscale.py::test_partition_one_step_matches_oracle -q -x 2>&1 | tail -3
python - <<'PY'
import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_2404_02300_b200 import gnnpart as gp
from benchdata import workloads as W
w = W.WORKLOADS['reddit_gcn']; prep = W.prepare(w, lambda *a: None); part = W.load_part(prep, 0)
ctx = gp.Context(0)
for i in range(3):
    t = time.time(); s = gp.Shard.from_part(part['ext'], part['owner'], part['role'], part['labels'], part['edges'], part['features'], ctx); ctx.synchronize(); print('shard load s', time.time() - t); s.close()
PY
