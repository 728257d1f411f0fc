#!/bin/bash
# ncu durations of k_score: normal vs no-row-math (JIT_SCORE_FLOOR) on a standalone-only C3 pool
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -c "
from paper_2504_20068_b200 import _build
_build.build_library(force=True, out='paper_2504_20068_b200/libjitsched_floor.so', defines=['-DJIT_SCORE_FLOOR'])" > /dev/null 2>&1
cat > /tmp/fl.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, workloads as W
from paper_2504_20068_b200 import Scheduler
d = W.pool_snapshot(3, 1 << 20, frac_compound=float(sys.argv[1]))
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
hs = []
for i in range(3):
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=max(nt, 1)); s.load(d["pool"], d["tasks"]); hs.append(s)
for k in range(9):
    hs[k % 3].step_async(d["now_ns"], d["v_token_ns"])
torch.cuda.synchronize()
PY
for lib in libjitsched libjitsched_floor; do for fc in 0.0 0.3; do
  JITSCHED_LIB=$PWD/paper_2504_20068_b200/$lib.so ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k_score -s 3 -c 4 --csv python /tmp/fl.py $fc 2>/dev/null | grep gpu__time_duration | awk -F'","' -v l=$lib -v f=$fc '{print l, "frac", f, $NF}'
done; done
