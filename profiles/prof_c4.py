"""Driver for an ncu launch list of C4 steps in big mode (chained step_async after the switch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_c4()
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
for _ in range(3):
    r = s.step(d["now_ns"], d["v_token_ns"])
print("n_spec", r["n_spec"], "n_candidates", r["n_candidates"], "b_star", r["b_star"])
for _ in range(4):
    s.step_async(d["now_ns"], d["v_token_ns"])
print(s.fetch()["n_selected"], s.counters())
torch.cuda.synchronize()
