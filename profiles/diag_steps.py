"""Per-step diagnostics on C3: length-bound refreshes, speculative fallback, selection sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
for k in range(6):
    r = s.step(d["now_ns"], d["v_token_ns"])
    print(k, {x: r[x] for x in ("n_pending", "n_refresh", "fallback", "b_star", "n_candidates", "n_selected",
                                "n_dropped_now", "n_spec")})
    print("   phases ns:", s.phase_times())
