"""Debug helper: a few steps on a small pool, in graph and direct-launch modes, printing the device
and host copies of the control block (JITSCHED_DEBUG_CTRL)."""
import os
import sys

os.environ["JITSCHED_DEBUG_CTRL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 14)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
for mode in ("graph", "direct"):
    print(mode, flush=True)
    if mode == "direct":
        os.environ["JITSCHED_NO_GRAPH"] = "1"
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
    s.load(d["pool"], d["tasks"])
    for k in range(3):
        try:
            r = s.step(d["now_ns"], d["v_token_ns"])
            print(k, {x: r[x] for x in ("n_pending", "fallback", "b_star", "n_selected", "n_spec")}, flush=True)
        except Exception as e:  # noqa: BLE001
            print(k, "error", e, flush=True)
