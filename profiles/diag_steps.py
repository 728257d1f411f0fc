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
    import ctypes as C
    t = (C.c_uint64 * 11)()
    s.lib.jit_sched_phase_times(s.h, t, 11)
    if t[9] and t[10] and t[3] > t[2]:
        print("   resolve phase 2->3: %d cycles in %d ns = %.0f MHz" % (t[10] - t[9], t[3] - t[2], (t[10] - t[9]) / (t[3] - t[2]) * 1e3))
