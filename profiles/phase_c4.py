"""C4 big-mode step phases (a -DJIT_PHASE_STAMPS build via JITSCHED_LIB): k_group's window over the
large Cd -- sort, prefix sums, window argmax, batch (ns between %globaltimer stamps 6..10)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_c4()
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
rows = []
for k in range(10):
    r = s.step(d["now_ns"], d["v_token_ns"])
    ts = (C.c_uint64 * 12)()
    s.lib.jit_sched_phase_times(s.h, ts, 11)
    v = np.array(list(ts)[:11], np.int64)
    if k >= 3 and v[6] and v[10]:
        rows.append(np.diff(v[6:11]))
print("n_candidates", r["n_candidates"], "n_spec", r["n_spec"])
print("k_group ns: sort, prefix sums, window argmax, batch+bookkeeping =", np.median(np.array(rows), axis=0).tolist())
