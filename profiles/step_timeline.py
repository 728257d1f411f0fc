"""Where the C3 step's time goes between k_score and k_spec (a build with -DJIT_TIMELINE
-DJIT_PHASE_STAMPS via JITSCHED_LIB): per step, on one %globaltimer clock, k_score's first warp
start and last warp end (per-warp stamps in the scratch), then k_spec's phase stamps (after its
dependency wait, set loaded, ranks, cutoff / Cd, prefix sums, window, batch written)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
rows = []
for k in range(16):
    s.debug_scratch(1)
    r = s.step(d["now_ns"], d["v_token_ns"])
    t = s.debug_scratch(16 * 148 * 64).reshape(-1, 16).astype(np.int64)
    t = t[t[:, 0] > 0]
    ts = (C.c_uint64 * 12)()
    s.lib.jit_sched_phase_times(s.h, ts, 11)
    v = np.array(list(ts)[:8], np.int64)
    if k < 3 or r["fallback"] or not v.all():
        continue
    t0 = t[:, 0].min()
    rows.append([t[:, 3].max() - t0, np.percentile(t[:, 3], 50) - t0] + (v - t0).tolist())
a = np.median(np.array(rows), axis=0)
names = ["k_score last warp end", "k_score median warp end", "k_spec after wait", "partials read",
         "set in smem", "ranks / B*", "Cd positions", "prefix sums", "window argmax", "batch written"]
print(f"{len(rows)} steps, median ns from k_score's first warp start:")
for nm, x in zip(names, a):
    print(f"  {nm:24s} {x:8.0f}")
