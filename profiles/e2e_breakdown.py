"""Where the serving-loop step's wall time goes (jit_sched_step with deltas), C3 pool: Python
marshalling vs the C call, and the C call with no deltas / progress only / arrivals only / both."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402
from paper_2504_20068_b200 import jitsched as J  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
per, steps = 256, 40
extra = W.pool_snapshot(77, per * (4 * steps + 16) + 64, frac_compound=0.0, table=d["table"])
extra["pool"]["id"] = (extra["pool"]["id"].astype(np.uint64) + (1 << 28)).astype(np.uint32)
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n + per * (4 * steps + 16), task_capacity=nt)
s.load(d["pool"], d["tasks"])
loop = bench.EngineLoop(d, extra, per)
now, v = d["now_ns"], d["v_token_ns"]
b = s.step(now, v)
for _ in range(3):
    b = s.step(now, v, progress=loop.progress(b), arrivals=loop.arrivals(now))
torch.cuda.synchronize()
for mode in ("none", "progress", "arrivals", "both"):
    walls, py = [], []
    for _ in range(steps):
        now += 20 * W.MS
        prog = loop.progress(b) if mode in ("progress", "both") else None
        arr = loop.arrivals(now) if mode in ("arrivals", "both") else None
        t0 = time.perf_counter()
        if arr is not None:                           # the marshalling alone (what step() does first)
            ap, keep = s.make_pool(arr, None)
        t1 = time.perf_counter()
        b = s.step(now, v, progress=prog, arrivals=arr)
        t2 = time.perf_counter()
        walls.append(t2 - t1); py.append(t1 - t0)
    print(f"{mode:9s} step wall median {statistics.median(walls) * 1e6:7.1f} us; make_pool alone {statistics.median(py) * 1e6:6.1f} us")
