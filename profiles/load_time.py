"""Wall time of jit_sched_load (C3 pool from pinned host memory) and of the first step after it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
pool = {k: (torch.from_numpy(np.ascontiguousarray(v)).pin_memory() if isinstance(v, np.ndarray) else v)
        for k, v in d["pool"].items()}
tasks = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in d["tasks"].items()}
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
for i in range(4):
    t0 = time.perf_counter(); s.load(pool, tasks); t1 = time.perf_counter()
    r = s.step(d["now_ns"], d["v_token_ns"]); t2 = time.perf_counter()
    print(f"load {1e3 * (t1 - t0):.3f} ms, first step {1e3 * (t2 - t1):.3f} ms (refresh {r['n_refresh']}, fallback {r['fallback']})")
