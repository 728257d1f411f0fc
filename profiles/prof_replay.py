"""Minimal driver for ncu on the replay kernel: C5 mixed traces, a subset of the sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

n_rep = int(sys.argv[1]) if len(sys.argv) > 1 else 296
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
traces = [W.trace_mixed(k) for k in range(4)]
sweep = W.c5_sweep(4096)
specs = [dict(sweep[(i * 13) % 4096], trace=i % 4) for i in range(n_rep)]
rc = dict(traces[0]["rcfg"], n_steps=steps)
s = Scheduler(traces[0]["cfg"], traces[0]["groups"], traces[0]["table"], capacity=64, task_capacity=8)
res, _ = s.replay([t["trace"] for t in traces], specs, rc)
print("steps", sum(r["steps"] for r in res))
