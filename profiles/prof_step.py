"""Minimal driver for ncu: C3 pool (2^20 rows), R rotated handles, a few warm steps then
`--steps` graph launches.  Used only under ncu (numbers printed here are not bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--rot", type=int, default=3)
ap.add_argument("--rows", type=int, default=1 << 20)
ap.add_argument("--frac-compound", type=float, default=0.3)
a = ap.parse_args()
d = W.pool_snapshot(3, a.rows, frac_compound=a.frac_compound)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
hs = []
for i in range(a.rot):
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
    s.load(d["pool"], d["tasks"])
    for _ in range(3):                     # first step: exact path (+ re-score); then the fast path
        r = s.step(d["now_ns"], d["v_token_ns"])
    print("handle", i, "fallback", r["fallback"], "n_spec", r["n_spec"])
    hs.append(s)
for k in range(a.steps):
    hs[k % a.rot].step_async(d["now_ns"], d["v_token_ns"])
torch.cuda.synchronize()
print("done")
