"""Per-warp timeline of one k_score launch (JIT_TIMELINE build via JITSCHED_LIB): start skew,
prologue, item loop (and the part of it spent waiting for slots), epilogue, end spread."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
hs = []
for i in range(6):
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
    s.load(d["pool"], d["tasks"])
    for _ in range(3):
        s.step(d["now_ns"], d["v_token_ns"])
    hs.append(s)
for rep in range(3):
    for h in hs:
        h.debug_scratch(1)
    ms = Scheduler.time_scoring(hs, d["now_ns"], d["v_token_ns"], 6)
    t = hs[-1].debug_scratch(16 * 148 * 64).reshape(-1, 16).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    st, pro, items, wait, epi, end = t[:, 0] - t0, t[:, 1] - t[:, 0], t[:, 2] - t[:, 1], t[:, 4], t[:, 3] - t[:, 2], t[:, 3] - t0
    q = lambda a: "p10 %6.0f p50 %6.0f p90 %6.0f max %6.0f" % tuple(np.percentile(a, [10, 50, 90, 100]))
    print(f"rep {rep}: b2b avg {ms * 1e3:.2f} us over 6 launches; warps {len(t)}; items/warp {np.bincount(t[:, 5])}")
    for name, a in (("start", st), ("prologue", pro), ("items", items), ("  waiting", wait), ("epilogue", epi), ("end", end)):
        print(f"  {name:10s} ns  {q(a)}")
    ts_, ns_ = t[:, 6] & ((1 << 48) - 1), t[:, 6] >> 48
    tc_, nc_ = t[:, 7] & ((1 << 48) - 1), t[:, 7] >> 48
    print(f"  prologue: persist in {q(t[:, 12])}; ring filled {q(t[:, 13])}; groups done {q(t[:, 14])}")
    nc = t[:, 11].sum()
    if nc:
        print(f"  cmp item phases ns: A {t[:, 8].sum() / nc:.0f}  per-task {t[:, 9].sum() / nc:.0f}  B {t[:, 10].sum() / nc:.0f}")
    print(f"  standalone phase ns {q(ts_)}; per chunk {ts_.sum() / max(ns_.sum(), 1):.0f} ({ns_.sum()} chunks)")
    print(f"  ring items ns {q(tc_)}; per item {tc_.sum() / max(nc_.sum(), 1):.0f} ({nc_.sum()} items)")
