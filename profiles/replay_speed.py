"""Replay speed per CTA and over the C5 sweep (device time, CUDA events): C1, C2 (one replay =
one CTA), a 592-replay slice of C5(i).  Compare libraries with JITSCHED_LIB."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402


def timed(s, traces, specs, rc):
    s.replay(traces, specs[:2], dict(rc, n_steps=min(rc["n_steps"], 50)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res, _ = s.replay(traces, specs, rc)
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1)


one = dict(trace=0, load_num=1, load_den=1, slo_num=1, slo_den=1)
for name, d, steps in (("C1", W.trace_c1(), None), ("C2", W.trace_c2(), 3000)):
    rc = dict(d["rcfg"], **({"n_steps": steps} if steps else {}))
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=64, task_capacity=8)
    res, ms = timed(s, [d["trace"]], [one], rc)
    st = int(res[0]["steps"])
    print(f"{name}: {st} steps in {ms:.2f} ms = {st / ms * 1e3:.0f} steps/s ({ms * 1e3 / st:.1f} us/step), goodput {int(res[0]['token_goodput'])}")
    s.close()
traces = [W.trace_mixed(k) for k in range(3)]
sweep = W.c5_sweep()
for n_rep in (592, 4096):
    specs = [dict(sweep[(i * 4096) // n_rep], trace=i % 3) for i in range(n_rep)]
    s = Scheduler(traces[0]["cfg"], traces[0]["groups"], traces[0]["table"], capacity=64, task_capacity=8)
    res, ms = timed(s, [t["trace"] for t in traces], specs, traces[0]["rcfg"])
    st = sum(int(r["steps"]) for r in res)
    print(f"C5 {n_rep} replays: {st} steps in {ms:.1f} ms = {st / ms * 1e3 / 1e6:.2f} M steps/s; goodput sum {sum(int(r['token_goodput']) for r in res)}")
    s.close()
