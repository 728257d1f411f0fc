"""C5(i) sweep throughput of the library's replay-CTA configuration (device time, CUDA events).

The sweep configurations in replay.cuh's table were compared with this script through a temporary
JIT_REPLAY_SWEEP switch (removed once 128 threads x 8 CTAs per SM won); each run printed its
steps/s and whether its per-replay results equalled the first configuration's.

usage (under gpurun): python profiles/sweep_variants.py [repeats, default 2]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

variants = list(range(int(sys.argv[1]) if len(sys.argv) > 1 else 2))
traces = [W.trace_mixed(k) for k in range(4)]
sweep = W.c5_sweep(4096)
specs = [dict(sp, trace=i % len(traces)) for i, sp in enumerate(sweep)]
rc = dict(traces[0]["rcfg"], n_steps=4096)
s = Scheduler(traces[0]["cfg"], traces[0]["groups"], traces[0]["table"], capacity=64, task_capacity=8)
ref = None
for v in variants:
    s.replay([t["trace"] for t in traces], specs[:400], dict(rc, n_steps=64))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res, _ = s.replay([t["trace"] for t in traces], specs, rc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = sum(int(r["steps"]) for r in res)
    key = [(int(r["token_goodput"]), int(r["steps"]), int(r["n_done"]), int(r["sim_end_ns"])) for r in res]
    same = ref is None or key == ref
    ref = ref or key
    print(f"run {v}: {st} steps in {ms:.1f} ms = {st / ms * 1e3 / 1e6:.2f} M steps/s; equal to run 0: {same}",
          flush=True)
s.close()
