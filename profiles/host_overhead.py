"""Host cost of one step launch vs device time per step (is the step loop host- or device-bound?).

Prints, for K back-to-back step_async calls on one C3 handle: wall-clock microseconds per call
spent on the host (no synchronisation inside the loop) and device microseconds per step
(CUDA events around the whole loop)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
now, v = d["now_ns"], d["v_token_ns"]
for _ in range(20):
    if os.environ.get("JITSCHED_EXPERIMENT"):
        s.step_async(now, v)        # results are not valid in experiment mode: never fetched
    else:
        s.step(now, v)
torch.cuda.synchronize()
K = 400
stream = torch.cuda.current_stream()
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(K):
        s.step_async(now, v)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"rep {rep}: host {1e6 * (t1 - t0) / K:.1f} us/call   device {1e3 * e0.elapsed_time(e1) / K:.1f} us/step",
          flush=True)
# raw ctypes call cost without the python wrapper
lib, h = s.lib, s.h
import ctypes as C  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(K):
    lib.jit_sched_step_async(h, C.c_int64(now), C.c_int64(v))
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"raw ctypes: host {1e6 * (t1 - t0) / K:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / K:.1f} us/step")
