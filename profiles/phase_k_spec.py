import os, sys, ctypes as C
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads as W
from paper_2504_20068_b200 import Scheduler
d = W.pool_snapshot(3, 1 << 20)
n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt)
s.load(d["pool"], d["tasks"])
acc = []
for k in range(12):
    r = s.step(d["now_ns"], d["v_token_ns"])
    t = (C.c_uint64 * 12)()
    s.lib.jit_sched_phase_times(s.h, t, 11)
    v = list(t)[:11]
    if k >= 3 and all(v[:9]): acc.append([x - v[0] for x in v])
    print(k, r["n_spec"], r["n_candidates"], r["n_selected"], r["fallback"], [x - v[0] if x else None for x in v])
a = np.array(acc)
print("median phases ns:", np.median(a, axis=0).tolist())
