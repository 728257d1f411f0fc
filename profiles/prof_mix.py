"""k_score / step device time vs pool composition (standalone vs compound rows), C3 generator.
Not a bench number: a diagnostic for where k_score's time goes (run under gpurun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402

K, ROT = 30, 4
for frac in [float(x) for x in (sys.argv[1:] or ["0.0", "0.3", "0.99"])]:
    d = W.pool_snapshot(3, 1 << 20, frac_compound=frac)
    n, nt = len(d["pool"]["input_len"]), len(d["tasks"]["arrival_ns"])
    hs = []
    for i in range(ROT):
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=max(nt, 1))
        s.load(d["pool"], d["tasks"])
        s.step(d["now_ns"], d["v_token_ns"])
        s.step(d["now_ns"], d["v_token_ns"])
        s.kernel_times(slots=K)
        hs.append(s)
    for k in range(K):
        hs[k % ROT].step_async(d["now_ns"], d["v_token_ns"])
    torch.cuda.synchronize()
    kt = np.mean([h.kernel_times() for h in hs], axis=0)
    print(f"frac_compound {frac:.2f} rows {n} tasks {nt}: k_score {kt[0] * 1e3:.2f} us, k_spec {kt[2] * 1e3:.2f} us, "
          f"step {kt[4] * 1e3:.2f} us", flush=True)
    for h in hs:
        h.close()
