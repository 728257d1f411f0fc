"""Debug helper: replay tests/test_shard_gpu.py::test_virtual_shards_random_pools step by step,
printing each shard's shape before its phases (run with CUDA_LAUNCH_BLOCKING=1 under gpurun)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2504_20068_b200 import Scheduler  # noqa: E402
from paper_2504_20068_b200.sharded import ShardedStep, shard_pool, virtual_shards_step  # noqa: E402

rng = np.random.default_rng(301)
for it in range(60):
    d = W.random_small_pool(rng, int(rng.integers(1, 80)), tie_heavy=(it % 6 == 0))
    world = int(rng.integers(1, 5))
    steps = []
    for r in range(world):
        sp, st = shard_pool(d["pool"], d["tasks"], r, world)
        n = max(len(sp["input_len"]), 1)
        nt = 0 if st is None else len(st["arrival_ns"])
        print(f"it {it} world {world} rank {r}: rows {len(sp['input_len'])} n_single {sp.get('n_single')} tasks {nt} "
              f"debug-cfg {d['cfg'].get('max_batch')} {d['cfg'].get('token_budget')}", flush=True)
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(n, world * (d["cfg"]["max_batch"] + 1)),
                      task_capacity=max(nt, 1))
        s.load(sp, st)
        steps.append(ShardedStep(s, r, world, None))
    outs = virtual_shards_step(steps, d["now_ns"], d["v_token_ns"])
    for st in steps:
        st.s.close()
print("done")
