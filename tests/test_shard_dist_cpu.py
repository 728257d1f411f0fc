"""World-size-2 gloo test of the sharded-step orchestration (paper_2504_20068_b200/sharded.py)
on CPU: two processes, each owning a shard, exchange round-1 / round-2 records through
torch.distributed allgathers and must both return the batch the oracle selects over the whole
pool (exact B*, bp, thr, |Cd| and batch ids)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.timeout(600) if hasattr(pytest.mark, "timeout") else []


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_allgather():
    import torch
    import torch.distributed as dist

    def gather(t):
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, t.contiguous())
        return torch.cat(parts)

    return gather


def _worker(rank, world, port, seed, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import oracle
    import workloads as W
    from paper_2504_20068_b200.sharded import ShardedStep, shard_pool
    from tests._fake_shard import FakeShardSched, FakeSpecShardSched
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        results = []
        for it in range(6):
            d = W.random_small_pool(rng, int(rng.integers(8, 60)))
            ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
            sp, st = shard_pool(d["pool"], d["tasks"], rank, world)
            dd = dict(d, pool=sp, tasks=st)
            fake = FakeShardSched(dd, d["cfg"]["max_batch"], max(len(sp["input_len"]), 1))
            step = ShardedStep(fake, rank, world, _gloo_allgather(), device="cpu")
            got = step.step(d["now_ns"], d["v_token_ns"])
            ok = True
            if ref["status"] == 0:
                ok = (list(got["batch_ids"]) == list(ref["batch_ids"]) and got["bp"] == ref["bp"] and
                      got["thr"] == ref["thr"] and got["b_star"] == ref["b_star"] and
                      got["n_candidates"] == ref["n_candidates"])
            results.append(bool(ok))
        # the speculative tier over gloo: a first step through the exact protocol leaves the
        # threshold, the next step on the same pool resolves the union of the exported sets
        n_spec = 0
        for it in range(4):
            d = W.random_small_pool(rng, int(rng.integers(20, 80)))
            ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
            sp, st = shard_pool(d["pool"], d["tasks"], rank, world)
            fake = FakeSpecShardSched(dict(d, pool=sp, tasks=st), d["cfg"]["max_batch"], max(len(sp["input_len"]), 1))
            step = ShardedStep(fake, rank, world, _gloo_allgather(), device="cpu")
            for k in range(2):
                got = step.step(d["now_ns"], d["v_token_ns"])
                ok = True
                if ref["status"] == 0:
                    ok = (list(got["batch_ids"]) == list(ref["batch_ids"]) and got["bp"] == ref["bp"] and
                          got["thr"] == ref["thr"] and got["b_star"] == ref["b_star"] and
                          got["n_candidates"] == ref["n_candidates"])
                    n_spec += got["path"] == "speculative"
                results.append(bool(ok))
        results.append(n_spec > 0)
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


def test_sharded_protocol_world2_gloo_matches_oracle():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 1234, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, oks in res:
        assert all(oks), (rank, oks)


def test_shard_pool_partition_is_exact():
    import workloads as W
    from paper_2504_20068_b200.sharded import shard_pool
    d = W.pool_snapshot(5, 5000, table_draws=1 << 12)
    parts = [shard_pool(d["pool"], d["tasks"], r, 3) for r in range(3)]
    ids = np.concatenate([p[0]["id"] for p in parts])
    assert sorted(ids.tolist()) == sorted(d["pool"]["id"].tolist())
    for p, t in parts:
        if t is not None:
            assert t["call_off"][0] == p["n_single"] and t["call_off"][-1] == len(p["input_len"])
