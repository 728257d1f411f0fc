"""Two-process runs of the multi-rank paths with the real kernels (one GPU here: both ranks on
cuda:0, records exchanged by a host-staged gloo allgather -- the same orchestration the N-GPU
runs drive over NCCL):
  * the sharded pool step (sharded.ShardedStep over two Schedulers, speculative tier included)
    against the unsharded oracle, consecutive steps;
  * NEXT-2 power-of-K with one replica per rank (jitsched.multi_step with an allgather) against
    the oracle's multi_step."""
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _host_allgather():
    import torch
    import torch.distributed as dist

    def gather(t):
        c = t.cpu()
        parts = [torch.empty_like(c) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, c)
        return torch.cat(parts).to(t.device)

    return gather


def _init(rank, world, port):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _shard_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    try:
        import oracle
        import workloads as W
        from paper_2504_20068_b200 import Scheduler
        from paper_2504_20068_b200.sharded import ShardedStep, shard_pool
        d = W.pool_snapshot(1401, 60_000, table_draws=1 << 15)
        sp, st = shard_pool(d["pool"], d["tasks"], rank, world)
        n, nt = len(sp["input_len"]), len(st["arrival_ns"])
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(n, world * (d["cfg"]["max_batch"] + 1)),
                      task_capacity=max(nt, 1))
        s.load(sp, st)
        step = ShardedStep(s, rank, world, _host_allgather())
        pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
        res = []
        for k in range(5):
            now = d["now_ns"] + k * 2_000_000
            ref = oracle.step(d["cfg"], d["groups"], d["table"], now, d["v_token_ns"], pool, d["tasks"])
            got = step.step(now, d["v_token_ns"])
            ok = got["status"] == ref["status"]
            if ok and ref["status"] == 0:
                ok = (np.array_equal(got["batch_ids"], ref["batch_ids"]) and got["b_star"] == ref["b_star"] and
                      np.float64(got["bp"]).view(np.uint64) == np.float64(ref["bp"]).view(np.uint64) and
                      got["n_candidates"] == ref["n_candidates"] and got["total_tokens"] == ref["total_tokens"])
            res.append((bool(ok), got.get("path")))
            pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        q.put((rank, res))
    except Exception as e:          # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _multi_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    try:
        import oracle
        import workloads as W
        from paper_2504_20068_b200 import Scheduler
        from paper_2504_20068_b200.jitsched import multi_step
        rng = np.random.default_rng(1402)
        d = W.random_small_pool(rng, 160, with_tasks=False)
        pools = W.replica_pools(d, world, 2, seed=11)
        vs = [10 * W.MS, 7 * W.MS][:world]
        ref_pools = [{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()} for p in pools]
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=len(pools[rank]["id"]), task_capacity=1)
        s.load(pools[rank], None)
        res = []
        for k in range(4):
            now = d["now_ns"] + k * 1000
            ref = oracle.multi_step(d["cfg"], d["groups"], d["table"], now, vs, ref_pools)
            got = multi_step([s], now, [vs[rank]], allgather=_host_allgather(), replica=rank)[0]
            rows = s.read_rows(debug=False)
            ok = (got["status"] == ref[rank]["status"] and np.array_equal(got["batch_ids"], ref[rank]["batch_ids"]) and
                  got["total_tokens"] == ref[rank]["total_tokens"] and np.array_equal(rows["meta"], ref[rank]["meta"]) and
                  np.array_equal(rows["aux"], ref[rank]["aux"]))
            res.append(bool(ok))
            for m in range(world):
                ref_pools[m]["meta"], ref_pools[m]["aux"] = ref[m]["meta"], ref[m]["aux"]
        q.put((rank, res))
    except Exception as e:
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(worker, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    return out


def test_sharded_step_two_processes():
    out = _run(_shard_worker)
    for r, res in out.items():
        assert isinstance(res, list), res
        assert all(ok for ok, _ in res), (r, res)
        assert any(path == "speculative" for _, path in res), res       # the fast tier ran


def test_power_of_k_one_replica_per_rank():
    out = _run(_multi_worker)
    for r, res in out.items():
        assert isinstance(res, list), res
        assert all(res), (r, res)
