"""GPU parity of the exact sharded step (shard.cuh) in virtual-shard mode: W handles on one
B200, each holding a shard, exchange records by concatenation (the allgather stand-in); every
rank's batch must equal the oracle's batch over the whole pool."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def _run(d, world, cap_extra=0):
    from paper_2504_20068_b200 import Scheduler
    from paper_2504_20068_b200.sharded import ShardedStep, shard_pool, virtual_shards_step
    steps = []
    for r in range(world):
        sp, st = shard_pool(d["pool"], d["tasks"], r, world)
        n = max(len(sp["input_len"]), 1)
        nt = 0 if st is None else len(st["arrival_ns"])
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(n, world * (d["cfg"]["max_batch"] + 1)) + cap_extra,
                      task_capacity=max(nt, 1))
        s.load(sp, st)
        steps.append(ShardedStep(s, r, world, None))
    outs = virtual_shards_step(steps, d["now_ns"], d["v_token_ns"])
    for st in steps:
        st.s.close()
    return outs


def _check(outs, ref, ctx):
    for o in outs:
        assert o["status"] == ref["status"], ctx
        if ref["status"] != 0:
            continue
        assert np.array_equal(o["batch_ids"], ref["batch_ids"]), ctx
        assert np.array_equal(o["batch_tokens"], ref["batch_tokens"]), ctx
        assert o["b_star"] == ref["b_star"] and o["n_candidates"] == ref["n_candidates"], ctx
        assert np.float64(o["bp"]).view(np.uint64) == np.float64(ref["bp"]).view(np.uint64), ctx
        assert np.float64(o["thr"]).view(np.uint64) == np.float64(ref["thr"]).view(np.uint64), ctx
        assert o["total_tokens"] == ref["total_tokens"], ctx


def test_virtual_shards_random_pools():
    rng = np.random.default_rng(301)
    for it in range(60):
        d = W.random_small_pool(rng, int(rng.integers(1, 80)), tie_heavy=(it % 6 == 0))
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        _check(_run(d, int(rng.integers(1, 5))), ref, f"iter {it}")


@pytest.mark.parametrize("world", [2, 8])
def test_virtual_shards_c3(world):
    d = W.pool_snapshot(3, 1 << 20)
    ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
    _check(_run(d, world), ref, f"C3 W={world}")


def test_virtual_shards_c5_pool_16m():
    """BASELINE config C5(ii): a 2^24-row pool sharded over 8 ranks (2^21 rows each)."""
    d = W.pool_snapshot(55, 1 << 24, table_draws=1 << 16)
    ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"],
                      rows_out=False)
    _check(_run(d, 8), ref, "C5(ii)")


@pytest.mark.parametrize("world,rows", [(2, 200_000), (4, 200_000), (4, 1 << 21)])
def test_virtual_shards_consecutive_steps_fast_path(world, rows):
    """Consecutive sharded steps: the first takes the exact two-round protocol (no threshold yet),
    later ones the speculative resolve across ranks (one exchange of speculative sets).  Every
    step must equal the oracle over the whole pool, run on the state its previous step left."""
    from paper_2504_20068_b200 import Scheduler
    from paper_2504_20068_b200.sharded import ShardedStep, shard_pool, virtual_shards_step
    d = W.pool_snapshot(31, rows, table_draws=1 << 16)
    if rows >= (1 << 21):
        # a union beyond the small-set path (> 256 entries, the histogram resolve): with the 3%
        # speculative margin tau = 8192 gives ~220 entries over 2^21 rows, so the C3 tau-sweep's
        # largest budget
        d["cfg"] = W.default_config(token_budget=65536, max_batch=65536)
    steps = []
    for r in range(world):
        sp, st = shard_pool(d["pool"], d["tasks"], r, world)
        n = max(len(sp["input_len"]), 1)
        nt = 0 if st is None else len(st["arrival_ns"])
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(n, world * (d["cfg"]["max_batch"] + 1)),
                      task_capacity=max(nt, 1))
        s.load(sp, st)
        steps.append(ShardedStep(s, r, world, None))
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    paths, sizes = [], []
    for k in range(4 if rows < (1 << 20) else 3):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"],
                          rows_out=False)
        outs = virtual_shards_step(steps, d["now_ns"], d["v_token_ns"])
        _check(outs, ref, f"W={world} step {k}")
        paths.append(outs[0]["path"])
        sizes.append(outs[0]["n_spec"])
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
    for st in steps:
        st.s.close()
    assert paths[0] == "exact" and "speculative" in paths[1:], paths
    if rows >= (1 << 21):        # a union larger than the small-set path: the histogram resolve ran
        assert max(sizes[1:]) > 256, sizes
