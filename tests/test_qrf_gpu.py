"""GPU parity of NEXT-4: the quantile regression forest as (a2)'s length estimator (reading A50)
-- the batch bound API, the pool step (streaming pass refresh, compound calls included) and the
replay -- bit-exact against the oracle (integer bounds, so every key follows exactly)."""
import numpy as np
import pytest

import oracle
import workloads as W
from .test_parity_gpu import _compare
from .test_replay_gpu import _cmp, _spec
from .test_oracle_qrf import _tiny_forest

pytestmark = pytest.mark.gpu


def _chain(d, s, n_steps, ctx, tab):
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    for k in range(n_steps):
        ref = oracle.step(d["cfg"], d["groups"], tab, d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        got = s.step(d["now_ns"], d["v_token_ns"])
        _compare(got, ref, s.read_rows(debug=s.debug), ctx=f"{ctx} step {k}")
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]


def test_batch_bounds():
    from paper_2504_20068_b200 import Scheduler
    F = W.build_forest(95)
    X, _ = W.forest_training_set(96, 3000)
    rng = np.random.default_rng(96)
    g = rng.integers(0, 3000, len(X)).astype(np.uint32)
    d = W.pool_snapshot(1, 256, table_draws=1 << 12)
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=64, task_capacity=8)
    s.attach_forest(F)
    got, ms = s.qrf_bound(X.astype(np.uint32), g)
    R, qn, qd, lm = d["cfg"]["refine_interval"], d["cfg"]["q_num"], d["cfg"]["q_den"], int(d["table"]["l_max"])
    for i in range(len(X)):
        a = R * (int(g[i]) // R)
        x = [int(X[i, 0]), int(X[i, 1]), a, int(X[i, 3])]
        assert got[i] == max(oracle.qrf_quantile(F, x, a, qn, qd, lm), int(g[i]) + 1), i
    assert ms > 0
    s.close()


def test_random_pools_with_tiny_forests():
    from paper_2504_20068_b200 import Scheduler
    rng = np.random.default_rng(1101)
    for it in range(40):
        d = W.random_small_pool(rng, int(rng.integers(1, 120)))
        F = _tiny_forest(rng, int(rng.integers(1, 8)), int(rng.integers(0, 4)))
        F["samples"] = np.minimum(F["samples"], d["table"]["l_max"]).astype(np.uint32)
        tab = dict(d["table"], forest=F)
        n = len(d["pool"]["id"])
        nt = 0 if d["tasks"] is None else len(d["tasks"]["arrival_ns"])
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(n, 1), task_capacity=max(nt, 1), debug=True)
        s.attach_forest(F)
        s.load(d["pool"], d["tasks"])
        _chain(d, s, 3, f"iter {it}", tab)
        s.close()


def test_c3_pool_with_forest_then_back_to_table():
    from paper_2504_20068_b200 import Scheduler
    d = W.pool_snapshot(97, 100_000, table_draws=1 << 16)
    F = W.build_forest(98)
    tab = dict(d["table"], forest=F)
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=len(d["pool"]["id"]),
                  task_capacity=len(d["tasks"]["arrival_ns"]), debug=False)
    s.load(d["pool"], d["tasks"])
    s.attach_forest(F)                    # after the load: every cached bound is invalidated
    _chain(d, s, 3, "forest", tab)
    s.load(d["pool"], d["tasks"])
    s.attach_forest(None)
    _chain(d, s, 2, "table again", d["table"])
    s.close()


def test_replay_with_forest():
    from paper_2504_20068_b200 import Scheduler
    F = W.build_forest(99)
    for it in range(3):
        d = W.trace_mixed(500 + it, n_rows=400)
        tab = dict(d["table"], forest=F)
        rc = dict(d["rcfg"], n_steps=1500)
        ref = oracle.replay(d["cfg"], d["groups"], tab, d["trace"], rc, log=True)
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=512, task_capacity=64)
        s.attach_forest(F)
        res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
        _cmp(res[0], log[0], ref, f"replay {it}")
        s.close()
