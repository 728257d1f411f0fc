"""GPU parity of NEXT-3 pattern-graph matching (jit_sched_match, reading A49) against the oracle.

The similarity is a mean of exp() terms: the device exp and the host libm exp may differ in the
last bit, so scores are compared within 1e-14 relative; the chosen pattern must equal the
oracle's except where the oracle's two best scores are themselves within that tolerance (then it
must be one of them).  Pruning (NoMatch) and exact ties are integer decisions: equal."""
import numpy as np
import pytest

import oracle
import workloads as W
from .test_parity_gpu import _compare

pytestmark = pytest.mark.gpu


def _sched(cfg=None, groups=None, table=None, cap=64, tcap=8):
    from paper_2504_20068_b200 import Scheduler
    d = W.pool_snapshot(1, 256, table_draws=1 << 12)
    return Scheduler(cfg or d["cfg"], groups if groups is not None else d["groups"],
                     table if table is not None else d["table"], capacity=cap, task_capacity=tcap)


def _check(store, queries, best, score):
    ob, os_ = oracle.match(store, queries)
    assert np.array_equal(best < 0, ob < 0)
    m = ob >= 0
    assert np.allclose(score[m], os_[m], rtol=1e-14, atol=0)
    scores = oracle.match_scores(store, queries) if (best != ob).any() else None
    for i in np.nonzero(best != ob)[0]:
        top = np.sort(scores[i])[::-1]
        assert top[0] - top[1] <= 1e-14 * top[0], (i, best[i], ob[i], top[:3])
        assert scores[i, best[i]] >= top[0] * (1 - 1e-14)


@pytest.mark.parametrize("n_patterns,n_queries", [(50, 500), (500, 4000), (1500, 2000)])
def test_random_stores(n_patterns, n_queries):
    store = W.pattern_store(71 + n_patterns, n_patterns=n_patterns)
    q = W.pattern_queries(72, store, n_queries)
    s = _sched()
    best, score = s.match(store, q)
    _check(store, q, best, score)
    assert (best < 0).sum() > 0 and (best >= 0).sum() > n_queries // 2
    s.close()


def test_exact_ties_and_no_match():
    T = W.TOOL
    store = {k: np.zeros((4, W.MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out", "t_ms")}
    store["n_stages"] = np.array([2, 2, 2, 3], np.uint32)
    for p in range(4):
        store["ident"][p, :3] = [1, T | 2, 3]
        store["in_len"][p, :3] = [100, 0, 50]
        store["out"][p, :3] = [200, 40, 10]
        store["t_ms"][p, :3] = [10, 20, 30]
    store["reuse"] = np.array([5, 9, 9, 1], np.uint32)
    q = {k: np.zeros((3, W.MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out")}
    q["stage"] = np.array([1, 0, 2], np.uint32)
    q["ident"][:, :3] = [1, T | 2, 3]
    q["ident"][1, 0] = 2                      # diverging identity: NoMatch
    q["out"][:, :2] = [200, 40]
    s = _sched()
    best, score = s.match(store, q)
    assert list(best) == [1, -1, 3] and score[0] == 1.0 and score[1] == -1.0
    _check(store, q, best, score)
    s.close()


def test_apply_to_resident_tasks_then_step():
    """matched stage structures become the tasks' (n_stages, stage times) -> phi -> D_s -> keys"""
    d = W.pool_snapshot(73, 30_000, table_draws=1 << 14)
    nt = len(d["tasks"]["arrival_ns"])
    store = W.pattern_store(74, n_patterns=400)
    q = W.pattern_queries(75, store, nt, foreign=0.1)
    tasks = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["tasks"].items()}
    tasks["cur_stage"] = q["stage"].copy()
    tasks["n_stages"] = np.maximum(tasks["n_stages"], q["stage"] + 1).astype(np.uint32)
    q["task"] = np.arange(nt, dtype=np.uint32)
    from paper_2504_20068_b200 import Scheduler
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=len(d["pool"]["id"]), task_capacity=nt, debug=True)
    s.load(d["pool"], tasks)
    best, score = s.match(store, q, apply=True)
    got = s.step(d["now_ns"], d["v_token_ns"])
    rows = s.read_rows()
    ob, _ = oracle.match(store, q)
    # where the device's choice differs only within the exp() tolerance, use the device's choice
    # (both are correct); its stage structure is what the oracle step then sees
    _check(store, q, best, score)
    t2 = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in tasks.items()}
    for t in np.nonzero(best >= 0)[0]:
        b = best[t]
        t2["n_stages"][t] = store["n_stages"][b]
        t2["pattern_ms"][t] = np.where(np.arange(W.MAX_STAGES) < store["n_stages"][b], store["t_ms"][b], 0)
    ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], t2)
    _compare(got, ref, rows, ctx="apply")
    # a query whose stage is not its task's current stage is refused
    bad = dict(q, stage=(q["stage"] + 1).astype(np.uint32))
    from paper_2504_20068_b200.jitsched import JitSchedError
    with pytest.raises(JitSchedError):
        s.match(store, bad, apply=True)
    s.close()
