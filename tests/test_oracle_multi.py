"""Pins of the oracle's NEXT-2 power-of-K step (§4.3; SPEC expand_multi_model S:322-330;
reading A51): K = M = 1 is the plain step; a request proposed by several replicas lands on the
fastest one; no request keeps a live dummy outside its replica; the proposals are exactly each
replica's plain GMAX step."""
import numpy as np

import oracle
import workloads as W


def _small(rng, n):
    d = W.random_small_pool(rng, n, with_tasks=False)
    return d


def test_single_replica_is_the_plain_step():
    rng = np.random.default_rng(1201)
    for it in range(40):
        d = _small(rng, int(rng.integers(1, 80)))
        pools = W.replica_pools(d, 1, 1, seed=it)
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pools[0], None)
        got = oracle.multi_step(d["cfg"], d["groups"], d["table"], d["now_ns"], [d["v_token_ns"]], pools)[0]
        for k in ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star"):
            assert got[k] == ref[k]
        for k in ("batch_ids", "batch_tokens", "meta", "aux"):
            assert np.array_equal(got[k], ref[k])


def test_assignment_to_the_fastest_replica_and_sibling_removal():
    rng = np.random.default_rng(1202)
    seen_conflict = 0
    for it in range(60):
        d = _small(rng, int(rng.integers(5, 90)))
        M = int(rng.integers(2, 5))
        K = int(rng.integers(1, M + 1))
        pools = W.replica_pools(d, M, K, seed=100 + it)
        vs = [int(x) for x in rng.choice([5, 10, 10, 20], M) * W.MS]
        # the proposals: each replica's plain step on its own dummies with its own v_token
        props = [oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], vs[m], pools[m], None) for m in range(M)]
        got = oracle.multi_step(d["cfg"], d["groups"], d["table"], d["now_ns"], vs, pools)
        winner = {}
        for m in range(M):
            if props[m]["status"] != 0:
                continue
            for i in props[m]["batch_ids"]:
                w = winner.get(int(i))
                if w is None or (vs[m], m) < (vs[w], w):
                    winner[int(i)] = m
        seen_conflict += sum(1 for i in winner if sum(int(i) in set(props[m]["batch_ids"]) for m in range(M)
                                                      if props[m]["status"] == 0) > 1)
        for m in range(M):
            if props[m]["status"] != 0:
                continue
            keep = np.array([winner[int(i)] == m for i in props[m]["batch_ids"]], bool)
            assert np.array_equal(got[m]["batch_ids"], props[m]["batch_ids"][keep])
            assert got[m]["total_tokens"] == int(props[m]["batch_tokens"][keep].sum())
            assert got[m]["b_star"] == props[m]["b_star"] and got[m]["bp"] == props[m]["bp"]
            # sibling removal: every dummy of a request assigned elsewhere is Moved
            st = (got[m]["meta"] >> 8) & 0xF
            for r, i in enumerate(pools[m]["id"]):
                w = winner.get(int(i))
                if w is not None and w != m:
                    assert st[r] == W.Q_MOVED
                elif st[r] == W.Q_MOVED:
                    raise AssertionError("moved without an assignment elsewhere")
        # no request is in two final batches
        ids = np.concatenate([g["batch_ids"] for g in got])
        assert len(ids) == len(set(ids.tolist()))
    assert seen_conflict > 20
