"""GPU parity of NEXT-2 power-of-K over M replicas (§4.3; reading A51): each replica's
handle steps over its dummies with its own v_token, the proposals are exchanged and reconciled on
the device (multi.cuh) -- batches, totals, Moved dummies and steps_waited compared with the
oracle's multi_step, bit-exact, over chains of steps."""
import numpy as np
import pytest

import oracle
import workloads as W
from paper_2504_20068_b200 import Scheduler
from paper_2504_20068_b200.jitsched import multi_step

pytestmark = pytest.mark.gpu


def _scheds(d, pools, debug=False):
    out = []
    for p in pools:
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=max(len(p["id"]), 1), task_capacity=1, debug=debug)
        s.load(p, None)
        out.append(s)
    return out


def _chain(d, pools, vs, n_steps, ctx, debug=False):
    M = len(pools)
    ref_pools = [{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()} for p in pools]
    ss = _scheds(d, pools, debug)
    n_conf = 0
    for k in range(n_steps):
        ref = oracle.multi_step(d["cfg"], d["groups"], d["table"], d["now_ns"] + k * 1000, vs, ref_pools)
        got = multi_step(ss, d["now_ns"] + k * 1000, vs)
        for m in range(M):
            c = f"{ctx} step {k} replica {m}"
            assert got[m]["status"] == ref[m]["status"], (c, got[m]["status"], ref[m]["status"])
            assert got[m]["n_pending"] == ref[m]["n_pending"], c
            if ref[m]["status"] == 0:
                for key in ("n_selected", "total_tokens", "b_star", "n_candidates"):
                    assert got[m][key] == ref[m][key], (c, key, got[m][key], ref[m][key])
                assert np.float64(got[m]["bp"]).view(np.uint64) == np.float64(ref[m]["bp"]).view(np.uint64), c
                assert np.array_equal(got[m]["batch_ids"], ref[m]["batch_ids"]), c
                assert np.array_equal(got[m]["batch_tokens"], ref[m]["batch_tokens"]), c
                assert np.array_equal(got[m]["batch_rows"], ref[m]["batch_rows"]), c
            rows = ss[m].read_rows(debug=False)
            assert np.array_equal(rows["meta"], ref[m]["meta"]), c
            assert np.array_equal(rows["aux"], ref[m]["aux"]), c
            ref_pools[m]["meta"], ref_pools[m]["aux"] = ref[m]["meta"], ref[m]["aux"]
            n_conf += int(((ref[m]["meta"] >> 8) & 0xF == W.Q_MOVED).sum())
        ids = np.concatenate([g["batch_ids"] for g in got])
        assert len(ids) == len(set(ids.tolist())), ctx            # no request in two batches
    for s in ss:
        s.close()
    return n_conf


def test_multi_random_pools():
    rng = np.random.default_rng(1301)
    moved = 0
    for it in range(40):
        d = W.random_small_pool(rng, int(rng.integers(5, 150)), with_tasks=False)
        M = int(rng.integers(1, 6))
        K = int(rng.integers(1, M + 1))
        pools = W.replica_pools(d, M, K, seed=300 + it)
        if any(len(p["id"]) == 0 for p in pools):
            continue
        vs = [int(x) for x in rng.choice([5, 10, 10, 20], M) * W.MS]
        moved += _chain(d, pools, vs, 3, f"iter {it} M={M} K={K}", debug=(it % 4 == 0))
    assert moved > 20                                              # sibling removal was exercised


def test_multi_equal_v_ties_to_lower_index():
    rng = np.random.default_rng(1302)
    d = W.random_small_pool(rng, 120, with_tasks=False)
    pools = W.replica_pools(d, 4, 4, seed=7)                       # every request on every replica
    assert _chain(d, pools, [10 * W.MS] * 4, 3, "equal v") > 0


@pytest.mark.parametrize("M,K", [(4, 2), (8, 2)])
def test_multi_c3_scale(M, K):
    d = W.pool_snapshot(1303, 200_000, table_draws=1 << 16)
    pools = W.replica_pools(d, M, K, seed=M * 10 + K)
    vs = [int(v) for v in np.linspace(0.8, 1.2, M) * d["v_token_ns"]]
    assert _chain(d, pools, vs, 2, f"C3 M={M} K={K}") > 0
