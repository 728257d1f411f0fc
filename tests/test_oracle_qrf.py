"""Pins of the oracle's NEXT-4 QRF length bound (§4.1; SPEC estimator S:92-158;
reading A50): worked values of predict_upper, the degenerate forest, the conditioning
on L > anchor and the clamp of (a2), quantile monotonicity, and brute force over tiny forests."""
import numpy as np

import oracle
import workloads as W
from . import _builders as B

LEAF = 0xFFFFFFFF


def _one_leaf(samples):
    return {"root": np.array([0], np.uint32), "feature": np.array([LEAF], np.uint32),
            "threshold": np.array([0], np.uint32), "left": np.array([len(samples)], np.uint32),
            "right": np.array([0], np.uint32), "samples": np.sort(np.array(samples, np.uint32))}


def test_spec_worked_values():
    F = _one_leaf(range(100, 201))                       # leaf pool {100..200}
    assert oracle.qrf_quantile(F, [1, 0, 0, 0], 0, 95, 100, 8192) == 195     # ceil(0.95 * 101) = 96th
    F = _one_leaf([100] * 40)                            # identical targets
    for qn in (1, 50, 95, 100):
        assert oracle.qrf_quantile(F, [7, 1, 0, 3], 0, qn, 100, 8192) == 100


def test_conditioning_and_l_max():
    F = _one_leaf([10, 20, 30, 40, 50])
    assert oracle.qrf_quantile(F, [1, 0, 20, 0], 20, 1, 1, 100) == 50     # q = 1: the largest above 20
    assert oracle.qrf_quantile(F, [1, 0, 20, 0], 20, 1, 3, 100) == 30     # ceil(3 / 3) = 1st above 20
    assert oracle.qrf_quantile(F, [1, 0, 50, 0], 50, 95, 100, 100) == 100  # nothing above: L_max (A7)


def _tiny_forest(rng, n_trees, depth):
    feat, thr, left, right, root, samples = [], [], [], [], [], []

    def grow(d):
        v = len(feat)
        feat.append(0); thr.append(0); left.append(0); right.append(0)
        if d < depth and rng.random() < 0.8:
            feat[v] = int(rng.integers(0, 4)); thr[v] = int(rng.integers(0, 60))
            left[v] = grow(d + 1); right[v] = grow(d + 1)
        else:
            ys = sorted(int(a) for a in rng.integers(1, 80, int(rng.integers(1, 7))))
            feat[v] = LEAF; thr[v] = len(samples); left[v] = len(ys)
            samples.extend(ys)
        return v
    for _ in range(n_trees):
        root.append(grow(0))
    u = lambda a: np.array(a, np.uint32)
    return {"root": u(root), "feature": u(feat), "threshold": u(thr), "left": u(left), "right": u(right),
            "samples": u(samples)}


def test_bruteforce_tiny_forests():
    rng = np.random.default_rng(1001)
    for it in range(300):
        F = _tiny_forest(rng, int(rng.integers(1, 6)), int(rng.integers(0, 4)))
        x = [int(a) for a in rng.integers(0, 60, 4)]
        anchor = int(rng.integers(0, 70))
        qn, qd = int(rng.integers(1, 101)), 100
        pooled = []
        for r in F["root"]:                                  # follow each tree by hand
            v = int(r)
            while F["feature"][v] != LEAF:
                v = int(F["left"][v] if x[F["feature"][v]] <= F["threshold"][v] else F["right"][v])
            off, cnt = int(F["threshold"][v]), int(F["left"][v])
            pooled += [int(a) for a in F["samples"][off:off + cnt]]
        above = sorted(a for a in pooled if a > anchor)
        exp = 90 if not above else above[-(-qn * len(above) // qd) - 1]
        assert oracle.qrf_quantile(F, x, anchor, qn, qd, 90) == exp, it


def test_monotone_in_q():
    F = W.build_forest(92, n_trees=8, n_train=2000)
    X, _ = W.forest_training_set(93, 200)
    for x in X:
        prev = 0
        for qn in (10, 50, 90, 95, 99, 100):
            v = oracle.qrf_quantile(F, x, int(x[2]), qn, 100, 8192)
            assert v >= prev
            prev = v


def test_step_uses_the_forest_with_the_clamp():
    """(a2) with a forest: L-hat = max(Q_q(forest pool | L > anchor), g + 1) for every pending row"""
    rng = np.random.default_rng(1002)
    for it in range(20):
        d = W.random_small_pool(rng, int(rng.integers(5, 80)))
        F = _tiny_forest(rng, 4, 3)
        tab = dict(d["table"], forest=F)
        out = oracle.step(d["cfg"], d["groups"], tab, d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        if out["status"] < 0:
            continue
        R = d["cfg"]["refine_interval"]
        for r in np.nonzero(out["pending"])[0]:
            g = int(d["pool"]["generated"][r])
            anchor = R * (g // R)
            x = [int(d["pool"]["input_len"][r]), int(d["pool"]["aux"][r]) & 0xFFFF, anchor,
                 int(d["pool"]["meta"][r]) & 0xFF]
            q = oracle.qrf_quantile(F, x, anchor, d["cfg"]["q_num"], d["cfg"]["q_den"], int(tab["l_max"]))
            assert out["lhat"][r] == max(q, g + 1)
    # the clamp of S:131: raw quantile 300 below generated 500 -> g + 1 (A5)
    groups = W.make_groups([(W.DDL, 0, 0, 100 * W.S_, 0)])
    tab = dict(B.table_from_counts([[1] * 8]), l_max=8, forest=_one_leaf([300] * 5))
    tab["l_max"] = 1000
    tab["edges"] = np.array([1000], np.uint32)
    tab["cum"] = np.array([[5]], np.uint32)
    p = B.pool([dict(id=1, L_i=10, g=500, pre=10, state=W.Q_RUNNING, flags=W.F_EVER)])
    cfg = W.default_config(token_budget=64, max_batch=4, prefill_chunk=8, refine_interval=1000)
    out = oracle.step(cfg, groups, tab, 10 * W.S_, W.MS, p, None)
    assert out["lhat"][0] == 501
