"""Pins of the oracle's NEXT-3 pattern-graph matcher (§4.1; SPEC patterns S:160-263;
reading A49): kernel values, prefix pruning, the mean aggregation, self-matches and the
tie-break, checked against closed forms and properties (not a second matcher)."""
import math

import numpy as np

import oracle
import workloads as W

T = W.TOOL


def _store(rows, reuse=None):
    """rows: list of stage lists [(ident, in_len, out, t_ms), ...]"""
    n = len(rows)
    st = {k: np.zeros((n, W.MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out", "t_ms")}
    st["n_stages"] = np.array([len(r) for r in rows], np.uint32)
    for p, r in enumerate(rows):
        for u, (i, a, o, t) in enumerate(r):
            st["ident"][p, u], st["in_len"][p, u], st["out"][p, u], st["t_ms"][p, u] = i, a, o, t
    st["reuse"] = np.array(reuse if reuse is not None else [1] * n, np.uint32)
    return st


def _query(stages, s):
    q = {k: np.zeros((1, W.MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out")}
    q["stage"] = np.array([s], np.uint32)
    for u, (i, a, o) in enumerate(stages):
        q["ident"][0, u], q["in_len"][0, u], q["out"][0, u] = i, a, o
    return q


def test_kernel_values():
    assert oracle.kernel_sim(100, 100) == 1.0                       # zero distance
    assert oracle.kernel_sim(300, 400) == math.exp(-0.5)            # sigma = 0.25 * 400 = 100
    assert oracle.kernel_sim(0, 1) == math.exp(-0.5)                # sigma floor 1 token
    assert oracle.kernel_sim(400, 300) == oracle.kernel_sim(300, 400)
    assert oracle.kernel_sim(100, 200) == math.exp(-(100 ** 2) / (2 * 50.0 ** 2))


def test_kind_mismatch_is_pruned():
    st = _store([[(0, 500, 200, 1000), (T | 2, 0, 300, 500)]])
    b, s = oracle.match(st, _query([(0, 500, 200), (2, 10, 0)], 1))      # an LLM where the pattern has a tool
    assert b[0] == -1 and s[0] == -1.0
    b, s = oracle.match(st, _query([(0, 500, 200), (T | 3, 0, 0)], 1))   # another tool id: diverging prefix
    assert b[0] == -1
    b, s = oracle.match(st, _query([(0, 500, 0)] * 3, 2))                # more stages than the pattern
    assert b[0] == -1


def test_mean_of_node_and_edge_terms():
    # stage 0 LLM out 300 vs 400 -> e^-1/2; stage 1 LLM edge in 100 vs 100 -> 1
    st = _store([[(1, 50, 400, 10), (2, 100, 10, 10), (3, 5, 5, 5)]])
    b, s = oracle.match(st, _query([(1, 50, 300), (2, 100, 0)], 1))
    assert b[0] == 0 and s[0] == (math.exp(-0.5) + 1.0) / 2.0
    # stage 1 a tool: no edge term
    st = _store([[(1, 50, 400, 10), (T | 2, 0, 10, 10)]])
    b, s = oracle.match(st, _query([(1, 50, 300), (T | 2, 0, 0)], 1))
    assert s[0] == math.exp(-0.5)
    # stage 0 revealed only: no term at all -> 1 for every surviving pattern
    b, s = oracle.match(st, _query([(1, 999, 0)], 0))
    assert b[0] == 0 and s[0] == 1.0


def test_tie_break_reuse_then_index():
    row = [(1, 50, 400, 10), (2, 100, 10, 10)]
    q = _query([(1, 50, 400), (2, 100, 0)], 1)
    assert oracle.match(_store([row, row, row], reuse=[3, 9, 9]), q)[0][0] == 1
    assert oracle.match(_store([row, row], reuse=[4, 4]), q)[0][0] == 0


def test_self_match_and_pruning_soundness():
    st = W.pattern_store(63, n_patterns=300)
    rng = np.random.default_rng(63)
    n = 200
    picks = rng.integers(0, 300, n)
    q = {k: np.zeros((n, W.MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out")}
    q["stage"] = np.zeros(n, np.uint32)
    for i, p in enumerate(picks):                   # exact prefixes of stored patterns
        s = int(rng.integers(0, st["n_stages"][p]))
        q["stage"][i] = s
        q["ident"][i, :s + 1] = st["ident"][p, :s + 1]
        q["in_len"][i, :s + 1] = st["in_len"][p, :s + 1]
        q["out"][i, :s] = st["out"][p, :s]
    best, score = oracle.match(st, q)
    scores = oracle.match_scores(st, q)
    for i, p in enumerate(picks):
        s = int(q["stage"][i])
        assert score[i] == 1.0 and scores[i, p] == 1.0
        # pruning is exactly "same identities on stages 0..s and more than s stages"
        same = (st["n_stages"] > s) & np.all(st["ident"][:, :s + 1] == q["ident"][i, :s + 1], axis=1)
        assert np.array_equal(scores[i] >= 0, same)
        assert np.all(scores[i][same] <= 1.0)
        # the best is a maximum, then the most reused, then the lowest index
        top = np.nonzero(scores[i] == scores[i].max())[0]
        r = st["reuse"][top]
        assert best[i] == top[r == r.max()][0]
