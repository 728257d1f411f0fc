"""Pins of the oracle's NEXT-2 rows: the fairness blend priority' = (1-f) priority + f Fair(r)
(§4.3; SPEC blend_fair S:331-338; reading A47) and the online adaptation of the cutoff
p (reading A48)."""
from fractions import Fraction

import numpy as np

import oracle
import workloads as W
from . import _builders as B

MS, S_ = W.MS, W.S_


def _rows_with_keys(Rs, fair):
    """DDL rows with R(k) set directly, L-hat 200 at g = 101 (len_rem 99), v = 10 ms, eps = 10 ms:
    t_gen + eps = 1 s, so key = R exactly (as in the gate pins)"""
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 4 * S_, 0)])
    tab = B.table_from_counts([[0] * 199 + [5]])
    p = B.pool([dict(id=10 + i, L_i=5, g=101, pre=5, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE, override=R)
                for i, R in enumerate(Rs)])
    p["fair"] = np.array(fair, np.uint32)
    return groups, tab, p


def _step(Rs, fair, num, den, **cfg_over):
    groups, tab, p = _rows_with_keys(Rs, fair)
    cfg = W.default_config(**{**dict(token_budget=64, max_batch=len(Rs), prefill_chunk=8, refine_interval=1,
                                      eps_ns=10 * MS, fair_num=num, fair_den=den), **cfg_over})
    return oracle.step(cfg, groups, tab, 100 * S_, 10 * MS, p, None)


def test_blend_spec_examples():
    out = _step([10], [2], 1, 2)                # priority 10, Fair 2, f = 0.5 -> 6
    assert out["key"][0] == 6.0
    out = _step([10, 7], [2, 9], 0, 1)          # f = 0: unchanged
    assert list(out["key"]) == [10.0, 7.0]
    out = _step([10, 7], [2, 9], 3, 3)          # f = 1: Fair only
    assert list(out["key"]) == [2.0, 9.0]


def test_blend_reorders_by_fairness():
    """f = 1: the one-slot batch goes to the highest Fair; f = 0 to the highest priority"""
    assert list(_step([100, 50], [1, 9], 0, 1, max_batch=1)["batch_ids"]) == [10]
    out = _step([100, 50], [1, 9], 1, 1)
    assert list(_step([100, 50], [1, 9], 1, 1, max_batch=1)["batch_ids"]) == [11]
    assert out["bp"] == 1.0


def test_blend_within_half_ulp_of_exact_rational():
    """random pools: the blended key is the exact rational (1-f) key + f Fair within the three
    roundings of its definition (|err| <= 2^-51 relative), and f = 0 changes nothing"""
    rng = np.random.default_rng(801)
    checked = 0
    for it in range(60):
        d = W.random_small_pool(rng, int(rng.integers(2, 80)))
        n = len(d["pool"]["id"])
        d["pool"]["fair"] = rng.integers(0, 5000, n).astype(np.uint32)
        base = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        zero = oracle.step(dict(d["cfg"], fair_num=0, fair_den=7), d["groups"], d["table"], d["now_ns"],
                           d["v_token_ns"], d["pool"], d["tasks"])
        assert np.array_equal(base["batch_ids"], zero["batch_ids"]) and np.array_equal(base["key"], zero["key"])
        num, den = int(rng.integers(1, 10)), 10
        bl = oracle.step(dict(d["cfg"], fair_num=num, fair_den=den), d["groups"], d["table"], d["now_ns"],
                         d["v_token_ns"], d["pool"], d["tasks"])
        if base["status"] < 0:
            continue
        for r in np.nonzero(base["pending"])[0]:
            exact = Fraction(den - num, den) * Fraction(float(base["key"][r])) + Fraction(num, den) * int(d["pool"]["fair"][r])
            got = Fraction(float(bl["key"][r]))
            assert abs(got - exact) <= abs(exact) * Fraction(1, 2 ** 51) + Fraction(1, 2 ** 1000)
            checked += 1
    assert checked > 500


# ------------------------------------------------------------------------------------------
# online p (A48)
# ------------------------------------------------------------------------------------------

GRID = [80, 90, 95, 100]


def _mix(x):
    m = (1 << 64) - 1
    z = (x * 0x9E3779B97F4A7C15 + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _adapt_inputs():
    d = W.trace_mixed(5, n_rows=600, rate_per_s=25.0)
    d["cfg"] = dict(d["cfg"], frame_steps=5, max_batch=24, token_budget=2048)
    return d


def test_online_p_grid_order_then_greedy_argmax():
    """eps = 0: windows 0-3 try the grid in order; every later window takes the arm of the highest
    mean window goodput so far.  The window goodputs come from independent replays cut at the
    window boundaries (token goodput is cumulative)."""
    d = _adapt_inputs()
    W_steps = 2 * d["cfg"]["frame_steps"]        # window = 2 frames
    n_win = 9
    rc = dict(d["rcfg"], p_adapt=1, eps_num=0, eps_den=1, window_frames=2, seed=5, n_steps=W_steps * n_win)
    full = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
    assert full["steps"] == W_steps * n_win
    arms = [int(full["log"]["p_num"][k * W_steps]) for k in range(n_win)]
    for k in range(n_win):                       # one arm per window
        assert np.all(full["log"]["p_num"][k * W_steps:(k + 1) * W_steps] == arms[k])
    assert arms[:4] == GRID
    cum = [0] + [oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], dict(rc, n_steps=W_steps * (k + 1)))
                 ["token_goodput"] for k in range(n_win)]
    gs = {a: [] for a in GRID}
    for k in range(n_win):
        if k >= 4:
            means = {a: Fraction(sum(gs[a]), len(gs[a])) for a in GRID}
            best = max(GRID, key=lambda a: (means[a], -GRID.index(a)))
            assert arms[k] == best, (k, arms, means)
        gs[arms[k]].append(cum[k + 1] - cum[k])


def test_online_p_full_exploration_follows_the_counter_generator():
    d = _adapt_inputs()
    W_steps = d["cfg"]["frame_steps"]
    rc = dict(d["rcfg"], p_adapt=1, eps_num=1, eps_den=1, window_frames=1, seed=1234, n_steps=W_steps * 12)
    out = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
    arms = [int(out["log"]["p_num"][k * W_steps]) for k in range(12)]
    assert arms[:4] == GRID
    for k in range(4, 12):
        assert arms[k] == GRID[(_mix(1234 + k) >> 32) % 4], k


def test_online_p_off_is_the_fixed_cutoff():
    d = _adapt_inputs()
    rc = dict(d["rcfg"], n_steps=400)
    a = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
    assert np.all(a["log"]["p_num"] == d["cfg"]["p_num"])
