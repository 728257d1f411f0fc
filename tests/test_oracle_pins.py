"""Pins of the CPU oracle against what the paper / SPEC worked examples / mathematics fix.

Every expected value comes from tests/golden/pins.json (hand-written, each with its citation),
from a closed form, or from an independent brute force over tiny inputs.  Nothing here
comes from the CUDA path.  Marked "not gpu" (runs on CPU).
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from tests import _builders as B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
S_, MS = W.S_, W.MS
V_UNIT = 999_999_000  # with len_rem = 1 and eps = 1000 ns: t_gen + eps = 10^9, so key == G' exactly


def _cfg(**kw):
    return W.default_config(**kw)


# ------------------------------------------------------------------------------------------
# (a2) conditional-quantile length bound, §4.1
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", GOLD["length_bound"], ids=lambda c: c["cite"][:40])
def test_length_bound_golden(case):
    tab = B.table_from_supports([case["support"]], case["l_max"])
    got = oracle.length_bound(tab, 0, case["g"], case["R"], *case["q"])
    assert got == case["expect"], case["cite"]


def _brute_bound(counts, g, R, qn, qd, l_max):
    anchor = R * (g // R)
    ms = [L for L in range(1, len(counts) + 1) for _ in range(int(counts[L - 1])) if L > anchor]
    if not ms:
        q = l_max
    else:
        ms.sort()
        k = (qn * len(ms) + qd - 1) // qd          # ceil(q M)-th order statistic (type 1)
        q = ms[k - 1]
    return max(q, g + 1)


def test_length_bound_bruteforce_random_histograms():
    rng = np.random.default_rng(11)
    for _ in range(400):
        l_max = int(rng.integers(1, 60))
        counts = rng.integers(0, 4, l_max) * (rng.random(l_max) < 0.6)
        tab = B.table_from_counts([counts])
        g = int(rng.integers(0, l_max + 5))
        R = int(rng.choice([1, 3, 50]))
        qd = int(rng.choice([100, 7, 1]))
        qn = int(rng.integers(1, qd + 1))
        assert oracle.length_bound(tab, 0, g, R, qn, qd) == _brute_bound(counts, g, R, qn, qd, l_max)


def test_length_bound_monotone_in_q_and_clamped():
    rng = np.random.default_rng(12)
    for _ in range(100):
        counts = rng.integers(0, 5, 40)
        tab = B.table_from_counts([counts])
        g = int(rng.integers(0, 45))
        vals = [oracle.length_bound(tab, 0, g, 1, qn, 100) for qn in (50, 80, 95, 100)]
        assert vals == sorted(vals)               # S:142 quantile monotonicity
        assert min(vals) >= g + 1                 # S:143 clamp safety (A5)


# ------------------------------------------------------------------------------------------
# (a3)/(a5) key, rate, starvation
# ------------------------------------------------------------------------------------------

def _one_ddl(G, len_rem_tab_point, g, v, waited=0, e2el=10 ** 6 * S_, delta=1, frame=50, eps=1000):
    groups = W.make_groups([(W.DDL, 0, 0, e2el, 0)])
    counts = np.zeros(max(len_rem_tab_point, 2), np.int64)
    counts[len_rem_tab_point - 1] = 1
    tab = B.table_from_counts([counts])
    p = B.pool([dict(id=7, L_i=3, pre=3, g=g, group=0, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE,
                     override=G, waited=waited, arrival=0)])
    cfg = _cfg(delta_starve=delta, frame_steps=frame, eps_ns=eps)
    return oracle.step(cfg, groups, tab, 10 * S_, v, p)


def test_key_spec_analyze_example():
    case = GOLD["key"][0]
    out = _one_ddl(case["G"], 1, 0, case["t_gen_ns"], eps=case["eps_ns"])
    assert out["key"][0] == case["expect"]
    # the exact rational, correctly rounded once
    assert out["key"][0] == float(Fraction(case["G"] * 10 ** 9, case["t_gen_ns"] + case["eps_ns"]))


def test_starvation_inflation_spec_example():
    case = GOLD["starvation"][0]
    out = _one_ddl(case["G"], 1, 0, V_UNIT, waited=case["frames"] * 50, delta=case["delta"], frame=50)
    assert out["key"][0] == case["expect_G"]
    out2 = _one_ddl(case["G"], 1, 0, V_UNIT, waited=case["frames"] * 50 - 1, delta=case["delta"], frame=50)
    assert out2["key"][0] == case["expect_G"] - 1      # floor(waited / Delta)


def test_lat_on_schedule_rate_is_one_over_tbt():
    """for latency-sensitive requests the TBT defines the per-token bandwidth; with reading
    A9 an on-schedule stream (now = a + TTFT + (g-1) TBT) has rate * TBT = 1 exactly."""
    ttft, tbt = 2 * S_, 100 * MS
    groups = W.make_groups([(W.LAT, ttft, tbt, 0, 0)])
    tab = B.table_from_supports([(300, 300)], 512)
    for g in (1, 7, 120):
        now = ttft + (g - 1) * tbt
        p = B.pool([dict(id=1, L_i=10, pre=10, g=g, group=0, state=W.Q_RUNNING, flags=W.F_EVER, arrival=0)])
        out = oracle.step(_cfg(), groups, tab, now, 15 * MS, p)
        assert out["lhat"][0] == 300
        assert out["t_rem"][0] == (300 - g) * tbt
        assert out["rate"][0] * tbt == 10 ** 9


def test_adversary_priorities():
    """with M=100, T=10, delta=1, A's priority is M/T = 10 per unit and B's 1/delta = 1."""
    e = W.edf_adversary()
    tr = e["trace"]
    p = B.pool([dict(id=i, L_i=1, g=0, pre=0, group=int(tr["group"][i]), dist_row=int(tr["dist_row"][i]),
                     flags=W.F_OVERRIDE, override=int(tr["override_R"][i]), arrival=0) for i in range(2)])
    out = oracle.step(e["cfg"], e["groups"], e["table"], 0, 10 * MS, p)
    ka, kb = out["key"]
    v = 10 * MS
    assert ka == float(Fraction(100 * 10 ** 9, 10 * v + 1000)) and kb == float(Fraction(10 ** 9, v + 1000))
    assert abs(ka / kb - 10.0) < 1e-3          # M/T : 1/delta = 10 : 1 up to eps


def test_expired_request_has_zero_goodput():
    groups = W.make_groups([(W.DDL, 0, 0, 5 * S_, 0)])
    tab = B.table_from_supports([(20, 20)], 64)
    p = B.pool([dict(id=1, L_i=4, pre=4, g=3, group=0, state=W.Q_RUNNING, flags=W.F_EVER, arrival=0, waited=100)])
    out = oracle.step(_cfg(delta_starve=1, frame_steps=50), groups, tab, 6 * S_, V_UNIT // 17, p)
    # G = 0 (A22), only starvation (2 frames) remains
    assert out["key"][0] == float(Fraction(2 * 10 ** 9, 17 * (V_UNIT // 17) + 1000))
    assert out["rate"][0] == float("inf")


# ------------------------------------------------------------------------------------------
# (a7)-(a9) selection
# ------------------------------------------------------------------------------------------

def _keyed_pool(keys, costs, lens, ids=None):
    """Rows whose key equals the given integer G' exactly (V_UNIT trick) with given cost/len."""
    rows = []
    for i, (k, c, L) in enumerate(zip(keys, costs, lens)):
        if c == 1:
            rows.append(dict(id=i if ids is None else ids[i], L_i=L, pre=L, g=5, group=0, state=W.Q_RUNNING,
                             flags=W.F_EVER | W.F_OVERRIDE, override=k))
        else:
            rows.append(dict(id=i if ids is None else ids[i], L_i=L, pre=L - c, g=0, group=0,
                             state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE, override=k))
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 6 * S_, 0)])
    tab = B.table_from_supports([(1, 1)], 8)    # point mass at 1: Lhat = g+1, len_rem = 1
    return B.pool(rows), groups, tab


def test_select_spec_length_window():
    case = GOLD["select_lengths"]
    n = len(case["lengths"])
    p, groups, tab = _keyed_pool([7] * n, [1] * n, case["lengths"])
    cfg = _cfg(token_budget=case["B"], max_batch=case["B"], prefill_chunk=1)
    out = oracle.step(cfg, groups, tab, S_, V_UNIT, p)
    assert list(p["input_len"][out["batch_rows"]]) == case["expect_lengths"]


@pytest.mark.parametrize("ci", [0, 1])
def test_select_budget_worked_example(ci):
    case = GOLD["select_budget"]
    c = case["cases"][ci]
    p, groups, tab = _keyed_pool(case["keys"], case["costs"], case["lens"])
    cfg = _cfg(token_budget=case["tau"], max_batch=8, prefill_chunk=8, p_num=c["p"][0], p_den=c["p"][1])
    out = oracle.step(cfg, groups, tab, S_, V_UNIT, p)
    assert out["b_star"] == c["expect_b_star"]
    assert out["bp"] == c["expect_bp"]
    assert sorted(out["batch_ids"].tolist()) == c["expect_batch"]


def test_select_p1_full_queue_is_topB():
    """p = 1 and |queue| = B -> exactly the top-B set."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(1, 10))
        keys = rng.choice(np.arange(1, 500), n, replace=False)
        p, groups, tab = _keyed_pool(keys.tolist(), [1] * n, rng.integers(1, 100, n).tolist())
        cfg = _cfg(token_budget=n, max_batch=n, prefill_chunk=1, p_num=1, p_den=1)
        out = oracle.step(cfg, groups, tab, S_, V_UNIT, p)
        assert sorted(out["batch_ids"].tolist()) == list(range(n))


def test_select_bruteforce_max_sum_subset():
    """p = 1, unit costs, distinct positive keys -> GMAX's batch is the
    max-sum subset of size <= B (exhaustive over all subsets, n <= 12)."""
    rng = np.random.default_rng(6)
    for _ in range(300):
        n = int(rng.integers(1, 13))
        Bsz = int(rng.integers(1, n + 1))
        keys = rng.choice(np.arange(1, 2000), n, replace=False)
        p, groups, tab = _keyed_pool(keys.tolist(), [1] * n, rng.integers(1, 50, n).tolist())
        cfg = _cfg(token_budget=Bsz, max_batch=Bsz, prefill_chunk=1, p_num=1, p_den=1)
        out = oracle.step(cfg, groups, tab, S_, V_UNIT, p)
        best = max(sum(keys[list(s)]) for r in range(0, Bsz + 1) for s in itertools.combinations(range(n), r))
        assert sum(keys[out["batch_ids"]]) == best


def _fx(k):
    return int(Fraction(min(k, 2 ** 31 - 1)) * 2 ** 32)


def _check_selection_properties(d, out):
    cfg, pool = d["cfg"], d["pool"]
    pend = out["pending"].astype(bool)
    if out["status"] == 1:
        assert not pend.any()
        return
    assert out["status"] == 0
    rows = np.nonzero(pend)[0]
    key, cost = out["key"], out["cost"]
    # B* and bp by definition (A14): order (key desc, id asc), largest prefix within tau and B_max
    order = sorted(rows, key=lambda r: (-key[r], pool["id"][r]))
    m, s = 0, 0
    while m < len(order) and m + 1 <= cfg["max_batch"] and s + cost[order[m]] <= cfg["token_budget"]:
        s += cost[order[m]]
        m += 1
    assert out["b_star"] == m
    assert out["bp"] == key[order[m - 1]]
    thr = (cfg["p_num"] / cfg["p_den"]) * out["bp"]
    assert out["thr"] == thr
    cd = [r for r in rows if key[r] >= thr]
    assert out["n_candidates"] == len(cd)
    lenf = (lambda r: int(pool["input_len"][r]) + int(pool["generated"][r])) if cfg["len_key"] else \
        (lambda r: int(pool["input_len"][r]))
    cd.sort(key=lambda r: (lenf(r), pool["id"][r]))
    sel = list(out["batch_rows"])
    # surrogate property: every selected key >= thr; budget respected
    assert all(key[r] >= thr for r in sel)
    assert sum(int(cost[r]) for r in sel) <= cfg["token_budget"] and len(sel) <= cfg["max_batch"]
    # contiguity in (len, id) order and optimality over EVERY feasible contiguous window
    i0 = cd.index(sel[0])
    assert cd[i0:i0 + len(sel)] == sel
    best, first = -1, None
    for i in range(len(cd)):
        acc, c = 0, 0
        for j in range(i, len(cd)):
            c += int(cost[cd[j]])
            if c > cfg["token_budget"] or j - i + 1 > cfg["max_batch"]:
                break
            acc += _fx(key[cd[j]])
            if acc > best:
                best, first = acc, i
    score = sum(_fx(key[r]) for r in sel)
    assert score == best and i0 == first     # first maximum (strict '>')


def test_selection_properties_random_pools():
    rng = np.random.default_rng(7)
    for it in range(400):
        d = W.random_small_pool(rng, int(rng.integers(1, 40)), tie_heavy=(it % 5 == 0))
        out = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        _check_selection_properties(d, out)


def test_delta_invariance_of_plan():
    """S:351 / P:463-467: the priority has no Delta, so the plan is Delta-invariant (no starvation)."""
    rng = np.random.default_rng(8)
    for _ in range(100):
        d = W.random_small_pool(rng, 20)
        outs = []
        for frame in (1, 50, 1000):
            cfg = dict(d["cfg"], frame_steps=frame, delta_starve=0)
            outs.append(oracle.step(cfg, d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"],
                                    d["tasks"])["batch_ids"].tolist())
        assert outs[0] == outs[1] == outs[2]


def test_cutoff_p1_large_budget_returns_whole_queue():
    """with p = 1 and B >= |queue| the whole queue is selected."""
    rng = np.random.default_rng(9)
    for _ in range(50):
        d = W.random_small_pool(rng, 15)
        cfg = dict(d["cfg"], p_num=1, p_den=1, token_budget=10 ** 6, max_batch=1000, prefill_chunk=1000)
        out = oracle.step(cfg, d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        if out["status"] == 0:
            assert out["n_selected"] == out["n_pending"]


def test_admission_strict_bound():
    """P:545 / S:410-412: waited 5.1 s -> dropped, 4.9 s and exactly 5.0 s (A29) kept; running never dropped."""
    groups = W.make_groups([(W.DDL, 0, 0, 100 * S_, 0)])
    tab = B.table_from_supports([(5, 5)], 8)
    now = 10 * S_
    p = B.pool([dict(id=0, L_i=2, arrival=now - 5_100_000_000), dict(id=1, L_i=2, arrival=now - 4_900_000_000),
                dict(id=2, L_i=2, arrival=now - 5 * S_),
                dict(id=3, L_i=2, pre=2, g=1, arrival=0, state=W.Q_RUNNING, flags=W.F_EVER)])
    out = oracle.step(_cfg(), groups, tab, now, 15 * MS, p)
    assert out["n_dropped_now"] == 1
    assert (out["meta"][0] >> 8) & 0xF == W.Q_DROPPED
    assert sorted(out["batch_ids"].tolist()) == [1, 2, 3]


# ------------------------------------------------------------------------------------------
# (a4) compound requests
# ------------------------------------------------------------------------------------------

def test_phi_sub_deadline_example():
    case = GOLD["phi"]
    groups = W.make_groups([(W.CMP, 0, 0, 10 * S_, 0)])
    tab = B.table_from_supports([(50, 50)], 64)
    a_c, now = 0, 7 * S_
    p = B.pool([dict(id=0, L_i=5, pre=5, g=2, group=0, state=W.Q_RUNNING, flags=W.F_EVER | W.F_COMPOUND, task=0)])
    pat = np.zeros((1, 8), np.uint32)
    pat[0, :3] = case["pattern_ms"]
    tasks = {"call_off": np.array([0, 1], np.uint32), "arrival_ns": np.array([a_c], np.int64),
             "deadline_ns": np.array([case["D_ns"]], np.int64), "cur_stage": np.array([case["s"]], np.uint32),
             "n_stages": np.array([3], np.uint32), "pattern_ms": pat, "goodput_done": np.zeros(1, np.uint64)}
    out = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, tasks)
    assert out["t_rem"][0] == a_c + case["expect_Ds_ns"] - now


def test_single_call_task_equals_ddl():
    """A single-call task is the plain DDL computation with E2EL = D_s."""
    rng = np.random.default_rng(10)
    for _ in range(50):
        L_i, g = int(rng.integers(1, 30)), int(rng.integers(0, 30))
        D = int(rng.integers(20, 200)) * S_
        a_c = 0
        now = int(rng.integers(1, 15)) * S_
        pat = np.zeros((1, 8), np.uint32)
        pat[0, :4] = rng.integers(1, 1000, 4)
        s = int(rng.integers(0, 4))
        Ds = D * int(pat[0, :s + 1].sum()) // int(pat[0, :4].sum())
        waited = int(rng.integers(0, 300))
        counts = rng.integers(0, 3, 64)
        counts[-1] += 1
        tab = B.table_from_counts([counts])
        groups = W.make_groups([(W.CMP, 0, 0, D, 0), (W.DDL, 0, 0, Ds, 0)])
        st = dict(L_i=L_i, pre=L_i, g=g, state=W.Q_RUNNING, waited=waited, arrival=a_c)
        p = B.pool([dict(id=0, group=0, flags=W.F_EVER | W.F_COMPOUND, task=0, **st),
                    dict(id=1, group=1, flags=W.F_EVER, **st)])
        tasks = {"call_off": np.array([0, 1], np.uint32), "arrival_ns": np.array([a_c], np.int64),
                 "deadline_ns": np.array([10 ** 6 * S_], np.int64), "cur_stage": np.array([s], np.uint32),
                 "n_stages": np.array([4], np.uint32), "pattern_ms": pat, "goodput_done": np.zeros(1, np.uint64)}
        # use the same D for the task deadline so that D_s = Ds
        tasks["deadline_ns"][0] = D
        out = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, tasks)
        if Ds + a_c - now > 0 and a_c + D > now:
            assert out["t_rem"][0] == out["t_rem"][1]
            assert out["key"][0] == out["key"][1]
            assert out["rate"][0] == out["rate"][1]


def test_compound_aggregation_bruteforce():
    """len_rem and bandwidth are aggregated over all pending calls of the current stage."""
    rng = np.random.default_rng(13)
    checked = 0
    for _ in range(300):
        d = W.random_small_pool(rng, int(rng.integers(6, 30)))
        if d["tasks"] is None:
            continue
        out = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        if out["status"] != 0:
            continue
        T, pool, cfg, G = d["tasks"], d["pool"], d["cfg"], d["groups"]
        for t in range(len(T["arrival_ns"])):
            rows = [r for r in range(T["call_off"][t], T["call_off"][t + 1]) if out["pending"][r]]
            if not rows:
                continue
            Tsum = sum(int(out["lhat"][r]) - int(pool["generated"][r]) for r in rows)
            gr = lambda r: int(pool["meta"][r]) & 0xFF
            Gcur = sum(int(G["w_in"][gr(r)]) * int(pool["input_len"][r]) + int(G["w_out"][gr(r)]) * int(out["lhat"][r])
                       for r in rows)
            Gt = int(T["goodput_done"][t]) + Gcur
            if T["arrival_ns"][t] + T["deadline_ns"][t] <= d["now_ns"]:
                Gt = 0
            t_gen = Tsum * d["v_token_ns"]
            S = int(T["n_stages"][t]); s = int(T["cur_stage"][t])
            Ds = int(T["deadline_ns"][t]) * int(T["pattern_ms"][t][:s + 1].sum()) // int(T["pattern_ms"][t][:S].sum())
            trem = int(T["arrival_ns"][t]) + Ds - d["now_ns"]
            if cfg["appb_filter"] and t_gen > max(trem, 0):
                Gt = 0
            for r in rows:
                Gp = Gt + cfg["delta_starve"] * ((int(pool["aux"][r]) >> 16) // cfg["frame_steps"])
                assert out["key"][r] == float(Fraction(Gp * 10 ** 9, t_gen + cfg["eps_ns"]))
                assert out["t_rem"][r] == trem
                checked += 1
    assert checked > 50


# ------------------------------------------------------------------------------------------
# (a10) replay and goodput accounting
# ------------------------------------------------------------------------------------------

def test_replay_single_ddl_closed_form():
    case = GOLD["replay_single_ddl"]
    groups = W.make_groups([(W.DDL, 0, 0, 20 * S_, 0)])
    tab = B.table_from_supports([(10, 10)], 64)
    tr = B.single_trace([dict(arrival_ns=0, input_len=case["L_i"], true_out=case["L_o"], group=0, dist_row=0)])
    out = oracle.replay(_cfg(token_budget=8192, max_batch=256), groups, tab, tr, B.default_rcfg())
    assert out["sim_end_ns"] == case["expect_end_ns"]
    assert out["token_goodput"] == case["expect_goodput"]
    assert out["steps"] == case["expect_steps"] and out["request_goodput"] == 1


@pytest.mark.parametrize("case", GOLD["base_goodput"], ids=lambda c: c["cite"][:30])
def test_replay_base_goodput(case):
    groups = W.make_groups([(W.DDL, 0, 0, 100 * S_, 0, case["w_in"], case["w_out"])])
    tab = B.table_from_supports([(case["L_o"], case["L_o"])], 1024)
    tr = B.single_trace([dict(arrival_ns=0, input_len=case["L_i"], true_out=case["L_o"], group=0)])
    out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg())
    assert out["token_goodput"] == case["expect"]


def test_replay_edf_adversary_gmax_completes_A():
    case = GOLD["edf_adversary"]
    e = W.edf_adversary(case["T"], case["N"], case["M"])
    out = oracle.replay(e["cfg"], e["groups"], e["table"], e["trace"], e["rcfg"])
    assert out["token_goodput"] == case["expect_goodput"]
    assert out["sim_end_ns"] >= case["T"] * 10 * MS


def test_replay_lat_token_timeline():
    """§3: token i counts iff it finishes by TTFT + i*TBT (measured from arrival)."""
    L_i, L_o = 100, 12
    t = [2_100_000]
    for k in range(1, L_o):
        t.append(t[-1] + 2_050_000 + 500 * (L_i + k))
    for ttft, tbt in ((2_100_000, 2_100_000), (3 * MS, 2_000_000), (S_, S_), (1, 1)):
        groups = W.make_groups([(W.LAT, ttft, tbt, 0, 0)])
        tab = B.table_from_supports([(L_o, L_o)], 64)
        tr = B.single_trace([dict(arrival_ns=0, input_len=L_i, true_out=L_o, group=0)])
        out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg())
        expect = sum(1 for i in range(L_o) if t[i] <= ttft + i * tbt)
        assert out["token_goodput"] == expect
        assert out["request_goodput"] == (1 if expect == L_o else 0)


def test_replay_invariants_and_determinism():
    for seed in range(3):
        d = W.trace_mixed(seed, n_rows=300, rate_per_s=6.0)
        rc = dict(d["rcfg"], n_steps=200000)
        a = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        b = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        assert a["status"] == 0
        assert {k: v for k, v in a.items() if k != "log"} == {k: v for k, v in b.items() if k != "log"}
        assert (a["log"] == b["log"]).all()                          # S:669 determinism
        tr, G = d["trace"], d["groups"]
        R = (G["w_in"][tr["group"]].astype(np.int64) * tr["input_len"] +
             G["w_out"][tr["group"]].astype(np.int64) * tr["true_out"])
        assert a["token_goodput"] <= int(R.sum())                   # S:496 goodput <= sum R(k)
        n_req = int((tr["task"] == W.NO_TASK).sum()) + len(tr["task_arrival_ns"])
        assert a["request_goodput"] <= n_req
        # drained: token conservation; every non-dropped request processed L_i + L_o - 1
        assert a["n_done"] + a["n_dropped"] == len(tr["input_len"])
        assert a["n_tasks_done"] + a["n_tasks_dropped"] == len(tr["task_arrival_ns"])


def test_replay_token_conservation_no_drops():
    d = W.trace_mixed(7, n_rows=200, rate_per_s=2.0)
    cfg = dict(d["cfg"], waiting_ns=10 ** 15)
    out = oracle.replay(cfg, d["groups"], d["table"], d["trace"], dict(d["rcfg"], n_steps=10 ** 6))
    tr = d["trace"]
    assert out["n_dropped"] == 0 and out["n_done"] == len(tr["input_len"])
    assert out["tokens_processed"] == int((tr["input_len"].astype(np.int64) + tr["true_out"] - 1).sum())


def test_replay_lone_lat_all_on_time():
    groups = W.make_groups([(W.LAT, 10 * S_, S_, 0, 0)])
    tab = B.table_from_supports([(30, 30)], 64)
    tr = B.single_trace([dict(arrival_ns=5 * MS, input_len=700, true_out=30, group=0)])
    out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg())
    assert out["token_goodput"] == 30 and out["request_goodput"] == 1
