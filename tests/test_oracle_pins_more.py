"""More pins of the CPU oracle (round 2): the parts the first pin set left to GPU == oracle.

Each expected value is a closed form written out here from the cited passage, or an independent
brute force over tiny inputs -- never a value produced by the oracle under test or by the CUDA
path.  Marked "not gpu" (runs on CPU).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from tests import _builders as B

S_, MS = W.S_, W.MS
C0, C_ATT, C_LIN = 2_000_000, 500, 50_000          # S:438 cost model (ns)


def _cfg(**kw):
    return W.default_config(**kw)


def _state(meta):
    return (np.asarray(meta) >> 8) & 0xF


def _waited(aux):
    return np.asarray(aux) >> 16


# ------------------------------------------------------------------------------------------
# steps_waited bookkeeping ("inflates ... by a small additive constant delta per frame";
# reading A12): a pending request left out of the batch waits one more step (counter saturating
# at 0xFFFF), a selected request keeps its counter.
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("frame", [1, 5, 50])
def test_steps_waited_rule_at_saturation(frame):
    """Counters near the 16-bit limit with Delta dividing 65535 (1, 5) and not (50)."""
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 6 * S_, 0)])
    tab = B.table_from_supports([(4, 4)], 8)
    near = [0xFFFD, 0xFFFE, 0xFFFF]
    rows = []
    # three selected rows (large overridden goodput) and three left out (goodput 0: starvation only)
    for i, w in enumerate(near):
        rows.append(dict(id=i, L_i=2, pre=2, g=1, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE,
                         override=2_000_000, waited=w))
    for i, w in enumerate(near):
        rows.append(dict(id=10 + i, L_i=2, pre=2, g=1, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE,
                         override=0, waited=w))
    cfg = _cfg(max_batch=3, token_budget=64, prefill_chunk=8, frame_steps=frame)
    out = oracle.step(cfg, groups, tab, 10 * S_, 15 * MS, B.pool(rows))
    assert out["status"] == 0
    assert sorted(out["batch_ids"].tolist()) == [0, 1, 2]
    assert _waited(out["aux"]).tolist() == near + [0xFFFE, 0xFFFF, 0xFFFF]
    # dist_row bits untouched
    assert (out["aux"] & 0xFFFF).tolist() == [0] * 6


def test_steps_waited_only_pending_rows_count():
    """Rows that are not pending (not yet arrived, Done, Dropped, Waiting) keep their counter."""
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 6 * S_, 0)])
    tab = B.table_from_supports([(4, 4)], 8)
    now = 10 * S_
    rows = [dict(id=0, L_i=2, pre=2, g=1, state=W.Q_RUNNING, flags=W.F_EVER, waited=7),
            dict(id=1, L_i=2, state=W.Q_QUEUED, waited=7, arrival=now + 1),
            dict(id=2, L_i=2, state=W.Q_DONE, flags=W.F_EVER, waited=7),
            dict(id=3, L_i=2, state=W.Q_DROPPED, waited=7),
            dict(id=4, L_i=2, pre=2, g=1, state=W.Q_PREEMPTED, flags=W.F_EVER, waited=7)]
    out = oracle.step(_cfg(max_batch=1, token_budget=64, prefill_chunk=8), groups, tab, now, 15 * MS, B.pool(rows))
    assert out["n_selected"] == 1
    sel = int(out["batch_rows"][0])
    expect = [7, 7, 7, 7, 7]
    for r in (0, 4):
        if r != sel:
            expect[r] = 8
    assert _waited(out["aux"]).tolist() == expect
    # selected: ever_scheduled set, Queued/Preempted -> Running
    assert _state(out["meta"])[sel] == W.Q_RUNNING and (out["meta"][sel] >> 12) & W.F_EVER


# ------------------------------------------------------------------------------------------
# admission for compound tasks, reading A40: a task is one API request; it is
# dropped when none of its calls was ever scheduled and now - a_c > waiting_time (strict).
# ------------------------------------------------------------------------------------------

def _tasks(offs, arrivals, D=100 * S_):
    nt = len(arrivals)
    pat = np.zeros((nt, 8), np.uint32)
    pat[:, 0] = 1
    return {"call_off": np.array(offs, np.uint32), "arrival_ns": np.array(arrivals, np.int64),
            "deadline_ns": np.full(nt, D, np.int64), "cur_stage": np.zeros(nt, np.uint32),
            "n_stages": np.ones(nt, np.uint32), "pattern_ms": pat, "goodput_done": np.zeros(nt, np.uint64)}


def test_compound_task_admission_drop():
    groups = W.make_groups([(W.DDL, 0, 0, 100 * S_, 0), (W.CMP, 0, 0, 100 * S_, 0)])
    tab = B.table_from_supports([(4, 4)], 8)
    now = 20 * S_
    C = W.F_COMPOUND
    rows = [dict(id=0, L_i=2, arrival=now - S_)]                       # standalone, young
    # task 0: never scheduled, a_c = now - 5.1 s -> dropped (its Queued and Waiting calls)
    rows += [dict(id=10, L_i=2, flags=C, group=1, task=0, arrival=now - S_),
             dict(id=11, L_i=2, flags=C, group=1, task=0, state=W.Q_WAITING, arrival=now - S_)]
    # task 1: never scheduled, a_c = now - 4.9 s -> kept
    rows += [dict(id=20, L_i=2, flags=C, group=1, task=1, arrival=now - S_)]
    # task 2: old, but one call was scheduled (ever) -> kept
    rows += [dict(id=30, L_i=2, flags=C, group=1, task=2, arrival=now - S_),
             dict(id=31, L_i=2, pre=2, g=1, flags=C | W.F_EVER, group=1, task=2, state=W.Q_RUNNING,
                  arrival=now - S_)]
    # task 3: never scheduled, exactly 5.0 s old -> kept (strict bound, A29)
    rows += [dict(id=40, L_i=2, flags=C, group=1, task=3, arrival=now - S_)]
    p = B.pool(rows)
    p["n_single"] = 1
    tasks = _tasks([1, 3, 4, 6, 7], [now - 5_100_000_000, now - 4_900_000_000, now - 60 * S_, now - 5 * S_])
    out = oracle.step(_cfg(max_batch=16, token_budget=64, prefill_chunk=8), groups, tab, now, 15 * MS, p, tasks)
    assert out["status"] == 0
    assert out["n_dropped_now"] == 2
    st = _state(out["meta"]).tolist()
    assert st[1] == W.Q_DROPPED and st[2] == W.Q_DROPPED
    assert st[3] != W.Q_DROPPED and st[4] != W.Q_DROPPED and st[6] != W.Q_DROPPED
    assert out["n_pending"] == 5
    assert sorted(out["batch_ids"].tolist()) == [0, 20, 30, 31, 40]


def test_replay_compound_task_dropped_when_never_scheduled():
    """A task whose calls never get a slot within waiting_time is dropped whole (A40): no goodput,
    every call counted as dropped, later stages never released."""
    groups = W.make_groups([(W.DDL, 0, 0, 100 * S_, 0), (W.CMP, 0, 0, 100 * S_, 0)])
    tab = B.table_from_supports([(3, 3)], 8)
    rows = [dict(arrival_ns=0, input_len=1, true_out=3, group=0, override_R=1_000_000)]
    for _ in range(4):
        rows.append(dict(arrival_ns=0, input_len=2, true_out=2, group=1, task=0))
    task = {"arrival": 0, "D": 100 * S_,
            "stages": [{"kind": 0, "b": 1, "e": 3, "pattern_ms": 100}, {"kind": 1, "exec": MS, "pattern_ms": 1},
                       {"kind": 0, "b": 3, "e": 5, "pattern_ms": 100}]}
    tr = B.single_trace(rows, [task])
    cfg = _cfg(max_batch=1, token_budget=64, prefill_chunk=8, waiting_ns=MS)
    out = oracle.replay(cfg, groups, tab, tr, B.default_rcfg())
    assert out["status"] == 0
    assert out["n_tasks_dropped"] == 1 and out["n_tasks_done"] == 0
    assert out["n_dropped"] == 4 and out["n_done"] == 1
    assert out["token_goodput"] == 1_000_000 and out["request_goodput"] == 1
    # the standalone request alone: prefill (emits token 0) + 2 decodes, B_max = 1
    t1 = C0 + C_ATT * 1 + C_LIN
    t2 = t1 + C0 + C_ATT * 2 + C_LIN
    t3 = t2 + C0 + C_ATT * 3 + C_LIN
    assert out["sim_end_ns"] == t3 and out["steps"] == 3


# ------------------------------------------------------------------------------------------
# replay: compound stage release, tool timers and CMP goodput at a_c + D (§3)
# ------------------------------------------------------------------------------------------

def _call_time(start, L_i, L_o):
    """Closed form of one call alone on the replica (A28: prefill end emits token 0;
    decode step k runs at context L_i + k)."""
    t = start + C0 + C_ATT * L_i + C_LIN
    for g in range(1, L_o):
        t += C0 + C_LIN + C_ATT * (L_i + g)
    return t


@pytest.mark.parametrize("slack", [0, -1])
def test_replay_llm_tool_llm_closed_form(slack):
    L1, O1, E, L2, O2 = 40, 6, 700 * MS, 25, 4
    t1 = _call_time(0, L1, O1)
    t2 = _call_time(t1 + E, L2, O2)
    D = t2 + slack                       # deadline exactly at completion -> counted (<=); 1 ns less -> 0
    groups = W.make_groups([(W.CMP, 0, 0, D, 0)])
    tab = B.table_from_supports([(8, 8)], 16)
    rows = [dict(arrival_ns=0, input_len=L1, true_out=O1, group=0, task=0),
            dict(arrival_ns=0, input_len=L2, true_out=O2, group=0, task=0)]
    task = {"arrival": 0, "D": D,
            "stages": [{"kind": 0, "b": 0, "e": 1, "pattern_ms": 100}, {"kind": 1, "exec": E, "pattern_ms": 700},
                       {"kind": 0, "b": 1, "e": 2, "pattern_ms": 100}]}
    tr = B.single_trace(rows, [task])
    out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg(), log=True)
    assert out["status"] == 0 and out["n_tasks_done"] == 1 and out["n_done"] == 2
    assert out["sim_end_ns"] == t2
    assert out["steps"] == O1 + O2
    expect = (L1 + O1 + L2 + O2) if slack == 0 else 0
    assert out["token_goodput"] == expect
    assert out["request_goodput"] == (1 if slack == 0 else 0)
    # the second call starts exactly when the tool ends (its first step's end time)
    assert out["log"]["now_ns"][O1] == t1 + E + C0 + C_ATT * L2 + C_LIN


# ------------------------------------------------------------------------------------------
# chunked prefill: L_i = 1300 with chunk 512 -> 512, 512, 276, then decodes
# ------------------------------------------------------------------------------------------

def test_replay_chunked_prefill_costs_and_ttft():
    L_i, L_o = 1300, 3
    ends = [C0 + C_ATT * 512 + C_LIN]
    ends.append(ends[-1] + C0 + C_ATT * 1024 + C_LIN)
    ends.append(ends[-1] + C0 + C_ATT * 1300 + C_LIN)        # token 0 (A28)
    ends.append(ends[-1] + C0 + C_LIN + C_ATT * (L_i + 1))
    ends.append(ends[-1] + C0 + C_LIN + C_ATT * (L_i + 2))
    ttft = ends[2]
    for ttft_slo, expect_tok0 in ((ttft, 1), (ttft - 1, 0)):
        groups = W.make_groups([(W.LAT, ttft_slo, 10 * S_, 0, 0)])
        tab = B.table_from_supports([(L_o, L_o)], 16)
        tr = B.single_trace([dict(arrival_ns=0, input_len=L_i, true_out=L_o, group=0)])
        out = oracle.replay(_cfg(prefill_chunk=512), groups, tab, tr, B.default_rcfg(), log=True)
        assert out["log"]["total_tokens"].tolist() == [512, 512, 276, 1, 1]
        assert out["log"]["now_ns"].tolist() == ends
        assert out["token_goodput"] == expect_tok0 + (L_o - 1)


def test_step_prefill_cost_is_capped_chunk():
    groups = W.make_groups([(W.DDL, 0, 0, 100 * S_, 0)])
    tab = B.table_from_supports([(4, 4)], 8)
    p = B.pool([dict(id=0, L_i=1300, pre=0), dict(id=1, L_i=1300, pre=512, state=W.Q_RUNNING, flags=W.F_EVER),
                dict(id=2, L_i=1300, pre=1024, state=W.Q_RUNNING, flags=W.F_EVER),
                dict(id=3, L_i=1300, pre=1300, g=1, state=W.Q_RUNNING, flags=W.F_EVER)])
    out = oracle.step(_cfg(prefill_chunk=512, token_budget=4096), groups, tab, S_, 15 * MS, p)
    assert out["cost"].tolist() == [512, 512, 276, 1]


# ------------------------------------------------------------------------------------------
# v_token = floor of the trailing mean of the last Delta iteration latencies (A24),
# v_token0 before the first iteration
# ------------------------------------------------------------------------------------------

@pytest.mark.parametrize("frame", [1, 3, 50])
def test_replay_v_token_trailing_mean(frame):
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 4 * S_, 0)])
    tab = B.table_from_supports([(40, 40)], 64)
    tr = B.single_trace([dict(arrival_ns=0, input_len=700, true_out=40, group=0),
                         dict(arrival_ns=3 * MS, input_len=90, true_out=25, group=0)])
    rc = B.default_rcfg(v_token0_ns=1_234_567)
    out = oracle.replay(_cfg(frame_steps=frame, prefill_chunk=256), groups, tab, tr, rc, log=True)
    now = out["log"]["now_ns"].astype(np.int64)
    v = out["log"]["v_token_ns"].astype(np.int64)
    lat = np.diff(np.concatenate([[0], now]))
    # no idle gaps in this trace: step k's latency is now_k - now_{k-1}
    assert v[0] == 1_234_567
    for k in range(1, len(v)):
        w = lat[max(0, k - frame):k]
        assert v[k] == int(w.sum()) // len(w), k


# ------------------------------------------------------------------------------------------
# load and SLO scaling of a replay (§6.4 sweep shape; rationals):
#   arrival' = floor(a * load_den / load_num), SLO' = floor(t * slo_num / slo_den)
# ------------------------------------------------------------------------------------------

def test_replay_load_and_slo_scaling():
    t_done = _call_time(0, 100, 10)                    # 21,022,500 ns: the single-DDL closed form
    tab = B.table_from_supports([(10, 10)], 64)
    for e2el, expect in ((2 * t_done, 110), (2 * t_done + 1, 110), (2 * t_done - 1, 0)):
        groups = W.make_groups([(W.DDL, 0, 0, e2el, 0)])
        tr = B.single_trace([dict(arrival_ns=0, input_len=100, true_out=10, group=0)])
        out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg(slo_num=1, slo_den=2))
        assert out["sim_end_ns"] == t_done and out["token_goodput"] == expect, e2el
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 3 * S_, 0)])
    tr = B.single_trace([dict(arrival_ns=1000, input_len=100, true_out=10, group=0)])
    out = oracle.replay(_cfg(), groups, tab, tr, B.default_rcfg(load_num=3, load_den=2))
    assert out["sim_end_ns"] == 666 + t_done            # floor(1000 * 2 / 3) = 666: idle jump first


# ------------------------------------------------------------------------------------------
# (a2) on coarse (non-unit) histogram bins, reading A42: the samples of bin k sit at its upper
# edge; condition on edge > anchor; type-1 quantile.  Brute force over the expanded multiset.
# ------------------------------------------------------------------------------------------

def _coarse_table(rng, n_bins, l_max):
    edges = np.sort(rng.choice(np.arange(1, l_max), n_bins - 1, replace=False)).tolist() + [l_max]
    counts = rng.integers(0, 4, n_bins) * (rng.random(n_bins) < 0.7)
    return np.array(edges, np.uint32), counts


def _brute_coarse(edges, counts, g, R, qn, qd, l_max):
    anchor = R * (g // R)
    ms = sorted(int(e) for e, c in zip(edges, counts) for _ in range(int(c)) if e > anchor)
    if not ms:
        q = l_max
    else:
        q = ms[(qn * len(ms) + qd - 1) // qd - 1]
    return max(q, g + 1)


def test_length_bound_coarse_bins_bruteforce():
    rng = np.random.default_rng(21)
    for _ in range(400):
        l_max = int(rng.integers(8, 300))
        nb = int(rng.integers(2, min(l_max, 40)))
        edges, counts = _coarse_table(rng, nb, l_max)
        tab = {"edges": edges, "cum": np.cumsum(counts)[None, :].astype(np.uint32), "l_max": l_max}
        g = int(rng.integers(0, l_max + 3))
        R = int(rng.choice([1, 7, 50]))
        qd = int(rng.choice([100, 3]))
        qn = int(rng.integers(1, qd + 1))
        assert oracle.length_bound(tab, 0, g, R, qn, qd) == _brute_coarse(edges, counts, g, R, qn, qd, l_max)


def test_step_lhat_matches_bruteforce_through_memo():
    """The step's L-hat goes through the per-call memo (oracle cond_quantile); compare every pending
    standalone row of random pools (random non-point-mass tables) with the brute force."""
    rng = np.random.default_rng(22)
    checked = 0
    for it in range(120):
        d = W.random_small_pool(rng, int(rng.integers(5, 80)))
        if it % 2:     # coarse bins on half of the pools
            l_max = int(d["table"]["l_max"])
            nb = int(rng.integers(2, l_max))
            edges = np.sort(rng.choice(np.arange(1, l_max), nb - 1, replace=False)).tolist() + [l_max]
            counts = rng.integers(0, 5, (d["table"]["cum"].shape[0], nb))
            d["table"] = {"edges": np.array(edges, np.uint32), "cum": np.cumsum(counts, 1).astype(np.uint32),
                          "l_max": l_max}
        out = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        if out["status"] < 0:
            continue
        tab = d["table"]
        cnt = np.diff(np.concatenate([np.zeros((tab["cum"].shape[0], 1), np.int64), tab["cum"].astype(np.int64)], 1), axis=1)
        for r in np.nonzero(out["pending"])[0]:
            row = int(d["pool"]["aux"][r]) & 0xFFFF
            g = int(d["pool"]["generated"][r])
            exp = _brute_coarse(tab["edges"], cnt[row], g, d["cfg"]["refine_interval"], d["cfg"]["q_num"],
                                d["cfg"]["q_den"], int(tab["l_max"]))
            assert int(out["lhat"][r]) == exp
            checked += 1
    assert checked > 500


# ------------------------------------------------------------------------------------------
# a stage sub-deadline given by the caller (SURVEY 8(b) task updates) replaces phi(s) D
# ------------------------------------------------------------------------------------------

def test_explicit_stage_deadline_replaces_pattern():
    groups = W.make_groups([(W.CMP, 0, 0, 40 * S_, 0)])
    tab = B.table_from_supports([(30, 30)], 64)
    a_c, now, D = 0, 7 * S_, 40 * S_
    p = B.pool([dict(id=0, L_i=5, pre=5, g=2, group=0, state=W.Q_RUNNING, flags=W.F_EVER | W.F_COMPOUND, task=0)])
    pat = np.zeros((1, 8), np.uint32)
    pat[0, :2] = [3, 1]                                   # stage 0: phi = 3/4 -> D_s = 30 s
    base = {"call_off": np.array([0, 1], np.uint32), "arrival_ns": np.array([a_c], np.int64),
            "deadline_ns": np.array([D], np.int64), "cur_stage": np.array([0], np.uint32),
            "n_stages": np.array([2], np.uint32), "pattern_ms": pat, "goodput_done": np.zeros(1, np.uint64)}
    ref = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, base)
    assert ref["t_rem"][0] == a_c + 30 * S_ - now
    same = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, dict(base, stage_deadline_ns=np.array([a_c + 30 * S_])))
    assert same["t_rem"][0] == ref["t_rem"][0] and same["key"][0] == ref["key"][0]
    neg = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, dict(base, stage_deadline_ns=np.array([-1])))
    assert neg["t_rem"][0] == ref["t_rem"][0]             # < 0: from the pattern
    other = oracle.step(_cfg(), groups, tab, now, 15 * MS, p, dict(base, stage_deadline_ns=np.array([12 * S_])))
    assert other["t_rem"][0] == 12 * S_ - now             # the key does not depend on t_rem (A1)
    assert other["key"][0] == ref["key"][0]
