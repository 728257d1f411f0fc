"""Pins of the oracle's NEXT-1 preemption gate (reading A46; §4.2, App. D.2
P:1073-1081; SPEC preemption_check S:313-321).

What the paper fixes, checked here without re-implementing the gate:
  * with nothing running the gate is transparent: the step equals plain GMAX;
  * between frame boundaries nothing running is preempted ("scheduling updates are
    restricted to discrete time frames");
  * the batch stays within tau and B_max, the running set is kept or evicted, never lost;
  * SPEC's three worked examples of preemption_check: equal goodputs -> no preemption;
    ratio 1.2 at delta 0.1 and zero KV -> preemption; gain 5 tokens against a 0.1 s stall at
    100 tokens/s (loss 10) -> no preemption;
  * a hand-derived two-request replay timeline (B_max = 1, 1 ms iterations, Delta = 4): the
    high-goodput arrival preempts at the first frame boundary, the KV stall (5 tokens at 10^6
    tokens/s = 5 us) lengthens that iteration, the evicted request resumes after it; with a
    huge delta or a slow swap link the schedule stays non-preemptive.
"""
import numpy as np

import oracle
import workloads as W
from . import _builders as B

MS, S_ = W.MS, W.S_


def _state(meta):
    return (np.asarray(meta) >> 8) & 0xF


def _with_states(d, fn):
    m = d["pool"]["meta"].copy()
    st = fn(_state(m))
    d["pool"]["meta"] = (m & ~np.uint32(0xF00)) | (st.astype(np.uint32) << np.uint32(8))


def test_gate_without_running_requests_is_plain_gmax():
    rng = np.random.default_rng(601)
    for it in range(150):
        d = W.random_small_pool(rng, int(rng.integers(1, 90)), tie_heavy=(it % 7 == 0))
        _with_states(d, lambda st: np.where(st == W.Q_RUNNING, W.Q_PREEMPTED, st))
        plain = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
        for frame_open in (True, False):
            cfg = dict(d["cfg"], preempt=1, pmtn_num=int(rng.integers(0, 3)), pmtn_den=10,
                       io_bw_tps=int(rng.choice([1, 10 ** 6])))
            g = oracle.step(cfg, d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"],
                            frame_open=frame_open)
            assert g["status"] == plain["status"]
            for k in ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star", "n_dropped_now"):
                assert g[k] == plain[k], (it, k)
            for k in ("batch_ids", "batch_tokens", "batch_rows", "meta", "aux"):
                assert np.array_equal(g[k], plain[k]), (it, k)
            assert g["n_preempted"] == 0 and g["stall_ns"] == 0


def test_gate_invariants_random_pools():
    rng = np.random.default_rng(602)
    seen_forced = seen_gated = 0
    for it in range(300):
        d = W.random_small_pool(rng, int(rng.integers(2, 90)))
        # a random running set: every pending-state row is Running with probability 1/3
        _with_states(d, lambda st: np.where((st <= W.Q_PREEMPTED) & (rng.random(len(st)) < 0.33), W.Q_RUNNING,
                                            np.where(st == W.Q_RUNNING, W.Q_QUEUED, st)))
        frame_open = bool(rng.random() < 0.5)
        cfg = dict(d["cfg"], preempt=1, pmtn_num=int(rng.choice([0, 1, 10 ** 6])), pmtn_den=10,
                   io_bw_tps=int(rng.choice([1000, 10 ** 9])))
        plain = oracle.step(dict(cfg, preempt=0), d["groups"], d["table"], d["now_ns"], d["v_token_ns"],
                            d["pool"], d["tasks"])
        g = oracle.step(cfg, d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"],
                        frame_open=frame_open)
        assert g["status"] == plain["status"]
        if g["status"] != 0:
            continue
        # GMAX's own outputs are the gate's input: unchanged
        for k in ("n_pending", "n_candidates", "b_star"):
            assert g[k] == plain[k]
        assert g["bp"] == plain["bp"] and g["thr"] == plain["thr"]
        pend = g["pending"].astype(bool)
        st0 = _state(d["pool"]["meta"])
        running = pend & (st0 == W.Q_RUNNING)
        F = np.zeros(len(pend), bool)
        F[g["batch_rows"]] = True
        Q = np.zeros(len(pend), bool)
        Q[plain["batch_rows"]] = True
        st1 = _state(g["meta"])
        evicted = running & ~F
        assert g["n_preempted"] == evicted.sum()
        assert np.all(st1[F] == W.Q_RUNNING) and np.all(st1[evicted] == W.Q_PREEMPTED)
        assert np.all(F <= (running | Q)), "a batch member is neither running nor proposed"
        assert g["total_tokens"] == int(g["cost"][F].sum()) <= cfg["token_budget"]
        assert g["n_selected"] == F.sum() <= cfg["max_batch"]
        # a selected request keeps its steps_waited; a pending one left out gets +1 (A12)
        w0, w1 = d["pool"]["aux"] >> 16, g["aux"] >> 16
        assert np.all(w1[F] == w0[F])
        out = pend & ~F
        assert np.all(w1[out] == np.minimum(w0[out] + 1, 0xFFFF))
        # batch order: window order (len asc, id asc; A20)
        L = d["pool"]["input_len"].astype(np.int64) + (d["pool"]["generated"] if cfg["len_key"] else 0)
        keys = list(zip(L[g["batch_rows"]], d["pool"]["id"][g["batch_rows"]]))
        assert keys == sorted(keys)
        fits = running.sum() <= cfg["max_batch"] and g["cost"][running].sum() <= cfg["token_budget"]
        if fits and (not frame_open or cfg["pmtn_num"] == 10 ** 6):
            assert not evicted.any(), "preempted outside a frame boundary / below the ratio"
        seen_forced += (not fits) and evicted.any()
        seen_gated += fits and evicted.any()
    assert seen_forced > 10 and seen_gated > 4, (seen_forced, seen_gated)


# ------------------------------------------------------------------------------------------
# SPEC S:318-321 worked examples.  Two DDL requests with R(k) set directly (App. D), the same
# length bound (point mass at 200, g = 101: L-hat 200, len_rem 99) and v = 10 ms (100 tokens/s),
# eps = 10 ms: t_gen + eps = 99 * 10 ms + 10 ms = 1 s, so key = R exactly.  A runs (B_max = 1),
# B is proposed; Delta = 50 steps of 10 ms: a frame is 0.5 s, so gain = (R_B - R_A) / 2 tokens.
# ------------------------------------------------------------------------------------------

def _pair(R_A, R_B, kv_A, io_bw, num, den):
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 4 * S_, 0)])
    tab = B.table_from_counts([[0] * 199 + [5]])
    L_A = kv_A - 101
    assert L_A >= 1
    p = B.pool([dict(id=1, L_i=L_A, g=101, pre=L_A, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE,
                     override=R_A),
                dict(id=2, L_i=5, g=101, pre=5, state=W.Q_PREEMPTED, flags=W.F_EVER | W.F_OVERRIDE, override=R_B)])
    cfg = W.default_config(token_budget=64, max_batch=1, prefill_chunk=8, refine_interval=1, eps_ns=10 * MS,
                           preempt=1, pmtn_num=num, pmtn_den=den, io_bw_tps=io_bw)
    out = oracle.step(cfg, groups, tab, 100 * S_, 10 * MS, p, None)
    assert out["key"][0] == R_A and out["key"][1] == R_B
    return out


def test_spec_example_equal_goodputs_no_preemption():
    out = _pair(1000, 1000, 200, 10 ** 9, 1, 10)
    assert list(out["batch_ids"]) == [1] and out["n_preempted"] == 0


def test_spec_example_ratio_1_2_zero_kv_preempts():
    # kv = 200 tokens at 10^12 tokens/s: floor(200e9 / 1e12) = 0 ns of stall
    out = _pair(1000, 1200, 200, 10 ** 12, 1, 10)
    assert list(out["batch_ids"]) == [2] and out["n_preempted"] == 1 and out["stall_ns"] == 0
    assert _state(out["meta"][0]) == W.Q_PREEMPTED and _state(out["meta"][1]) == W.Q_RUNNING
    # the same ratio is not enough at delta = 0.25
    out = _pair(1000, 1200, 200, 10 ** 12, 1, 4)
    assert list(out["batch_ids"]) == [1] and out["n_preempted"] == 0


def test_spec_example_net_loss_blocks_preemption():
    # gain (110 - 100) / 2 = 5 tokens; stall 200 tokens at 2000 tokens/s = 0.1 s = 10 tokens at
    # 100 tokens/s -> no preemption (ratio 1.1 > 1.05 passes)
    out = _pair(100, 110, 200, 2000, 1, 20)
    assert list(out["batch_ids"]) == [1] and out["n_preempted"] == 0
    # a faster link: stall 200 / 5000 s = 40 ms = 4 tokens < 5 -> preempt, stall reported
    out = _pair(100, 110, 200, 5000, 1, 20)
    assert list(out["batch_ids"]) == [2] and out["n_preempted"] == 1 and out["stall_ns"] == 40 * MS
    # at exactly gain == loss (stall 50 ms = 5 tokens) the strict '>' keeps A
    out = _pair(100, 110, 200, 4000, 1, 20)
    assert list(out["batch_ids"]) == [1]


def test_frame_closed_never_preempts():
    out_open = _pair(1000, 1200, 200, 10 ** 12, 1, 10)
    assert out_open["n_preempted"] == 1
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 4 * S_, 0)])
    tab = B.table_from_counts([[0] * 199 + [5]])
    p = B.pool([dict(id=1, L_i=99, g=101, pre=99, state=W.Q_RUNNING, flags=W.F_EVER | W.F_OVERRIDE, override=1000),
                dict(id=2, L_i=5, g=101, pre=5, state=W.Q_PREEMPTED, flags=W.F_EVER | W.F_OVERRIDE, override=1200)])
    cfg = W.default_config(token_budget=64, max_batch=1, prefill_chunk=8, refine_interval=1, eps_ns=10 * MS,
                           preempt=1, pmtn_num=1, pmtn_den=10, io_bw_tps=10 ** 12)
    out = oracle.step(cfg, groups, tab, 100 * S_, 10 * MS, p, None, frame_open=False)
    assert list(out["batch_ids"]) == [1] and out["n_preempted"] == 0


# ------------------------------------------------------------------------------------------
# Hand-derived replay timeline.  B_max = 1, iteration = c0 = 1 ms (c_att = c_lin = 0),
# Delta = 4.  A: DDL, arrives at 0, L_i = 1, L_o = 20, R(A) = 100.  B: arrives at 2.5 ms,
# L_i = 1, L_o = 5, R(B) = 10^4.  Steps 0-3 run A (B arrives during step 2; step 3 is not a
# boundary).  Step 4 (4 % 4 == 0) is a boundary: B preempts A (ratio 100; gain ~ 625 tokens,
# loss = stall / v = 5 us / 1 ms); A's KV is pre + gen = 1 + 4 = 5 tokens -> stall
# floor(5e9 / 1e6) = 5000 ns added to step 4.  B runs steps 4-8 (5 tokens), A resumes at step 9
# and needs 16 more tokens: steps 9-24.  25 steps, end at 25 ms + 5 us; both meet their
# deadlines: token goodput = 100 + 10^4.
# ------------------------------------------------------------------------------------------

def _toy(num, den, io_bw):
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 3 * S_, 0)])
    tab = B.table_from_counts([[0] * 63 + [3]])
    tr = B.single_trace([dict(arrival_ns=0, input_len=1, true_out=20, group=0, override_R=100),
                         dict(arrival_ns=2 * MS + MS // 2, input_len=1, true_out=5, group=0, override_R=10 ** 4)])
    cfg = W.default_config(token_budget=64, max_batch=1, prefill_chunk=8, refine_interval=1, frame_steps=4,
                           preempt=1, pmtn_num=num, pmtn_den=den, io_bw_tps=io_bw)
    rc = B.default_rcfg(v_token0_ns=MS, c0_ns=MS, c_att_ns=0, c_lin_ns=0)
    return oracle.replay(cfg, groups, tab, tr, rc, log=True, log_ids=True)


def test_toy_replay_preemption_timeline():
    out = _toy(1, 10, 10 ** 6)
    ids = out["log_ids"][:, 0]
    assert list(ids) == [0] * 4 + [1] * 5 + [0] * 16
    assert out["steps"] == 25 and out["n_preempted"] == 1 and out["n_done"] == 2
    assert out["sim_end_ns"] == 25 * MS + 5000
    L = out["log"]
    assert L["n_preempted"][4] == 1 and L["stall_ns"][4] == 5000 and L["stall_ns"].sum() == 5000
    assert L["now_ns"][4] - L["now_ns"][3] == MS + 5000
    assert out["token_goodput"] == 100 + 10 ** 4 and out["request_goodput"] == 2


def test_toy_replay_no_preemption_when_gated_out():
    for num, den, io_bw in [(10 ** 6, 1, 10 ** 6),      # delta = 10^6: the ratio never passes
                            (1, 10, 1)]:                 # 1 token/s: a 5 s stall = 5000 tokens of loss
        out = _toy(num, den, io_bw)
        ids = out["log_ids"][:, 0]
        assert list(ids) == [0] * 20 + [1] * 5
        assert out["n_preempted"] == 0 and out["sim_end_ns"] == 25 * MS


def test_gated_replay_runs_are_contiguous_without_preemption():
    """delta huge: once admitted, a request runs until it finishes (non-preemptive), so each
    request's appearances in the batch log form one contiguous run"""
    d = W.trace_c1()
    cfg = dict(d["cfg"], preempt=1, pmtn_num=10 ** 9, pmtn_den=1, max_batch=4)
    cfg, groups, tab, tr, rc = cfg, d["groups"], d["table"], d["trace"], d["rcfg"]
    out = oracle.replay(cfg, groups, tab, tr, dict(rc, n_steps=3000), log=True, log_ids=True)
    assert out["n_preempted"] == 0
    LI = out["log_ids"]
    n = out["log"]["n_selected"]
    last = {}
    for k in range(out["steps"]):
        for r in LI[k, :n[k]]:
            r = int(r)
            if r in last:
                assert last[r] == k - 1, f"request {r} left the batch at step {last[r]} and came back at {k}"
            last[r] = k
