"""GPU parity: libjitsched.so (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bar: integer / index outputs bit-exact; fp64 keys, rates, bp and thr compared
by bit pattern (the exactness contract makes them identical; the north_star tolerance 1e-9
relative is therefore met with zero error).
"""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

SCALARS = ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star", "n_dropped_now")


def _sched(d, capacity=None, tasks_cap=None, debug=True):
    from paper_2504_20068_b200 import Scheduler
    n = len(d["pool"]["input_len"])
    nt = 0 if d["tasks"] is None else len(d["tasks"]["arrival_ns"])
    return Scheduler(d["cfg"], d["groups"], d["table"], capacity=capacity or max(n, 1),
                     task_capacity=tasks_cap if tasks_cap is not None else max(nt, 1), debug=debug)


def _compare(got, ref, rows=None, pool=None, ctx=""):
    assert got["status"] == ref["status"], (ctx, got["status"], ref["status"])
    assert got["n_pending"] == ref["n_pending"], ctx
    if ref["status"] == 0:
        for k in SCALARS:
            assert got[k] == ref[k], (ctx, k, got[k], ref[k])
        assert np.float64(got["bp"]).view(np.uint64) == np.float64(ref["bp"]).view(np.uint64), ctx
        assert np.float64(got["thr"]).view(np.uint64) == np.float64(ref["thr"]).view(np.uint64), ctx
        assert np.array_equal(got["batch_ids"], ref["batch_ids"]), ctx
        assert np.array_equal(got["batch_tokens"], ref["batch_tokens"]), ctx
        assert np.array_equal(got["batch_rows"], ref["batch_rows"]), ctx
    if rows is not None and "key" in rows:
        pend = ref["pending"].astype(bool)
        assert np.array_equal(rows["pending"].astype(bool), pend), ctx
        assert np.array_equal(rows["key"].view(np.uint64)[pend], ref["key"].view(np.uint64)[pend]), ctx
        assert np.array_equal(rows["cost"][pend], ref["cost"][pend]), ctx
        if "lhat" in rows:
            assert np.array_equal(rows["lhat"][pend], ref["lhat"][pend]), ctx
            assert np.array_equal(rows["t_rem"][pend], ref["t_rem"][pend]), ctx
            assert np.array_equal(rows["rate"].view(np.uint64)[pend], ref["rate"].view(np.uint64)[pend]), ctx
    if rows is not None:
        assert np.array_equal(rows["meta"], ref["meta"]), ctx
        assert np.array_equal(rows["aux"], ref["aux"]), ctx


def _run_both(d, s=None, debug=True):
    ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], d["pool"], d["tasks"])
    own = s is None
    if own:
        s = _sched(d, debug=debug)
    s.load(d["pool"], d["tasks"])
    got = s.step(d["now_ns"], d["v_token_ns"])
    rows = s.read_rows(debug=debug)
    if own:
        s.close()
    return got, ref, rows


def test_random_small_pools_exact():
    rng = np.random.default_rng(101)
    for it in range(300):
        d = W.random_small_pool(rng, int(rng.integers(1, 60)), tie_heavy=(it % 7 == 0))
        got, ref, rows = _run_both(d)
        _compare(got, ref, rows, ctx=f"iter {it}")


def test_reuse_handle_across_pools_and_shapes():
    rng = np.random.default_rng(102)
    d0 = W.random_small_pool(rng, 50)
    s = _sched(d0, capacity=400, tasks_cap=16)
    for it in range(60):
        d = W.random_small_pool(rng, int(rng.integers(1, 300)))
        d["cfg"] = d0["cfg"]
        d["groups"], d["table"] = d0["groups"], d0["table"]
        got, ref, rows = _run_both(d, s)
        _compare(got, ref, rows, ctx=f"iter {it}")
    s.close()


@pytest.mark.parametrize("n", [4097, 65536 + 13, 200_003])
def test_c3_shaped_pools_full_compare(n):
    """several tiles + ragged tail; compound tasks of 16 calls; every row compared."""
    d = W.pool_snapshot(30 + n % 7, n, table_draws=1 << 16)
    got, ref, rows = _run_both(d)
    _compare(got, ref, rows, ctx=f"n={n}")


def test_c3_full_size_1m():
    """BASELINE config C3 (2^20 pending-pool rows, 16 SLO groups, tau 8192) in the launch
    configuration bench.py times: every key, the batch, bp, thr, B* and |Cd| compared."""
    d = W.pool_snapshot(3, 1 << 20)
    got, ref, rows = _run_both(d, debug=False)
    _compare(got, ref, rows, ctx="C3")


@pytest.mark.parametrize("tau,bmax", [(2048, 2048), (65536, 65536), (8192, 256)])
def test_c3_budget_sweep(tau, bmax):
    d = W.pool_snapshot(3, 300_000, table_draws=1 << 16)
    d["cfg"] = W.default_config(token_budget=tau, max_batch=bmax)
    got, ref, rows = _run_both(d, debug=False)
    _compare(got, ref, rows, ctx=f"tau={tau}")


def test_c4_compound_dag():
    """BASELINE config C4 (100K tasks, 64-call fan-out): compound aggregation over every task."""
    d = W.pool_c4(n_tasks=100_000, table_draws=1 << 16)
    got, ref, rows = _run_both(d, debug=True)
    _compare(got, ref, rows, ctx="C4")


def test_multi_step_engine_loop():
    """A serving loop: each step's batch advances (prefill chunk or one decode token) in both
    implementations; state (drops, steps_waited, cached bounds, ever_scheduled) must stay equal."""
    d = W.pool_snapshot(9, 30_000, table_draws=1 << 16)
    d["cfg"] = W.default_config(token_budget=4096, max_batch=1024, refine_interval=7)
    s = _sched(d)
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    s.load(pool, d["tasks"])
    now = d["now_ns"]
    progress = None
    for step in range(25):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], now, d["v_token_ns"], pool, d["tasks"])
        got = s.step(now, d["v_token_ns"], progress=progress)
        rows = s.read_rows()
        _compare(got, ref, rows, ctx=f"step {step}")
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        # engine progress of the executed batch
        r = ref["batch_rows"]
        gen, pre = pool["generated"], pool["prefilled"]
        dec = pre[r] >= pool["input_len"][r]
        pre[r[~dec]] += ref["batch_tokens"][~dec]
        done_pf = (~dec) & (pre[r] >= pool["input_len"][r])
        gen[r[dec | done_pf]] += 1
        st = (pool["meta"][r] >> 8) & 0xF
        finished = gen[r] >= pool["true_out"][r]
        st = np.where(finished, W.Q_DONE, st)
        pool["meta"][r] = (pool["meta"][r] & ~np.uint32(0xF00)) | (st.astype(np.uint32) << 8)
        progress = {"row": r, "generated": gen[r], "prefilled": pre[r], "state": st}
        now += 20 * W.MS
    s.close()


def test_empty_and_degenerate():
    rng = np.random.default_rng(104)
    d = W.random_small_pool(rng, 10, with_tasks=False)
    d["pool"]["meta"] = (d["pool"]["meta"] & ~np.uint32(0xF00)) | np.uint32(W.Q_DONE << 8)
    got, ref, rows = _run_both(d)
    assert ref["status"] == 1 and got["status"] == 1 and got["n_selected"] == 0
    # single row
    d = W.random_small_pool(rng, 1, with_tasks=False)
    got, ref, rows = _run_both(d)
    _compare(got, ref, rows, ctx="single")


def test_all_ties_force_deep_radix_passes():
    """Every key equal (best effort, no starvation): the select must resolve the boundary on
    request ids (all 8 digits) and the candidate set is the whole pool (bp = 0)."""
    n = 50_000
    rng = np.random.default_rng(105)
    groups = W.make_groups([(W.BE, 0, 0, 0, 600 * W.S_)])
    table = {"edges": np.arange(1, 65, dtype=np.uint32), "cum": np.cumsum(np.ones((1, 64), np.int64), axis=1).astype(np.uint32),
             "l_max": 64}
    pool = {"id": rng.permutation(n).astype(np.uint32), "arrival_ns": np.zeros(n, np.int64),
            "input_len": rng.integers(1, 5000, n).astype(np.uint32), "generated": np.ones(n, np.uint32),
            "prefilled": np.zeros(n, np.uint32), "meta": W._pack_meta(np.zeros(n), np.full(n, W.Q_RUNNING), np.full(n, W.F_EVER)),
            "aux": W._pack_aux(np.zeros(n), np.zeros(n)), "task": np.full(n, W.NO_TASK, np.uint32),
            "override_R": np.zeros(n, np.uint32), "n_single": n}
    pool["prefilled"] = pool["input_len"].copy()
    d = {"pool": pool, "tasks": None, "groups": groups, "table": table, "now_ns": 10 * W.S_, "v_token_ns": 10 * W.MS,
         "cfg": W.default_config(token_budget=3000, max_batch=3000, delta_starve=0)}
    got, ref, rows = _run_both(d)
    assert ref["bp"] == 0.0 and ref["n_candidates"] == n
    _compare(got, ref, rows, ctx="ties")


def test_determinism_double_run():
    d = W.pool_snapshot(11, 100_000, table_draws=1 << 16)
    a, _, ra = _run_both(d)
    b, _, rb = _run_both(d)
    assert np.array_equal(a["batch_ids"], b["batch_ids"]) and a["bp"] == b["bp"]
    assert np.array_equal(ra["key"].view(np.uint64), rb["key"].view(np.uint64))


def test_speculative_paths_against_oracle_chain():
    """Consecutive steps on one handle: the first step after a load takes the exact radix path
    (no threshold yet), later steps resolve from the speculative set -- in k_spec's fast path
    (|S| <= 256) or in k_spec_big (larger sets).  Every step is checked against the oracle run on
    the state the previous oracle step left (meta / aux bookkeeping), and both speculative paths
    must have been exercised."""
    seen_fast = seen_big = False
    for tau, bmax, n in [(8192, 8192, 200_000), (65536, 65536, 200_000), (4096, 64, 100_000)]:
        d = W.pool_snapshot(21, n, table_draws=1 << 16)
        d["cfg"] = W.default_config(token_budget=tau, max_batch=bmax)
        s = _sched(d, debug=False)
        s.load(d["pool"], d["tasks"])
        pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
        for k in range(4):
            ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
            got = s.step(d["now_ns"], d["v_token_ns"])
            _compare(got, ref, ctx=f"tau={tau} step {k} n_spec={got['n_spec']} fallback={got['fallback']}")
            if k > 0 and not got["fallback"]:
                seen_fast |= got["n_spec"] <= 256
                seen_big |= got["n_spec"] > 256
            pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        s.close()
    assert seen_fast and seen_big, (seen_fast, seen_big)


def test_time_scoring_leaves_state_consistent():
    """bench.py's roofline timing (jit_sched_time_scoring: back-to-back k_score launches over
    several handles) must leave each handle's pool as it was: the pass writes no per-row state in
    the steady state and the step counter (steps_waited stamps) only moves with a resolved step;
    the per-step partials / speculative set are consumed -- the next step equals the oracle's."""
    from paper_2504_20068_b200 import Scheduler
    L = 5
    ds, hs, pools = [], [], []
    for seed in (31, 32):
        d = W.pool_snapshot(seed, 150_000, table_draws=1 << 16)
        d["cfg"] = W.default_config(token_budget=8192, max_batch=8192)
        s = _sched(d, debug=True)
        s.load(d["pool"], d["tasks"])
        pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
        for _ in range(2):                       # second step: a speculative threshold exists
            ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
            _compare(s.step(d["now_ns"], d["v_token_ns"]), ref)
            pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        ds.append(d); hs.append(s); pools.append(pool)
    ms = Scheduler.time_scoring(hs, ds[0]["now_ns"], ds[0]["v_token_ns"], L * len(hs))
    assert ms > 0
    for d, s, pool in zip(ds, hs, pools):
        rows = s.read_rows(debug=True)
        assert np.array_equal(rows["meta"], pool["meta"])
        assert np.array_equal(rows["aux"], pool["aux"])
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        got = s.step(d["now_ns"], d["v_token_ns"])
        _compare(got, ref, ctx=f"after time_scoring n_spec={got['n_spec']} fallback={got['fallback']}")
        s.close()


def test_large_prefill_chunk_routes_small_sets_to_histogram_resolve():
    """The small-set resolve keeps 32-bit cost prefixes, valid while |S| * chunk < 2^32
    (kSpecFastChunk); a larger chunk (here 2^24 with tau = 2^26) must route even small speculative
    sets through k_spec_big -- every step still equal to the oracle (S:417 allows any chunk <= tau)."""
    d = W.pool_snapshot(23, 60_000, table_draws=1 << 16)
    d["cfg"] = W.default_config(token_budget=1 << 26, max_batch=64, prefill_chunk=1 << 24)
    s = _sched(d, debug=False)
    s.load(d["pool"], d["tasks"])
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    resolved = 0
    for k in range(3):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        got = s.step(d["now_ns"], d["v_token_ns"])
        _compare(got, ref, ctx=f"step {k} n_spec={got['n_spec']} fallback={got['fallback']}")
        resolved += int(k > 0 and not got["fallback"])
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
    s.close()
    assert resolved >= 1
