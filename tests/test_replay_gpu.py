"""GPU parity of the trace replay (a10): jit_sched_replay vs oracle.replay, per-step logs
(time, batch size, tokens, |Cd|, B*, bp bits, FNV hash of the batch ids in order) and
goodput counters bit-exact."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests import _builders as B

pytestmark = pytest.mark.gpu

RES_KEYS = ("token_goodput", "tokens_processed", "sim_end_ns", "request_goodput", "n_done", "n_dropped", "steps",
            "n_tasks_done", "n_tasks_dropped")


def _sched(d, cap=64):
    from paper_2504_20068_b200 import Scheduler
    return Scheduler(d["cfg"], d["groups"], d["table"], capacity=cap, task_capacity=8)


def _spec(rc, trace=0):
    return dict(trace=trace, load_num=rc["load_num"], load_den=rc["load_den"], slo_num=rc["slo_num"], slo_den=rc["slo_den"])


def _cmp(got, glog, ref, ctx):
    for k in RES_KEYS:
        assert got[k] == ref[k], (ctx, k, got[k], ref[k])
    assert got["error"] == 0
    if glog is not None:
        L = ref["log"]
        n = len(L)
        for f in ("now_ns", "n_selected", "total_tokens", "n_candidates", "b_star", "ids_hash"):
            assert np.array_equal(glog[f][:n], L[f]), (ctx, f, np.nonzero(glog[f][:n] != L[f])[0][:5])
        assert np.array_equal(glog["bp"][:n].view(np.uint64), L["bp"].view(np.uint64)), ctx


def test_c1_toy_full_log():
    d = W.trace_c1()
    ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], d["rcfg"], log=True)
    s = _sched(d)
    res, log = s.replay([d["trace"]], [_spec(d["rcfg"])], d["rcfg"], log_steps=d["rcfg"]["n_steps"])
    _cmp(res[0], log[0], ref, "C1")
    s.close()


def test_single_ddl_and_edf_adversary():
    e = W.edf_adversary()
    ref = oracle.replay(e["cfg"], e["groups"], e["table"], e["trace"], e["rcfg"], log=True)
    s = _sched(e)
    res, log = s.replay([e["trace"]], [_spec(e["rcfg"])], e["rcfg"], log_steps=64)
    _cmp(res[0], log[0], ref, "edf")
    assert res[0]["token_goodput"] == 100
    s.close()
    groups = W.make_groups([(W.DDL, 0, 0, 20 * W.S_, 0)])
    tab = B.table_from_supports([(10, 10)], 64)
    tr = B.single_trace([dict(arrival_ns=0, input_len=100, true_out=10, group=0, dist_row=0)])
    d = {"cfg": W.default_config(token_budget=8192, max_batch=256), "groups": groups, "table": tab}
    s = _sched(d)
    res, _ = s.replay([tr], [_spec(B.default_rcfg())], B.default_rcfg())
    assert res[0]["sim_end_ns"] == 21_022_500 and res[0]["token_goodput"] == 110
    s.close()


def test_c5_sampled_replays_full_logs():
    """C5(i): sampled (load, SLO-scale) points of the sweep, 4096 steps each, full logs."""
    traces = [W.trace_mixed(k) for k in range(3)]
    d = traces[0]
    sweep = W.c5_sweep()
    picks = [0, 63, 64 * 31 + 17, 64 * 63, 4095, 2222]
    specs = [dict(sweep[i], trace=i % 3) for i in picks]
    s = _sched(d)
    res, log = s.replay([t["trace"] for t in traces], specs, d["rcfg"], log_steps=d["rcfg"]["n_steps"])
    for j, sp in enumerate(specs):
        rc = dict(d["rcfg"], **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
        t = traces[sp["trace"]]
        ref = oracle.replay(t["cfg"], t["groups"], t["table"], t["trace"], rc, log=True)
        _cmp(res[j], log[j], ref, f"C5 pick {picks[j]}")
    s.close()


@pytest.mark.parametrize("n_rep", [640, 1024])
def test_c5_sweep_path_sampled(n_rep):
    """More replays than two per SM take a sweep configuration, state in global slices: 256-thread
    CTAs (3 per SM) below 6 replays per SM (640), 128-thread CTAs (8 per SM, 512 sort rows in
    shared memory) from there (1024): a sample of them, full logs, against the oracle."""
    traces = [W.trace_mixed(k) for k in range(3)]
    d = traces[0]
    sweep = W.c5_sweep()
    specs = [dict(sweep[(i * 4096) // n_rep], trace=i % 3) for i in range(n_rep)]
    rc0 = dict(d["rcfg"], n_steps=1024)
    s = _sched(d)
    res, log = s.replay([t["trace"] for t in traces], specs, rc0, log_steps=1024)
    for j in (0, 1, 97, 331, 500, 777 % n_rep, n_rep - 1):
        sp = specs[j]
        rc = dict(rc0, **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
        t = traces[sp["trace"]]
        ref = oracle.replay(t["cfg"], t["groups"], t["table"], t["trace"], rc, log=True)
        _cmp(res[j], log[j], ref, f"C5 sweep replay {j}")
    s.close()


def test_c2_10k_until_drained():
    """BASELINE config C2: 10K chat + deadline mix, 8 SLO groups, tau 8192 -- one serial replay."""
    d = W.trace_c2()
    ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], d["rcfg"], log=True)
    s = _sched(d)
    res, log = s.replay([d["trace"]], [_spec(d["rcfg"])], d["rcfg"], log_steps=ref["steps"])
    _cmp(res[0], log[0], ref, "C2")
    s.close()


def test_many_small_random_traces():
    rng = np.random.default_rng(77)
    for it in range(6):
        d = W.trace_mixed(100 + it, n_rows=int(rng.integers(20, 400)), rate_per_s=float(rng.uniform(2, 40)))
        d["cfg"] = W.default_config(token_budget=int(rng.integers(600, 4000)), max_batch=int(rng.integers(1, 64)),
                                    prefill_chunk=512, refine_interval=int(rng.choice([1, 50])))
        rc = dict(d["rcfg"], n_steps=3000)
        ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        s = _sched(d)
        res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
        _cmp(res[0], log[0], ref, f"random {it}")
        s.close()


def test_task_drops_in_the_same_step_as_scoring():
    """Mixed traces whose compound tasks are dropped by admission (A40) while other rows are
    scored: the dropped calls must leave the pending set in that very step (regression: the
    compound-row cleanup once raced the task pass)."""
    rng = np.random.default_rng(701)
    for it in range(4):
        d = W.trace_mixed(300 + it, n_rows=int(rng.integers(20, 500)), rate_per_s=float(rng.uniform(2, 60)))
        d["cfg"] = W.default_config(token_budget=int(rng.integers(600, 4000)), max_batch=int(rng.integers(1, 48)),
                                    prefill_chunk=512, refine_interval=int(rng.choice([1, 50])),
                                    frame_steps=int(rng.choice([1, 2, 7, 50])))
        rc = dict(d["rcfg"], n_steps=3000)
        ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        s = _sched(d, cap=512)
        res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
        _cmp(res[0], log[0], ref, f"drops {it}")
        s.close()


@pytest.mark.parametrize("n_rep", [400, 900])
def test_sweep_configs_short(n_rep):
    """Both sweep configurations (256-thread CTAs below 6 replays per SM, 128-thread CTAs x 8 per
    SM from there) on short replays -- sized for the sanitizers (profiles/sanitize.sh): sampled
    replays against the oracle, full logs."""
    traces = [W.trace_mixed(k) for k in range(2)]
    d = traces[0]
    sweep = W.c5_sweep()
    specs = [dict(sweep[(i * 4093) % 4096], trace=i % 2) for i in range(n_rep)]
    rc0 = dict(d["rcfg"], n_steps=24)
    s = _sched(d)
    res, log = s.replay([t["trace"] for t in traces], specs, rc0, log_steps=24)
    for j in (0, n_rep // 2, n_rep - 1):
        sp = specs[j]
        rc = dict(rc0, **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
        t = traces[sp["trace"]]
        ref = oracle.replay(t["cfg"], t["groups"], t["table"], t["trace"], rc, log=True)
        _cmp(res[j], log[j], ref, f"short sweep replay {j}")
    s.close()
