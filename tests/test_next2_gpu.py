"""GPU parity of the NEXT-2 rows: the fairness blend (A47) in the pool step (streaming pass,
speculative and exact resolves, arrivals) and in the replay, and the online adaptation of p (A48)
in the replay -- bit-exact against the oracle."""
import numpy as np
import pytest

import oracle
import workloads as W
from .test_parity_gpu import _compare, _sched
from .test_replay_gpu import _cmp, _spec
from .test_gate_gpu import _cmp_gate

pytestmark = pytest.mark.gpu


def _chain(d, s, n_steps, ctx):
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    for k in range(n_steps):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        got = s.step(d["now_ns"], d["v_token_ns"])
        _compare(got, ref, s.read_rows(debug=s.debug), ctx=f"{ctx} step {k}")
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]


def test_blend_random_pools():
    rng = np.random.default_rng(901)
    for it in range(60):
        d = W.random_small_pool(rng, int(rng.integers(1, 120)), tie_heavy=(it % 8 == 0))
        d["pool"]["fair"] = rng.integers(0, 3000, len(d["pool"]["id"])).astype(np.uint32)
        den = int(rng.choice([2, 10, 7]))
        d["cfg"] = dict(d["cfg"], fair_num=int(rng.integers(0, den + 1)), fair_den=den)
        s = _sched(d)
        s.load(d["pool"], d["tasks"])
        _chain(d, s, 3, f"iter {it}")
        s.close()


@pytest.mark.parametrize("num,den", [(1, 2), (1, 10), (1, 1)])
def test_blend_c3_speculative_chain(num, den):
    d = W.pool_snapshot(902, 200_000, table_draws=1 << 16)
    rng = np.random.default_rng(num * 10 + den)
    d["pool"]["fair"] = rng.integers(0, 400, len(d["pool"]["id"])).astype(np.uint32)
    d["cfg"] = dict(d["cfg"], fair_num=num, fair_den=den)
    s = _sched(d, debug=False)
    s.load(d["pool"], d["tasks"])
    _chain(d, s, 4, f"f={num}/{den}")
    s.close()


def test_blend_with_arrivals():
    base = W.pool_snapshot(903, 20_000, table_draws=1 << 14)
    rng = np.random.default_rng(903)
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base["pool"].items()}
    ns = int(pool["n_single"])
    n = len(pool["id"])
    fair = rng.integers(0, 500, n).astype(np.uint32)
    cfg = dict(base["cfg"], fair_num=3, fair_den=10)
    # the GPU starts with the compound rows + the first half of the standalone rows; the second
    # half arrives with its Fair scores
    half = ns // 2
    keys = ("id", "arrival_ns", "input_len", "generated", "prefilled", "meta", "aux", "task", "override_R")
    first = {k: np.concatenate([pool[k][:half], pool[k][ns:]]) for k in keys}
    first["n_single"] = half
    first["fair"] = np.concatenate([fair[:half], fair[ns:]])
    tasks = dict(base["tasks"])
    tasks["call_off"] = (np.asarray(tasks["call_off"], np.int64) - (ns - half)).astype(np.uint32)
    arr = {k: pool[k][half:ns].copy() for k in keys}
    arr["n_single"] = ns - half
    arr["fair"] = fair[half:ns]
    from paper_2504_20068_b200 import Scheduler
    s = Scheduler(cfg, base["groups"], base["table"], capacity=n, task_capacity=len(tasks["arrival_ns"]), debug=True)
    s.load(first, tasks)
    got = s.step(base["now_ns"], base["v_token_ns"], arrivals=arr)
    # the oracle's pool in the GPU's row order: first, then the arrivals
    opool = {k: np.concatenate([first[k], arr[k]]) for k in keys}
    opool["n_single"] = half
    opool["fair"] = np.concatenate([first["fair"], arr["fair"]])
    # compound rows sit between the two standalone blocks: the oracle needs standalone rows first
    perm = np.concatenate([np.arange(half), np.arange(n - (ns - half), n), np.arange(half, n - (ns - half))])
    opool = {k: (v[perm] if isinstance(v, np.ndarray) else v) for k, v in opool.items()}
    opool["n_single"] = ns
    otasks = dict(tasks)
    otasks["call_off"] = (np.asarray(tasks["call_off"], np.int64) + (ns - half)).astype(np.uint32)
    ref = oracle.step(cfg, base["groups"], base["table"], base["now_ns"], base["v_token_ns"], opool, otasks)
    for k in ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star"):
        assert got[k] == ref[k], k
    assert np.array_equal(got["batch_ids"], ref["batch_ids"])
    assert np.float64(got["bp"]).view(np.uint64) == np.float64(ref["bp"]).view(np.uint64)
    s.close()


def test_replay_blend_and_online_p():
    rng = np.random.default_rng(904)
    for it in range(6):
        d = W.trace_mixed(400 + it, n_rows=int(rng.integers(40, 600)), rate_per_s=float(rng.uniform(5, 40)))
        d["trace"]["fair"] = rng.integers(0, 800, len(d["trace"]["input_len"])).astype(np.uint32)
        d["cfg"] = W.default_config(token_budget=int(rng.integers(600, 4000)), max_batch=int(rng.integers(1, 48)),
                                    prefill_chunk=512, frame_steps=int(rng.choice([2, 5, 50])),
                                    fair_num=int(rng.integers(0, 4)), fair_den=4,
                                    preempt=int(it % 2), pmtn_num=1, pmtn_den=10)
        rc = dict(d["rcfg"], n_steps=2500, p_adapt=int(it != 0), eps_num=int(rng.integers(0, 3)), eps_den=4,
                  window_frames=int(rng.choice([1, 3, 10])), seed=int(rng.integers(0, 1 << 40)))
        ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        from paper_2504_20068_b200 import Scheduler
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=1024, task_capacity=8)
        res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
        _cmp_gate(res[0], log[0], ref, f"replay {it}")
        assert np.array_equal(log[0]["p_num"][:len(ref["log"])], ref["log"]["p_num"])
        s.close()


def test_c5_sampled_online_p():
    traces = [W.trace_mixed(k) for k in range(2)]
    d = traces[0]
    sweep = W.c5_sweep()
    picks = [5, 64 * 40 + 3]
    specs = [dict(sweep[i], trace=i % 2) for i in picks]
    rc0 = dict(d["rcfg"], p_adapt=1, eps_num=1, eps_den=10, window_frames=4, seed=77)
    from paper_2504_20068_b200 import Scheduler
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=4096, task_capacity=1024)
    res, log = s.replay([t["trace"] for t in traces], specs, rc0, log_steps=rc0["n_steps"])
    for j, sp in enumerate(specs):
        rc = dict(rc0, **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
        t = traces[sp["trace"]]
        ref = oracle.replay(t["cfg"], t["groups"], t["table"], t["trace"], rc, log=True)
        _cmp(res[j], log[j], ref, f"C5 pick {picks[j]}")
        assert np.array_equal(log[j]["p_num"][:len(ref["log"])], ref["log"]["p_num"])
    s.close()
