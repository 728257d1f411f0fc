"""GPU parity of the NEXT-1 preemption gate in the trace replay (reading A46; §4.2 P:482-490,
App. D.2): jit_sched_replay with the gate on vs oracle.replay, per-step logs
(including evictions and KV stall) and goodput counters bit-exact."""
import numpy as np
import pytest

import oracle
import workloads as W
from tests import _builders as B
from .test_replay_gpu import _cmp, _sched, _spec

pytestmark = pytest.mark.gpu

MS, S_ = W.MS, W.S_


def _cmp_gate(got, glog, ref, ctx):
    _cmp(got, glog, ref, ctx)
    assert got["n_preempted"] == ref["n_preempted"], (ctx, got["n_preempted"], ref["n_preempted"])
    L = ref["log"]
    n = len(L)
    for f in ("n_preempted", "stall_ns", "v_token_ns"):
        assert np.array_equal(glog[f][:n], L[f]), (ctx, f, np.nonzero(glog[f][:n] != L[f])[0][:5])


def test_toy_timeline():
    groups = W.make_groups([(W.DDL, 0, 0, 10 ** 3 * S_, 0)])
    tab = B.table_from_counts([[0] * 63 + [3]])
    tr = B.single_trace([dict(arrival_ns=0, input_len=1, true_out=20, group=0, override_R=100),
                         dict(arrival_ns=2 * MS + MS // 2, input_len=1, true_out=5, group=0, override_R=10 ** 4)])
    rc = B.default_rcfg(v_token0_ns=MS, c0_ns=MS, c_att_ns=0, c_lin_ns=0, n_steps=100)
    for num, den, bw, pre in [(1, 10, 10 ** 6, 1), (10 ** 6, 1, 10 ** 6, 0), (1, 10, 1, 0)]:
        cfg = W.default_config(token_budget=64, max_batch=1, prefill_chunk=8, refine_interval=1, frame_steps=4,
                               preempt=1, pmtn_num=num, pmtn_den=den, io_bw_tps=bw)
        d = {"cfg": cfg, "groups": groups, "table": tab}
        ref = oracle.replay(cfg, groups, tab, tr, rc, log=True)
        assert ref["n_preempted"] == pre
        s = _sched(d)
        res, log = s.replay([tr], [_spec(rc)], rc, log_steps=64)
        _cmp_gate(res[0], log[0], ref, f"toy {num}/{den} bw {bw}")
        s.close()


@pytest.mark.parametrize("frame,num,bw", [(1, 0, 10 ** 9), (4, 1, 10 ** 6), (50, 1, 10 ** 6), (3, 0, 2000)])
def test_c1_gated(frame, num, bw):
    d = W.trace_c1()
    cfg = dict(d["cfg"], max_batch=6, token_budget=600, frame_steps=frame, preempt=1, pmtn_num=num, pmtn_den=10,
               io_bw_tps=bw)
    rc = dict(d["rcfg"], n_steps=2000)
    ref = oracle.replay(cfg, d["groups"], d["table"], d["trace"], rc, log=True)
    s = _sched(dict(d, cfg=cfg))
    res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
    _cmp_gate(res[0], log[0], ref, f"C1 frame {frame}")
    s.close()


def test_random_traces_gated():
    rng = np.random.default_rng(701)
    seen = 0
    for it in range(8):
        d = W.trace_mixed(300 + it, n_rows=int(rng.integers(20, 500)), rate_per_s=float(rng.uniform(2, 60)))
        d["cfg"] = W.default_config(token_budget=int(rng.integers(600, 4000)), max_batch=int(rng.integers(1, 48)),
                                    prefill_chunk=512, refine_interval=int(rng.choice([1, 50])),
                                    frame_steps=int(rng.choice([1, 2, 7, 50])), preempt=1,
                                    pmtn_num=int(rng.choice([0, 1, 3])), pmtn_den=10,
                                    io_bw_tps=int(rng.choice([10 ** 4, 10 ** 6, 10 ** 9])))
        rc = dict(d["rcfg"], n_steps=3000)
        ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc, log=True)
        seen += ref["n_preempted"] > 0
        s = _sched(d, cap=512)
        res, log = s.replay([d["trace"]], [_spec(rc)], rc, log_steps=rc["n_steps"])
        _cmp_gate(res[0], log[0], ref, f"random {it}")
        s.close()
    assert seen >= 3, seen


def test_c5_sampled_gated():
    """C5 sweep points with the gate on (default delta 0.1, 10^6 tokens/s, Delta = 50)."""
    traces = [W.trace_mixed(k) for k in range(2)]
    d = traces[0]
    cfg = dict(d["cfg"], preempt=1)
    sweep = W.c5_sweep()
    picks = [0, 64 * 31 + 17, 4095]
    specs = [dict(sweep[i], trace=i % 2) for i in picks]
    s = _sched(dict(d, cfg=cfg))
    res, log = s.replay([t["trace"] for t in traces], specs, d["rcfg"], log_steps=d["rcfg"]["n_steps"])
    for j, sp in enumerate(specs):
        rc = dict(d["rcfg"], **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
        t = traces[sp["trace"]]
        ref = oracle.replay(dict(t["cfg"], preempt=1), t["groups"], t["table"], t["trace"], rc, log=True)
        _cmp_gate(res[j], log[j], ref, f"C5 pick {picks[j]}")
    s.close()
