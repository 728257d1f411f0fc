"""More GPU parity: coarse (non-unit) histogram bins on the device (reading
A42), compound tasks larger than one work item of the streaming pass (a task of 300+ calls read
in several chunks), the configuration bench.py times (steps 2..K on the 2^20 pool through chained
async steps over rotated handles), steps_waited saturation at 0xFFFF over many steps, and the
device step counter's wrap at 2^32 with the stamp rebase.  Every step is compared with the
oracle run on the state the previous oracle step left."""
import numpy as np
import pytest

import oracle
import workloads as W
from .test_parity_gpu import _compare, _sched

pytestmark = pytest.mark.gpu


def _coarsen(table, edges):
    """a unit-bin table regrouped into bins ending at `edges` (the last = l_max): the counts of
    bin k are those of the unit bins (edges[k-1], edges[k]] (A42: they sit at the upper edge)"""
    cum = table["cum"]
    return {"edges": np.asarray(edges, np.uint32), "cum": np.ascontiguousarray(cum[:, np.asarray(edges) - 1]),
            "l_max": int(table["l_max"])}


def _chain(d, s, n_steps, ctx, rows=True, per_step=None):
    """n_steps synchronous steps on handle s (already loaded) vs the oracle chain"""
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    outs = []
    for k in range(n_steps):
        if per_step:
            per_step(k)
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        got = s.step(d["now_ns"], d["v_token_ns"])
        _compare(got, ref, s.read_rows(debug=s.debug) if rows else None, ctx=f"{ctx} step {k}")
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        outs.append(got)
    return outs


def test_coarse_bins_random_pools():
    rng = np.random.default_rng(501)
    for it in range(80):
        d = W.random_small_pool(rng, int(rng.integers(1, 150)), tie_heavy=(it % 9 == 0))
        l_max = int(d["table"]["l_max"])
        nb = int(rng.integers(1, l_max))
        edges = np.sort(rng.choice(np.arange(1, l_max), nb - 1, replace=False)).tolist() + [l_max]
        d["table"] = _coarsen(d["table"], edges)
        s = _sched(d)
        s.load(d["pool"], d["tasks"])
        _chain(d, s, 3, f"iter {it} bins {nb}")
        s.close()


@pytest.mark.parametrize("n_bins", [2, 64, 700])
def test_coarse_bins_c3(n_bins):
    d = W.pool_snapshot(502, 150_000, table_draws=1 << 16)
    l_max = int(d["table"]["l_max"])
    edges = np.unique(np.geomspace(1, l_max, n_bins).astype(np.int64))
    edges = np.unique(np.concatenate([edges[edges < l_max], [l_max]]))
    d["table"] = _coarsen(d["table"], edges)
    s = _sched(d)
    s.load(d["pool"], d["tasks"])
    _chain(d, s, 3, f"bins {len(edges)}")
    s.close()


def _merge_tasks(parts):
    """one pool from C3 snapshots that share a table: standalone rows of the first, then the tasks
    of every part in order (task sizes mix); ids made unique per part"""
    rows_keys = ("id", "arrival_ns", "input_len", "generated", "prefilled", "meta", "aux", "task",
                 "override_R", "true_out")
    tkeys = ("arrival_ns", "deadline_ns", "cur_stage", "n_stages", "pattern_ms", "goodput_done")
    p0 = parts[0]["pool"]
    ns = int(p0["n_single"])
    blocks = [{k: np.asarray(p0[k])[:ns] for k in rows_keys}]
    tk = {k: [] for k in tkeys}
    off = [ns]
    t_base = 0
    for j, d in enumerate(parts):
        p, t = d["pool"], d["tasks"]
        b = int(p["n_single"])
        blk = {k: np.asarray(p[k])[b:].copy() for k in rows_keys}
        blk["id"] = blk["id"] + np.uint32(j * 10 ** 7)
        blk["task"] = blk["task"] + np.uint32(t_base)
        blocks.append(blk)
        n_t = len(t["arrival_ns"])
        for k in tkeys:
            tk[k].append(np.asarray(t[k]))
        co = np.asarray(t["call_off"], np.int64)
        off += list(off[-1] + (co[1:] - co[0]))
        t_base += n_t
    pool = {k: np.concatenate([b[k] for b in blocks]) for k in rows_keys}
    pool["n_single"] = ns
    tasks = {k: np.concatenate(v) for k, v in tk.items()}
    tasks["call_off"] = np.array(off, np.uint32)
    d = dict(parts[0])
    d["pool"], d["tasks"] = pool, tasks
    return d


def test_big_tasks_multi_chunk():
    """tasks of 300, 1000, 129, 128, 127 calls among tasks of 5 and 16: the streaming pass reads a
    task of more rows than one item holds in several chunks and sums its calls across them"""
    base = W.pool_snapshot(503, 60_000, table_draws=1 << 16)
    parts = [base]
    for j, (cpt, n) in enumerate([(300, 3000), (1000, 3000), (129, 1290), (128, 1280), (127, 1270), (5, 2000)]):
        parts.append(W.pool_snapshot(510 + j, n, frac_compound=1.0, calls_per_task=cpt, table=base["table"]))
    d = _merge_tasks(parts)
    d["cfg"] = W.default_config(token_budget=16384, max_batch=2048)
    s = _sched(d)
    s.load(d["pool"], d["tasks"])
    _chain(d, s, 4, "big tasks")
    s.close()


def test_timed_configuration_chained_async():
    """what bench.py times: the 2^20 C3 pool on rotated handles, first step exact, warm-up steps
    synchronous, then chained step_async steps with no fetch in between; each handle's last batch
    and its per-row state must equal the oracle chain of as many steps, and no step of the chain
    may have needed the host (device fallback / skip counters)."""
    d = W.pool_snapshot(3, 1 << 20)
    rot, warm, K = 2, 3, 6
    hs = []
    for _ in range(rot):
        s = _sched(d, debug=False)
        s.load(d["pool"], d["tasks"])
        s.step(d["now_ns"], d["v_token_ns"])
        hs.append(s)
    for i in range(warm):
        hs[i % rot].step(d["now_ns"], d["v_token_ns"])
    c0 = [s.counters() for s in hs]
    for k in range(K):
        hs[k % rot].step_async(d["now_ns"], d["v_token_ns"])
    got = [s.fetch() for s in hs]
    c1 = [s.counters() for s in hs]
    assert sum(b["skipped"] - a["skipped"] for a, b in zip(c0, c1)) == 0
    assert sum(b["fallbacks"] - a["fallbacks"] for a, b in zip(c0, c1)) == 0
    # oracle chains: handle i ran 1 + |{warm-up steps on i}| + |{chained steps on i}| steps
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    refs = []
    n_max = 1 + max(len(range(i, warm, rot)) + len(range(i, K, rot)) for i in range(rot))
    for k in range(n_max):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        refs.append(ref)
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
    for i, s in enumerate(hs):
        n_i = 1 + len(range(i, warm, rot)) + len(range(i, K, rot))
        _compare(got[i], refs[n_i - 1], s.read_rows(debug=False), ctx=f"handle {i} after {n_i} steps")
        s.close()


def test_waited_saturation_many_steps():
    """steps_waited at 0xFFFD / 0xFFFE / 0xFFFF and rows starting at 0, over 60 steps with no
    progress: the count saturates at 0xFFFF (A12) and the key's waiting term follows it"""
    rng = np.random.default_rng(504)
    for it in range(6):
        d = W.random_small_pool(rng, int(rng.integers(40, 120)))
        aux = d["pool"]["aux"].copy()
        n = len(aux)
        w = rng.choice([0, 1, 0xFFFD, 0xFFFE, 0xFFFF, 0xFFF0], n).astype(np.uint32)
        d["pool"]["aux"] = (aux & np.uint32(0xFFFF)) | (w << np.uint32(16))
        d["cfg"] = dict(d["cfg"], max_batch=1 + it % 3)
        s = _sched(d)
        s.load(d["pool"], d["tasks"])
        _chain(d, s, 60 if it < 2 else 12, f"iter {it}")
        s.close()


def test_step_counter_wrap_and_stamp_rebase():
    """the device step counter wraps at 2^32 and the stamp rebase (every 2^30 launches) runs
    inside this chain; counts and keys must not notice either"""
    rng = np.random.default_rng(505)
    for it, (steps0, launched0) in enumerate([(0xFFFFFFF0, (1 << 30) - 5), (0x7FFFFFF8, (2 << 30) - 1),
                                             (0xFFFFFFFF, (1 << 30) - 1)]):
        d = W.random_small_pool(rng, 100)
        aux = d["pool"]["aux"].copy()
        w = rng.choice([0, 3, 0xFFFC, 0xFFFF], len(aux)).astype(np.uint32)
        d["pool"]["aux"] = (aux & np.uint32(0xFFFF)) | (w << np.uint32(16))
        d["cfg"] = dict(d["cfg"], max_batch=2)
        s = _sched(d)
        s.load(d["pool"], d["tasks"])
        s.debug_set_counter(steps0 - 3, launched0 - 3)
        _chain(d, s, 3, f"case {it} before")
        s.debug_set_counter(steps0, launched0)            # mid-chain: stamps move with the counter
        pool = d["pool"]
        d2 = dict(d)
        d2["pool"] = dict(pool)
        # continue the oracle chain from the state after 3 steps (re-run it to get there)
        st = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in pool.items()}
        for _ in range(3):
            r = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], st, d["tasks"])
            st["meta"], st["aux"] = r["meta"], r["aux"]
        d2["pool"] = st
        _chain(d2, s, 30, f"case {it} across the wrap")
        s.close()


def test_big_sets_resolve_on_device_in_chained_steps():
    """Speculative sets larger than k_spec's fast path (C4-shaped pool): after the first such step
    the handle chains the big-set resolve in its step graph, so chained step_async steps resolve on
    the device (no host path, nothing skipped); every step still equals the oracle chain."""
    from .test_parity_gpu import _compare, _sched
    d = W.pool_c4(n_tasks=20_000, table_draws=1 << 15)
    s = _sched(d, debug=False)
    s.load(d["pool"], d["tasks"])
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    refs = []
    for k in range(6):
        ref = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"])
        pool["meta"], pool["aux"] = ref["meta"], ref["aux"]
        refs.append(ref)
    for k in range(2):                                   # exact path, then a host-resolved big set
        _compare(s.step(d["now_ns"], d["v_token_ns"]), refs[k], ctx=f"C4 step {k}")
    c0 = s.counters()
    for k in range(2, 5):
        s.step_async(d["now_ns"], d["v_token_ns"])
    got = s.fetch()
    c1 = s.counters()
    assert got["n_spec"] > 256, got["n_spec"]
    assert c1["fallbacks"] == c0["fallbacks"] and c1["skipped"] == c0["skipped"], (c0, c1)
    assert c1["steps"] == c0["steps"] + 3
    _compare(got, refs[4], s.read_rows(debug=False), ctx="C4 chained step 4")
    _compare(s.step(d["now_ns"], d["v_token_ns"]), refs[5], ctx="C4 step 5")
    s.close()
