"""GPU parity of the per-step deltas of jit_sched_step (the API of P:544): arrivals
appended to the resident pool (standalone requests and whole new compound tasks), task updates
(stage release, goodput of finished calls, an explicit stage sub-deadline) and progress keyed by
request id.  The oracle runs every step on the same requests in the load layout (standalone rows
first, then the tasks' calls), so rows differ: batches, per-request state and every scalar are
compared through the request ids."""
import numpy as np
import pytest

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

ROW_KEYS = ("id", "arrival_ns", "input_len", "generated", "prefilled", "meta", "aux", "task", "override_R")
TASK_KEYS = ("arrival_ns", "deadline_ns", "cur_stage", "n_stages", "pattern_ms", "goodput_done")


def _split(d):
    """standalone rows and per-task call blocks of a pool snapshot"""
    p, t = d["pool"], d["tasks"]
    ns = int(p["n_single"])
    std = {k: np.asarray(p[k])[:ns].copy() for k in ROW_KEYS + ("true_out",)}
    tasks = []
    for i in range(len(t["arrival_ns"])):
        b, e = int(t["call_off"][i]), int(t["call_off"][i + 1])
        rows = {k: np.asarray(p[k])[b:e].copy() for k in ROW_KEYS + ("true_out",)}
        tasks.append((rows, {k: np.asarray(t[k])[i].copy() for k in TASK_KEYS}))
    return std, tasks


def _assemble(std, tasks):
    """a pool in the load layout from standalone rows and (rows, task constants) blocks; the rows'
    task fields are renumbered 0.. in block order"""
    parts = [std] + [b[0] for b in tasks]
    pool = {k: np.concatenate([p[k] for p in parts]) for k in ROW_KEYS + ("true_out",)}
    ns = len(std["input_len"])
    pool["n_single"] = ns
    off = [ns]
    for i, (rows, _) in enumerate(tasks):
        pool["task"][off[-1]:off[-1] + len(rows["input_len"])] = i
        off.append(off[-1] + len(rows["input_len"]))
    if not tasks:
        return pool, None
    tk = {k: np.stack([b[1][k] for b in tasks]) for k in TASK_KEYS}
    tk["call_off"] = np.array(off, np.uint32)
    return pool, tk


def test_engine_loop_with_arrivals_task_updates_and_progress_by_id():
    base = W.pool_snapshot(41, 20_000, table_draws=1 << 16)
    extra = W.pool_snapshot(42, 12_000, table=base["table"])
    extra["pool"]["id"] = extra["pool"]["id"] + np.uint32(10 ** 6)          # ids stay unique
    cfg = W.default_config(token_budget=4096, max_batch=1024, refine_interval=7)
    b_std, b_tasks = _split(base)
    e_std, e_tasks = _split(extra)
    from paper_2504_20068_b200 import Scheduler
    cap = 40_000
    s = Scheduler(cfg, base["groups"], base["table"], capacity=cap, task_capacity=4096, debug=True)
    pool0, tasks0 = _assemble(b_std, b_tasks)
    s.load(pool0, tasks0)
    gpu_ids = pool0["id"].copy()                       # the GPU's rows in order (appends go to the end)
    o_std = {k: v.copy() for k, v in b_std.items()}      # the oracle's requests (load layout)
    o_tasks = [(dict(r), dict(t)) for r, t in b_tasks]
    stage_dl = [-1] * len(o_tasks)
    now, v = base["now_ns"], base["v_token_ns"]
    progress = None
    n_std_step, n_task_step = 600, 20
    for step in range(12):
        arrivals = arrival_tasks = task_updates = None
        a_std = {k: vv[step * n_std_step:(step + 1) * n_std_step] for k, vv in e_std.items()}
        a_tasks = e_tasks[step * n_task_step:(step + 1) * n_task_step]
        if len(a_std["input_len"]) or a_tasks:
            arrivals, arrival_tasks = _assemble(a_std, a_tasks)
            gpu_ids = np.concatenate([gpu_ids, arrivals["id"]])
            o_std = {k: np.concatenate([o_std[k], a_std[k]]) for k in o_std}
            o_tasks += [(dict(r), dict(t)) for r, t in a_tasks]
            stage_dl += [-1] * len(a_tasks)
        if step % 3 == 2:                              # advance a few tasks to their next stage
            sel = [i for i, (_, t) in enumerate(o_tasks) if int(t["cur_stage"]) + 1 < int(t["n_stages"])][:8]
            tu = {"task": np.array(sel, np.uint32), "cur_stage": np.zeros(len(sel), np.uint32),
                  "goodput_done": np.zeros(len(sel), np.uint64), "stage_deadline_ns": np.full(len(sel), -1, np.int64)}
            for j, i in enumerate(sel):
                t = o_tasks[i][1]
                t["cur_stage"] = np.uint32(int(t["cur_stage"]) + 1)
                t["goodput_done"] = np.uint64(int(t["goodput_done"]) + 100 + j)
                tu["cur_stage"][j] = t["cur_stage"]
                tu["goodput_done"][j] = t["goodput_done"]
                if j % 2:                               # an explicit stage sub-deadline
                    stage_dl[i] = int(t["arrival_ns"]) + (j + 1) * W.S_
                    tu["stage_deadline_ns"][j] = stage_dl[i]
                else:
                    stage_dl[i] = -1
            task_updates = tu
        opool, otasks = _assemble(o_std, o_tasks)
        if otasks is not None:
            otasks["stage_deadline_ns"] = np.array(stage_dl, np.int64)
        ref = oracle.step(cfg, base["groups"], base["table"], now, v, opool, otasks)
        got = s.step(now, v, progress=progress, arrivals=arrivals, arrival_tasks=arrival_tasks,
                     task_updates=task_updates)
        ctx = f"step {step}"
        assert got["status"] == ref["status"], ctx
        for k in ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star", "n_dropped_now"):
            assert got[k] == ref[k], (ctx, k, got[k], ref[k])
        assert np.float64(got["bp"]).view(np.uint64) == np.float64(ref["bp"]).view(np.uint64), ctx
        assert np.float64(got["thr"]).view(np.uint64) == np.float64(ref["thr"]).view(np.uint64), ctx
        assert np.array_equal(got["batch_ids"], ref["batch_ids"]), ctx
        assert np.array_equal(got["batch_tokens"], ref["batch_tokens"]), ctx
        # per-request state, by id
        rows = s.read_rows()
        o_index = {int(i): r for r, i in enumerate(opool["id"])}
        perm = np.array([o_index[int(i)] for i in gpu_ids])
        assert np.array_equal(rows["meta"], ref["meta"][perm]), ctx
        assert np.array_equal(rows["aux"], ref["aux"][perm]), ctx
        pend = ref["pending"][perm].astype(bool)
        assert np.array_equal(rows["key"].view(np.uint64)[pend], ref["key"][perm].view(np.uint64)[pend]), ctx
        # carry the oracle's bookkeeping over and run the batch (engine progress, keyed by id)
        std_n = len(o_std["input_len"])
        where = {}                                     # id -> (block holding the request, index)
        o_std["meta"], o_std["aux"] = ref["meta"][:std_n].copy(), ref["aux"][:std_n].copy()
        for j in range(std_n):
            where[int(o_std["id"][j])] = (o_std, j)
        off = std_n
        for rows_t, _ in o_tasks:
            m = len(rows_t["input_len"])
            rows_t["meta"], rows_t["aux"] = ref["meta"][off:off + m].copy(), ref["aux"][off:off + m].copy()
            for j in range(m):
                where[int(rows_t["id"][j])] = (rows_t, j)
            off += m
        sel_ids = ref["batch_ids"]
        gen_upd, pre_upd, st_upd = [], [], []
        for bid, tok in zip(sel_ids, ref["batch_tokens"]):
            holder, j = where[int(bid)]
            pre, gen, L_in = int(holder["prefilled"][j]), int(holder["generated"][j]), int(holder["input_len"][j])
            if pre < L_in:                             # a prefill chunk; its end emits token 0 (A28)
                pre = min(pre + int(tok), L_in)
                if pre == L_in:
                    gen += 1
            else:
                gen += 1
            st = (int(holder["meta"][j]) >> 8) & 0xF
            if gen >= int(holder["true_out"][j]):
                st = W.Q_DONE
            holder["prefilled"][j], holder["generated"][j] = pre, gen
            holder["meta"][j] = (int(holder["meta"][j]) & ~0xF00) | (st << 8)
            gen_upd.append(gen); pre_upd.append(pre); st_upd.append(st)
        progress = {"id": np.asarray(sel_ids, np.uint32), "generated": np.array(gen_upd, np.uint32),
                    "prefilled": np.array(pre_upd, np.uint32), "state": np.array(st_upd, np.uint32)}
        now += 20 * W.MS
    s.close()


def test_progress_validation_fails_the_step():
    """Done is final and unknown ids are errors (S:37 state machine; ADVICE k_progress)."""
    from paper_2504_20068_b200 import Scheduler
    from paper_2504_20068_b200.jitsched import JitSchedError
    d = W.pool_snapshot(43, 4096, table_draws=1 << 14)
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=4096, task_capacity=1024)
    s.load(d["pool"], d["tasks"])
    s.step(d["now_ns"], d["v_token_ns"])
    done = int(np.nonzero(((d["pool"]["meta"] >> 8) & 0xF) == W.Q_DONE)[0][0])
    bad = {"id": np.array([d["pool"]["id"][done]], np.uint32), "generated": np.array([1], np.uint32),
           "prefilled": np.array([0], np.uint32), "state": np.array([W.Q_RUNNING], np.uint32)}
    with pytest.raises(JitSchedError):
        s.step(d["now_ns"], d["v_token_ns"], progress=bad)
    s.load(d["pool"], d["tasks"])
    unknown = dict(bad, id=np.array([0xFFFFFFF0], np.uint32), state=np.array([W.Q_RUNNING], np.uint32))
    with pytest.raises(JitSchedError):
        s.step(d["now_ns"], d["v_token_ns"], progress=unknown)
    s.load(d["pool"], d["tasks"])
    dup = dict(d["pool"])
    dup["id"] = dup["id"].copy()
    dup["id"][1] = dup["id"][0]
    with pytest.raises(JitSchedError):
        s.load(dup, d["tasks"])
    s.close()
