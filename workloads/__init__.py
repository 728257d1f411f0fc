"""Seeded synthetic inputs shared by the oracle and the CUDA path (configs C1-C5).

This module holds NONE of the method's arithmetic: it only draws requests, SLO groups,
length-distribution tables, compound DAGs and configuration constants.  Both ``oracle/``
and ``paper_2504_20068_b200`` consume its dicts of numpy arrays; neither is imported here.

Recipe:
  * RNG: numpy PCG64, seed 250420068 + k for config k.
  * Lengths: lognormal moment-matched to Table 3; output mu shifted by
    +0.25*z where z is the standardized log input-bucket centre (gives the table rows signal).
  * Length tables: histogram (width-1 bins up to L_max) of independent draws per row;
    a request's true L_o is drawn from its own row.
  * SLOs: TTFT ~2 s, TBT ~100 ms, E2EL 20 s, compound 20 s x stages; mix 1:1:1.
  * Arrivals: Poisson.
"""
from __future__ import annotations

import numpy as np

SEED0 = 250420068
NO_TASK = 0xFFFFFFFF
MAX_STAGES = 8
LAT, DDL, CMP, BE = 0, 1, 2, 3
Q_QUEUED, Q_RUNNING, Q_PREEMPTED, Q_DONE, Q_DROPPED, Q_WAITING, Q_MOVED = 0, 1, 2, 3, 4, 5, 6
F_EVER, F_COMPOUND, F_OVERRIDE = 1, 2, 4
MS = 1_000_000
S_ = 1_000_000_000

# (mu, sigma) of ln(length), moment-matched to Table 3, SURVEY.md §8(d)
LOGN = {
    "chat_in": (3.5002, 1.4369), "chat_out": (5.4233, 0.8231),
    "chatc_in": (6.9700, 0.6326), "chatc_out": (8.3688, 0.2594),
    "dr_in": (6.9868, 1.0664), "dr_out": (5.8315, 0.9476),
    "drc_in": (9.2174, 0.6224), "drc_out": (7.9871, 0.6084),
}
# apps: (input key, output key); compound apps are per task, spread over its calls
APPS = [("chat_in", "chat_out"), ("dr_in", "dr_out"), ("chatc_in", "chatc_out"), ("drc_in", "drc_out")]


def rng_for(k: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED0 + k))


def default_config(**over) -> dict:
    """Appendix A of SURVEY.md: paper constants (p=0.95 P:472, R=50 P:283, Delta=50 P:489,
    waiting 5 s P:545) and the readings for the unspecified ones (q, eps, delta_starve)."""
    cfg = dict(token_budget=8192, max_batch=8192, prefill_chunk=512, refine_interval=50, frame_steps=50,
               q_num=95, q_den=100, p_num=95, p_den=100, delta_starve=1, len_key=0, appb_filter=0,
               eps_ns=1000, waiting_ns=5 * S_,
               # NEXT-1 gate (reading A46): off by default; delta_pmtn = 0.1, KV swap
               # bandwidth 10^6 tokens/s
               preempt=0, pmtn_num=1, pmtn_den=10, io_bw_tps=10 ** 6)
    cfg.update(over)
    return cfg


def make_groups(spec) -> dict:
    """spec: list of (type, ttft_ns, tbt_ns, e2el_ns, be_deadline_ns[, w_in, w_out])."""
    g = {k: [] for k in ("type", "w_in", "w_out", "ttft_ns", "tbt_ns", "e2el_ns", "be_deadline_ns")}
    for s in spec:
        t, ttft, tbt, e2el, be = s[:5]
        wi, wo = (s[5], s[6]) if len(s) > 5 else (1, 1)
        for k, v in zip(g, (t, wi, wo, ttft, tbt, e2el, be)):
            g[k].append(v)
    return {k: np.array(v, dtype=np.int64 if k.endswith("_ns") else np.uint32) for k, v in g.items()}


def _bucket(input_len, n_buckets):
    b = np.floor(np.log2(np.maximum(input_len, 1))).astype(np.int64)
    return np.clip(b, 0, n_buckets - 1)


def _out_mu(app, bucket, n_buckets):
    mu = np.array([LOGN[a[1]][0] for a in APPS])[np.asarray(app)]
    z = (np.asarray(bucket) - (n_buckets - 1) / 2.0) / max(n_buckets / 4.0, 1.0)
    return mu + 0.25 * z


def _draw_out(rng, app, bucket, n_buckets, l_max, scale=1.0, size=None):
    mu = _out_mu(app, bucket, n_buckets) + np.log(scale)
    sig = LOGN[APPS[app][1]][1]
    x = np.rint(rng.lognormal(mu, sig, size=size))
    return np.clip(x, 1, l_max).astype(np.uint32)


def make_table(rng, n_apps, n_buckets, l_max, draws=1 << 18, scales=None) -> dict:
    """Length-distribution table: rows = app x input-length bucket; width-1 bins up to L_max;
    cum[row][k] = number of draws with L <= k+1 (a cumulative histogram)."""
    n_rows = n_apps * n_buckets
    cum = np.zeros((n_rows, l_max), np.uint32)
    for a in range(n_apps):
        for b in range(n_buckets):
            sc = scales[a] if scales is not None else 1.0
            x = _draw_out(rng, a, b, n_buckets, l_max, scale=sc, size=draws)
            h = np.bincount(x, minlength=l_max + 1)[1:]
            cum[a * n_buckets + b] = np.cumsum(h).astype(np.uint32)
    edges = np.arange(1, l_max + 1, dtype=np.uint32)
    return {"edges": edges, "cum": cum, "l_max": l_max, "n_buckets": n_buckets, "scales": scales}


def _draw_in(rng, key, size, lo=1, hi=32768, scale=1.0):
    mu, sig = LOGN[key]
    return np.clip(np.rint(rng.lognormal(mu + np.log(scale), sig, size=size)), lo, hi).astype(np.uint32)


def _pack_meta(group, state, flags):
    return (np.asarray(group, np.uint32) | (np.asarray(state, np.uint32) << 8) |
            (np.asarray(flags, np.uint32) << 12)).astype(np.uint32)


def _pack_aux(dist_row, waited):
    return (np.asarray(dist_row, np.uint32) | (np.minimum(np.asarray(waited, np.int64), 0xFFFF).astype(np.uint32) << 16)).astype(np.uint32)


# ----------------------------------------------------------------------------------------
# Pool snapshots (C3, C4, random small pools)
# ----------------------------------------------------------------------------------------

def groups_c3() -> dict:
    spec = []
    for ttft, tbt in [(1, 50), (2, 50), (2, 100), (2, 150), (5, 200), (5, 300)]:
        spec.append((LAT, ttft * S_, tbt * MS, 0, 0))
    for e in (5, 10, 20, 40, 80, 160):
        spec.append((DDL, 0, 0, e * S_, 0))
    for e in (10, 20, 40):
        spec.append((CMP, 0, 0, e * S_, 0))
    spec.append((BE, 0, 0, 0, 600 * S_))
    return make_groups(spec)


def pool_snapshot(seed: int, n: int, frac_compound: float = 0.3, calls_per_task: int = 16,
                  n_buckets: int = 16, l_max: int = 8192, now_ns: int = 1000 * S_, table_draws=1 << 18,
                  done_frac_calls: float = 0.1, table=None) -> dict:
    """C3-shaped pool: 40% chat-single, 30% DR-single, 30% compound calls (tasks of 16);
    25% queued / 10% mid-prefill / 65% decoding; ids a random permutation."""
    rng = rng_for(seed)
    groups = groups_c3()
    if table is None:
        table = make_table(rng, 4, n_buckets, l_max, draws=table_draws)
    n_tasks = int(round(n * frac_compound / calls_per_task))
    n_calls = n_tasks * calls_per_task
    n_single = n - n_calls
    # --- standalone rows
    app = np.where(rng.random(n_single) < 0.4 / 0.7, 0, 1)
    L_in = np.where(app == 0, _draw_in(rng, "chat_in", n_single), _draw_in(rng, "dr_in", n_single))
    bucket = _bucket(L_in, n_buckets)
    mu = _out_mu(app, bucket, n_buckets)
    sig = np.where(app == 0, LOGN["chat_out"][1], LOGN["dr_out"][1])
    L_out = np.clip(np.rint(rng.lognormal(mu, sig)), 1, l_max).astype(np.uint32)
    u = rng.random(n_single)
    gsel = np.where(u < 0.475, rng.integers(0, 6, n_single),
                    np.where(u < 0.95, rng.integers(6, 12, n_single), 15)).astype(np.uint32)
    # --- compound rows (tasks of calls_per_task calls of the current stage)
    t_app = rng.integers(2, 4, n_tasks)
    c_app = np.repeat(t_app, calls_per_task)
    c_in = np.where(c_app == 2, _draw_in(rng, "chatc_in", n_calls, scale=1 / calls_per_task),
                    _draw_in(rng, "drc_in", n_calls, scale=1 / calls_per_task))
    c_bucket = _bucket(c_in, n_buckets)
    c_mu = _out_mu(c_app, c_bucket, n_buckets) - np.log(calls_per_task)
    c_sig = np.where(c_app == 2, LOGN["chatc_out"][1], LOGN["drc_out"][1])
    c_out = np.clip(np.rint(rng.lognormal(c_mu, c_sig)), 1, l_max).astype(np.uint32)
    t_group = rng.integers(12, 15, n_tasks).astype(np.uint32)
    # --- concatenate
    L_in = np.concatenate([L_in, c_in]).astype(np.uint32)
    L_out = np.concatenate([L_out, c_out]).astype(np.uint32)
    apps = np.concatenate([app, c_app])
    buckets = np.concatenate([bucket, c_bucket])
    group = np.concatenate([gsel, np.repeat(t_group, calls_per_task)]).astype(np.uint32)
    dist_row = (apps * n_buckets + buckets).astype(np.uint32)
    # --- progress state
    u = rng.random(n)
    state = np.full(n, Q_QUEUED, np.uint32)
    gen = np.zeros(n, np.uint32)
    pre = np.zeros(n, np.uint32)
    dec = (u >= 0.35) & (L_out >= 2)
    pf = (u >= 0.25) & (u < 0.35) & (L_in >= 2)
    gen[dec] = rng.integers(1, L_out[dec])
    pre[dec] = L_in[dec]
    pre[pf] = rng.integers(1, L_in[pf])
    running = dec | pf
    state[running] = Q_RUNNING
    flags = np.where(running, F_EVER, 0).astype(np.uint32)
    arrival = np.where(running, now_ns - rng.integers(0, 60 * S_, n), now_ns - rng.integers(0, 6 * S_, n))
    waited = np.where(running, rng.poisson(10, n), rng.poisson(60, n))
    task = np.full(n, NO_TASK, np.uint32)
    task[n_single:] = np.repeat(np.arange(n_tasks, dtype=np.uint32), calls_per_task)
    flags[n_single:] |= F_COMPOUND
    done = np.zeros(n, bool)
    done[n_single:] = rng.random(n_calls) < done_frac_calls
    state[done] = Q_DONE
    meta = _pack_meta(group, state, flags)
    aux = _pack_aux(dist_row, waited)
    ids = rng.permutation(n).astype(np.uint32)
    pool = {"id": ids, "arrival_ns": arrival.astype(np.int64), "input_len": L_in, "generated": gen,
            "prefilled": pre, "meta": meta, "aux": aux, "task": task,
            "override_R": np.zeros(n, np.uint32), "true_out": L_out, "n_single": n_single}
    n_st = rng.integers(2, MAX_STAGES + 1, n_tasks).astype(np.uint32)
    cur = (rng.random(n_tasks) * n_st).astype(np.uint32)
    pat = np.zeros((n_tasks, MAX_STAGES), np.uint32)
    for s in range(MAX_STAGES):
        pat[:, s] = np.where(s < n_st, np.clip(np.rint(rng.lognormal(np.log(1000) - 0.5, 1.0, n_tasks)), 1, 60000), 0)
    e2el = groups["e2el_ns"][t_group]
    tasks = {"call_off": (n_single + np.arange(n_tasks + 1, dtype=np.int64) * calls_per_task).astype(np.uint32),
             "arrival_ns": (now_ns - rng.integers(0, 120 * S_, n_tasks)).astype(np.int64),
             "deadline_ns": (e2el * n_st).astype(np.int64), "cur_stage": cur, "n_stages": n_st,
             "pattern_ms": pat, "goodput_done": rng.integers(0, 20000, n_tasks).astype(np.uint64)}
    return {"pool": pool, "tasks": tasks, "groups": groups, "table": table, "now_ns": now_ns,
            "v_token_ns": 15 * MS, "cfg": default_config()}


def pool_c4(seed: int = 4, n_tasks: int = 100_000, l_max: int = 8192, table_draws=1 << 18) -> dict:
    """C4: 100K compound tasks (50% deep-research, 50% agentic); half in a 64-call fan-out
    stage (30% of those calls already done), half in a 1-call stage."""
    rng = rng_for(seed)
    groups = groups_c3()
    n_buckets = 16
    table = make_table(rng, 4, n_buckets, l_max, draws=table_draws)
    fan = rng.random(n_tasks) < 0.5
    calls = np.where(fan, 64, 1).astype(np.int64)
    off = np.zeros(n_tasks + 1, np.int64)
    off[1:] = np.cumsum(calls)
    n = int(off[-1])
    t_app = np.where(rng.random(n_tasks) < 0.5, 3, 2)
    c_app = np.repeat(t_app, calls)
    c_in = np.where(c_app == 3, _draw_in(rng, "drc_in", n, scale=1 / 16), _draw_in(rng, "chatc_in", n, scale=1 / 16))
    c_bucket = _bucket(c_in, n_buckets)
    c_out = np.clip(np.rint(rng.lognormal(_out_mu(c_app, c_bucket, n_buckets) - np.log(16),
                                          np.where(c_app == 3, LOGN["drc_out"][1], LOGN["chatc_out"][1]))),
                    1, l_max).astype(np.uint32)
    now_ns = 1000 * S_
    u = rng.random(n)
    state = np.full(n, Q_QUEUED, np.uint32)
    gen = np.zeros(n, np.uint32)
    pre = np.zeros(n, np.uint32)
    dec = (u >= 0.35) & (c_out >= 2)
    pf = (u >= 0.25) & (u < 0.35) & (c_in >= 2)
    gen[dec] = rng.integers(1, c_out[dec])
    pre[dec] = c_in[dec]
    pre[pf] = rng.integers(1, c_in[pf])
    state[dec | pf] = Q_RUNNING
    fan_row = np.repeat(fan, calls)
    state[fan_row & (rng.random(n) < 0.3)] = Q_DONE
    flags = (np.where(dec | pf, F_EVER, 0) | F_COMPOUND).astype(np.uint32)
    t_group = rng.integers(12, 15, n_tasks).astype(np.uint32)
    group = np.repeat(t_group, calls).astype(np.uint32)
    pool = {"id": rng.permutation(n).astype(np.uint32),
            "arrival_ns": np.repeat(now_ns - rng.integers(0, 120 * S_, n_tasks), calls).astype(np.int64),
            "input_len": c_in, "generated": gen, "prefilled": pre,
            "meta": _pack_meta(group, state, flags),
            "aux": _pack_aux((c_app * n_buckets + c_bucket).astype(np.uint32), rng.poisson(20, n)),
            "task": np.repeat(np.arange(n_tasks, dtype=np.uint32), calls),
            "override_R": np.zeros(n, np.uint32), "true_out": c_out, "n_single": 0}
    n_st = rng.integers(2, MAX_STAGES + 1, n_tasks).astype(np.uint32)
    pat = np.zeros((n_tasks, MAX_STAGES), np.uint32)
    for s in range(MAX_STAGES):
        pat[:, s] = np.where(s < n_st, np.clip(np.rint(rng.lognormal(np.log(1000) - 0.5, 1.0, n_tasks)), 1, 60000), 0)
    tasks = {"call_off": off.astype(np.uint32), "arrival_ns": (now_ns - rng.integers(0, 120 * S_, n_tasks)).astype(np.int64),
             "deadline_ns": (groups["e2el_ns"][t_group] * n_st).astype(np.int64),
             "cur_stage": (rng.random(n_tasks) * n_st).astype(np.uint32), "n_stages": n_st, "pattern_ms": pat,
             "goodput_done": rng.integers(0, 50000, n_tasks).astype(np.uint64)}
    return {"pool": pool, "tasks": tasks, "groups": groups, "table": table, "now_ns": now_ns,
            "v_token_ns": 15 * MS, "cfg": default_config()}


def random_small_pool(rng: np.random.Generator, n: int, n_groups_each: int = 2, l_max: int = 64,
                      n_rows: int = 3, with_tasks: bool = True, tie_heavy: bool = False) -> dict:
    """Small random pool for property / brute-force parity tests (<= a few hundred rows)."""
    spec = []
    for _ in range(n_groups_each):
        spec.append((LAT, int(rng.integers(1, 2000)) * MS, int(rng.integers(1, 200)) * MS, 0, 0,
                     int(rng.integers(0, 3)), int(rng.integers(1, 3))))
        spec.append((DDL, 0, 0, int(rng.integers(1, 60)) * S_, 0, int(rng.integers(0, 3)), int(rng.integers(1, 3))))
    spec.append((BE, 0, 0, 0, 600 * S_))
    spec.append((CMP, 0, 0, 20 * S_, 0))
    groups = make_groups(spec)
    g_cmp = len(spec) - 1
    # random histogram table
    cum = np.zeros((n_rows, l_max), np.uint32)
    for r in range(n_rows):
        h = rng.integers(0, 5, l_max) * (rng.random(l_max) < 0.5)
        if rng.random() < 0.2:
            h = np.zeros(l_max, np.int64)
            h[int(rng.integers(0, l_max))] = 7
        cum[r] = np.cumsum(h)
    table = {"edges": np.arange(1, l_max + 1, dtype=np.uint32), "cum": cum, "l_max": l_max}
    now = 100 * S_
    n_tasks = int(rng.integers(0, 3)) if (with_tasks and n >= 6) else 0
    calls = [int(rng.integers(1, 4)) for _ in range(n_tasks)]
    n_calls = sum(calls)
    n_single = n - n_calls
    L_in = rng.integers(1, 40, n).astype(np.uint32)
    gen = np.zeros(n, np.uint32)
    pre = np.zeros(n, np.uint32)
    state = np.zeros(n, np.uint32)
    flags = np.zeros(n, np.uint32)
    u = rng.random(n)
    dec = u < 0.5
    pre[dec] = L_in[dec]
    gen[dec] = rng.integers(1, l_max, dec.sum())
    pf = (u >= 0.5) & (u < 0.65) & (L_in > 1)
    pre[pf] = rng.integers(1, np.maximum(L_in[pf], 2))
    state[dec | pf] = Q_RUNNING
    flags[dec | pf] = F_EVER
    state[u > 0.95] = rng.choice([Q_DONE, Q_DROPPED, Q_PREEMPTED], (u > 0.95).sum())
    group = rng.integers(0, len(spec) - 1, n).astype(np.uint32)
    arrival = now - rng.integers(0, 8 * S_, n)
    arrival[rng.random(n) < 0.05] = now + S_  # not yet arrived
    waited = rng.integers(0, 400, n)
    task = np.full(n, NO_TASK, np.uint32)
    pos = n_single
    for t, c in enumerate(calls):
        task[pos:pos + c] = t
        group[pos:pos + c] = g_cmp
        flags[pos:pos + c] |= F_COMPOUND
        pos += c
    override = np.zeros(n, np.uint32)
    if rng.random() < 0.3:
        m = (rng.random(n) < 0.3) & (task == NO_TASK)
        override[m] = rng.integers(1, 500, m.sum())
        flags[m] |= F_OVERRIDE
    if tie_heavy:
        gen[:] = 0
        pre[:] = 0
        state[:] = Q_QUEUED
        flags &= ~np.uint32(F_EVER)
        arrival[:] = now - S_
        waited[:] = rng.integers(0, 3, n) * 50
    pool = {"id": rng.permutation(np.arange(1000, 1000 + 3 * n))[:n].astype(np.uint32),
            "arrival_ns": arrival.astype(np.int64), "input_len": L_in, "generated": gen, "prefilled": pre,
            "meta": _pack_meta(group, state, flags),
            "aux": _pack_aux(rng.integers(0, n_rows, n), waited), "task": task, "override_R": override,
            "n_single": n_single}
    tasks = None
    if n_tasks:
        off = np.concatenate([[n_single], n_single + np.cumsum(calls)]).astype(np.uint32)
        n_st = rng.integers(1, MAX_STAGES + 1, n_tasks).astype(np.uint32)
        pat = np.zeros((n_tasks, MAX_STAGES), np.uint32)
        for s in range(MAX_STAGES):
            pat[:, s] = np.where(s < n_st, rng.integers(1, 5000, n_tasks), 0)
        tasks = {"call_off": off, "arrival_ns": (now - rng.integers(0, 50 * S_, n_tasks)).astype(np.int64),
                 "deadline_ns": rng.integers(1, 80, n_tasks).astype(np.int64) * S_,
                 "cur_stage": (rng.random(n_tasks) * n_st).astype(np.uint32), "n_stages": n_st,
                 "pattern_ms": pat, "goodput_done": rng.integers(0, 300, n_tasks).astype(np.uint64)}
    B = int(rng.integers(1, 9))
    cfg = default_config(token_budget=int(rng.integers(40, 200)), max_batch=B,
                         prefill_chunk=int(rng.integers(1, 40)), refine_interval=int(rng.choice([1, 5, 50])),
                         frame_steps=int(rng.choice([1, 50])), p_num=int(rng.choice([95, 70, 100])),
                         len_key=int(rng.integers(0, 2)), appb_filter=int(rng.random() < 0.2))
    return {"pool": pool, "tasks": tasks, "groups": groups, "table": table, "now_ns": now,
            "v_token_ns": int(rng.integers(1, 30)) * MS, "cfg": cfg}


# ----------------------------------------------------------------------------------------
# Replay traces (C1 toy, C2 10K mix, C5 mixed 1:1:1)
# ----------------------------------------------------------------------------------------

def _empty_trace():
    return {k: [] for k in ("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task")}


def _finish_trace(rows, tasks):
    tr = {k: np.array(v, dtype=np.int64 if k == "arrival_ns" else np.uint32) for k, v in rows.items()}
    nt = len(tasks)
    tr["task_arrival_ns"] = np.array([t["arrival"] for t in tasks], np.int64)
    tr["task_deadline_ns"] = np.array([t["D"] for t in tasks], np.int64)
    tr["task_n_stages"] = np.array([len(t["stages"]) for t in tasks], np.uint32)
    for k, dt in (("stage_kind", np.uint32), ("stage_exec_ns", np.int64), ("stage_pattern_ms", np.uint32),
                  ("stage_call_begin", np.uint32), ("stage_call_end", np.uint32)):
        tr[k] = np.zeros(nt * MAX_STAGES, dt)
    for i, t in enumerate(tasks):
        for s, st in enumerate(t["stages"]):
            k = i * MAX_STAGES + s
            tr["stage_kind"][k] = st["kind"]
            tr["stage_exec_ns"][k] = st.get("exec", 0)
            tr["stage_pattern_ms"][k] = st["pattern_ms"]
            tr["stage_call_begin"][k] = st.get("b", 0)
            tr["stage_call_end"][k] = st.get("e", 0)
    return tr


def _add_task(rng, rows, tasks, arrival, group, D, stage_calls, in_key, out_row_of, l_max, in_hi, tool_prob=0.0,
              n_buckets=1, app=2, in_scale=1.0, out_scale=1.0):
    t = {"arrival": int(arrival), "D": int(D), "stages": []}
    tid = len(tasks)
    for s, ncall in enumerate(stage_calls):
        if s > 0 and rng.random() < tool_prob:
            t["stages"].append({"kind": 1, "exec": int(rng.lognormal(np.log(S_) - 0.5, 1.0)),
                                "pattern_ms": int(rng.integers(200, 3000))})
            continue
        b = len(rows["input_len"])
        for _ in range(ncall):
            L_in = int(_draw_in(rng, in_key, None, hi=in_hi, scale=in_scale))
            bucket = int(_bucket(np.array([L_in]), n_buckets)[0])
            row = out_row_of(app, bucket)
            L_o = int(_draw_out(rng, app, bucket, n_buckets, l_max, scale=out_scale))
            for k, v in zip(("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"),
                            (0, L_in, L_o, group, row, 0, tid)):
                rows[k].append(v)
        t["stages"].append({"kind": 0, "b": b, "e": len(rows["input_len"]),
                            "pattern_ms": int(rng.integers(500, 6000))})
    tasks.append(t)


def trace_c1(seed: int = 1) -> dict:
    """C1 toy (SPEC scale): 12 LAT + 12 DDL chat-single requests and 2 compound tasks
    (1 call -> 3 calls); SLOs scaled by 1/40 so they bind; L_max 256; 200 steps."""
    rng = rng_for(seed)
    l_max, nb = 256, 1
    table = make_table(rng, 3, nb, l_max, draws=1 << 16, scales=[0.25, 1.0, 0.01])
    groups = make_groups([(LAT, 50 * MS, 2_500_000, 0, 0), (DDL, 0, 0, 500 * MS, 0), (CMP, 0, 0, 500 * MS, 0),
                          (BE, 0, 0, 0, 15 * S_)])
    rows, tasks = _empty_trace(), []
    t = 0
    kinds = [LAT] * 12 + [DDL] * 12 + [CMP] * 2
    rng.shuffle(kinds)
    for k in kinds:
        t += int(rng.exponential(10 * MS))
        if k == CMP:
            _add_task(rng, rows, tasks, t, 2, 2 * 500 * MS, [1, 3], "chat_in", lambda a, b: 2, l_max, 512,
                      n_buckets=nb, app=2, in_scale=0.05, out_scale=0.01)
            continue
        L_in = int(_draw_in(rng, "chat_in", None, hi=512))
        L_o = int(_draw_out(rng, 0, 0, nb, l_max, scale=0.25))
        for key, v in zip(("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"),
                          (t, L_in, L_o, 0 if k == LAT else 1, 0, 0, NO_TASK)):
            rows[key].append(v)
    tr = _finish_trace(rows, tasks)
    cfg = default_config(token_budget=512, max_batch=512, prefill_chunk=512)
    rcfg = dict(n_steps=200, v_token0_ns=2_050_000, c0_ns=2_000_000, c_att_ns=500, c_lin_ns=50_000,
                load_num=1, load_den=1, slo_num=1, slo_den=1)
    return {"trace": tr, "groups": groups, "table": table, "cfg": cfg, "rcfg": rcfg}


def groups_c2() -> dict:
    spec = [(LAT, 2 * S_, tbt * MS, 0, 0) for tbt in (50, 100, 200)]
    spec += [(DDL, 0, 0, e * S_, 0) for e in (10, 20, 40, 80)]
    spec += [(BE, 0, 0, 0, 600 * S_)]
    return make_groups(spec)


def trace_c2(seed: int = 2, n_req: int = 10_000, rate_per_s: float = 30.0, l_max: int = 8192) -> dict:
    """C2: 10K requests, 50% LAT / 45% DDL / 5% BE, 70% chat / 30% DR lengths, 8 SLO groups,
    token budget 8192, B_max 256, Poisson arrivals; replay until drained."""
    rng = rng_for(seed)
    nb = 8
    table = make_table(rng, 2, nb, l_max, draws=1 << 18)
    groups = groups_c2()
    gap = rng.exponential(S_ / rate_per_s, n_req)
    arrival = np.cumsum(gap).astype(np.int64)
    app = np.where(rng.random(n_req) < 0.7, 0, 1)
    L_in = np.where(app == 0, _draw_in(rng, "chat_in", n_req, hi=16384), _draw_in(rng, "dr_in", n_req, hi=16384))
    bucket = _bucket(L_in, nb)
    L_o = np.clip(np.rint(rng.lognormal(_out_mu(app, bucket, nb),
                                        np.where(app == 0, LOGN["chat_out"][1], LOGN["dr_out"][1]))), 1, l_max)
    u = rng.random(n_req)
    group = np.where(u < 0.5, rng.integers(0, 3, n_req), np.where(u < 0.95, rng.integers(3, 7, n_req), 7))
    rows = {"arrival_ns": arrival, "input_len": L_in, "true_out": L_o.astype(np.uint32),
            "group": group.astype(np.uint32), "dist_row": (app * nb + bucket).astype(np.uint32),
            "override_R": np.zeros(n_req, np.uint32), "task": np.full(n_req, NO_TASK, np.uint32)}
    tr = _finish_trace({k: list(v) for k, v in rows.items()}, [])
    cfg = default_config(token_budget=8192, max_batch=256)
    rcfg = dict(n_steps=1_000_000, v_token0_ns=2_050_000, c0_ns=2_000_000, c_att_ns=500, c_lin_ns=50_000,
                load_num=1, load_den=1, slo_num=1, slo_den=1)
    return {"trace": tr, "groups": groups, "table": table, "cfg": cfg, "rcfg": rcfg}


def groups_c5() -> dict:
    return make_groups([(LAT, 2 * S_, 100 * MS, 0, 0), (DDL, 0, 0, 20 * S_, 0), (CMP, 0, 0, 20 * S_, 0),
                        (BE, 0, 0, 0, 600 * S_)])


def trace_mixed(seed: int, n_rows: int = 2048, rate_per_s: float = 12.0, l_max: int = 8192, table=None) -> dict:
    """C5 base trace: mixed 1:1:1 (LAT : DDL : compound task) by request count, Poisson
    arrivals, compound tasks of 2-4 stages with 1-4 calls per LLM stage and occasional
    tool stages; exactly n_rows rows."""
    rng = rng_for(5 * 7919 + seed)
    nb = 8
    if table is None:
        table = make_table(rng_for(5), 4, nb, l_max, draws=1 << 17)
    groups = groups_c5()
    rows, tasks = _empty_trace(), []
    t = 0
    i = 0
    while len(rows["input_len"]) < n_rows:
        t += int(rng.exponential(S_ / rate_per_s))
        kind = i % 3
        i += 1
        if kind == 2:
            S = int(rng.integers(2, 5))
            calls = [int(rng.integers(1, 5)) for _ in range(S)]
            if len(rows["input_len"]) + sum(calls) > n_rows:
                kind = int(rng.integers(0, 2))
            else:
                app = int(rng.integers(2, 4))
                _add_task(rng, rows, tasks, t, 2, 20 * S_ * S, calls, "chatc_in" if app == 2 else "drc_in",
                          lambda a, b: a * nb + b, l_max, 16384, tool_prob=0.25, n_buckets=nb, app=app,
                          in_scale=0.1, out_scale=0.1)
                continue
        app = 0 if rng.random() < 0.7 else 1
        L_in = int(_draw_in(rng, "chat_in" if app == 0 else "dr_in", None, hi=16384))
        bucket = int(_bucket(np.array([L_in]), nb)[0])
        L_o = int(_draw_out(rng, app, bucket, nb, l_max))
        for key, v in zip(("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"),
                          (t, L_in, L_o, kind, app * nb + bucket, 0, NO_TASK)):
            rows[key].append(v)
    tr = _finish_trace(rows, tasks)
    cfg = default_config(token_budget=2048, max_batch=128)
    rcfg = dict(n_steps=4096, v_token0_ns=2_050_000, c0_ns=2_000_000, c_att_ns=500, c_lin_ns=50_000,
                load_num=1, load_den=1, slo_num=1, slo_den=1)
    return {"trace": tr, "groups": groups, "table": table, "cfg": cfg, "rcfg": rcfg}


def c5_sweep(n_replays: int = 4096, n_load: int = 64, n_slo: int = 64):
    """C5(i) sweep grid: load factors geometric 0.25x-4x, SLO scales geometric 0.5x-2x (covers
    the paper's 0.8x/1.5x), as exact rationals over 1024.  Replay i -> (load i//n_slo,
    slo i%n_slo)."""
    loads = np.rint(1024 * np.geomspace(0.25, 4.0, n_load)).astype(np.uint64)
    slos = np.rint(1024 * np.geomspace(0.5, 2.0, n_slo)).astype(np.uint64)
    out = []
    for i in range(n_replays):
        li, si = (i // n_slo) % n_load, i % n_slo
        out.append(dict(load_num=int(loads[li]), load_den=1024, slo_num=int(slos[si]), slo_den=1024))
    return out


def edf_adversary(T: int = 10, N: int = 9, M: int = 100, v_ns: int = 10 * MS) -> dict:
    """App. D.1 mapped onto the replay: time unit = one iteration of
    v_ns; L_i = 1, L_o = t_comp/unit; B_max = tau = 1; c0 = v, c_att = c_lin = 0; R via
    override.  A: arrival 0, t_comp = T, SLO T, R = M.  B_i: arrival i*delta, t_comp = delta,
    absolute SLO (i+1)*delta (reading A34), R = 1; delta = T/(N+1)."""
    delta = T // (N + 1)
    assert delta * (N + 1) == T
    groups = make_groups([(DDL, 0, 0, T * v_ns, 0), (DDL, 0, 0, delta * v_ns, 0)])
    l_max = max(T, 2)
    cum = np.zeros((2, l_max), np.uint32)
    cum[0, T - 1:] = 1          # point mass at T tokens (A's length)
    cum[1, delta - 1:] = 1      # point mass at delta tokens (B's length)
    table = {"edges": np.arange(1, l_max + 1, dtype=np.uint32), "cum": cum, "l_max": l_max}
    rows = _empty_trace()
    for k, v in zip(("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"),
                    (0, 1, T, 0, 0, M, NO_TASK)):
        rows[k].append(v)
    for i in range(N):
        for k, v in zip(("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"),
                        (i * delta * v_ns, 1, delta, 1, 1, 1, NO_TASK)):
            rows[k].append(v)
    tr = _finish_trace(rows, [])
    cfg = default_config(token_budget=1, max_batch=1, prefill_chunk=1, waiting_ns=10 ** 15)
    rcfg = dict(n_steps=1000, v_token0_ns=v_ns, c0_ns=v_ns, c_att_ns=0, c_lin_ns=0,
                load_num=1, load_den=1, slo_num=1, slo_den=1)
    return {"trace": tr, "groups": groups, "table": table, "cfg": cfg, "rcfg": rcfg}


# ----------------------------------------------------------------------------------------
# NEXT-3 pattern graphs (§4.1): a store of ~500 stage-structured graphs drawn from
# families (deep-research / agentic shapes: LLM plan -> tool -> LLM fan-out -> ... -> LLM
# summary), and queries = fresh instances revealed up to a random stage.
# ----------------------------------------------------------------------------------------

TOOL = 1 << 31


def _pattern_families(rng, n_families):
    fams = []
    for f in range(n_families):
        S = int(rng.integers(2, MAX_STAGES + 1))
        ident, base_in, base_out, base_t = [], [], [], []
        for u in range(S):
            tool = u % 2 == 1 and rng.random() < 0.7
            ident.append((TOOL | int(rng.integers(0, 6))) if tool else int(rng.integers(0, 4)))
            base_in.append(0 if tool else int(rng.lognormal(np.log(800), 0.8)))
            base_out.append(int(rng.lognormal(np.log(300 if tool else 250), 0.7)))   # tool: exec ms
            base_t.append(int(rng.lognormal(np.log(1500), 0.8)))
        fams.append((S, ident, base_in, base_out, base_t))
    return fams


def _instance(rng, fam, noise=0.3, swap=0.15):
    S, ident, bi, bo, bt = fam
    ident = list(ident)
    if rng.random() < swap:                       # a divergent branch of the family
        u = int(rng.integers(0, S))
        ident[u] = (ident[u] & TOOL) | int(rng.integers(0, 6 if ident[u] & TOOL else 4))
    jit = lambda x: max(1, int(round(x * rng.lognormal(0.0, noise)))) if x else 0
    return S, ident, [jit(x) for x in bi], [jit(x) for x in bo], [jit(x) for x in bt]


def pattern_store(seed: int = 61, n_patterns: int = 500, n_families: int = 24) -> dict:
    rng = rng_for(seed)
    fams = _pattern_families(rng, n_families)
    st = {k: np.zeros((n_patterns, MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out", "t_ms")}
    st["n_stages"] = np.zeros(n_patterns, np.uint32)
    for p in range(n_patterns):
        S, ident, i_, o_, t_ = _instance(rng, fams[int(rng.integers(0, n_families))])
        st["n_stages"][p] = S
        for u in range(S):
            st["ident"][p, u], st["in_len"][p, u], st["out"][p, u], st["t_ms"][p, u] = ident[u], i_[u], o_[u], t_[u]
    st["reuse"] = rng.integers(1, 60, n_patterns).astype(np.uint32)
    st["families"] = fams
    return st


def pattern_queries(seed: int, store: dict, n_queries: int, foreign: float = 0.05) -> dict:
    """fresh instances of the store's families (a few of unknown families: NoMatch), revealed up
    to a random stage s: identities and input lengths of stages 0..s, outputs of stages 0..s-1"""
    rng = rng_for(seed)
    fams = store["families"]
    other = _pattern_families(rng, 4)
    q = {k: np.zeros((n_queries, MAX_STAGES), np.uint32) for k in ("ident", "in_len", "out")}
    q["stage"] = np.zeros(n_queries, np.uint32)
    q["true_t_ms"] = np.zeros((n_queries, MAX_STAGES), np.uint32)
    for i in range(n_queries):
        fam = other[int(rng.integers(0, 4))] if rng.random() < foreign else fams[int(rng.integers(0, len(fams)))]
        S, ident, i_, o_, t_ = _instance(rng, fam)
        s = int(rng.integers(0, S))
        q["stage"][i] = s
        for u in range(S):
            if u <= s:
                q["ident"][i, u], q["in_len"][i, u] = ident[u], i_[u]
            if u < s:
                q["out"][i, u] = o_[u]
            q["true_t_ms"][i, u] = t_[u]
    return q


# ----------------------------------------------------------------------------------------
# NEXT-4: a quantile regression forest over (L_i, dist_row, anchor, group) -> L_o, trained on
# synthetic requests drawn like the pool's (extremely randomized splits, bootstrap rows, leaves
# keep their sorted targets: Meinshausen-style QRF).  Input generation only: the
# method's arithmetic (the quantile at inference) lives in the oracle and the kernels.
# ----------------------------------------------------------------------------------------

def forest_training_set(seed: int, n: int, n_buckets: int = 16, l_max: int = 8192, R: int = 50):
    rng = rng_for(seed)
    app = rng.integers(0, 4, n)
    keys = [APPS[a][0] for a in app]
    L_in = np.array([int(_draw_in(rng, k, None)) for k in keys], np.int64)
    b = _bucket(L_in, n_buckets)
    mu = _out_mu(app, b, n_buckets)
    sig = np.array([LOGN[APPS[a][1]][1] for a in app])
    L_o = np.clip(np.rint(rng.lognormal(mu, sig)), 1, l_max).astype(np.int64)
    g = (rng.random(n) * L_o).astype(np.int64)                   # generated so far, < L_o
    anchor = R * (g // R)
    group = rng.integers(0, 16, n)
    X = np.stack([L_in, app * n_buckets + b, anchor, group], 1).astype(np.int64)
    return X, L_o


def build_forest(seed: int = 91, n_trees: int = 32, max_depth: int = 10, min_leaf: int = 5, n_train: int = 6000,
                 X=None, y=None) -> dict:
    rng = rng_for(seed)
    if X is None:
        X, y = forest_training_set(seed + 1, n_train)
    feat, thr, left, right, root, samples = [], [], [], [], [], []

    def grow(idx, depth):
        v = len(feat)
        feat.append(0); thr.append(0); left.append(0); right.append(0)
        if depth < max_depth and len(idx) >= 2 * min_leaf:
            for _ in range(8):                                  # a few random (feature, threshold) draws
                f = int(rng.integers(0, X.shape[1]))
                vals = X[idx, f]
                t = int(vals[int(rng.integers(0, len(idx)))])
                m = vals <= t
                if min_leaf <= m.sum() <= len(idx) - min_leaf:
                    feat[v], thr[v] = f, t
                    left[v] = grow(idx[m], depth + 1)
                    right[v] = grow(idx[~m], depth + 1)
                    return v
        feat[v] = 0xFFFFFFFF
        thr[v] = len(samples)
        ys = np.sort(y[idx])
        samples.extend(int(a) for a in ys)
        left[v] = len(ys)
        return v

    for _ in range(n_trees):
        boot = rng.integers(0, len(y), len(y))
        root.append(grow(boot, 0))
    u = lambda a: np.array(a, np.uint32)
    return {"root": u(root), "feature": u(feat), "threshold": u(thr), "left": u(left), "right": u(right),
            "samples": u(samples)}


def replica_pools(d: dict, M: int, K: int, seed: int = 7):
    """NEXT-2 power-of-K inputs: the standalone rows of pool snapshot d, each given dummies on K
    of M replicas sampled without replacement; returns M standalone pools (rows in id
    order of the base pool)."""
    rng = rng_for(seed)
    p = d["pool"]
    ns = int(p["n_single"])
    keys = ("id", "arrival_ns", "input_len", "generated", "prefilled", "meta", "aux", "task", "override_R")
    pick = np.zeros((ns, M), bool)
    choice = np.argsort(rng.random((ns, M)), axis=1)[:, :K]     # K of M without replacement per row
    np.put_along_axis(pick, choice, True, axis=1)
    pools = []
    for m in range(M):
        sel = np.nonzero(pick[:, m])[0]
        q = {k: np.asarray(p[k])[:ns][sel].copy() for k in keys}
        q["n_single"] = len(sel)
        pools.append(q)
    return pools
