"""CPU oracle of the JITServe GMAX step and trace replay (arXiv 2504.20068).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The product path
(``paper_2504_20068_b200``) never imports it and shares no code with it.

The arithmetic lives in ``gmax_oracle.c`` (plain single-threaded C, ``-O2 -ffp-contract=off``);
this module only compiles it on demand with gcc and marshals numpy arrays through ctypes.
Every function in the C file cites the PAPER.md / SPEC.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gmax_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

NO_TASK = 0xFFFFFFFF
MAX_STAGES = 8


def build(force: bool = False) -> str:
    """Compile liboracle.so next to the source (gcc, -O2 -ffp-contract=off)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Group(C.Structure):
    _fields_ = [("type", C.c_uint32), ("w_in", C.c_uint32), ("w_out", C.c_uint32), ("_pad", C.c_uint32),
                ("ttft_ns", C.c_int64), ("tbt_ns", C.c_int64), ("e2el_ns", C.c_int64),
                ("be_deadline_ns", C.c_int64)]


class _Config(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("token_budget", "max_batch", "prefill_chunk", "refine_interval",
                                          "frame_steps", "q_num", "q_den", "p_num", "p_den", "delta_starve",
                                          "len_key", "appb_filter")] + \
               [("eps_ns", C.c_int64), ("waiting_ns", C.c_int64)] + \
               [(k, C.c_uint32) for k in ("preempt", "pmtn_num", "pmtn_den", "_pad2")] + [("io_bw_tps", C.c_uint64)] + \
               [(k, C.c_uint32) for k in ("fair_num", "fair_den")]


class _Forest(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("n_trees", "n_nodes", "n_samples", "n_features")] + \
               [(k, C.c_void_p) for k in ("root", "feature", "threshold", "left", "right", "samples")]


class _Table(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_bins", C.c_uint32), ("l_max", C.c_uint32), ("_pad", C.c_uint32),
                ("edges", C.c_void_p), ("cum", C.c_void_p), ("forest", C.c_void_p)]


def _mk_forest(forest, keep):
    F = _Forest()
    F.n_trees, F.n_nodes = len(forest["root"]), len(forest["feature"])
    F.n_samples, F.n_features = len(forest["samples"]), 4
    for k in ("root", "feature", "threshold", "left", "right", "samples"):
        a = _arr(forest[k], np.uint32)
        if a.size == 0:
            a = np.zeros(1, np.uint32)
        keep.append(a)
        setattr(F, k, _ptr(a))
    keep.append(F)
    return F


class _Pool(C.Structure):
    _fields_ = [("n", C.c_uint32), ("_pad", C.c_uint32)] + \
               [(k, C.c_void_p) for k in ("id", "arrival_ns", "input_len", "generated", "prefilled", "meta",
                                          "aux", "task", "override_R", "fair")]


class _Tasks(C.Structure):
    _fields_ = [("n", C.c_uint32), ("_pad", C.c_uint32)] + \
               [(k, C.c_void_p) for k in ("call_off", "arrival_ns", "deadline_ns", "cur_stage", "n_stages",
                                          "pattern_ms", "goodput_done", "stage_deadline_ns")]


class _Result(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("n_pending", "n_selected", "total_tokens", "n_candidates", "b_star",
                                          "n_dropped_now", "error", "n_preempted")] + \
               [("bp", C.c_double), ("thr", C.c_double), ("stall_ns", C.c_int64)]


class _RowsOut(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("key", "rate", "t_rem", "lhat", "cost", "pending")]


class _Trace(C.Structure):
    _fields_ = [("n_rows", C.c_uint32), ("n_tasks", C.c_uint32)] + \
               [(k, C.c_void_p) for k in ("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R",
                                          "task", "task_arrival_ns", "task_deadline_ns", "task_n_stages",
                                          "stage_kind", "stage_exec_ns", "stage_pattern_ms", "stage_call_begin",
                                          "stage_call_end", "fair")]


class _ReplayCfg(C.Structure):
    _fields_ = [("n_steps", C.c_uint32), ("log_ids", C.c_uint32)] + \
               [(k, C.c_int64) for k in ("v_token0_ns", "c0_ns", "c_att_ns", "c_lin_ns")] + \
               [(k, C.c_uint64) for k in ("load_num", "load_den", "slo_num", "slo_den")] + \
               [(k, C.c_uint32) for k in ("p_adapt", "eps_num", "eps_den", "window_frames")] + [("seed", C.c_uint64)]


class _ReplayResult(C.Structure):
    _fields_ = [("token_goodput", C.c_uint64), ("tokens_processed", C.c_uint64), ("sim_end_ns", C.c_int64)] + \
               [(k, C.c_uint32) for k in ("request_goodput", "n_done", "n_dropped", "steps", "n_tasks_done",
                                          "n_tasks_dropped", "error", "n_preempted")]


STEP_LOG_DTYPE = np.dtype([("now_ns", "<i8"), ("n_selected", "<u4"), ("total_tokens", "<u4"),
                           ("n_candidates", "<u4"), ("b_star", "<u4"), ("bp", "<f8"), ("ids_hash", "<u8"),
                           ("v_token_ns", "<i8"), ("n_preempted", "<u4"), ("p_num", "<u4"), ("stall_ns", "<i8")])


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.og_step.restype = C.c_int
        _lib.og_replay.restype = C.c_int
        _lib.og_length_bound.restype = C.c_uint32
        _lib.og_length_bound.argtypes = [C.POINTER(_Table), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint32]
    return _lib


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _mk_config(cfg):
    c = _Config()
    gate_defaults = {"preempt": 0, "pmtn_num": 1, "pmtn_den": 10, "_pad2": 0, "io_bw_tps": 10 ** 6,
                     "fair_num": 0, "fair_den": 1}
    for k, _ in _Config._fields_:
        setattr(c, k, int(cfg.get(k, gate_defaults.get(k, 0)) if k in gate_defaults else cfg[k]))
    return c


def _mk_groups(groups):
    n = len(groups["type"])
    arr = (_Group * max(n, 1))()
    for i in range(n):
        for k in ("type", "w_in", "w_out", "ttft_ns", "tbt_ns", "e2el_ns", "be_deadline_ns"):
            setattr(arr[i], k, int(groups[k][i]))
    return arr, n


def _mk_table(table, keep):
    edges = _arr(table["edges"], np.uint32)
    cum = _arr(table["cum"], np.uint32)
    keep += [edges, cum]
    t = _Table()
    t.n_rows, t.n_bins = cum.shape
    t.l_max = int(table["l_max"])
    t.edges = _ptr(edges)
    t.cum = _ptr(cum)
    if table.get("forest") is not None:          # NEXT-4: (a2) from the QRF (A50)
        F = _mk_forest(table["forest"], keep)
        t.forest = C.cast(C.pointer(F), C.c_void_p)
    return t


def length_bound(table, row: int, g: int, R: int, q_num: int, q_den: int) -> int:
    """Lhat = max(Q_q(L | L > R*floor(g/R)), g+1) on one length-table row (§4.1)."""
    lib = _load()
    keep = []
    t = _mk_table(table, keep)
    return int(lib.og_length_bound(C.byref(t), row, g, R, q_num, q_den))


def step(cfg, groups, table, now_ns: int, v_token_ns: int, pool, tasks=None, rows_out: bool = True,
         frame_open: bool = True):
    """One GMAX step (Alg. 1 Schedule) over a pool snapshot.

    ``pool`` is a dict of numpy arrays (id, arrival_ns, input_len, generated, prefilled, meta, aux,
    task, override_R).  meta/aux are copied and the updated copies are returned.  With
    ``cfg["preempt"]`` the preemption gate (NEXT-1, reading A46) filters the proposal;
    ``frame_open`` says whether this step is a frame boundary (preemption allowed).
    """
    lib = _load()
    keep = []
    c = _mk_config(cfg)
    g, ng = _mk_groups(groups)
    t = _mk_table(table, keep)
    n = len(pool["id"])
    cols = {
        "id": _arr(pool["id"], np.uint32), "arrival_ns": _arr(pool["arrival_ns"], np.int64),
        "input_len": _arr(pool["input_len"], np.uint32), "generated": _arr(pool["generated"], np.uint32),
        "prefilled": _arr(pool["prefilled"], np.uint32), "meta": np.array(pool["meta"], dtype=np.uint32),
        "aux": np.array(pool["aux"], dtype=np.uint32), "task": _arr(pool["task"], np.uint32),
        "override_R": _arr(pool["override_R"], np.uint32),
    }
    if pool.get("fair") is not None:
        cols["fair"] = _arr(pool["fair"], np.uint32)
    p = _Pool()
    p.n = n
    for k, v in cols.items():
        setattr(p, k, _ptr(v))
    tp = None
    if tasks is not None and len(tasks["arrival_ns"]):
        tcols = {
            "call_off": _arr(tasks["call_off"], np.uint32), "arrival_ns": _arr(tasks["arrival_ns"], np.int64),
            "deadline_ns": _arr(tasks["deadline_ns"], np.int64), "cur_stage": _arr(tasks["cur_stage"], np.uint32),
            "n_stages": _arr(tasks["n_stages"], np.uint32), "pattern_ms": _arr(tasks["pattern_ms"], np.uint32),
            "goodput_done": _arr(tasks["goodput_done"], np.uint64),
        }
        if tasks.get("stage_deadline_ns") is not None:
            tcols["stage_deadline_ns"] = _arr(tasks["stage_deadline_ns"], np.int64)
        keep.append(tcols)
        tp = _Tasks()
        tp.n = len(tcols["arrival_ns"])
        for k, v in tcols.items():
            setattr(tp, k, _ptr(v))
    res = _Result()
    ids = np.zeros(max(n, 1), np.uint32)
    toks = np.zeros(max(n, 1), np.uint32)
    rows = np.zeros(max(n, 1), np.uint32)
    ro = None
    out_rows = {}
    if rows_out:
        out_rows = {"key": np.zeros(n, np.float64), "rate": np.zeros(n, np.float64),
                    "t_rem": np.zeros(n, np.int64), "lhat": np.zeros(n, np.uint32),
                    "cost": np.zeros(n, np.uint32), "pending": np.zeros(n, np.uint32)}
        ro = _RowsOut(*[_ptr(out_rows[k]) for k in ("key", "rate", "t_rem", "lhat", "cost", "pending")])
    rc = lib.og_step(C.byref(c), g, C.c_uint32(ng), C.byref(t), C.c_int64(now_ns), C.c_int64(v_token_ns),
                     C.byref(p), C.byref(tp) if tp is not None else None, C.byref(res),
                     _ptr(ids), _ptr(toks), _ptr(rows), C.byref(ro) if ro is not None else None,
                     C.c_uint32(1 if frame_open else 0))
    k = res.n_selected
    out = {"status": rc, "n_pending": res.n_pending, "n_selected": k, "total_tokens": res.total_tokens,
           "n_candidates": res.n_candidates, "b_star": res.b_star, "n_dropped_now": res.n_dropped_now,
           "bp": res.bp, "thr": res.thr, "batch_ids": ids[:k].copy(), "batch_tokens": toks[:k].copy(),
           "batch_rows": rows[:k].copy(), "meta": cols["meta"], "aux": cols["aux"],
           "n_preempted": res.n_preempted, "stall_ns": res.stall_ns}
    out.update(out_rows)
    return out


def replay(cfg, groups, table, trace, rcfg, log: bool = False, log_ids: bool = False):
    """Replay one trace under GMAX (a10): cost model S:395-403/S:438, goodput §3 P:209-216."""
    lib = _load()
    keep = []
    c = _mk_config(cfg)
    g, ng = _mk_groups(groups)
    t = _mk_table(table, keep)
    tr = _Trace()
    types = {"arrival_ns": np.int64, "input_len": np.uint32, "true_out": np.uint32, "group": np.uint32,
             "dist_row": np.uint32, "override_R": np.uint32, "task": np.uint32, "task_arrival_ns": np.int64,
             "task_deadline_ns": np.int64, "task_n_stages": np.uint32, "stage_kind": np.uint32,
             "stage_exec_ns": np.int64, "stage_pattern_ms": np.uint32, "stage_call_begin": np.uint32,
             "stage_call_end": np.uint32}
    cols = {}
    if trace.get("fair") is not None:
        types = dict(types, fair=np.uint32)
    for k, dt in types.items():
        a = _arr(trace[k], dt)
        if a.size == 0:
            a = np.zeros(1, dt)
        cols[k] = a
        setattr(tr, k, _ptr(a))
    tr.n_rows = len(trace["input_len"])
    tr.n_tasks = len(trace["task_arrival_ns"])
    rc = _ReplayCfg()
    rc.n_steps = int(rcfg["n_steps"])
    rc.log_ids = 1 if log_ids else 0
    for k in ("v_token0_ns", "c0_ns", "c_att_ns", "c_lin_ns", "load_num", "load_den", "slo_num", "slo_den"):
        setattr(rc, k, int(rcfg[k]))
    for k, dflt in (("p_adapt", 0), ("eps_num", 1), ("eps_den", 10), ("window_frames", 100), ("seed", 0)):
        setattr(rc, k, int(rcfg.get(k, dflt)))
    res = _ReplayResult()
    L = np.zeros(max(rc.n_steps, 1), STEP_LOG_DTYPE) if log else None
    LI = np.zeros(max(rc.n_steps, 1) * int(cfg["max_batch"]), np.uint32) if log_ids else None
    st = lib.og_replay(C.byref(c), g, C.c_uint32(ng), C.byref(t), C.byref(tr), C.byref(rc), C.byref(res),
                       _ptr(L), _ptr(LI))
    out = {"status": st, "token_goodput": res.token_goodput, "tokens_processed": res.tokens_processed,
           "sim_end_ns": res.sim_end_ns, "request_goodput": res.request_goodput, "n_done": res.n_done,
           "n_dropped": res.n_dropped, "steps": res.steps, "n_tasks_done": res.n_tasks_done,
           "n_tasks_dropped": res.n_tasks_dropped, "n_preempted": res.n_preempted}
    if log:
        out["log"] = L[:res.steps].copy()
    if log_ids:
        out["log_ids"] = LI.reshape(max(rc.n_steps, 1), int(cfg["max_batch"]))[:res.steps].copy()
    return out


class _Patterns(C.Structure):
    _fields_ = [("n", C.c_uint32), ("_pad", C.c_uint32)] + \
               [(k, C.c_void_p) for k in ("n_stages", "ident", "in_len", "out", "t_ms", "reuse")]


class _Queries(C.Structure):
    _fields_ = [("n", C.c_uint32), ("_pad", C.c_uint32)] + [(k, C.c_void_p) for k in ("stage", "ident", "in_len", "out")]


def _mk_patterns(store, keep):
    P = _Patterns()
    P.n = len(store["n_stages"])
    for k in ("n_stages", "ident", "in_len", "out", "t_ms", "reuse"):
        a = _arr(store[k], np.uint32)
        keep.append(a)
        setattr(P, k, _ptr(a))
    return P


def _mk_queries(queries, keep):
    Q = _Queries()
    Q.n = len(queries["stage"])
    for k in ("stage", "ident", "in_len", "out"):
        a = _arr(queries[k], np.uint32)
        keep.append(a)
        setattr(Q, k, _ptr(a))
    return Q


def kernel_sim(a: int, b: int) -> float:
    """Gaussian-kernel similarity of two attributes (§4.1, sigma of S:250)."""
    lib = _load()
    lib.og_kernel_sim.restype = C.c_double
    return float(lib.og_kernel_sim(C.c_uint32(a), C.c_uint32(b)))


def match_scores(store, queries) -> np.ndarray:
    """[n_queries, n_patterns] similarity scores (-1 = pruned), NEXT-3 (reading A49)."""
    lib = _load()
    lib.og_match_score.restype = C.c_double
    keep = []
    P = _mk_patterns(store, keep)
    Q = _mk_queries(queries, keep)
    out = np.zeros((Q.n, P.n), np.float64)
    for q in range(Q.n):
        for p in range(P.n):
            out[q, p] = lib.og_match_score(C.byref(P), C.c_uint32(p), C.byref(Q), C.c_uint32(q))
    return out


def match(store, queries):
    """Best stored pattern per query and its score (-1 / -1.0 = NoMatch), NEXT-3 (A49)."""
    lib = _load()
    keep = []
    P = _mk_patterns(store, keep)
    Q = _mk_queries(queries, keep)
    best = np.zeros(max(Q.n, 1), np.int32)
    score = np.zeros(max(Q.n, 1), np.float64)
    lib.og_match(C.byref(P), C.byref(Q), _ptr(best), _ptr(score))
    return best[:Q.n].copy(), score[:Q.n].copy()


def qrf_quantile(forest, x, anchor: int, q_num: int, q_den: int, l_max: int) -> int:
    """NEXT-4 (A50): Q_q of the pooled leaf samples above `anchor` for features x (4 ints)."""
    lib = _load()
    lib.og_qrf_quantile.restype = C.c_uint32
    keep = []
    F = _mk_forest(forest, keep)
    xa = _arr(np.asarray(x), np.uint32)
    return int(lib.og_qrf_quantile(C.byref(F), _ptr(xa), C.c_uint32(anchor), C.c_uint32(q_num), C.c_uint32(q_den),
                                   C.c_uint32(l_max)))


def multi_step(cfg, groups, table, now_ns: int, v_tokens, pools):
    """NEXT-2 power-of-K (A51): one GMAX step on each of M replicas' pools of dummies (replica m
    keyed with v_tokens[m]), cross-replica assignment (smallest v, then lower index) and sibling
    removal (other replicas' dummies of an assigned request become Moved).  Returns per replica a
    dict like step()'s (meta / aux updated copies)."""
    lib = _load()
    keep = []
    c = _mk_config(cfg)
    g, ng = _mk_groups(groups)
    t = _mk_table(table, keep)
    M = len(pools)
    parr = (C.c_void_p * M)()
    cols_all = []
    for m, pool in enumerate(pools):
        cols = {
            "id": _arr(pool["id"], np.uint32), "arrival_ns": _arr(pool["arrival_ns"], np.int64),
            "input_len": _arr(pool["input_len"], np.uint32), "generated": _arr(pool["generated"], np.uint32),
            "prefilled": _arr(pool["prefilled"], np.uint32), "meta": np.array(pool["meta"], dtype=np.uint32),
            "aux": np.array(pool["aux"], dtype=np.uint32), "task": _arr(pool["task"], np.uint32),
            "override_R": _arr(pool["override_R"], np.uint32),
        }
        if pool.get("fair") is not None:
            cols["fair"] = _arr(pool["fair"], np.uint32)
        p = _Pool()
        p.n = len(cols["id"])
        for k, vv in cols.items():
            setattr(p, k, _ptr(vv))
        keep.append(p)
        cols_all.append(cols)
        parr[m] = C.cast(C.pointer(p), C.c_void_p)
    res = (_Result * M)()
    rows = [np.zeros(max(len(cl["id"]), 1), np.uint32) for cl in cols_all]
    toks = [np.zeros(max(len(cl["id"]), 1), np.uint32) for cl in cols_all]
    rptr = (C.c_void_p * M)(*[_ptr(a) for a in rows])
    tptr = (C.c_void_p * M)(*[_ptr(a) for a in toks])
    va = _arr(np.asarray(v_tokens), np.int64)
    rc = lib.og_multi_step(C.byref(c), g, C.c_uint32(ng), C.byref(t), C.c_int64(now_ns), C.c_uint32(M), _ptr(va),
                           parr, res, rptr, tptr)
    out = []
    for m in range(M):
        k = res[m].n_selected
        r = rows[m][:k].copy()
        out.append({"status": rc if rc < 0 else (1 if res[m].n_pending == 0 else 0), "n_pending": res[m].n_pending,
                    "n_selected": k, "total_tokens": res[m].total_tokens, "n_candidates": res[m].n_candidates,
                    "b_star": res[m].b_star, "n_dropped_now": res[m].n_dropped_now, "bp": res[m].bp, "thr": res[m].thr,
                    "batch_rows": r, "batch_ids": cols_all[m]["id"][r].copy(), "batch_tokens": toks[m][:k].copy(),
                    "meta": cols_all[m]["meta"], "aux": cols_all[m]["aux"]})
    return out
