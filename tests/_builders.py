"""Tiny hand-built inputs for the pin tests (no method arithmetic here)."""
import numpy as np

import workloads as W

S_ = W.S_
MS = W.MS


def table_from_supports(supports, l_max):
    """Rows with uniform counts (1 each) on the closed integer ranges given."""
    cum = np.zeros((len(supports), l_max), np.uint32)
    for r, (lo, hi) in enumerate(supports):
        h = np.zeros(l_max, np.int64)
        h[lo - 1:hi] = 1
        cum[r] = np.cumsum(h)
    return {"edges": np.arange(1, l_max + 1, dtype=np.uint32), "cum": cum, "l_max": l_max}


def table_from_counts(counts):
    counts = np.asarray(counts, np.int64)
    cum = np.cumsum(counts, axis=1).astype(np.uint32)
    return {"edges": np.arange(1, counts.shape[1] + 1, dtype=np.uint32), "cum": cum, "l_max": counts.shape[1]}


def pool(rows):
    """rows: list of dicts with keys id, arrival, L_i, g, pre, group, state, flags, dist_row,
    waited, task, override (defaults filled)."""
    d = dict(arrival=0, g=0, pre=0, group=0, state=W.Q_QUEUED, flags=0, dist_row=0, waited=0, task=W.NO_TASK, override=0)
    R = [{**d, **r} for r in rows]
    n = len(R)
    out = {
        "id": np.array([r["id"] for r in R], np.uint32),
        "arrival_ns": np.array([r["arrival"] for r in R], np.int64),
        "input_len": np.array([r["L_i"] for r in R], np.uint32),
        "generated": np.array([r["g"] for r in R], np.uint32),
        "prefilled": np.array([r["pre"] for r in R], np.uint32),
        "meta": W._pack_meta([r["group"] for r in R], [r["state"] for r in R], [r["flags"] for r in R]),
        "aux": W._pack_aux([r["dist_row"] for r in R], [r["waited"] for r in R]),
        "task": np.array([r["task"] for r in R], np.uint32),
        "override_R": np.array([r["override"] for r in R], np.uint32),
        "n_single": n,
    }
    return out


def single_trace(rows, tasks=()):
    tr = W._empty_trace()
    for r in rows:
        for k in ("arrival_ns", "input_len", "true_out", "group", "dist_row", "override_R", "task"):
            tr[k].append(r.get(k, 0 if k != "task" else W.NO_TASK))
    return W._finish_trace(tr, list(tasks))


def default_rcfg(**over):
    r = dict(n_steps=100000, v_token0_ns=2_050_000, c0_ns=2_000_000, c_att_ns=500, c_lin_ns=50_000,
             load_num=1, load_den=1, slo_num=1, slo_den=1)
    r.update(over)
    return r
