"""CPU stand-in for libjitsched's four shard phases (TEST ONLY).

It lets the sharded-step orchestration (paper_2504_20068_b200/sharded.py) and its exchange
pattern run on CPU with gloo: per-row keys and costs come from the oracle on the rank's shard,
the record formats are jit_rec1 / jit_rec2, and the selection logic follows the definitions of
DESIGN.md §3 (A14-A20).  The real kernels are checked against the oracle in
tests/test_shard_gpu.py.
"""
import numpy as np

import oracle

REC1_DT = np.dtype([("img", "<u8"), ("id", "<u4"), ("cost", "<u4")])
REC2_DT = np.dtype([("img", "<u8"), ("id", "<u4"), ("cost", "<u4"), ("len", "<u4"), ("row", "<u4"), ("rank", "<u4"),
                    ("pad", "<u4")])
NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


def _fx(key):
    return int(np.floor(min(float(key), 2.0 ** 31 - 1) * 2.0 ** 32))


class FakeShardSched:
    def __init__(self, d, max_batch, capacity):
        self.d = d
        self.max_batch = max_batch
        self.capacity = capacity
        self.device = "cpu"

    def shard_prefix(self, now, v, rec1):
        d = self.d
        self.out = oracle.step(d["cfg"], d["groups"], d["table"], now, v, d["pool"], d["tasks"])
        key, cost, pend = self.out["key"], self.out["cost"], self.out["pending"].astype(bool)
        ids = d["pool"]["id"]
        rows = sorted(np.nonzero(pend)[0], key=lambda r: (-key[r], ids[r]))
        cfg = d["cfg"]
        m, s = 0, 0
        while m < len(rows) and m + 1 <= cfg["max_batch"] and s + cost[rows[m]] <= cfg["token_budget"]:
            s += cost[rows[m]]
            m += 1
        exp = rows[:min(m + 1, len(rows))]
        r1 = rec1.numpy().view(REC1_DT)
        r1[:] = np.array([(NONE, 0, 0)], REC1_DT)
        for i, r in enumerate(exp):
            r1[i] = (np.float64(key[r]).view(np.uint64), ids[r], cost[r])
        return len(exp)

    def shard_merge(self, all1):
        a = all1.numpy().view(REC1_DT)
        a = a[a["img"] != NONE]
        cfg = self.d["cfg"]
        order = sorted(range(len(a)), key=lambda i: (-a["img"][i].view(np.float64), a["id"][i]))
        m, s = 0, 0
        while m < len(order) and m + 1 <= cfg["max_batch"] and s + a["cost"][order[m]] <= cfg["token_budget"]:
            s += int(a["cost"][order[m]])
            m += 1
        self.b_star = m
        self.bp = float(a["img"][order[m - 1]].view(np.float64)) if len(order) else 0.0
        self.thr = (cfg["p_num"] / cfg["p_den"]) * self.bp

    def shard_candidates(self, rec2, rank):
        d, key, pend = self.d, self.out["key"], self.out["pending"].astype(bool)
        pool, cfg = d["pool"], d["cfg"]
        rows = [r for r in np.nonzero(pend)[0] if key[r] >= self.thr]
        r2 = rec2.numpy().view(REC2_DT)
        for i, r in enumerate(rows):
            ln = int(pool["input_len"][r]) + (int(pool["generated"][r]) if cfg["len_key"] else 0)
            r2[i] = (np.float64(key[r]).view(np.uint64), pool["id"][r], self.out["cost"][r], ln, r, rank, 0)
        return len(rows)

    def shard_finish(self, all2, rank):
        cfg = self.d["cfg"]
        a = all2.numpy().view(REC2_DT)
        a = a[a["img"] != NONE]
        o = sorted(range(len(a)), key=lambda i: (int(a["len"][i]), int(a["id"][i])))
        best, bi, bj = -1, 0, 0
        j = 0
        for i in range(len(o)):
            j = max(j, i)
            c = sum(int(a["cost"][o[k]]) for k in range(i, j + 1))
            while j + 1 < len(o) and c + int(a["cost"][o[j + 1]]) <= cfg["token_budget"] and j + 2 - i <= cfg["max_batch"]:
                j += 1
                c += int(a["cost"][o[j]])
            sc = sum(_fx(a["img"][o[k]].view(np.float64)) for k in range(i, j + 1))
            if sc > best:
                best, bi, bj = sc, i, j
        sel = [o[k] for k in range(bi, bj + 1)]
        return {"status": 0, "n_selected": len(sel), "batch_ids": np.array([a["id"][k] for k in sel], np.uint32),
                "batch_tokens": np.array([a["cost"][k] for k in sel], np.uint32), "b_star": self.b_star, "bp": self.bp,
                "thr": self.thr, "n_candidates": len(a),
                "total_tokens": int(sum(int(a["cost"][k]) for k in sel))}


SPEC_DT = np.dtype([("img", "<u8"), ("id", "<u4"), ("cost", "<u4"), ("len", "<u4"), ("pad", "<u4")])
SPEC_CAP = 1024


class FakeSpecShardSched(FakeShardSched):
    """Adds the speculative tier (jit_shard_spec_export / _resolve): every rank exports its rows
    with key >= t (t = fl(0.97 x the previous cutoff), identical on every rank), and every rank
    resolves the union -- exact when the budget walk stops inside the union (or the union holds
    every pending request) and thr >= t; otherwise None (the exact protocol)."""

    def __init__(self, d, max_batch, capacity):
        super().__init__(d, max_batch, capacity)
        self.t = None

    def shard_spec_bytes(self):
        return 16 + SPEC_DT.itemsize * SPEC_CAP

    def shard_spec_export(self, now, v, buf, rank):
        d, cfg = self.d, self.d["cfg"]
        self.out = oracle.step(cfg, d["groups"], d["table"], now, v, d["pool"], d["tasks"])
        key, pend = self.out["key"], self.out["pending"].astype(bool)
        b = buf.numpy()
        hdr = b[:16].view(np.uint32)
        hdr[0] = int(pend.sum())
        if self.t is None:
            hdr[1] = 0xFFFFFFFF                               # no threshold yet: exact protocol
            return
        rows = [r for r in np.nonzero(pend)[0] if np.float64(key[r]).view(np.uint64) >= self.t]
        assert len(rows) <= SPEC_CAP
        hdr[1] = len(rows)
        rec = b[16:].view(SPEC_DT)
        for i, r in enumerate(rows):
            ln = int(d["pool"]["input_len"][r]) + (int(d["pool"]["generated"][r]) if cfg["len_key"] else 0)
            rec[i] = (np.float64(key[r]).view(np.uint64), d["pool"]["id"][r], self.out["cost"][r], ln, 0)

    def shard_spec_resolve(self, allb, world, rank):
        cfg = self.d["cfg"]
        b = allb.numpy().reshape(world, -1)
        hdrs = [b[w, :16].view(np.uint32) for w in range(world)]
        if any(h[1] == 0xFFFFFFFF for h in hdrs):
            return None
        n_pend = sum(int(h[0]) for h in hdrs)
        u = np.concatenate([b[w, 16:].view(SPEC_DT)[:int(hdrs[w][1])] for w in range(world)])
        if n_pend == 0 or len(u) == 0:
            return None
        whole = len(u) == n_pend
        order = sorted(range(len(u)), key=lambda i: (-u["img"][i].view(np.float64), int(u["id"][i])))
        m, s = 0, 0
        while m < len(order) and m + 1 <= cfg["max_batch"] and s + int(u["cost"][order[m]]) <= cfg["token_budget"]:
            s += int(u["cost"][order[m]])
            m += 1
        if m == 0 or (m == len(order) and not whole):
            return None
        bp = float(u["img"][order[m - 1]].view(np.float64))
        thr = (cfg["p_num"] / cfg["p_den"]) * bp
        if not whole and np.float64(thr).view(np.uint64) < self.t:
            return None
        cd = u[[i for i in range(len(u)) if u["img"][i].view(np.float64) >= thr]]
        a = np.zeros(len(cd), REC2_DT)
        for f in ("img", "id", "cost", "len"):
            a[f] = cd[f]
        self.b_star, self.bp, self.thr = m, bp, thr
        out = self.shard_finish(_as_rec2(a), rank)
        return out

    def shard_finish(self, all2, rank):
        out = super().shard_finish(all2, rank)
        self.t = np.float64(0.97 * self.thr).view(np.uint64)   # identical on every rank
        return out


class _as_rec2:
    """numpy REC2 array in the shape shard_finish expects (a tensor-like with .numpy())."""

    def __init__(self, a):
        self.a = a

    def numpy(self):
        return self.a.view(np.uint8)
