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
