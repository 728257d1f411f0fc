"""Exact GMAX step over a request pool sharded across ranks (shard.cuh).

One process per GPU.  Each rank's Scheduler holds its shard (request ids unique across
ranks).  A step first tries the speculative resolve across ranks: each rank exports its
speculative set {key >= t} (t is the same on every rank), one allgather, and every rank resolves
the union (jit_shard_spec_export / jit_shard_spec_resolve).  When that cannot be exact (first
step, a set too large, a failed check) the step continues -- without rescoring -- with the exact
protocol of two rounds, each a fixed-size allgather of records over NCCL/NVLink:

  round 1  jit_shard_prefix  -> first min(B*_r+1, |P_r|) local requests (key desc, id asc)
           allgather         -> every rank: jit_shard_merge -> exact global B*, bp, thr
  round 2  jit_shard_candidates -> local {key >= thr}; counts allgathered, records padded to
           the max count and allgathered -> jit_shard_finish: the same window (a9) on every
           rank -> identical batch; the bookkeeping lands on the rank owning each request.

The allgather is injected so the same orchestration runs with NCCL (torch.distributed),
with a single-GPU "virtual shard" concatenation, or (in tests) with gloo on CPU.
"""
from __future__ import annotations

REC1, REC2 = 16, 32


def nccl_allgather(group=None):
    import torch
    import torch.distributed as dist

    def gather(t):
        ws = dist.get_world_size(group)
        out = torch.empty(t.numel() * ws, dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out

    return gather


class ShardedStep:
    """Drives one rank's Scheduler through the two exchange rounds."""

    def __init__(self, sched, rank: int, world: int, allgather, device=None):
        import torch
        self.s, self.rank, self.world, self.allgather = sched, rank, world, allgather
        dev = device if device is not None else f"cuda:{sched.device}"
        self.rec1 = torch.full(((sched.max_batch + 1) * REC1,), 0xFF, dtype=torch.uint8, device=dev)
        self.rec2 = torch.full((max(sched.capacity, 1) * REC2,), 0xFF, dtype=torch.uint8, device=dev)
        self.cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        self.fast = hasattr(sched, "shard_spec_export")
        self.spec = torch.zeros(sched.shard_spec_bytes() if self.fast else 1, dtype=torch.uint8, device=dev)
        self.last = {}
        self.n_fast = self.n_exact = 0

    def step(self, now_ns: int, v_token_ns: int) -> dict:
        s = self.s
        if self.fast:
            # fast path: one allgather of the speculative sets, resolved identically on every rank
            s.shard_spec_export(now_ns, v_token_ns, self.spec, self.rank)
            out = s.shard_spec_resolve(self.allgather(self.spec), self.world, self.rank)
            if out is not None:
                out["path"] = "speculative"
                self.n_fast += 1
                self.last = out
                return out
        self.n_exact += 1
        return self._exact(now_ns, v_token_ns)

    def _exact(self, now_ns: int, v_token_ns: int) -> dict:
        s = self.s
        self.rec1.fill_(0xFF)                                # unused slots: img = ~0 (invalid)
        n1 = s.shard_prefix(now_ns, v_token_ns, self.rec1)
        all1 = self.allgather(self.rec1)
        s.shard_merge(all1)
        n2 = s.shard_candidates(self.rec2, self.rank)
        self.cnt.fill_(n2)
        counts = self.allgather(self.cnt)
        m = max(1, int(counts.max().item()))
        self.rec2[n2 * REC2:m * REC2].fill_(0xFF)
        all2 = self.allgather(self.rec2[:m * REC2])
        out = s.shard_finish(all2, self.rank)
        out["n_export1"] = n1
        out["n_candidates_local"] = n2
        out["n_candidates"] = int(counts.sum().item())
        out["path"] = "exact"
        self.last = out
        return out


def virtual_shards_step(steps, now_ns: int, v_token_ns: int):
    """Run the protocol for W ShardedStep-like drivers living on ONE device (test mode): the
    allgather is a concatenation of the W ranks' buffers, executed phase by phase."""
    import torch
    W = len(steps)
    if all(st.fast for st in steps):
        for st in steps:
            st.s.shard_spec_export(now_ns, v_token_ns, st.spec, st.rank)
        allspec = torch.cat([st.spec for st in steps])
        outs = [st.s.shard_spec_resolve(allspec, W, st.rank) for st in steps]
        if all(o is not None for o in outs):
            for o in outs:
                o["path"] = "speculative"
            return outs
        assert all(o is None for o in outs), "ranks disagree on the fast path"
    for st in steps:
        st.rec1.fill_(0xFF)
    n1 = [st.s.shard_prefix(now_ns, v_token_ns, st.rec1) for st in steps]
    all1 = torch.cat([st.rec1 for st in steps])
    for st in steps:
        st.s.shard_merge(all1)
    n2 = [st.s.shard_candidates(st.rec2, st.rank) for st in steps]
    m = max(1, max(n2))
    for st, k in zip(steps, n2):
        st.rec2[k * REC2:m * REC2].fill_(0xFF)
    all2 = torch.cat([st.rec2[:m * REC2] for st in steps])
    outs = [st.s.shard_finish(all2, st.rank) for st in steps]
    for o, a, b in zip(outs, n1, n2):
        o["n_export1"], o["n_candidates_local"], o["n_candidates"] = a, b, sum(n2)
        o["path"] = "exact"
    del W
    return outs


def shard_pool(pool: dict, tasks, rank: int, world: int):
    """Split a pool snapshot by request owner: standalone rows by id mod world, compound calls
    with their whole task (task index mod world).  Returns (pool, tasks) for `rank`."""
    import numpy as np
    n_single = int(pool.get("n_single", len(pool["input_len"])))
    ids = np.asarray(pool["id"])
    keep_s = np.nonzero((ids[:n_single] % world) == rank)[0]
    rows = [keep_s]
    t_keep = []
    if tasks is not None and len(tasks["arrival_ns"]):
        off = np.asarray(tasks["call_off"], np.int64)
        for t in range(len(tasks["arrival_ns"])):
            if t % world == rank:
                t_keep.append(t)
                rows.append(np.arange(off[t], off[t + 1]))
    sel = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    out = {}
    for k, v in pool.items():
        out[k] = v[sel] if isinstance(v, np.ndarray) and len(v) == len(ids) else v
    out["n_single"] = len(keep_s)
    tout = None
    if t_keep:
        tk = np.asarray(t_keep)
        sizes = off[tk + 1] - off[tk]
        tout = {k: np.asarray(v)[tk] for k, v in tasks.items() if k != "call_off"}
        tout["call_off"] = (len(keep_s) + np.concatenate([[0], np.cumsum(sizes)])).astype(np.uint32)
        newt = np.repeat(np.arange(len(tk), dtype=np.uint32), sizes)
        out["task"] = out["task"].copy()
        out["task"][len(keep_s):] = newt
    return out, tout
