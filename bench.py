#!/usr/bin/env python
"""bench.py -- the JITServe GMAX scheduling step on B200 (contract: DESIGN.md §8).

Headline (N=1): BASELINE config C3 -- one GMAX step (a1-a9) over a pool of 2^20 pending
requests resident in HBM (16 SLO groups, token budget 8192, B_max 8192), timed on the device
with CUDA events over K chained steps rotating over pool copies that together exceed 4x the L2.
`value` = pending requests scheduled per second, summed over ranks.  Also on the line:
  * roofline of the dominant kernel (k_score) against the measured HBM copy bandwidth, its
    forced-refresh variant (every cached length bound stale), and the device counters that prove
    every timed step resolved on the device (no exact-path fallback, no skipped chained step);
  * e2e: the serving loop through the public API -- every step carries that step's arrivals and
    the previous batch's progress (keyed by request id) host->device and reads the batch back;
  * configs: C1 (toy trace replay), C2 (10K-request replay), C4 (compound DAG pool step);
  * replay: BASELINE config C5(i), replayed serving steps per second, with its CPU baseline (the
    oracle over every host core on a bounded sample of the sweep);
  * cpu_baseline: the CPU oracle (oracle/, plain C, 1 core) on a bounded sample of C3 steps.
N > 1 (torchrun): C5(ii) -- one pool of N x 2^21 requests sharded by request id; every step is the
speculative union over an NCCL allgather (exact two-round protocol as fallback).
`--impl reference` runs the oracle as the reference arm (rank 0 only) on the same config.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "pending requests scheduled/sec (1M pool)"
UNIT = "requests/s"
# algorithmic bytes of k_score: per standalone row its 32-B hot row read (arrival 8,
# input_len, generated, prefilled, dist_row | cached bound, meta, steps_waited stamp), nothing
# written in the steady state; per compound call the same + 4 B read (task id); per task 32 B of
# constants + 4 B ever flag.  SURVEY §8(d) counts 40 B per request (32 B read + an 8-B key write
# this design does not need): `frac_8d` reports that accounting too.
BYTES_ROW, BYTES_CALL, BYTES_TASK = 32, 36, 36
BYTES_8D = 40
L2_BYTES = 126 * (1 << 20)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=0, help="pool rows per GPU (default 2^20 at N=1, 2^21 per rank at N>1)")
    ap.add_argument("--rot", type=int, default=0, help="pool copies rotated (default: enough for 4x the L2)")
    ap.add_argument("--replays", type=int, default=4096)
    ap.add_argument("--replay-steps", type=int, default=4096)
    ap.add_argument("--e2e-steps", type=int, default=40)
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1/C2/C4 lines")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: exercise the N>1 code path with all ranks on one GPU (test mode; the "
                         "exchange goes through host memory, numbers are not NVLink numbers)")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of k_score per launch, from the committed
    ncu --set full capture summary (profiles/k_score_traffic.json); None when absent."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "k_score_traffic.json")))
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={idx}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}



def c3_config(n, nt, ws, rot, extra=None):
    """the config dict both arms print (same workload, same keys)"""
    cfg = {"workload": "C3: 2^20-row pending pool per GPU (40% chat, 30% deep-research, 30% compound calls "
                       "in 16-call tasks), 16 SLO groups, tau 8192, B_max 8192, v_token 15 ms",
           "rows_per_gpu": n, "tasks_per_gpu": nt,
           "l2": f"inputs larger than L2: {rot} rotated pool copies (>= 4x the 126 MB L2 of hot state)",
           "parallelism": "single GPU" if ws == 1 else f"{ws} shards"}
    if extra:
        cfg.update(extra)
    return cfg


def c5ii_config(ws, n, rot):
    """the N > 1 config dict both arms print (the sharded C5(ii) pool)"""
    return {"workload": f"C5(ii): {ws} x {n}-row shards of one pool (C3 generator), sharded by request id, "
                        "tau 8192, B_max 8192", "rows_total": ws * n, "rows_per_gpu": n,
            "l2": f"{rot} rotated shard copies per rank (>= 4x the L2 of hot state)",
            "parallelism": f"sharded pool over {ws} ranks: speculative sets allgathered over NCCL and resolved "
                           "identically on every rank (exact 2-round protocol as fallback)"}


def rot_for(args, hot):
    """pool copies rotated so that their hot state exceeds 4x the L2 (at least 6)"""
    return args.rot or max(6, -(-4 * L2_BYTES // hot))


def alg_bytes(d):
    n = len(d["pool"]["input_len"])
    n_single = int(d["pool"]["n_single"])
    nt = 0 if d["tasks"] is None else len(d["tasks"]["arrival_ns"])
    return n_single * BYTES_ROW + (n - n_single) * BYTES_CALL + nt * BYTES_TASK


def oracle_step_timing(d, budget_s=10.0, max_steps=40):
    """CPU oracle on a pool (bounded sample), pinned to one host core."""
    import oracle
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    pool = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in d["pool"].items()}
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_steps and (not times or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        out = oracle.step(d["cfg"], d["groups"], d["table"], d["now_ns"], d["v_token_ns"], pool, d["tasks"],
                          rows_out=False)
        times.append(time.perf_counter() - t0)
        pool["meta"], pool["aux"] = out["meta"], out["aux"]
    return sum(times) / len(times), len(times)


def run_reference(args, ws, rank):
    """The reference arm: the CPU oracle as it stands, on this arm's config (rank 0 only)."""
    if rank != 0:
        return
    rows = args.rows or (1 << 20 if ws == 1 else 1 << 21)
    d = W.pool_snapshot(3, rows)
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    import oracle
    oracle.build()
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_step_timing(d, budget_s=0.0, max_steps=1)
    t, k = oracle_step_timing(d, budget_s=60.0, max_steps=max(1, min(args.steps, 20)))
    v = n / t
    if ws == 1:
        cfg = c3_config(n, nt, 1, rot_for(args, alg_bytes(d)))
        sample = f"{k} oracle steps over the full C3 pool ({n} rows), 1 core of {cpu_model()}"
    else:                                   # the sharded pool's config; the sample: one rank's shard
        cfg = c5ii_config(ws, n, args.rot or max(2, -(-4 * L2_BYTES // alg_bytes(d))))
        sample = f"{k} oracle steps over one {n}-row shard of the C5(ii) pool, 1 core of {cpu_model()}"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": k,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# the serving loop through the public API (e2e): each step carries its arrivals and the previous
# batch's progress (keyed by request id) from pinned host memory and reads the batch back
# ------------------------------------------------------------------------------------------
class EngineLoop:
    def __init__(self, d, extra, arrivals_per_step):
        self.d = d
        p = d["pool"]
        self.L_in = {}
        self.state = {}
        ids = p["id"]
        self.gen = dict(zip(ids.tolist(), p["generated"].astype(np.int64).tolist()))
        self.pre = dict(zip(ids.tolist(), p["prefilled"].astype(np.int64).tolist()))
        self.L_in = dict(zip(ids.tolist(), p["input_len"].astype(np.int64).tolist()))
        self.L_o = dict(zip(ids.tolist(), p["true_out"].astype(np.int64).tolist()))
        ep = extra["pool"]
        ns = int(ep["n_single"])
        self.extra = {k: np.asarray(ep[k])[:ns] for k in ("id", "arrival_ns", "input_len", "generated", "prefilled",
                                                           "meta", "aux", "task", "override_R", "true_out")}
        self.k = arrivals_per_step
        self.next = 0

    def arrivals(self, now):
        e, a, b = self.extra, self.next, self.next + self.k
        if b > len(e["id"]):
            return None
        self.next = b
        arr = {k: v[a:b].copy() for k, v in e.items()}
        arr["arrival_ns"][:] = now                      # they arrive now, queued, never scheduled
        arr["generated"][:] = 0
        arr["prefilled"][:] = 0
        arr["meta"] = (arr["meta"] & ~np.uint32(0xFF00)).astype(np.uint32)
        arr["aux"] = (arr["aux"] & np.uint32(0xFFFF)).astype(np.uint32)
        arr["n_single"] = b - a
        for i, L, Lo in zip(arr["id"].tolist(), arr["input_len"].tolist(), arr["true_out"].tolist()):
            self.gen[i], self.pre[i], self.L_in[i], self.L_o[i] = 0, 0, L, Lo
        return arr

    def progress(self, batch):
        ids = batch["batch_ids"][:batch["n_selected"]].tolist()
        toks = batch["batch_tokens"][:batch["n_selected"]].tolist()
        g, p_, st = [], [], []
        for i, t in zip(ids, toks):
            pre, gen, L = self.pre[i], self.gen[i], self.L_in[i]
            if pre < L:
                pre = min(pre + t, L)
                if pre == L:
                    gen += 1                              # token 0 at the end of the prefill (A28)
            else:
                gen += 1
            self.pre[i], self.gen[i] = pre, gen
            g.append(gen); p_.append(pre)
            st.append(W.Q_DONE if gen >= self.L_o[i] else W.Q_RUNNING)
        return {"id": np.array(ids, np.uint32), "generated": np.array(g, np.uint32),
                "prefilled": np.array(p_, np.uint32), "state": np.array(st, np.uint32)}


def e2e_leg(args, d, dev, stream, Scheduler):
    """the serving loop, wall clock per synchronous step (the host marshals and reads the batch)"""
    import torch
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    per_step = 256
    extra = W.pool_snapshot(77, per_step * (args.e2e_steps + 8) + 64, frac_compound=0.0, table=d["table"])
    extra["pool"]["id"] = (extra["pool"]["id"].astype(np.uint64) + (1 << 28)).astype(np.uint32)
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n + per_step * (args.e2e_steps + 8), task_capacity=nt,
                  device=dev, stream=stream)
    s.load(d["pool"], d["tasks"])
    loop = EngineLoop(d, extra, per_step)
    now, v = d["now_ns"], d["v_token_ns"]
    b = s.step(now, v)
    for _ in range(3):                                   # warm-up of the loop itself
        b = s.step(now, v, progress=loop.progress(b), arrivals=loop.arrivals(now))
    torch.cuda.synchronize()
    walls, h2d, d2h, fb0 = [], [], [], s.counters()["fallbacks"]
    for _ in range(args.e2e_steps):
        now += 20 * W.MS
        prog = loop.progress(b)
        arr = loop.arrivals(now)
        t0 = time.perf_counter()
        b = s.step(now, v, progress=prog, arrivals=arr)
        walls.append(time.perf_counter() - t0)
        h2d.append(sum(int(a.nbytes) for a in prog.values()) +
                   (sum(int(a.nbytes) for k, a in arr.items() if isinstance(a, np.ndarray) and k != "true_out")
                    if arr is not None else 0))
        d2h.append(12 * b["n_selected"] + 256)          # batch (id, tokens, row) + the control block
    fb = s.counters()["fallbacks"] - fb0
    s.close()
    med = statistics.median(walls)
    return {"value": n / med, "unit": UNIT, "h2d_bytes_per_step": int(np.mean(h2d)),
            "d2h_bytes_per_step": int(np.mean(d2h)), "ms_per_step": med * 1e3,
            "ms_per_step_mean": float(np.mean(walls)) * 1e3, "steps": args.e2e_steps, "exact_path_steps": fb,
            "how": f"the serving loop through jit_sched_step: every step {per_step} new requests arrive and the "
                   "previous batch's progress (keyed by request id) is reported (one pinned H2D of the deltas), the "
                   "batch is read back (pinned mirror written by the GPU); wall clock per synchronous step, median"}


def full_reload_e2e(d, dev, stream, Scheduler, steps=5):
    """secondary: the whole pool H2D from pinned memory + a step (the round-1 e2e, worst case)"""
    import torch
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    hp = {k: (torch.from_numpy(np.ascontiguousarray(v)).pin_memory() if isinstance(v, np.ndarray) else v)
          for k, v in d["pool"].items()}
    ht = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in d["tasks"].items()}
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt, device=dev, stream=stream)
    s.load(hp, ht)
    s.step(d["now_ns"], d["v_token_ns"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        s.load(hp, ht)
        s.step(d["now_ns"], d["v_token_ns"])
    te = (time.perf_counter() - t0) / steps
    h2d = sum(int(t.numel() * t.element_size()) for k, t in hp.items() if hasattr(t, "numel") and k != "true_out")
    h2d += sum(int(t.numel() * t.element_size()) for t in ht.values())
    s.close()
    return {"value": n / te, "ms_per_step": te * 1e3, "h2d_bytes_per_step": h2d,
            "how": "jit_sched_load(whole pinned host pool) + jit_sched_step (first step after a load: exact path)"}


# ------------------------------------------------------------------------------------------
# replays (C1, C2, C5(i)) and their CPU baselines
# ------------------------------------------------------------------------------------------
def _oracle_replay_worker(job):
    import oracle
    d, spec, n_steps = job
    rc = dict(d["rcfg"], n_steps=n_steps, **{k: spec[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
    t0 = time.perf_counter()
    out = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc)
    return out["steps"], time.perf_counter() - t0


def replay_cpu_baseline(traces, specs, n_steps, budget_s=20.0):
    """the oracle replaying a bounded sample of the C5(i) sweep on every host core (process pool)"""
    import multiprocessing as mp
    import oracle
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    jobs = [(traces[i % len(traces)], specs[i], n_steps) for i in range(len(specs))]
    # size the sample: time one replay, then take ~budget_s of CPU work per core
    st, t1 = _oracle_replay_worker(jobs[0])
    per = max(1, int(budget_s / max(t1, 1e-3)))
    sample = jobs[1:1 + min(len(jobs) - 1, per * cores)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_replay_worker, sample, chunksize=1)
    wall = time.perf_counter() - t0
    steps = sum(r[0] for r in res)
    return {"value": steps / wall, "unit": "steps/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(sample)} C5(i) replays (the first ones of the sweep, up to {n_steps} steps each) on "
                      f"{cores} cores of {cpu_model()} (process pool), {steps} replayed steps in {wall:.1f} s",
            "us_per_step_per_core": wall * cores / max(steps, 1) * 1e6}


def replay_leg(args, ws, rank, dev, stream, barrier, allmax, allsum, cpu=True):
    """C5(i): the load x SLO-scale sweep of independent replays; replay i -> rank i mod N (no
    communication; total work fixed, i.e. strong scaling over N)."""
    import torch
    from paper_2504_20068_b200 import Scheduler
    traces = [W.trace_mixed(k) for k in range(4)]
    sweep = W.c5_sweep(args.replays)
    specs = [dict(sp, trace=i % len(traces)) for i, sp in enumerate(sweep)]
    mine = specs[rank::ws]
    rc = dict(traces[0]["rcfg"], n_steps=args.replay_steps)
    rs = Scheduler(traces[0]["cfg"], traces[0]["groups"], traces[0]["table"], capacity=64, task_capacity=8,
                   device=dev, stream=stream)
    rs.replay([t["trace"] for t in traces], mine[:min(len(mine), 64)], rc)     # warm-up
    barrier()
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    res, _ = rs.replay([t["trace"] for t in traces], mine, rc)
    r1.record(stream)
    torch.cuda.synchronize()
    barrier()
    rms = allmax(r0.elapsed_time(r1))
    steps_done = allsum(float(sum(r["steps"] for r in res)))
    rs.close()
    out = {"metric": "replayed serving steps/sec", "value": steps_done / (rms / 1e3), "unit": "steps/s",
           "workload": f"C5(i): {args.replays} replays (64 load x 64 SLO-scale points, 4 base mixed 1:1:1 traces "
                       f"of 2048 rows), up to {args.replay_steps} steps each, tau 2048, B_max 128",
           "ms": rms, "steps_total": int(steps_done), "scaling": "strong (fixed sweep, replay i -> rank i mod N)",
           "goodput_tokens_sum": int(allsum(float(sum(r["token_goodput"] for r in res)))), "gpu_launches": 1}
    if cpu and rank == 0 and ws == 1:
        out["cpu_baseline"] = replay_cpu_baseline([{"trace": t["trace"], "groups": t["groups"], "table": t["table"],
                                                    "cfg": t["cfg"], "rcfg": rc} for t in traces], specs,
                                                  args.replay_steps)
    return out


def config_lines(args, dev, stream, Scheduler):
    """C1 (toy trace), C2 (10K requests), C4 (compound DAG pool): GPU and oracle side by side"""
    import torch
    import oracle
    oracle.build()
    out = {}
    # ---- C1 and C2: one replay each (GPU: one CTA), replayed steps / s; the oracle on one core
    for name, d, cap_steps in (("C1", W.trace_c1(), 200), ("C2", W.trace_c2(), 3000)):
        rc = dict(d["rcfg"], n_steps=min(d["rcfg"]["n_steps"], cap_steps))
        rs = Scheduler(d["cfg"], d["groups"], d["table"], capacity=64, task_capacity=8, device=dev, stream=stream)
        spec = [dict(trace=0, load_num=1, load_den=1, slo_num=1, slo_den=1)]
        rs.replay([d["trace"]], spec, rc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res, _ = rs.replay([d["trace"]], spec, rc)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rs.close()
        t0 = time.perf_counter()
        ref = oracle.replay(d["cfg"], d["groups"], d["table"], d["trace"], rc)
        tc = time.perf_counter() - t0
        same = all(int(res[0][k]) == int(ref[k]) for k in ("token_goodput", "tokens_processed", "sim_end_ns", "steps"))
        out[name] = {"metric": "replayed serving steps/sec (one replay)", "value": res[0]["steps"] / (ms / 1e3),
                     "unit": "steps/s", "steps": int(res[0]["steps"]), "ms": ms, "token_goodput": int(res[0]["token_goodput"]),
                     "equal_to_oracle": bool(same),
                     "cpu_baseline": {"value": ref["steps"] / tc, "unit": "steps/s", "cores": 1, "kind": "oracle",
                                      "sample": f"the same replay ({ref['steps']} steps) on 1 core"},
                     "workload": ("C1: SPEC toy trace, 32 requests, 200 steps, tau 512" if name == "C1" else
                                  f"C2: 10K-request chat + deadline mix, 8 SLO groups, tau 8192, B_max 256, first "
                                  f"{rc['n_steps']} steps"),
                     "note": "one replay is one CTA: latency-bound, not an HBM workload (SURVEY 8(d))"}
    # ---- C4: the compound DAG pool (100K tasks, ~3.25M call rows): the step and k_score
    d = W.pool_c4()
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    hs = []
    for _ in range(3):
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt, device=dev, stream=stream)
        s.load(d["pool"], d["tasks"])
        for _ in range(3):
            s.step(d["now_ns"], d["v_token_ns"])
        hs.append(s)
    torch.cuda.synchronize()
    c0 = [h.counters() for h in hs]
    # synchronous steps: C4's speculative set is larger than k_spec's one-CTA fast path, so every
    # step also runs the host-launched resolve (k_spec_big); wall clock per step
    K = 30
    t0 = time.perf_counter()
    for k in range(K):
        last = hs[k % 3].step(d["now_ns"], d["v_token_ns"])
    torch.cuda.synchronize()
    ms_sync = (time.perf_counter() - t0) / K * 1e3
    # device-resolved chained steps (the handles chain the big-set resolve in their graphs once a
    # set outgrew k_spec's fast path): CUDA events around K step_async launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(K):
        hs[k % 3].step_async(d["now_ns"], d["v_token_ns"])
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    for h in hs:
        last = h.fetch()
    c1 = [h.counters() for h in hs]
    k_ms = Scheduler.time_scoring(hs, d["now_ns"], d["v_token_ns"], 30)
    ab = alg_bytes(d)
    pk = peaks()
    hbm = pk["hbm_gbs"] if pk else 6650.0
    out["C4"] = {"metric": "call rows scheduled/sec", "value": n / (ms / 1e3), "unit": "rows/s", "rows": n, "tasks": nt,
                 "ms_per_step": ms, "tasks_per_s": nt / (ms / 1e3), "n_spec": int(last["n_spec"]),
                 "ms_per_step_synchronous_wall": ms_sync,
                 "how": "device time of chained jit_sched_step_async steps over 3 rotated copies (CUDA events; the "
                        "big speculative set resolved by k_spec_big_chain inside the step graph); the synchronous "
                        "wall-clock step beside it",
                 "k_score": {"ms": k_ms, "alg_bytes": ab, "achieved_gbs": ab / (k_ms / 1e3) / 1e9,
                             "frac": ab / (k_ms / 1e3) / 1e9 / hbm,
                             "survey_8d_bytes": n * 52 + nt * 24, "frac_8d": (n * 52 + nt * 24) / (k_ms / 1e3) / 1e9 / hbm},
                 "fallbacks": sum(b["fallbacks"] - a["fallbacks"] for a, b in zip(c0, c1)),
                 "skipped": sum(b["skipped"] - a["skipped"] for a, b in zip(c0, c1)),
                 "workload": "C4: 100K compound tasks (50% in a 64-call fan-out stage, 30% of those calls done; "
                             "50% in a 1-call stage), tau 8192, B_max 8192; 3 rotated copies"}
    for h in hs:
        h.close()
    # ---- C3 token-budget sweep (tau 2,048 to 65,536, B_max = tau): synchronous steps
    d3 = W.pool_snapshot(3, 1 << 20)
    n3, nt3 = len(d3["pool"]["input_len"]), len(d3["tasks"]["arrival_ns"])
    sweep = {}
    for tau in (2048, 8192, 65536):
        cfg = dict(d3["cfg"], token_budget=tau, max_batch=tau)
        hs = []
        for _ in range(4):                               # 4 x 36 MB > L2
            s = Scheduler(cfg, d3["groups"], d3["table"], capacity=n3, task_capacity=nt3, device=dev, stream=stream)
            s.load(d3["pool"], d3["tasks"])
            for _ in range(3):
                s.step(d3["now_ns"], d3["v_token_ns"])
            hs.append(s)
        torch.cuda.synchronize()
        K = 24
        t0 = time.perf_counter()
        for k in range(K):
            last = hs[k % 4].step(d3["now_ns"], d3["v_token_ns"])
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / K * 1e3
        sweep[str(tau)] = {"ms_per_step_wall": ms, "requests_per_s": n3 / (ms / 1e3), "b_star": int(last["b_star"]),
                           "n_candidates": int(last["n_candidates"]), "n_selected": int(last["n_selected"]),
                           "n_spec": int(last["n_spec"]), "fallback": int(last["fallback"])}
        for h in hs:
            h.close()
    out["C3_tau_sweep"] = {"metric": "pending requests scheduled/sec (1M pool) vs token budget", "unit": "requests/s",
                           "points": sweep,
                           "how": "synchronous jit_sched_step (host round trip included), wall clock, 4 rotated copies",
                           "workload": "C3 pool (2^20 rows) with tau = B_max in {2048, 8192, 65536}"}
    return out


def next_lines(args, dev, stream, Scheduler):
    """SURVEY 8(f) rows built this round, each measured beside the oracle:
    NEXT-1 preemption gate (C5 replays), NEXT-2 fairness blend (C3 k_score) and online p
    (C5 replays), NEXT-3 pattern matching (C4-scale queries x a 500-graph store)."""
    import torch
    import oracle
    out = {}
    # ---- NEXT-1 / NEXT-2 in the replay: a slice of the C5 sweep with the gate, with online p
    traces = [W.trace_mixed(k) for k in range(3)]
    d = traces[0]
    sweep = W.c5_sweep()
    specs = [dict(sweep[i], trace=i % 3) for i in range(0, 4096, 8)]         # 512 sweep points
    variants = {"plain": (d["cfg"], d["rcfg"]),
                "gate": (dict(d["cfg"], preempt=1), d["rcfg"]),
                "online_p": (d["cfg"], dict(d["rcfg"], p_adapt=1, eps_num=1, eps_den=10, window_frames=4, seed=1))}
    for name, (cfg, rc) in variants.items():
        rs = Scheduler(cfg, d["groups"], d["table"], capacity=4096, task_capacity=1024, device=dev, stream=stream)
        rs.replay([t["trace"] for t in traces], specs[:8], rc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res, _ = rs.replay([t["trace"] for t in traces], specs, rc)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        rs.close()
        steps = sum(int(r["steps"]) for r in res)
        # the oracle on a bounded sample (4 replays), to check and to time
        t0 = time.perf_counter()
        same, osteps = True, 0
        for j in range(4):
            sp = specs[j * 128]
            rcj = dict(rc, **{k: sp[k] for k in ("load_num", "load_den", "slo_num", "slo_den")})
            t = traces[sp["trace"]]
            ref = oracle.replay(cfg, t["groups"], t["table"], t["trace"], rcj)
            same &= all(int(res[j * 128][k]) == int(ref[k]) for k in ("token_goodput", "steps", "sim_end_ns"))
            osteps += ref["steps"]
        tc = time.perf_counter() - t0
        out[f"replay_{name}"] = {
            "metric": "replayed serving steps/sec (C5 sweep slice)", "value": steps / (ms / 1e3), "unit": "steps/s",
            "replays": len(specs), "token_goodput_sum": int(sum(int(r["token_goodput"]) for r in res)),
            "n_preempted_sum": int(sum(int(r["n_preempted"]) for r in res)), "equal_to_oracle_sample": bool(same),
            "cpu_baseline": {"value": osteps / tc, "unit": "steps/s", "cores": 1, "kind": "oracle",
                             "sample": "4 of the replays on 1 core"},
            "workload": "C5(i) slice: 512 (load, SLO-scale) points x 4096 steps of 2048-row mixed traces"}
    # ---- NEXT-2 blend in the pool step: k_score over C3 with f = 1/10 (every pending row keyed exactly)
    dd = W.pool_snapshot(3, 1 << 20)
    rng = np.random.default_rng(3)
    pool = dict(dd["pool"], fair=rng.integers(0, 400, len(dd["pool"]["id"])).astype(np.uint32))
    hs = []
    for _ in range(6):
        sb = Scheduler(dict(dd["cfg"], fair_num=1, fair_den=10), dd["groups"], dd["table"], capacity=len(pool["id"]),
                       task_capacity=len(dd["tasks"]["arrival_ns"]), device=dev, stream=stream)
        sb.load(pool, dd["tasks"])
        for _ in range(3):
            sb.step(dd["now_ns"], dd["v_token_ns"])
        hs.append(sb)
    k_ms = Scheduler.time_scoring(hs, dd["now_ns"], dd["v_token_ns"], 30)
    for sb in hs:
        sb.close()
    out["blend_k_score"] = {"metric": "k_score ms per 2^20-row C3 pool with the fairness blend (f = 1/10)",
                            "value": k_ms, "unit": "ms", "alg_bytes": alg_bytes(dd) + 4 * len(pool["id"]),
                            "note": "the blend needs every pending key exactly (no fp32 pre-test) plus Fair(r)"}
    # ---- NEXT-2 power-of-K: the C3 standalone requests, each with dummies on K = 2 of M = 8
    # replicas (replica v_token 0.8-1.2x), one multi-replica step = 8 replica steps + the proposal
    # exchange + 8 reconciles (all replicas on this GPU; across GPUs the exchange is an allgather)
    from paper_2504_20068_b200.jitsched import multi_step
    M, K = 8, 2
    pools = W.replica_pools(dd, M, K, seed=5)
    vs = [int(v) for v in np.linspace(0.8, 1.2, M) * dd["v_token_ns"]]
    reps = [Scheduler(dd["cfg"], dd["groups"], dd["table"], capacity=len(p["id"]), task_capacity=1, device=dev,
                      stream=stream) for p in pools]
    for r_, p in zip(reps, pools):
        r_.load(p, None)
    ref = oracle.multi_step(dd["cfg"], dd["groups"], dd["table"], dd["now_ns"], vs,
                            [{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()} for p in pools])
    got = multi_step(reps, dd["now_ns"], vs)
    same = all(np.array_equal(g_["batch_ids"], r_["batch_ids"]) for g_, r_ in zip(got, ref))
    t0 = time.perf_counter()
    n_mstep = 20
    for _ in range(n_mstep):
        got = multi_step(reps, dd["now_ns"], vs)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n_mstep
    tc0 = time.perf_counter()
    oracle.multi_step(dd["cfg"], dd["groups"], dd["table"], dd["now_ns"], vs,
                      [{k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in p.items()} for p in pools])
    tc = time.perf_counter() - tc0
    rows_m = sum(len(p["id"]) for p in pools)
    for r_ in reps:
        r_.close()
    out["power_of_k"] = {"metric": "dummy rows scheduled/sec (power-of-K, M = 8 replicas, K = 2)",
                         "value": rows_m / wall, "unit": "rows/s", "ms_per_multi_step": wall * 1e3,
                         "rows": rows_m, "selected_total": int(sum(g_["n_selected"] for g_ in got)),
                         "first_step_equal_to_oracle": bool(same),
                         "how": "wall clock of synchronous multi_step calls (8 jit_sched_step + exports + 8 "
                                "jit_multi_reconcile on one GPU)",
                         "cpu_baseline": {"value": rows_m / tc, "unit": "rows/s", "cores": 1, "kind": "oracle",
                                          "sample": "one oracle multi_step over the same 8 replica pools"},
                         "workload": "C3's 2^20-row pool, its standalone rows with dummies on 2 of 8 replicas"}
    # ---- NEXT-3: pattern matching, C4-scale
    store = W.pattern_store(61, n_patterns=500)
    q = W.pattern_queries(62, store, 100_000)
    ms_ = Scheduler(dd["cfg"], dd["groups"], dd["table"], capacity=64, task_capacity=8, device=dev, stream=stream)
    ms_.match(store, q)
    kms = []
    for _ in range(5):
        t0 = time.perf_counter()
        best, score = ms_.match(store, q)
        wall = (time.perf_counter() - t0) * 1e3
        kms.append(ms_.last_match_ms())
    ms_.close()
    sub = {k: v[:200] for k, v in q.items()}
    t0 = time.perf_counter()
    ob, _ = oracle.match(store, sub)
    tc = time.perf_counter() - t0
    out["match"] = {"metric": "compound tasks matched/sec (500-graph store)", "value": 100_000 / (np.median(kms) / 1e3),
                    "unit": "queries/s", "kernel_ms": float(np.median(kms)), "call_ms_wall": wall,
                    "pairs_per_s": 100_000 * 500 / (np.median(kms) / 1e3),
                    "agree_with_oracle_sample": float((ob == best[:200]).mean()),
                    "cpu_baseline": {"value": 200 / tc, "unit": "queries/s", "cores": 1, "kind": "oracle",
                                     "sample": "200 queries x 500 graphs on 1 core"},
                    "workload": "100K queries (C4's task count) revealed at random stages, 500 stored graphs "
                                "from 24 families"}
    # ---- NEXT-4: QRF length bounds for a 2^20-request refresh (every bound of a fresh pool)
    F = W.build_forest(91)
    X, _ = W.forest_training_set(5, 1 << 20)
    g = (np.random.default_rng(5).random(len(X)) * 2000).astype(np.uint32)
    qs = Scheduler(dd["cfg"], dd["groups"], dd["table"], capacity=64, task_capacity=8, device=dev, stream=stream)
    qs.attach_forest(F)
    qs.qrf_bound(X[:1024].astype(np.uint32), g[:1024])
    kq = []
    for _ in range(3):
        bounds, kms_q = qs.qrf_bound(X.astype(np.uint32), g)
        kq.append(kms_q)
    qs.close()
    t0 = time.perf_counter()
    R = dd["cfg"]["refine_interval"]
    ok = 0
    for i in range(300):
        a = R * (int(g[i]) // R)
        v = max(oracle.qrf_quantile(F, [int(X[i, 0]), int(X[i, 1]), a, int(X[i, 3])], a, 95, 100, 8192), int(g[i]) + 1)
        ok += int(v == bounds[i])
    tc = time.perf_counter() - t0
    out["qrf"] = {"metric": "QRF length bounds/sec (2^20 requests)", "value": len(X) / (np.median(kq) / 1e3),
                  "unit": "bounds/s", "kernel_ms": float(np.median(kq)), "trees": len(F["root"]),
                  "nodes": len(F["feature"]), "samples": len(F["samples"]), "agree_with_oracle_sample": ok / 300,
                  "cpu_baseline": {"value": 300 / tc, "unit": "bounds/s", "cores": 1, "kind": "oracle",
                                   "sample": "300 requests on 1 core"},
                  "workload": "2^20 synthetic requests (C3 input mix), 32-tree forest of depth 10 on 6K samples"}
    return out


# ------------------------------------------------------------------------------------------
# N = 1: the C3 step
# ------------------------------------------------------------------------------------------
def run_single(args, dev, stream):
    import torch
    from paper_2504_20068_b200 import Scheduler
    rows = args.rows or (1 << 20)
    d = W.pool_snapshot(3, rows)
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    now, v = d["now_ns"], d["v_token_ns"]
    K, Wm = args.steps, max(3, args.warmup)
    hot = alg_bytes(d)
    rot = rot_for(args, hot)
    hs, first_ms = [], []
    for i in range(rot):
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt, device=dev, stream=stream)
        s.load(d["pool"], d["tasks"])
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s.step(now, v)                                     # first step after a load: exact path
        f1.record(stream)
        torch.cuda.synchronize()
        first_ms.append(f0.elapsed_time(f1))
        hs.append(s)
    for i in range(Wm):
        sel = hs[i % rot].step(now, v)
    torch.cuda.synchronize()
    c_before = [s.counters() for s in hs]
    clk = Clocks(dev)
    t_soak = time.perf_counter() + 0.6                     # clocks sampled under this load
    j = 0
    while time.perf_counter() < t_soak:
        for _ in range(20):
            hs[j % rot].step_async(now, v)
            j += 1
        torch.cuda.synchronize()
    host_us = []

    def timed_block():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        for k in range(K):
            hs[k % rot].step_async(now, v)
        host_us.append((time.perf_counter() - h0) / K * 1e6)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    ms = timed_block()                                     # (1) the headline
    for s in hs:
        s.kernel_times(slots=K)
    ms_events = timed_block()                              # (2) with event nodes around each kernel
    for s in hs:
        s.fetch()
    c_after = [s.counters() for s in hs]
    kt = np.zeros(5)
    for i, s in enumerate(hs):
        steps_i = len(range(i, K, rot))
        if steps_i:
            kt += np.array(s.kernel_times()) * steps_i
    kt /= K
    for s in hs:
        s.kernel_times(slots=0)
    n_b2b = max(60, K)
    k_b2b = Scheduler.time_scoring(hs, now, v, n_b2b)      # (3) k_score back to back
    k_refresh = Scheduler.time_scoring(hs, now, v, 12, force_refresh=True)   # (4) every bound stale
    k_refresh2 = Scheduler.time_scoring(hs, now, v, 30, refresh_2pct=True)  # (5) every 50th bound stale
    k_floor = Scheduler.time_scoring(hs, now, v, n_b2b, read_floor=True)   # (6) the rows read, nothing else
    for _ in range(3):
        for k in range(20):
            hs[k % rot].step_async(now, v)
        torch.cuda.synchronize()
        time.sleep(0.1)
    for s in hs:
        s.fetch()
    clocks = clk.stop()
    fallback = sum(b["fallbacks"] - a["fallbacks"] for a, b in zip(c_before, c_after))
    skipped = sum(b["skipped"] - a["skipped"] for a, b in zip(c_before, c_after))
    steps_dev = sum(b["steps"] - a["steps"] for a, b in zip(c_before, c_after))
    tr = ncu_traffic()
    pk = peaks()
    hbm = pk["hbm_gbs"] if pk else 6650.0
    achieved = hot / (k_b2b / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_score", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_source": tr["source"] if tr else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if pk else "fallback 6650 GB/s",
                "alg_bytes_per_launch": hot, "k_score_ms": k_b2b,
                "alg_bytes_how": f"{BYTES_ROW} B per standalone row, {BYTES_CALL} B per compound call, {BYTES_TASK} B "
                                 "per task, read; no per-row write in the steady state (DESIGN.md §7)",
                "frac_8d": n * BYTES_8D / (k_b2b / 1e3) / 1e9 / hbm,
                "frac_8d_how": f"SURVEY 8(d)'s {BYTES_8D} B per request over the same time",
                "how": f"{n_b2b} back-to-back k_score launches rotating over the {rot} L2-defeating pool copies, CUDA "
                       "events on the library stream around the sequence (jit_sched_time_scoring)",
                "forced_refresh": {"k_score_ms": k_refresh, "frac": hot / (k_refresh / 1e3) / 1e9 / hbm,
                                   "how": "every cached length bound invalidated before each launch (untimed); each "
                                          "launch timed alone, so it also carries its launch latency"},
                "read_floor": {"ms": k_floor, "gbs": n * 32 / (k_floor / 1e3) / 1e9,
                               "frac_of_peak": n * 32 / (k_floor / 1e3) / 1e9 / hbm,
                               "k_score_over_floor": k_floor / k_b2b * (hot / (n * 32)),
                               "how": "the pool's 32-B hot rows read with k_score's load pattern (256-bit loads, next "
                                      "chunk in flight) and nothing else, back to back over the same rotated copies: "
                                      "the achievable time of this footprint; k_score_over_floor = the floor's GB/s "
                                      "over k_score's"},
                "refresh_2pct": {"k_score_ms": k_refresh2, "frac": hot / (k_refresh2 / 1e3) / 1e9 / hbm,
                                 "how": "every 50th row's cached bound invalidated before each launch (SURVEY 8(d)'s "
                                        "steady state of about 2% refresh); each launch timed alone"},
                "kernel_ms_event_nodes": {"k_score": kt[0], "k_spec": kt[2], "step_graph": kt[4]},
                "first_step_after_load_ms": float(np.median(first_ms)), "ms_per_step_with_event_nodes": ms_events}
    for s in hs:
        s.close()
    e2e = e2e_leg(args, d, dev, stream, Scheduler)
    e2e["full_reload"] = full_reload_e2e(d, dev, stream, Scheduler)
    configs = None if args.no_configs else config_lines(args, dev, stream, Scheduler)
    if configs is not None:
        configs["next"] = next_lines(args, dev, stream, Scheduler)
    replay = None if args.no_replay else replay_leg(args, 1, 0, dev, stream, lambda: None, lambda x: x, lambda x: x,
                                                    cpu=not args.no_cpu)
    cpu = None
    if not args.no_cpu:
        t, k = oracle_step_timing(d, budget_s=12.0, max_steps=30)
        cpu = {"value": n / t, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{k} oracle steps over the full C3 pool ({n} rows), pinned to 1 core of {cpu_model()}",
               "ms_per_step": t * 1e3}
    line = {"metric": METRIC, "value": n / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": Wm,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": c3_config(n, nt, 1, rot),
            "run": {"device_steps_resolved": steps_dev, "fast_path_fallbacks": fallback,
                    "chained_steps_skipped": skipped, "host_submit_us_per_step": round(host_us[0], 2),
                    "last_batch": {"n_selected": sel["n_selected"], "b_star": sel["b_star"],
                                   "n_candidates": sel["n_candidates"]}},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "configs": configs,
            "gpu_launches": 2 * K, "clocks": clocks, "replay": replay}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# N > 1: C5(ii), one pool sharded by request id
# ------------------------------------------------------------------------------------------
def run_sharded(args, ws, rank, dev, stream, barrier, allmax, allsum):
    """one pool of N x 2^21 requests sharded by request id (each rank owns 2^21 rows; weak
    scaling); every step tries the speculative union (one allgather), else the exact protocol"""
    import torch
    import torch.distributed as dist
    from paper_2504_20068_b200 import Scheduler
    from paper_2504_20068_b200.sharded import ShardedStep, nccl_allgather
    rows = args.rows or (1 << 21)
    d = W.pool_snapshot(3 + 1000 * rank, rows)
    d["pool"]["id"] = (d["pool"]["id"].astype(np.uint64) * ws + rank).astype(np.uint32)   # globally unique ids
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    now, v = d["now_ns"], d["v_token_ns"]
    cap = max(n, ws * (d["cfg"]["max_batch"] + 1))
    hot = alg_bytes(d)
    rot = args.rot or max(2, -(-4 * L2_BYTES // hot))
    hs, sts = [], []
    for i in range(rot):
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=cap, task_capacity=nt, device=dev, stream=stream)
        s.load(d["pool"], d["tasks"])
        if args.backend == "gloo":
            def gather(t):                               # test mode: through host memory
                c = t.cpu()
                out = [torch.empty_like(c) for _ in range(ws)]
                dist.all_gather(out, c)
                return torch.cat(out).to(t.device)
            st = ShardedStep(s, rank, ws, gather)
        else:
            st = ShardedStep(s, rank, ws, nccl_allgather())
        hs.append(s); sts.append(st)
    K, Wm = args.steps, max(3, args.warmup)
    for i in range(Wm * rot):
        out = sts[i % rot].step(now, v)
    for st in sts:
        st.n_fast = st.n_exact = 0
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(K):
        out = sts[k % rot].step(now, v)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms = allmax(e0.elapsed_time(e1) / K)
    total = allsum(float(n))
    n_fast = sum(st.n_fast for st in sts)
    n_exact = sum(st.n_exact for st in sts)
    roofline = None
    try:
        k_ms = allmax(Scheduler.time_scoring(hs, now, v, 30))
        pk = peaks()
        hbm = pk["hbm_gbs"] if pk else 6650.0
        achieved = hot / (k_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": "k_score", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                    "frac": achieved / hbm, "traffic": None, "alg_bytes_per_launch": hot, "k_score_ms": k_ms,
                    "frac_8d": n * BYTES_8D / (k_ms / 1e3) / 1e9 / hbm,
                    "how": f"per rank: 30 back-to-back k_score launches over {rot} copies of its shard, max over ranks"}
    except Exception as ex:  # pragma: no cover
        roofline = {"error": str(ex)[:200]}
    # C5(ii)'s local / collective / merge breakdown: CUDA events on the stream around the export
    # (k_score + the speculative set), the allgather and the union resolve; speculative steps only
    breakdown = None
    try:
        parts = []
        for k in range(2 * rot):
            st = sts[k % rot]
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            barrier()
            ev[0].record(stream)
            st.s.shard_spec_export(now, v, st.spec, st.rank)
            ev[1].record(stream)
            allb = st.allgather(st.spec)
            ev[2].record(stream)
            r = st.s.shard_spec_resolve(allb, st.world, st.rank)
            ev[3].record(stream)
            if r is None:                                # exact protocol this step: not part of the breakdown
                st._exact(now, v)
                continue
            torch.cuda.synchronize()
            parts.append([ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])])
        if parts:
            med = np.median(np.array(parts), axis=0)
            breakdown = {"local_ms": allmax(float(med[0])), "collective_ms": allmax(float(med[1])),
                         "merge_ms": allmax(float(med[2])), "steps": len(parts),
                         "how": "median over speculative steps of CUDA-event intervals on the library stream around "
                                "jit_shard_spec_export (k_score + set export), the allgather, jit_shard_spec_resolve "
                                "(union resolve + batch readback); max over ranks"}
    except Exception as ex:  # pragma: no cover
        breakdown = {"error": str(ex)[:200]}
    for s in hs[1:]:
        s.close()
    # e2e: the sharded step with each step's deltas... the exchange is the step; wall clock, max over ranks
    e2e = None
    try:
        s0, st0 = hs[0], sts[0]
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.e2e_steps):
            rr = st0.step(now, v)
            d2h += 256 + 12 * rr["n_selected"]
        torch.cuda.synchronize()
        te = allmax((time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": total / te, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(d2h / args.e2e_steps),
               "ms_per_step": te * 1e3,
               "how": "per rank: the sharded step through the public API (speculative export, NCCL allgather, union "
                      "resolve, batch read back), synchronous, wall clock, max over ranks; no deltas"}
    except Exception as ex:  # pragma: no cover
        e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}
    hs[0].close()
    replay = None if args.no_replay else replay_leg(args, ws, rank, dev, stream, barrier, allmax, allsum, cpu=False)
    if rank == 0:
        line = {"metric": METRIC, "value": total / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": Wm,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": c5ii_config(ws, n, rot),
                "run": {"rows_total": int(total), "steps_speculative": n_fast, "steps_exact_protocol": n_exact,
                        "breakdown": breakdown,
                        "last_batch": {"n_selected": out["n_selected"], "b_star": out["b_star"],
                                       "n_candidates": out["n_candidates"]}},
                "roofline": roofline, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": 3 * n_fast + 18 * n_exact, "clocks": clocks, "replay": replay}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    import torch.distributed as dist
    if args.backend == "gloo":
        local = 0                                        # test mode: every rank on GPU 0
    torch.cuda.set_device(local)
    if ws > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = local
    stream = torch.cuda.current_stream(dev)
    if ws == 1:
        return run_single(args, dev, stream)

    def barrier():
        dist.barrier()

    red_dev = "cpu" if args.backend == "gloo" else f"cuda:{dev}"

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    return run_sharded(args, ws, rank, dev, stream, barrier, allmax, allsum)


if __name__ == "__main__":
    main()
