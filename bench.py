#!/usr/bin/env python
"""bench.py -- the JITServe GMAX scheduling step on B200 (contract: DESIGN.md §8).

Headline (N=1): BASELINE config C3 -- one GMAX step (a1-a9) over a pool of 2^20 pending
requests resident in HBM (16 SLO groups, token budget 8192, B_max 8192), timed on the device
with CUDA events.  `value` = pending requests scheduled per second, summed over ranks (weak
scaling: every rank owns a 2^20-row shard).  Also reported:
  * roofline of the dominant kernel (k_score) against the measured HBM copy bandwidth;
  * e2e: the same step through the C ABI from pinned HOST buffers (pool H2D + batch D2H);
  * replay: BASELINE config C5(i) -- the load x SLO-scale sweep of independent trace replays,
    replayed serving steps per second (replays sharded i -> rank i mod N, no communication);
  * cpu_baseline: the CPU oracle (oracle/, plain C, 1 core) on a bounded sample of C3.
`--impl reference` runs the oracle as the reference arm (rank 0 only).
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
# written in the steady state; per compound call the same + 4 B read (task id); per task 32 B read
# (its constants).  SURVEY §8(d) counts 40 B per request (32 B read + an 8-B key write this design
# does not need); `frac_8d` reports that accounting too.
BYTES_ROW, BYTES_CALL, BYTES_TASK = 32, 36, 32
BYTES_8D = 40


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of k_score per launch, from the committed
    ncu --set full capture summary (profiles/k_score_traffic.json, written by
    profiles/summarize.py); None when absent."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "k_score_traffic.json")))
        return t
    except Exception:
        return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--rot", type=int, default=6, help="pool copies rotated to defeat the 126 MB L2")
    ap.add_argument("--replays", type=int, default=4096)
    ap.add_argument("--replay-steps", type=int, default=4096)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-replay", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
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


def build_c3(rank, rows):
    d = W.pool_snapshot(3 + 1000 * rank, rows)
    return d


def oracle_step_timing(d, budget_s=10.0, max_steps=40):
    """CPU oracle on the C3 pool, pinned to one host core (bounded sample)."""
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
    t = sum(times) / len(times)
    return t, len(times)


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, ws, rank):
    if rank != 0:
        return
    d = build_c3(0, args.rows)
    n = len(d["pool"]["input_len"])
    import oracle
    oracle.build()
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_step_timing(d, budget_s=0.0, max_steps=1)
    t, k = oracle_step_timing(d, budget_s=60.0, max_steps=max(1, min(args.steps, 20)))
    v = n / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": k,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3: 2^20-row pending pool, 16 SLO groups, tau 8192, B_max 8192", "rows": n},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{k} oracle steps over the full C3 pool ({n} rows), 1 core of {cpu_model()}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pinned_pool(d):
    import torch
    out = {}
    for k, v in d["pool"].items():
        if isinstance(v, np.ndarray):
            t = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
            out[k] = t
        else:
            out[k] = v
    tasks = {}
    for k, v in d["tasks"].items():
        tasks[k] = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
    return out, tasks


def replay_leg(args, ws, rank, dev, stream, barrier, allmax, allsum):
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
    return {"metric": "replayed serving steps/sec", "value": steps_done / (rms / 1e3), "unit": "steps/s",
            "workload": f"C5(i): {args.replays} replays (64 load x 64 SLO-scale points, 4 base mixed 1:1:1 traces "
                        f"of 2048 rows), up to {args.replay_steps} steps each, tau 2048, B_max 128",
            "ms": rms, "steps_total": int(steps_done), "scaling": "strong (fixed sweep, replay i -> rank i mod N)",
            "goodput_tokens_sum": int(allsum(float(sum(r["token_goodput"] for r in res)))),
            "gpu_launches": 1}


def run_sharded(args, ws, rank, dev, stream, barrier, allmax, allsum):
    """N > 1: one pool of N x 2^20 requests sharded by request id (each rank owns 2^20 rows;
    weak scaling); every step is the exact two-round protocol of shard.cuh with NCCL
    allgathers over NVLink (torch.distributed), identical batch on every rank."""
    import torch
    import torch.distributed as dist
    from paper_2504_20068_b200 import Scheduler
    from paper_2504_20068_b200.sharded import ShardedStep, nccl_allgather
    d = build_c3(rank, args.rows)
    d["pool"]["id"] = (d["pool"]["id"].astype(np.uint64) * ws + rank).astype(np.uint32)   # globally unique ids
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    now, v = d["now_ns"], d["v_token_ns"]
    cap = max(n, ws * (d["cfg"]["max_batch"] + 1))
    s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=cap, task_capacity=nt, device=dev, stream=stream)
    s.load(d["pool"], d["tasks"])
    if args.backend == "gloo":
        def gather(t):                                   # test mode: through host memory
            c = t.cpu()
            out = [torch.empty_like(c) for _ in range(ws)]
            dist.all_gather(out, c)
            return torch.cat(out).to(t.device)
        st = ShardedStep(s, rank, ws, gather)
    else:
        st = ShardedStep(s, rank, ws, nccl_allgather())
    K, Wm = args.steps, max(3, args.warmup)
    for _ in range(Wm):
        out = st.step(now, v)
    st.n_fast = st.n_exact = 0
    barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(K):
        out = st.step(now, v)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    ms = allmax(e0.elapsed_time(e1) / K)
    total = allsum(float(n))
    n_fast, n_exact = st.n_fast, st.n_exact              # the timed steps' paths (before the e2e leg)
    # roofline of k_score on every rank (as at N = 1: back-to-back launches rotating over this
    # rank's shard and 5 more copies of it, to defeat the L2), max over ranks
    roofline = None
    try:
        extra = []
        for _ in range(5):
            s2 = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt, device=dev, stream=stream)
            s2.load(d["pool"], d["tasks"])
            s2.step(now, v)
            extra.append(s2)
        torch.cuda.synchronize()
        k_ms = allmax(Scheduler.time_scoring([s] + extra, now, v, 60))
        for s2 in extra:
            s2.close()
        n_single = int(d["pool"]["n_single"])
        alg_bytes = n_single * BYTES_ROW + (n - n_single) * BYTES_CALL + nt * BYTES_TASK
        pk = peaks()
        hbm_peak = pk["hbm_gbs"] if pk else 6650.0
        tr = ncu_traffic()
        achieved = alg_bytes / (k_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": "k_score", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "traffic": tr["bytes_per_launch"] if tr else None,
                    "alg_bytes_per_launch": alg_bytes, "k_score_ms": k_ms,
                    "how": "per rank: 60 back-to-back k_score launches over 6 copies of its shard "
                           "(jit_sched_time_scoring), max over ranks"}
    except Exception as ex:  # pragma: no cover
        roofline = {"error": str(ex)[:200]}
    # e2e through the C ABI: every rank loads its shard from pinned host buffers (H2D) and runs the
    # sharded step (exchange + batch D2H); wall clock, max over ranks
    e2e = None
    try:
        hp, ht = pinned_pool(d)
        h2d = sum(int(t.numel() * t.element_size()) for k, t in hp.items() if hasattr(t, "numel") and k != "true_out")
        h2d += sum(int(t.numel() * t.element_size()) for t in ht.values())
        s.load(hp, ht)
        st.step(now, v)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.e2e_steps):
            s.load(hp, ht)
            rr = st.step(now, v)
            d2h += 248 + 12 * rr["n_selected"]
        torch.cuda.synchronize()
        te = allmax((time.perf_counter() - t0) / args.e2e_steps)
        e2e = {"value": total / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h / args.e2e_steps), "ms_per_step": te * 1e3,
               "how": "per rank: jit_sched_load(pinned host shard) + the sharded step (NCCL exchange, batch D2H); "
                      "wall clock, max over ranks"}
    except Exception as ex:  # pragma: no cover
        e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}
    s.close()
    replay = None if args.no_replay else replay_leg(args, ws, rank, dev, stream, barrier, allmax, allsum)
    if rank == 0:
        line = {"metric": METRIC, "value": total / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": Wm,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"C5(ii)-shaped: {ws} x 2^20-row shards of one pool (C3 generator), sharded by "
                                       "request id, tau 8192, B_max 8192", "rows_total": int(total),
                           "l2": "inputs larger than L2 (2^20 rows x ~100 B workspace per rank plus exchange buffers)",
                           "parallelism": f"sharded pool over {ws} ranks: speculative sets allgathered over NCCL and "
                                          "resolved identically on every rank (exact 2-round protocol as fallback)",
                           "steps_speculative": n_fast, "steps_exact_protocol": n_exact,
                           "last_batch": {"n_selected": out["n_selected"], "b_star": out["b_star"],
                                          "n_candidates": out["n_candidates"]}},
                "roofline": roofline, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": 3 * n_fast + 18 * n_exact, "clocks": clocks,
                "replay": replay}
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
    from paper_2504_20068_b200 import Scheduler
    dev = local
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    red_dev = "cpu" if args.backend == "gloo" else f"cuda:{dev}"

    def allmax(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if ws == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    if ws > 1:
        return run_sharded(args, ws, rank, dev, stream, barrier, allmax, allsum)
    # ------------------------------------------------------------------ C3 pool step
    d = build_c3(rank, args.rows)
    n = len(d["pool"]["input_len"])
    nt = len(d["tasks"]["arrival_ns"])
    now, v = d["now_ns"], d["v_token_ns"]
    K, Wm = args.steps, max(3, args.warmup)
    hs = []
    first_ms = []
    for i in range(args.rot):
        s = Scheduler(d["cfg"], d["groups"], d["table"], capacity=n, task_capacity=nt, device=dev, stream=stream)
        s.load(d["pool"], d["tasks"])
        # first step after load: every row computes its length bound (cold cache) -- timed apart
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        s.step(now, v)
        f1.record(stream)
        torch.cuda.synchronize()
        first_ms.append(f0.elapsed_time(f1))
        hs.append(s)
    # warm-up (synchronous: validates that every step resolves on the graph's fast path)
    statuses = []
    for i in range(Wm):
        r = hs[i % args.rot].step(now, v)
        statuses.append(r["status"])
    sel = r
    barrier()
    torch.cuda.synchronize()
    # clocks: the sampler runs through a ~0.6 s soak of the same step loop, the timed blocks
    # and a short tail, so that nvidia-smi has samples under this load (B200_PROFILING.md)
    c_before = [s.counters() for s in hs]
    clk = Clocks(dev)
    t_soak = time.perf_counter() + 0.6
    j = 0
    while time.perf_counter() < t_soak:
        for _ in range(20):
            hs[j % args.rot].step_async(now, v)
            j += 1
        torch.cuda.synchronize()

    host_us = []                                          # host time to submit one step (launch loop)

    def timed_block():
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h0 = time.perf_counter()
        for k in range(K):
            hs[k % args.rot].step_async(now, v)
        host_us.append((time.perf_counter() - h0) / K * 1e6)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1) / K

    # (1) the headline: K steps with no per-kernel event nodes in the graphs
    ms = timed_block()
    # (2) the same K steps again with CUDA-event nodes around each kernel (for the roofline)
    for s in hs:
        s.kernel_times(slots=K)
    ms_events = timed_block()
    # every timed step must have resolved on the device's fast path: the device counters of every
    # handle over the soak + timed blocks (exact-path steps, and chained steps skipped because an
    # earlier one needed the host) must not have moved
    for s in hs:
        s.fetch()
    c_after = [s.counters() for s in hs]
    # (3) k_score alone, back to back over the rotated pools (launch overlapped by the previous
    # kernel, as inside the step where k_spec hides it): the roofline's kernel duration
    barrier()
    n_b2b = max(60, K)
    k_b2b = Scheduler.time_scoring(hs, now, v, n_b2b)
    for _ in range(3):
        for k in range(20):
            hs[k % args.rot].step_async(now, v)
        torch.cuda.synchronize()
        time.sleep(0.1)
    for s in hs:
        s.fetch()
    clocks = clk.stop()
    ms_max = allmax(ms)
    fallback = sum(b["fallbacks"] - a["fallbacks"] for a, b in zip(c_before, c_after))
    skipped = sum(b["skipped"] - a["skipped"] for a, b in zip(c_before, c_after))
    steps_dev = sum(b["steps"] - a["steps"] for a, b in zip(c_before, c_after))
    kt = np.zeros(5)
    for i, s in enumerate(hs):
        steps_i = len(range(i, K, args.rot))
        if steps_i:
            kt += np.array(s.kernel_times()) * steps_i
    kt /= K
    tr = ncu_traffic()
    total_rows = allsum(float(n))
    value = total_rows / (ms_max / 1e3)
    n_single = int(d["pool"]["n_single"])
    alg_bytes = n_single * BYTES_ROW + (n - n_single) * BYTES_CALL + nt * BYTES_TASK
    pk = peaks()
    hbm_peak = pk["hbm_gbs"] if pk else 6650.0
    achieved = alg_bytes / (k_b2b / 1e3) / 1e9
    achieved_nodes = alg_bytes / (kt[0] / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_score", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_source": tr["source"] if tr else None,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if pk else "fallback 6650 GB/s",
                "alg_bytes_per_launch": alg_bytes, "k_score_ms": k_b2b,
                "frac_8d": n * BYTES_8D / (k_b2b / 1e3) / 1e9 / hbm_peak,
                "how": f"{n_b2b} back-to-back k_score launches rotating over the {args.rot} L2-defeating pool "
                       "copies, CUDA events on the library stream around the sequence (jit_sched_time_scoring)",
                "kernel_ms_event_nodes": {"k_score": kt[0], "k_spec": kt[2], "step_graph": kt[4]},
                "frac_event_nodes": achieved_nodes / hbm_peak,
                "how_event_nodes": "CUDA event nodes around each kernel inside the step graph, averaged over "
                                   "the K steps of a second timed block; each node pair also counts the "
                                   "kernel node's launch latency (~5 us)",
                "frac_of_8tbs_datasheet": achieved / 8000.0,
                "first_step_after_load_ms": float(np.median(first_ms)),
                "ms_per_step_with_event_nodes": ms_events}

    # ------------------------------------------------------------------ steady state with progress
    # the engine loop: every step reports the progress of each handle's previous batch (decode
    # +1 token, or the next prefill chunk; host mirror of the pool), so cached length bounds go
    # stale as rows cross a multiple of R tokens and k_score refreshes them (SURVEY §8(d)'s
    # "steady state"); wall clock per synchronous step, progress H2D + batch D2H included
    steady = None
    try:
        mirror = [{"gen": d["pool"]["generated"].astype(np.int64).copy(),
                   "pre": d["pool"]["prefilled"].astype(np.int64).copy()} for _ in hs]
        L_in = d["pool"]["input_len"].astype(np.int64)
        last = [None] * len(hs)
        for i, s in enumerate(hs):
            last[i] = s.step(now, v)
        torch.cuda.synchronize()
        refresh, fb, ms_s = [], 0, []
        KS = max(10, K)
        for k in range(KS):
            i = k % len(hs)
            b, m = last[i], mirror[i]
            rows = np.asarray(b["batch_rows"][:b["n_selected"]], np.int64)
            tok = np.asarray(b["batch_tokens"][:b["n_selected"]], np.int64)
            dec = m["pre"][rows] >= L_in[rows]
            m["gen"][rows] += np.where(dec, 1, 0)
            newpre = np.minimum(m["pre"][rows] + np.where(dec, 0, tok), L_in[rows])
            m["gen"][rows] += np.where(~dec & (newpre >= L_in[rows]), 1, 0)      # token 0 at prefill end (A28)
            m["pre"][rows] = newpre
            prog = {"row": rows, "generated": m["gen"][rows], "prefilled": m["pre"][rows],
                    "state": np.full(len(rows), W.Q_RUNNING)}
            t0 = time.perf_counter()
            last[i] = hs[i].step(now, v, prog)
            ms_s.append((time.perf_counter() - t0) * 1e3)
            refresh.append(last[i]["n_refresh"])
            fb += int(last[i]["fallback"])
        ms_med = float(np.median(ms_s))
        steady = {"ms_per_step_wall_median": ms_med, "value": n / (ms_med / 1e3), "unit": UNIT, "steps": KS,
                  "refresh_per_step_mean": float(np.mean(refresh)), "fallback_steps": fb,
                  "how": "synchronous jit_sched_step with the previous batch's progress (one pinned H2D) and the batch (written by the GPU into pinned host memory), "
                         "wall clock, median over steps, 6 rotated pools"}
    except Exception as ex:  # pragma: no cover
        steady = {"error": str(ex)[:200]}

    # ------------------------------------------------------------------ e2e through the C ABI
    e2e = None
    try:
        hp, ht = pinned_pool(d)
        s0 = hs[0]
        h2d = sum(int(t.numel() * t.element_size()) for k, t in hp.items() if hasattr(t, "numel") and k != "true_out")
        h2d += sum(int(t.numel() * t.element_size()) for t in ht.values())
        for _ in range(2):
            s0.load(hp, ht)
            s0.step(now, v)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for _ in range(args.e2e_steps):
            s0.load(hp, ht)
            rr = s0.step(now, v)
            d2h += 248 + 12 * rr["n_selected"]
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / args.e2e_steps
        te = allmax(te)
        e2e = {"value": total_rows / te, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h / args.e2e_steps), "ms_per_step": te * 1e3,
               "how": "wall clock around jit_sched_load(pinned host pool) + jit_sched_step (batch D2H), synchronized"}
    except Exception as ex:  # pragma: no cover
        e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}
    for s in hs:
        s.close()

    replay = None if args.no_replay else replay_leg(args, ws, rank, dev, stream, barrier, allmax, allsum)

    # ------------------------------------------------------------------ CPU oracle baseline
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        import oracle
        t, k = oracle_step_timing(d, budget_s=12.0, max_steps=30)
        cpu = {"value": n / t, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{k} oracle steps over the full C3 pool ({n} rows), pinned to 1 core of {cpu_model()}",
               "ms_per_step": t * 1e3}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": Wm,
                "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": "C3: 2^20-row pending pool per GPU (40% chat, 30% deep-research, 30% compound "
                                       "calls in 16-call tasks), 16 SLO groups, tau 8192, B_max 8192, v_token 15 ms",
                           "rows_per_gpu": n, "tasks_per_gpu": nt,
                           "l2": f"inputs larger than L2: {args.rot} rotated pool copies of ~{(n * 100) >> 20} MiB workspace each",
                           "parallelism": f"{ws} independent 2^20-row shards (no data-path collective)" if ws > 1 else "single GPU",
                           "fast_path_fallbacks": fallback, "chained_steps_skipped": skipped,
                           "device_steps_resolved": steps_dev,
                           "host_submit_us_per_step": round(host_us[0], 2), "last_batch": {"n_selected": sel["n_selected"],
                                                                         "b_star": sel["b_star"],
                                                                         "n_candidates": sel["n_candidates"]}},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "steady_with_progress": steady,
                "gpu_launches": 2 * K,
                "clocks": clocks, "replay": replay}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
