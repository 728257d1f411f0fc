"""Summarise ncu outputs from gpurun_out/ into a markdown table (run here, no GPU needed).

usage: python profiles/summarize.py gpurun_out/launches.csv [gpurun_out/prof_score.ncu-rep ...] > profiles/rNN_ncu.md
"""
import collections
import json
import os
import csv
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "lts__t_bytes.sum", "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
       "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_barrier",
       "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
       "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_membar", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
       "smsp__pcsamp_warps_issue_stalled_dispatch_stall", "smsp__pcsamp_warps_issue_stalled_not_selected",
       "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_sample_count"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"]
    if not hi:
        return "(no launch data)\n"
    h = rows[hi[0]]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    order = []
    for r in rows[hi[0] + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].replace("void ", "")
        if k not in order:
            order.append(k)
        try:
            agg[k][r[mi]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    tot = sum(sum(agg[k]["gpu__time_duration.sum"]) for k in order)
    out = ["| kernel | launches | mean µs | share of all kernel time | DRAM read MB/launch | DRAM write MB/launch |",
           "|---|---|---|---|---|---|"]
    for k in order:
        t = agg[k]["gpu__time_duration.sum"]
        rd = agg[k].get("dram__bytes_read.sum", [0])
        wr = agg[k].get("dram__bytes_write.sum", [0])
        out.append(f"| {k} | {len(t)} | {sum(t) / len(t) / 1e3:.2f} | {sum(t) / tot * 100:.1f}% | "
                   f"{sum(rd) / len(rd) / 1e6:.2f} | {sum(wr) / len(wr) / 1e6:.2f} |")
    return "\n".join(out) + "\n"


def report(path):
    try:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    except Exception as e:  # pragma: no cover
        return f"({path}: {e})\n"
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        return f"({path}: empty)\n"
    h = rows[0]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0] if "Kernel Name" in h else "?"
        out.append(f"**{name}** ({path.split('/')[-1]})\n")
        out.append("| metric | value |\n|---|---|")
        for m in RAW:
            if m in h:
                out.append(f"| {m} | {r[h.index(m)]} |")
        out.append("")
    return "\n".join(out) + "\n"


def traffic_json(path, out_json):
    """k_score's DRAM traffic per launch (read + write) from a --set full capture -> json for bench.py."""
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    if len(rows) < 3:
        return
    h = rows[0]
    for row in rows[2:]:
        name = row[h.index("Kernel Name")]
        if "k_score" not in name:
            continue
        units = rows[1]
        def val(m):
            v = float(row[h.index(m)].replace(",", ""))
            u = units[h.index(m)]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        json.dump({"bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                   "gpu_time_us": float(row[h.index("gpu__time_duration.sum")]),
                   "source": f"ncu --set full capture {os.path.basename(path)} (one launch, cold L2)"},
                  open(out_json, "w"), indent=1)
        return


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--traffic":
        traffic_json(sys.argv[2], sys.argv[3])
        sys.exit(0)
    print("## Launch list (ncu, cold-cache, serialised)\n")
    print(launches(sys.argv[1]))
    for p in sys.argv[2:]:
        print(report(p))
