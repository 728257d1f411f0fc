"""Aggregate an ncu --set full capture (imported source, -lineinfo) per CUDA source line:
instructions executed and warp-stall samples, top lines first.
usage: python profiles/src_lines.py <rep.ncu-rep> [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, agg, tot_i, tot_s = None, [], 0, 0
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[0] != "":                       # a CUDA source line (its metrics aggregate its SASS)
        try:
            ie = int(r[hdr.index("Instructions Executed")])
            ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except Exception:
            continue
        agg.append((ie, ss, f"{cur_file}:{r[0]}", r[1].strip()[:100]))
        tot_i += ie
        tot_s += ss
print(f"total instructions executed {tot_i}, stall samples {tot_s}")
for ie, ss, where, src in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{ie:10d} {100.0 * ie / max(tot_i, 1):5.1f}%  {ss:6d} {100.0 * ss / max(tot_s, 1):5.1f}%  {where:18s} {src}")
