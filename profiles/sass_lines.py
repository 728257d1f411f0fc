"""Attribute ncu per-instruction counts (source page, SASS) of k_score to source lines / functions
using the line table of the local build (same sources and flags).  Run here (no GPU):
  python profiles/sass_lines.py gpurun_out/prof_score.ncu-rep [kernel-mangled-prefix] [cubin-prefix]
(k_spec: python profiles/sass_lines.py gpurun_out/prof_spec.ncu-rep _ZN3jit6k_spec exact)"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "_ZN3jit7k_scoreILb0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2504_20068_b200", "libjitsched.so")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the source page lists the kernel, then any non-inlined callee: keep the kernel's section
ends = [i for i, r in enumerate(rows) if i > 1 and r and r[0] == "Kernel Name"]
if ends:
    rows = rows[:ends[0]]
h = rows[1]
ie, smp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = [(r[1], int(r[ie] or 0), int(r[smp] or 0)) for r in rows[2:] if len(r) > ie]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.startswith(sys.argv[3] if len(sys.argv) > 3 else "abi")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
start = [i for i, l in enumerate(sass) if l.startswith(".text." + kern)][0]
seq, cur = [], None
for l in sass[start + 1:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        seq.append((cur, m.group(2)))
print("sass", len(seq), "profiled", len(data))
funcs = {}
for fn in set(loc[0] for loc, _ in seq if loc):
    p = os.path.join(ROOT, "paper_2504_20068_b200", "csrc", fn)
    if os.path.exists(p):
        lst = []
        for i, l in enumerate(open(p).read().splitlines(), 1):
            m = re.search(r"__device__ (?:__forceinline__ |__noinline__ )?(?:static )?[\w:<>]+ (\w+)\(|__global__ .*? (k_\w+)\(", l)
            if m:
                lst.append((i, m.group(1) or m.group(2)))
        funcs[fn] = lst
def fname(loc):
    if not loc:
        return "?"
    f, l = loc
    name = f
    for i, n in funcs.get(f, []):
        if i <= l:
            name = f + ":" + n
    return name
tot = sum(n for _, n, _ in data)
N = float(os.environ.get("ROWS", 1 << 20))
byf, byl, ops = collections.Counter(), collections.Counter(), collections.Counter()
for (loc, ins), (s, n, k) in zip(seq, data):
    byf[fname(loc)] += n
    byl[loc] += n
    o = s.split()
    o = o[1] if o and o[0].startswith("@") else (o[0] if o else "")
    ops[o.split(".")[0]] += n
print(f"total {tot} warp-inst = {tot * 32 / N:.1f} thread-inst/row")
for k, n in byf.most_common(25):
    print(f"  {k:40s} {n * 32 / N:7.1f}/row")
print("lines:")
for k, n in byl.most_common(25):
    print(f"  {k}  {n * 32 / N:7.1f}/row")
print("ops:", [(o, round(n * 32 / N, 1)) for o, n in ops.most_common(20)])

# stall hot spots (the stall is charged to the instruction after a deferred BAR / BSYNC)
hs = out and list(csv.reader(io.StringIO(out)))[1]
cols = [c for c in ("stall_barrier", "stall_wait", "stall_long_sb", "stall_short_sb", "stall_branch_resolving")
        if c in hs]
for cname in cols:
    ci = hs.index(cname)
    vals = [(int(r[ci] or 0), i) for i, r in enumerate(rows[2:]) if len(r) > ci]
    top = sorted(vals, reverse=True)[:5]
    print(cname, [(v, seq[i][0], seq[i - 1][1][:28]) for v, i in top if i < len(seq)])

# warp-stall samples per source line (all reasons), top 30
byls = collections.Counter()
for (loc, ins), (s, n, k) in zip(seq, data):
    byls[loc] += k
print("samples by line:", sum(byls.values()))
for k, v in byls.most_common(30):
    print(f"  {k}  {v}")
