#!/bin/bash
# Build k_score tuning variants (extra -D flags) beside the default library and time each with a
# short bench run (no replay / cpu legs).  usage: VARIANTS="name:-DX=1 name2:-DY=2" bash profiles/variants.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for v in base ${VARIANTS}; do
  name=${v%%:*}; defs=${v#*:}; [ "$v" = base ] && defs=""
  lib=$PWD/paper_2504_20068_b200/libjitsched_$name.so
  python -c "
from paper_2504_20068_b200 import _build
_build.build_library(force=True, out='$lib', defines='$defs'.replace(',', ' ').split())" > gpurun_out/build_$name.log 2>&1 || { echo "$name build failed"; tail -5 gpurun_out/build_$name.log; continue; }
  JITSCHED_LIB=$lib timeout 300 python bench.py --no-replay --no-cpu --steps 30 --e2e-steps 2 > gpurun_out/bench_$name.log 2>&1
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/bench_$name.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("$name", "defs=$defs", "ms/step %.4f" % d["ms_per_step"], "k_score b2b us %.2f" % (r["k_score_ms"] * 1e3), "nodes", {k: round(v * 1e3, 2) for k, v in r["kernel_ms_event_nodes"].items()}, "frac %.3f" % r["frac"])
except Exception as e:
    print("$name failed", e, open("gpurun_out/bench_$name.log").read()[-800:])
PY
done
