#!/bin/bash
# Time every library in profiles/variants/ (built by tune_build.sh) with a short bench run.
mkdir -p gpurun_out
for lib in profiles/variants/lib_*.so; do
  name=$(basename $lib .so); name=${name#lib_}
  JITSCHED_LIB=$PWD/$lib timeout 300 python bench.py --no-replay --no-cpu --steps 30 --e2e-steps 2 > gpurun_out/tune_$name.log 2>&1
  python - <<PY
import json
try:
    d = json.loads(open("gpurun_out/tune_$name.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print("$name", "ms/step %.4f" % d["ms_per_step"], "k_score b2b us %.2f" % (r["k_score_ms"] * 1e3),
          "nodes", {k: round(v * 1e3, 2) for k, v in r["kernel_ms_event_nodes"].items()}, "frac %.3f" % r["frac"],
          "fb", d["run"]["fast_path_fallbacks"], "skip", d["run"]["chained_steps_skipped"])
except Exception as e:
    print("$name failed", e, open("gpurun_out/tune_$name.log").read()[-800:])
PY
done
