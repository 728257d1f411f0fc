#!/bin/bash
# Build k_score tuning variants HERE (CPU, nvcc cross-compiles) into profiles/variants/ so that a
# gpurun call only times them (profiles/tune_run.sh).  usage:
#   VARIANTS="name:-DX=1,-DY=2 name2:-DZ=3" bash profiles/tune_build.sh
mkdir -p profiles/variants
pids=()
for v in ${VARIANTS}; do
  name=${v%%:*}; defs=${v#*:}
  ( python -c "
from paper_2504_20068_b200 import _build
_build.build_library(force=True, out='$PWD/profiles/variants/lib_$name.so', defines='$defs'.replace(',', ' ').split())" \
      > profiles/variants/build_$name.log 2>&1 && echo "built $name" || { echo "$name build failed"; tail -5 profiles/variants/build_$name.log; } ) &
  pids+=($!)
done
wait
