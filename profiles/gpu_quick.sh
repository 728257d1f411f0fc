#!/bin/bash
# quick GPU check: build, parity tests, bench without the replay/cpu legs (outputs in gpurun_out/)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-replay --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench_quick.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bench_quick.log
