#!/bin/bash
# Full GPU round (under gpurun): build, GPU tests, smoke, the default bench line, ncu evidence.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
timeout 900 bash profiles/run_ncu.sh; echo ncu rc=$?
tail -3 gpurun_out/pytest_gpu.log
