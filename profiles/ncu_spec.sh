#!/bin/bash
# one `--set full` capture of k_spec (source-correlated) -> gpurun_out/prof_spec.ncu-rep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"^k_spec" -s 4 -c 1 -o gpurun_out/prof_spec -f \
    python profiles/prof_step.py --steps 6 --rot 3 > gpurun_out/ncu_spec.log 2>&1
tail -2 gpurun_out/ncu_spec.log
