#!/bin/bash
# one `--set full` capture of k_score (source-correlated) -> gpurun_out/prof_score.ncu-rep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_score -s 16 -c 1 -o gpurun_out/prof_score -f \
    python profiles/prof_step.py --steps 8 --rot 3 > gpurun_out/ncu_score.log 2>&1
tail -3 gpurun_out/ncu_score.log
