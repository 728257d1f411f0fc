#!/bin/bash
# ncu evidence for the C3 step (run under gpurun on ONE GPU).  Outputs in gpurun_out/.
#  1. launch list: every kernel of a few steps with device time + DRAM bytes (cold-cache,
#     serialised -- compare SHARES, not absolute times, with bench.py's CUDA-event numbers)
#  2. one `--set full` capture of k_score (the dominant kernel) and of k_spec
# The step graph holds kernel nodes only, so ncu profiles the graph as bench.py runs it.
P="python profiles/prof_step.py --steps 6 --rot 3"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $P > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_score -s 4 -c 1 -o gpurun_out/prof_score -f $P \
    > gpurun_out/ncu_full.log 2>&1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"^k_spec" -s 4 -c 1 \
    -o gpurun_out/prof_spec -f $P >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
