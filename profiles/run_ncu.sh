#!/bin/bash
# ncu evidence for the C3 step (run under gpurun on ONE GPU).  Outputs in gpurun_out/.
#  1. launch list of bench.py itself (device time per launch; cold-cache, serialised -- compare
#     SHARES with bench.py's CUDA-event numbers, not absolute times)
#  2. one `--set full` capture of a steady-state k_score (the dominant kernel) and of k_spec
#  3. profiles/k_score_traffic.json (DRAM bytes per k_score launch) for bench.py's roofline.traffic
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 6 --warmup 3 --no-replay --no-configs --no-cpu \
    --e2e-steps 4 > gpurun_out/ncu_launch.log 2>&1
P="python profiles/prof_step.py --steps 8 --rot 3"
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_score -s 16 -c 1 \
    -o gpurun_out/prof_score -f $P > gpurun_out/ncu_full.log 2>&1
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"^k_spec" -s 12 -c 1 \
    -o gpurun_out/prof_spec -f $P >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out | tail -5
# the replay kernel: one capture of the C5 sweep configuration (256-thread CTAs)
ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_replay -c 1 \
    -o gpurun_out/prof_replay -f python profiles/prof_replay.py 640 512 >> gpurun_out/ncu_full.log 2>&1
