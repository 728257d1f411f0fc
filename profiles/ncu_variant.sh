#!/bin/bash
# ncu --set full capture of one steady-state k_score launch of a library variant
# usage: bash profiles/ncu_variant.sh <lib path> <out name>
lib=${1:-$PWD/paper_2504_20068_b200/libjitsched.so}; out=${2:-prof_score}; shift 2; extra="$@"
JITSCHED_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:k_score -s 16 -c 1 -o gpurun_out/$out -f \
    python profiles/prof_step.py --steps 8 --rot 3 $extra > gpurun_out/ncu_$out.log 2>&1
tail -2 gpurun_out/ncu_$out.log
