# A/B: conditional-node graph vs flat graph (all fallback kernels launched, early exit)
python profiles/diag_steps.py 2>&1 | tail -7
for mode in cond flat; do
  if [ $mode = flat ]; then export JITSCHED_FLAT_GRAPH=1; fi
  timeout 300 python bench.py --no-replay --no-cpu --steps 200 > gpurun_out/ab_$mode.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/ab_$mode.json'));print('$mode', d['ms_per_step'], d['roofline']['kernel_ms'])" || tail -3 gpurun_out/ab_$mode.json
done
