#!/bin/bash
# compute-sanitizer over small GPU parity cases (memcheck / racecheck / synccheck /
# initcheck on small configs).  Logs in gpurun_out/sanitizer_*.log.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="tests/test_parity_gpu.py::test_empty_and_degenerate tests/test_parity_gpu.py::test_c3_shaped_pools_full_compare tests/test_replay_gpu.py::test_c1_toy_full_log tests/test_replay_gpu.py::test_many_small_random_traces tests/test_replay_gpu.py::test_sweep_configs_short tests/test_parity_gpu.py::test_speculative_paths_against_oracle_chain tests/test_multi_gpu.py::test_multi_equal_v_ties_to_lower_index tests/test_deltas_gpu.py::test_engine_loop_with_arrivals_task_updates_and_progress_by_id"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 python -m pytest -q -x $T \
      > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -m1 'ERROR SUMMARY' gpurun_out/sanitizer_$tool.log)"
done
