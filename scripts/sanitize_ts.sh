#!/bin/bash
# compute-sanitizer over the TS engine (bulk-copy ring + mbarriers, hpr_tsell.cuh): the C1 engine
# and edge-shape cases (memcheck / synccheck: every engine; racecheck: the TS cases only -- the
# tool terminates the process on the opt-in CB engine's pipeline); logs in gpurun_out/sanitize_ts_*.log
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 7"
T=tests/test_gpu_parity.py
TS_IDS="$T::test_iteration_bit_exact_c1[hpr-2-ts] $T::test_iteration_bit_exact_c1[hdr-1-ts] $T::test_iteration_bit_exact_c1[dr-0-ts] $T::test_edge_shapes_bit_exact[ineq_only-ts] $T::test_edge_shapes_bit_exact[empty_rows_cols-ts] $T::test_edge_shapes_bit_exact[long_rows-ts]"
for tool in memcheck synccheck; do
  t0=$(date +%s)
  timeout 900 $CS --tool $tool python -m pytest -x -q $T -k "test_iteration_bit_exact_c1 or test_edge_shapes_bit_exact" > gpurun_out/sanitize_ts_$tool.log 2>&1
  echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/sanitize_ts_$tool.log
done
t0=$(date +%s)
timeout 1500 $CS --tool racecheck python -m pytest -x -q $TS_IDS > gpurun_out/sanitize_ts_racecheck.log 2>&1
echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/sanitize_ts_racecheck.log
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed\|rc=" gpurun_out/sanitize_ts_*.log > gpurun_out/sanitize_ts_summary.txt
