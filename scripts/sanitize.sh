#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over smoke()
# and the C1-size engine, power-step, batch, row-block and exact-path parity tests.
# Logs land in gpurun_out/sanitize_*.log; summaries are copied to profiles/.
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 7"
SMOKE='import __graft_entry__ as g; g.smoke()'
run() {   # name tool args...
  local name=$1 tool=$2; shift 2
  local t0=$(date +%s)
  timeout 900 $CS --tool $tool "$@" > gpurun_out/sanitize_${name}_${tool}.log 2>&1
  echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/sanitize_${name}_${tool}.log
}
for tool in memcheck racecheck synccheck initcheck; do
  run smoke $tool python -c "$SMOKE"
done
# the SELL / CB / split / STG engines (x 3 variants), power method, batch, row-block, exact path
for tool in memcheck racecheck synccheck; do
  run engines $tool python -m pytest -x -q tests/test_gpu_parity.py -k "test_iteration_bit_exact_c1 or test_scaling_and_power or test_spmv_abi or test_edge_shapes_bit_exact"
  run batch $tool python -m pytest -x -q tests/test_gpu_batch.py -k "small_cases or matches_single or deterministic"
  run rowblock $tool python -m pytest -x -q tests/test_gpu_rowblock.py -k "test_partitioned_trajectory_c1 or test_partitioned_scaling_and_power or test_nccl_transport_world1"
  run exact $tool python -m pytest -x -q tests/test_exact.py -k "reports_vs_reference or normal_equations"
done
grep -H "ERROR SUMMARY\|rc=" gpurun_out/sanitize_*.log > gpurun_out/sanitize_summary.txt
