#!/bin/bash
# C2 engines vs the oracle; compute-sanitizer memcheck / synccheck over the TS
# index-word kernel (HPR_TS_AW=1: C1 / edge-shape TS cases + the flow-LP case).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "c2_engines" > gpurun_out/c2_engines.log 2>&1; echo "rc=$?" >> gpurun_out/c2_engines.log
CS="compute-sanitizer --target-processes all --print-limit 50 --error-exitcode 7"
T=tests/test_gpu_parity.py
for tool in memcheck synccheck; do
  t0=$(date +%s)
  HPR_TS_AW=1 timeout 900 $CS --tool $tool python -m pytest -x -q $T -k "(test_iteration_bit_exact_c1 and ts) or (test_edge_shapes_bit_exact and ts) or test_flow_lp_compact_many_blocks" > gpurun_out/sanitize_aw_$tool.log 2>&1
  echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/sanitize_aw_$tool.log
done
grep -H "ERROR SUMMARY\|passed\|failed\|rc=" gpurun_out/sanitize_aw_*.log > gpurun_out/sanitize_aw_summary.txt
