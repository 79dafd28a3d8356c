#!/bin/bash
# C3 solve breakdown (report phases vs device iteration time); C4 TS A/B interleaved; row-block tests.
mkdir -p gpurun_out
timeout 300 python scripts/c1_breakdown.py c3 > gpurun_out/breakdown_c3.log 2>&1
: > gpurun_out/c4_ab.log
for ts in 0 1 0 1; do
  echo "== HPR_TS=$ts" >> gpurun_out/c4_ab.log
  HPR_TS=$ts timeout 300 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> gpurun_out/c4_ab.log
done
timeout 600 python -m pytest tests/test_gpu_rowblock.py -m gpu -x -q -rf > gpurun_out/pytest_rb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rb.log
