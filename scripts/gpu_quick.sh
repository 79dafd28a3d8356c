#!/bin/bash
# full GPU test suite + per-iteration timing of C2 / C3
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for c in c2 c3; do timeout 600 python scripts/prof_iter.py --config $c --reps 3 > gpurun_out/prof_$c.log 2>&1; done
