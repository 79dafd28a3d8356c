#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 scripts/microbench/stage_bw > gpurun_out/stage_bw.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/e2e_profile.py > gpurun_out/e2e_profile.log 2>&1
