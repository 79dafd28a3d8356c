#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_exact.py tests/test_gpu_rowblock.py -m gpu -x -q -rf > gpurun_out/pytest_ssm.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ssm.log
: > gpurun_out/ssm.log
for mode in 1 0; do echo "== HPR_SMALL_SMEM=$mode" >> gpurun_out/ssm.log; HPR_SMALL_SMEM=$mode timeout 200 python scripts/c1_breakdown.py c1 >> gpurun_out/ssm.log 2>&1; done
