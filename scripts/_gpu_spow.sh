#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_config_scale.py tests/test_exact.py -m gpu -x -q -rf > gpurun_out/pytest_spow.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_spow.log
for mode in 1 0; do echo "== HPR_SMALL=$mode" >> gpurun_out/spow.log; HPR_SMALL=$mode timeout 200 python scripts/c1_breakdown.py c1 >> gpurun_out/spow.log 2>&1; done
