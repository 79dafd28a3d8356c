#!/bin/bash
# TS in the row-block path: row-block + parity GPU tests, C4 (1 GPU) with / without TS.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowblock.py tests/test_gpu_parity.py -m gpu -x -q -rf > gpurun_out/pytest_rb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rb.log
for ts in 2 0; do
HPR_TS=$ts timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c4_ts$ts.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_ts$ts.log
done
