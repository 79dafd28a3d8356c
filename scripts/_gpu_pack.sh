#!/bin/bash
mkdir -p gpurun_out
nproc > gpurun_out/pack_ab.log
for nat in 1 0; do
  echo "== HPR_PACK_NATIVE=$nat" >> gpurun_out/pack_ab.log
  HPR_PACK_NATIVE=$nat timeout 400 python scripts/c5_pipe_sweep.py >> gpurun_out/pack_ab.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -x -q -rf > gpurun_out/pytest_batch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batch.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
