#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/c5_ab.log; : > $out
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/libhprlp_b200_noreg.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 300 python scripts/batch_time.py >> $out 2>&1
done
timeout 600 python -m pytest tests/test_gpu_batch.py -m gpu -x -q -rf > gpurun_out/pytest_batch.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_batch.log
