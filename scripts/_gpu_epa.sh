#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/epa_ab.log; : > $out
for rep in 1 2; do
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 150 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
done
done
for so in paper_2408_12179_b200/variants/libhprlp_b200_epa_w16.so paper_2408_12179_b200/variants/libhprlp_b200_epa_w18.so; do
HPR_LIB_PATH=$PWD/$so timeout 300 python -m pytest tests/test_gpu_parity.py -k "many_blocks or ts" -x -q > gpurun_out/pytest_$(basename $so).log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$(basename $so).log
done
