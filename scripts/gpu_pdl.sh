#!/bin/bash
mkdir -p gpurun_out
#timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/variants5.log; : > $out
for rep in 1 2; do
for cfg in c2 c3; do
  for so in paper_2408_12179_b200/variants/*.so; do
    echo "== $cfg $(basename $so)" >> $out
    HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1
  done
done
done
timeout 600 python scripts/e2e_breakdown.py > gpurun_out/e2e_breakdown.log 2>&1
