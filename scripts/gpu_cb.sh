#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
out=gpurun_out/cb.log; : > $out
for cfg in c1 c2 c3; do
  for cb in 0 auto; do
    echo "== $cfg HPR_CB=$cb" >> $out
    if [ $cb = auto ]; then timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1; else HPR_CB=0 timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1; fi
  done
done
