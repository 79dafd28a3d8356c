#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/variants4.log; : > $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu --format=csv >> $out
for rep in 1 2; do
for cfg in c2 c3; do
  for so in paper_2408_12179_b200/variants/*.so; do
    echo "== $cfg $(basename $so)" >> $out
    HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep -E "per-it|clocks" >> $out
  done
done
done
