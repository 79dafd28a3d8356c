#!/bin/bash
# per-iteration timing of each built variant on C2 and C3
mkdir -p gpurun_out
out=gpurun_out/variants.log; : > $out
for cfg in c2 c3; do
  for so in paper_2408_12179_b200/variants/*.so; do
    echo "== $cfg $(basename $so)" >> $out
    HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 2>&1 | grep per-it >> $out
  done
done
