#!/bin/bash
# A/B timing of the variants built by scripts/build_variants.sh (same box, same
# call: compare within one run only -- box-to-box variance is ~10-20 %).
#   usage (under gpurun): bash scripts/gpu_variants.sh [configs...]   default: c2 c3  (c4: scripts/prof_c4.py)
mkdir -p gpurun_out
out=gpurun_out/variants.log; : > $out
cfgs=${@:-c2 c3}
for rep in 1 2; do
  for cfg in $cfgs; do
    for so in paper_2408_12179_b200/variants/*.so; do
      echo "== $cfg $(basename $so)" >> $out
      if [ "$cfg" = c4 ]; then
        HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_c4.py --reps 3 >> $out 2>&1
      else
        HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1
      fi
    done
  done
done
