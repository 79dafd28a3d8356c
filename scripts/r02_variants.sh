#!/bin/bash
# Round-2 A/B of the SELL gather-ahead register budget / lean pipeline (C2, C3),
# the persisting-L2 window on y (C3), then ncu --set full of the C2 and C3 iteration kernels.
mkdir -p gpurun_out
out=gpurun_out/r02_variants.log; : > $out
for rep in 1 2; do
  for cfg in c2 c3; do
    for so in paper_2408_12179_b200/variants/*.so; do
      echo "== $cfg $(basename $so)" >> $out
      HPR_LIB_PATH=$PWD/$so timeout 600 python scripts/prof_iter.py --config $cfg --reps 3 >> $out 2>&1
    done
  done
  for w in 0 1; do
    echo "== c3 HPR_L2WIN=$w base" >> $out
    HPR_L2WIN=$w HPR_LIB_PATH=$PWD/paper_2408_12179_b200/variants/libhprlp_b200_base.so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  done
done
for c in c2 c3; do
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:EpiXIter|EpiYIter' -s 20 -c 2 -o gpurun_out/r02_${c}_iter python scripts/prof_iter.py --config $c --reps 1 --steps 20 > gpurun_out/r02_ncu_full_$c.log 2>&1
done
