#!/bin/bash
# gather-ahead instances at 7 CTAs/SM (ga7) and the A_g^T partial store at 8 (store8) vs the
# current library: C2 / C4 per-iteration, alternating on one box.
mkdir -p gpurun_out
out=gpurun_out/minb3_ab.log; : > $out
V=$PWD/paper_2408_12179_b200/variants
for rep in 1 2; do
  echo "== c2 default" >> $out; timeout 600 python scripts/prof_iter.py --config c2 --reps 3 2>&1 | grep per-iter >> $out
  echo "== c2 ga7" >> $out; HPR_LIB_PATH=$V/libhprlp_b200_ga7.so timeout 600 python scripts/prof_iter.py --config c2 --reps 3 2>&1 | grep per-iter >> $out
  for v in default ga7 store8; do
    if [ $v = default ]; then L=""; else L="HPR_LIB_PATH=$V/libhprlp_b200_$v.so"; fi
    echo "== c4 $v" >> $out; env $L timeout 600 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
  done
done
