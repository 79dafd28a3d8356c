#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/gamin_ab.log; : > $out
for rep in 1 2; do
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 150 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
  HPR_LIB_PATH=$PWD/$so timeout 150 python scripts/prof_iter.py --config c2 --reps 5 2>&1 | grep per-iter >> $out
done
done
