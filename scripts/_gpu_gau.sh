#!/bin/bash
# gather-ahead batch size (spill-free U=3 / U=2 vs U=4 with spills): C2, C4 rank, C3.
mkdir -p gpurun_out
out=gpurun_out/gau_ab.log; : > $out
for rep in 1 2; do
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  echo "== $(basename $so)" >> $out
  HPR_LIB_PATH=$PWD/$so timeout 150 python scripts/prof_iter.py --config c2 --reps 5 2>&1 | grep per-iter >> $out
  HPR_LIB_PATH=$PWD/$so timeout 300 python scripts/prof_c4.py --reps 3 2>&1 | grep per-iter >> $out
done
done
