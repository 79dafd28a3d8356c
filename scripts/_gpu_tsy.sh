#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/tsy_ab.log; : > $out
for so in paper_2408_12179_b200/libhprlp_b200.so paper_2408_12179_b200/variants/*.so; do
  for m in "0 2" "1 2"; do
    set -- $m
    echo "== $(basename $so) HPR_TS_A=$1 HPR_TS_AT=$2" >> $out
    HPR_LIB_PATH=$PWD/$so HPR_TS_A=$1 HPR_TS_AT=$2 timeout 150 python scripts/prof_iter.py --config c3 --reps 3 2>&1 | grep per-iter >> $out
  done
done
