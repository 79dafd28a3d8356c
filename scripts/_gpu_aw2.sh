#!/bin/bash
# TS index words, round 2: U=3 batches for the index-word kernel (U=4 spilled):
# C3 per-iteration A/B vs the pre-change library, alternating, same box.
mkdir -p gpurun_out
out=gpurun_out/aw_ab2.log; : > $out
V=paper_2408_12179_b200/variants
for rep in 1 2; do
  echo "== head" >> $out; HPR_LIB_PATH=$PWD/$V/libhprlp_b200_head.so timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== aw1_u3_w24" >> $out; HPR_TS_AW=1 timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== aw1_u3_w23" >> $out; HPR_LIB_PATH=$PWD/$V/libhprlp_b200_w23u3.so HPR_TS_AW=1 timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
  echo "== aw0" >> $out; HPR_TS_AW=0 timeout 600 python scripts/prof_iter.py --config c3 --reps 3 >> $out 2>&1
done
